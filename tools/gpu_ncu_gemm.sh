mkdir -p gpurun_out
Q="./tools/gemm_bench 1 square"
timeout 120 $Q > gpurun_out/gb_sq.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zgemm -c 1 -o gpurun_out/prof_gemm_sq $Q > gpurun_out/ncu_gemm.log 2>&1; echo "ncu rc=$?"
Q="./tools/gemm_bench 1 cfg3"
timeout 120 $Q > gpurun_out/gb_c3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zgemm -c 6 -o gpurun_out/prof_gemm_c3 $Q > gpurun_out/ncu_gemm3.log 2>&1; echo "ncu rc=$?"
