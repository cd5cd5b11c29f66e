# ncu --set full of the config-3 step's largest zgemm launches (after the same command ran clean)
mkdir -p gpurun_out
Q="python bench.py --config 3 --quick --steps 1 --warmup 1"
timeout 300 $Q > gpurun_out/quick3.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:zgemm_grouped -s ${1:-38} -c ${2:-6} -o gpurun_out/prof_zgemm_r1 $Q > gpurun_out/ncu_full_r1.log 2>&1; echo "ncu rc=$?"; ls -la gpurun_out/prof_zgemm_r1.ncu-rep
