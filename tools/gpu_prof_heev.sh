mkdir -p gpurun_out
Q="python bench.py --config 3 --quick --steps 1 --warmup 1"
timeout 300 $Q > gpurun_out/quick3.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:heev -s 40 -c 10 -o gpurun_out/prof_heev_final $Q > gpurun_out/ncu_heev_final.log 2>&1; echo "ncu rc=$?"; ls -la gpurun_out/prof_heev_final.ncu-rep
