mkdir -p gpurun_out
Q="python bench.py --config 3 --quick --steps 1 --warmup 1"
timeout 300 $Q > gpurun_out/quick3.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:heev_tridiag -s 5 -c 2 -o gpurun_out/prof_tri2 $Q > gpurun_out/ncu_tri.log 2>&1; echo "ncu rc=$?"
