mkdir -p gpurun_out
Q="python bench.py --config 2 --quick --steps 1 --warmup 1"
timeout 300 $Q > gpurun_out/quick2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $Q > gpurun_out/ncu_l2.log 2>&1; echo "rc=$?"
