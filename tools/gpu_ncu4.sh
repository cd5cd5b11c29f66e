mkdir -p gpurun_out
Q="python bench.py --config 4 --quick --steps 1 --warmup 1"
timeout 300 $Q > gpurun_out/quick4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches4.csv $Q > gpurun_out/ncu_launch4.log 2>&1; echo "ncu launches rc=$?"
