mkdir -p gpurun_out
Q="python bench.py --config 3 --quick --steps 1 --warmup 1"
timeout 300 $Q > gpurun_out/quick3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches3.csv $Q > gpurun_out/ncu_launch3.log 2>&1; echo "ncu launches rc=$?"
TTN_DEBUG_GEMM=1 timeout 300 python bench.py --config 3 --quick --steps 1 --warmup 0 --batch 64 > gpurun_out/dbg3.json 2> gpurun_out/dbg3.err; echo rc=$?
