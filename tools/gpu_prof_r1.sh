# launch list (cold, serialised) of one config-3 step + full capture of the largest zgemm launches
mkdir -p gpurun_out
Q="python bench.py --config 3 --quick --steps 1 --warmup 1"
timeout 300 $Q > gpurun_out/quick3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_c3_new.csv $Q > gpurun_out/ncu_launch_new.log 2>&1; echo "ncu launches rc=$?"
