# Round-end evidence: default bench line, launch lists (+ DRAM bytes) of configs 3 and 4, and
# one ncu --set full capture of config 3's largest zgemm launches.  Each ncu pass runs only after
# the same command exited 0 without ncu.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active
timeout 1200 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
for c in 3 4; do
Q="python bench.py --config $c --quick --steps 1 --warmup 1"
timeout 600 $Q > gpurun_out/quick$c.log 2>&1 && \
timeout 1200 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_final_c$c.csv $Q > gpurun_out/ncu_launch_final_c$c.log 2>&1; echo "ncu launches c$c rc=$?"
done
Q="python bench.py --config 3 --quick --steps 1 --warmup 1"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:zgemm_grouped -s 39 -c 5 -o gpurun_out/prof_zgemm_final $Q > gpurun_out/ncu_full_final.log 2>&1; echo "ncu full rc=$?"
ls -la gpurun_out/*.ncu-rep gpurun_out/launches_final_c*.csv
