# one GPU call: parity tests, smoke, full bench line, ncu launch list, per-launch DRAM traffic of
# every zgemm launch of one step, and one --set full capture of the heaviest zgemm launches.
# (gpurun copies gpurun_out/ back only below 64 MiB: keep the full capture small)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/bench.err
Q="python bench.py --quick --steps 1 --warmup 1"
timeout 300 $Q > gpurun_out/quick.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $Q > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
N=$(python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/launches.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name')
print(sum(1 for r in rows[1:] if 'zgemm_grouped' in r[ki]) // 2)
PY
)
echo "zgemm launches per step: $N"
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:zgemm_grouped -s $N -c $N --csv --log-file gpurun_out/zgemm_traffic.csv $Q > gpurun_out/ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:zgemm_grouped -s $((N + 10)) -c 4 -o gpurun_out/prof_zgemm $Q > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ls -la gpurun_out | head -30; du -sh gpurun_out
