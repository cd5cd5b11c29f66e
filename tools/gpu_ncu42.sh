mkdir -p gpurun_out
for c in 4 2; do
Q="python bench.py --config $c --quick --steps 1 --warmup 1"
timeout 300 $Q > gpurun_out/quick$c.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches$c.csv $Q > gpurun_out/ncu_launch$c.log 2>&1; echo "ncu launches $c rc=$?"
done
