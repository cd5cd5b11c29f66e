mkdir -p gpurun_out
for c in 1 2 4 5; do
timeout 900 python bench.py --config $c > gpurun_out/bench_final_c$c.json 2> gpurun_out/bench_final_c$c.err; echo "cfg$c rc=$?"
done
