timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for c in 5 3; do
timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "bench$c rc=$?"; tail -3 gpurun_out/bench_c$c.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c$c.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac']); [print(k, round(v['ms'],1), v['launches']) for k,v in d['kernels'].items()]"
done
