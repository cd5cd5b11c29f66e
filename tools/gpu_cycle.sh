timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -3 gpurun_out/bench_c3.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c3.json')); print(d['value'], d['ms_per_step']); [print(k, round(v['ms'],1), v['launches']) for k,v in d['kernels'].items()]"
