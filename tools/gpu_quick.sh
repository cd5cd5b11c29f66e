# full GPU tests, then short benches of the given configs (default 3 2 5); kernel-family split
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
for c in ${@:-3 2 5}; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q_c$c.json 2> gpurun_out/q_c$c.err; echo "bench$c rc=$?"; tail -3 gpurun_out/q_c$c.err
python -c "
import json; d=json.load(open('gpurun_out/q_c$c.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac']); [print(k, round(v['ms'],1), v['launches'], round(v['tflops'],2)) for k,v in d['kernels'].items()]"
done
