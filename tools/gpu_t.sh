mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for c in 4 2 3; do
timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "bench$c rc=$?"; tail -3 gpurun_out/bench_c$c.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c$c.json')); print(d['value'], d['ms_per_step'], d['fp64_tflops_end_to_end'], d['roofline']['frac']); [print(k, round(v['ms'],1), v['launches'], v['tflops']) for k,v in d['kernels'].items()]"
done
