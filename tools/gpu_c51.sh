mkdir -p gpurun_out
for c in 5 1; do
timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "bench$c rc=$?"; tail -3 gpurun_out/bench_c$c.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c$c.json')); print(d['value'], d['ms_per_step'], d['fp64_tflops_end_to_end'], d['roofline']['frac'], d['e2e'], d['cpu_baseline']); [print(k, round(v['ms'],1), v['launches'], v['tflops']) for k,v in d['kernels'].items()]"
done
