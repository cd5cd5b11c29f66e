mkdir -p gpurun_out
for c in ${@:-3}; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-showcase > gpurun_out/b_c$c.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/b_c$c.json')); print('cfg$c', round(d['value'],2), round(d['ms_per_step'],2), round(d['roofline']['frac'],3), {k:round(v['ms'],1) for k,v in d['kernels'].items()})"
done
