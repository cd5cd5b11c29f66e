mkdir -p gpurun_out
for v in 0 1; do for c in 3 4 5; do
if [ $v = 1 ]; then export TTN_PLAN_PAD16=1; else unset TTN_PLAN_PAD16; fi
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-showcase > gpurun_out/pad_${v}_c$c.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/pad_${v}_c$c.json')); print('pad=$v cfg$c', round(d['value'],2), round(d['ms_per_step'],2), round(d['roofline']['frac'],3), round(d['kernels']['zgemm']['ms'],1))"
done; done
