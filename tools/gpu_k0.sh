mkdir -p gpurun_out
for k in 0 24 48; do for c in 3 4 5 2; do
TTN_PLAN_K0=$k timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/k0_${k}_c$c.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/k0_${k}_c$c.json')); print('k0=$k cfg$c', round(d['value'],2), round(d['ms_per_step'],2), round(d['roofline']['frac'],3), round(d['kernels']['zgemm']['ms'],1))"
done; done
