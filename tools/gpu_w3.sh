mkdir -p gpurun_out
for w in 1 2 4; do for c in 3; do
timeout 600 python bench.py --config $c --workers $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/w_${w}_c$c.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/w_${w}_c$c.json')); print('w=$w cfg$c', round(d['value'],2), round(d['ms_per_step'],2), round(d['roofline']['frac'],3), round(d['kernels']['all']['ms'],1))"
done; done
