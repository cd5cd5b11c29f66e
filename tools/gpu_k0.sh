#!/bin/bash
# planner derating sweep (TTN_PLAN_K0) on configs 3 / 4: step time, zgemm time, algorithmic frac
mkdir -p gpurun_out/k0
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/k0/build.log 2>&1 || exit 1
for c in ${CONFIGS:-3}; do
for k in ${K0S:-0 8 16 24 40}; do
  TTN_PLAN_K0=$k timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-showcase > gpurun_out/k0/c${c}_k$k.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/k0/c${c}_k$k.json')); k=d['kernels']; r=d['roofline']
print('c$c K0=$k', round(d['value'],2), 'ms/step', round(d['ms_per_step'],2), 'zgemm', round(k['zgemm']['ms']/d['steps'],2), 'heev', round(k['heev']['ms']/d['steps'],2), 'frac', round(r['frac'],3), 'keff', round(r['kernel_efficiency']['frac'],3))"
done; done
