#!/bin/bash
# A/B of the factor leg order (TTN_FAC_BA): parity subset, bench lines, TMA coverage
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for e in TTN_FAC_BA=1; do
  env $e timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "config1 or small_trees or mixed or config3_batch or config2 or tolerance or degenerate or zero_state or config5_circuit or config4" 2>&1 | tail -2
done
for e in TTN_FAC_BA=0 TTN_FAC_BA=1; do for c in 3 4 2; do
  env $e timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-showcase > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/b.json')); k=d['kernels']; r=d['roofline']
print('$e c$c', round(d['value'],2), 'ms/step', round(d['ms_per_step'],2), 'zgemm', round(k['zgemm']['ms']/d['steps'],2), 'heev', round(k['heev']['ms']/d['steps'],2), 'frac', round(r['frac'],3), 'keff', round(r['kernel_efficiency']['frac'],3))"
done; done
TTN_FAC_BA=1 TTN_DEBUG_GEMM=1 timeout 300 python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-showcase 2>&1 >/dev/null | grep gemm-tma | awk '{n++; p+=$2; t+=$4; f+=$6} END {print "c3 BA tma problems", p, "of", t, "mean MNK frac", f/n}'
