#!/bin/bash
# TMA coverage of a config (TTN_DEBUG_TMA fold failures, TTN_DEBUG_GEMM coverage) and a
# planner-derating sweep (TTN_PLAN_K0) of its bench line
mkdir -p gpurun_out/cov
C=${C:-3}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cov/build.log 2>&1 || exit 1
TTN_DEBUG_TMA=1 TTN_DEBUG_GEMM=1 timeout 300 python bench.py --config $C --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-showcase 2> gpurun_out/cov/dbg_c$C.err > /dev/null
grep gemm-tma gpurun_out/cov/dbg_c$C.err | awk '{n++; p+=$2; t+=$4; f+=$6} END {print "tma problems", p, "of", t, "mean MNK frac", f/n}'
grep tma-fail gpurun_out/cov/dbg_c$C.err | sed 's/^\[tma-fail\] //' | sort | uniq -c | sort -rn | head -20 > gpurun_out/cov/fail_c$C.txt
for k in ${K0S:-24 40 64}; do
  TTN_PLAN_K0=$k timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-showcase > gpurun_out/cov/k$k.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/cov/k$k.json')); k=d['kernels']; r=d['roofline']
print('K0=$k c$C', round(d['value'],2), 'ms/step', round(d['ms_per_step'],2), 'zgemm', round(k['zgemm']['ms']/d['steps'],2), 'frac', round(r['frac'],3), 'keff', round(r['kernel_efficiency']['frac'],3))"
done
