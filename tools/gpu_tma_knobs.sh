#!/bin/bash
# A/B of the TMA staging knobs on config 4 / 3 zgemm time
mkdir -p gpurun_out/tma
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/tma/build.log 2>&1 || { tail -30 gpurun_out/tma/build.log; exit 1; }
run() {  # label, env...
  local lab=$1; shift
  for c in ${CONFIGS:-4 3}; do
    env "$@" timeout 300 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/tma/k_${lab}_c$c.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/tma/k_${lab}_c$c.json')); k=d['kernels']
print('$lab c$c', round(d['value'],2), 'zgemm ms/step', round(k['zgemm']['ms']/d['steps'],2), 'keff', round(d['roofline']['kernel_efficiency']['frac'],3))"
  done
}
run base TTN_GEMM_TMA=0
run tma TTN_GEMM_TMA=1
run rank5 TTN_TMA_RANK5=1
