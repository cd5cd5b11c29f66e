#!/bin/bash
# TMA routing thresholds (TTN_TMA_MIN_K, TTN_TMA_MIN_MNK): bench lines per config
source tools/gpu_ab.sh
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
export STEPS=${STEPS:-3}
for c in ${CONFIGS:-5 3 2}; do
  run c${c}_base $c "" X=1
  for k in 32 64 128 256; do run c${c}_mink$k $c "" TTN_TMA_MIN_K=$k; done
  run c${c}_notma $c "" TTN_GEMM_TMA=0
done
