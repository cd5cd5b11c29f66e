#!/bin/bash
# config-5 regression hunt (round 2: 2319 -> 1356 applies/s): bench lines under each knob
source tools/gpu_ab.sh
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
export STEPS=3
run c5_base 5 "" X=1
run c5_notma 5 "" TTN_GEMM_TMA=0
run c5_nospec 5 "" TTN_NO_SPECULATE=1
run c5_no2s 5 "" TTN_HEEV_2S=0
run c5_facab 5 "" TTN_FAC_BA=0
run c5_w1 5 "--workers 1" X=1
run c5_w1_notma 5 "--workers 1" TTN_GEMM_TMA=0
run c5_nofork 5 "" TTN_GEMM_NO_FORK=1
