#!/bin/bash
# The round-2 A/B measurements behind DESIGN.md §6 / §9: bench lines under the library's
# measurement knobs (run under gpurun).  Results: gpurun_out/ab_<name>.json.
#   TTN_JACOBI_MAX_N  route Grams up to this order to the one-warp Jacobi kernel (default off)
#   TTN_HEEV_WY       blocked WY back-transform on the GEMM kernel (default off)
#   TTN_GEMM_NO_FORK  variant kernels of a launch set on one stream (default: forked)
#   TTN_PDL           programmatic dependent launch (default off)
#   TTN_GEMM_TMA=0    cp.async staging for every GEMM problem (default: TMA where operands fold)
#   TTN_TMA_RANK5=1   tensor maps padded to rank 5 (one instruction form; default exact rank)
#   TTN_PLAN_K0       the planner's short-contraction derating (default 24)
#   TTN_CHFSI_MIN_N   Grams above this order take the Chebyshev solver (default 512)
source tools/gpu_ab.sh
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in 1 3 5; do
  run c${c}_base $c "" X=1
  run c${c}_jac12 $c "" TTN_JACOBI_MAX_N=12
  run c${c}_wy $c "" TTN_HEEV_WY=1
  run c${c}_nofork $c "" TTN_GEMM_NO_FORK=1
  run c${c}_pdl $c "" TTN_PDL=1
done
run c3_w2 3 "--workers 2" X=1
run c2_base 2 "" X=1
run c2_pdl 2 "" TTN_PDL=1
for c in 3 4; do
  run c${c}_notma $c "" TTN_GEMM_TMA=0
  run c${c}_rank5 $c "" TTN_TMA_RANK5=1
  run c${c}_k0_40 $c "" TTN_PLAN_K0=40
done
