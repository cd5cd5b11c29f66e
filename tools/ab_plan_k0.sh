source tools/gpu_ab.sh
export STEPS=5
for k in 0 12 16 24 32 48; do run c3_k0_$k 3 "" TTN_PLAN_K0=$k; done
for k in 0 16 24 48; do run c4_k0_$k 4 "" TTN_PLAN_K0=$k; done
