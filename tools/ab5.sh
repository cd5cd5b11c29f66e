source tools/gpu_ab.sh
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
STEPS=5 run c5_s5 5 "" X=1
STEPS=10 run c5_s10 5 "" X=1
STEPS=20 run c5_s20 5 "" X=1
STEPS=10 run c5_s10_nofork 5 "" TTN_GEMM_NO_FORK=1
STEPS=10 run c5_s10_w2 5 "--workers 2" X=1
STEPS=10 run c5_s10_w8 5 "--workers 8" X=1
STEPS=10 run c5_s10_nospec 5 "" TTN_NO_SPECULATE=1
nproc; cat /proc/loadavg
