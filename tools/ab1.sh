source tools/gpu_ab.sh
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run c5_base 5 "" X=1
run c5_nofork 5 "" TTN_GEMM_NO_FORK=1
run c5_jac12 5 "" TTN_JACOBI_MAX_N=12
run c5_nofork_jac12 5 "" TTN_GEMM_NO_FORK=1 TTN_JACOBI_MAX_N=12
run c1_base 1 "" X=1
run c1_nofork 1 "" TTN_GEMM_NO_FORK=1
run c1_jac12 1 "" TTN_JACOBI_MAX_N=12
run c1_nofork_jac12 1 "" TTN_GEMM_NO_FORK=1 TTN_JACOBI_MAX_N=12
run c3_w1 3 "--workers 1" X=1
run c3_w2 3 "--workers 2" X=1
run c3_w3 3 "--workers 3" X=1
run c3_w2_nofork 3 "--workers 2" TTN_GEMM_NO_FORK=1
run c3_nofork 3 "--workers 1" TTN_GEMM_NO_FORK=1
run c2_base 2 "" X=1
run c2_nofork 2 "" TTN_GEMM_NO_FORK=1
