source tools/gpu_ab.sh
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py -k "config3 or small_trees or large_gram or degenerate" 2>&1 | tail -2
TTN_TRIDIAG_PAIR4=1 timeout 900 python -m pytest -x -q tests/test_gpu_parity.py -k "config3_batch or small_trees or degenerate" 2>&1 | tail -2
run c3_pair6 3 "" X=1
run c3_nopair6 3 "" TTN_TRIDIAG_NOPAIR6=1
run c3_pair6_pair4 3 "" TTN_TRIDIAG_PAIR4=1
run c3_pair6_b 3 "" X=1
run c3_nopair6_b 3 "" TTN_TRIDIAG_NOPAIR6=1
run c5_pair4 5 "" TTN_TRIDIAG_PAIR4=1
run c5_base 5 "" X=1
