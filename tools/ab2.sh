source tools/gpu_ab.sh
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest -x -q tests/test_gpu_schedule.py tests/test_gpu_edges.py tests/test_gpu_loopback.py tests/test_gpu_parity.py -k "not config4 and not full_batch" 2>&1 | tail -2
run c1_pdl 1 "" X=1
run c1_nopdl 1 "" TTN_NO_PDL=1
run c2_pdl 2 "" X=1
run c2_nopdl 2 "" TTN_NO_PDL=1
run c3_pdl 3 "" X=1
run c3_nopdl 3 "" TTN_NO_PDL=1
run c5_pdl 5 "" X=1
run c5_nopdl 5 "" TTN_NO_PDL=1
run c5_pdl_b 5 "" X=1
