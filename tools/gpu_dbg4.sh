TTN_DEBUG_GEMM=1 TTN_DEBUG_CHFSI=1 timeout 300 python bench.py --config 4 --quick --steps 1 --warmup 0 > gpurun_out/dbg4.json 2> gpurun_out/dbg4.err; echo rc=$?
grep chfsi gpurun_out/dbg4.err
