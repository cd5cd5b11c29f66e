mkdir -p gpurun_out
Q="python bench.py --config 3 --quick --steps 1 --warmup 1"
timeout 300 $Q > gpurun_out/quick3.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:zgemm_grouped<\(int\)128, \(int\)16, \(int\)4, \(int\)1, \(bool\)0, \(bool\)0>" -s 4 -c 2 -o gpurun_out/prof_skinny $Q > gpurun_out/ncu_skinny.log 2>&1; echo "ncu rc=$?"; ls -la gpurun_out/prof_skinny.ncu-rep; tail -3 gpurun_out/ncu_skinny.log
