#!/bin/bash
# final round-2 evidence: bench lines of every config, ncu launch lists + full capture, f1 and
# f2 sweeps (run under gpurun)
set -x
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final/build.log 2>&1
timeout 900 python bench.py > gpurun_out/final/bench_c3.json 2> gpurun_out/final/bench_c3.err
for c in 1 2 4 5; do
  timeout 900 python bench.py --config $c > gpurun_out/final/bench_c$c.json 2> gpurun_out/final/bench_c$c.err
done
timeout 1200 python tools/f1_circuit.py > gpurun_out/final/f1_circuit_r02.jsonl 2> gpurun_out/final/f1.err
timeout 900 python tools/paper_random.py > gpurun_out/final/paper_random_r02.jsonl 2> gpurun_out/final/f2.err
PCONFIGS="3 2 1" bash tools/gpu_profile.sh > gpurun_out/final/prof.log 2>&1
mv gpurun_out/launches_r02_* gpurun_out/ncu_zgemm_traffic_r02_* gpurun_out/ncu_r02_c3_full.md gpurun_out/prof_r02_c3_raw.csv.gz gpurun_out/final/ 2>/dev/null
rm -f gpurun_out/final/*.csv
ls -la gpurun_out/final
