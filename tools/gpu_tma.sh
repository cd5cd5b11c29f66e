#!/bin/bash
# TMA staging check (run under gpurun): parity subset, TMA coverage per config, A/B bench
#   CONFIGS="3 4"  FULL=1 (whole -m gpu suite)
mkdir -p gpurun_out/tma
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/tma/build.log 2>&1 || { tail -30 gpurun_out/tma/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "config1 or small_trees or mixed or errors or degenerate or zero_state or tolerance" > gpurun_out/tma/pytest1.log 2>&1; echo "pytest1 rc=$?"; tail -3 gpurun_out/tma/pytest1.log
for c in ${CONFIGS:-3 4}; do
  for t in 1 0; do
    TTN_GEMM_TMA=$t timeout 300 python bench.py --config $c > gpurun_out/tma/bench_c${c}_tma$t.json 2> gpurun_out/tma/bench_c${c}_tma$t.err
    python - <<PY
import json
d = json.load(open("gpurun_out/tma/bench_c${c}_tma$t.json"))
k = d.get("kernels", {})
print("c$c tma=$t", round(d["value"], 2), "ms/step", round(d["ms_per_step"], 2), "frac", round(d["roofline"].get("frac", 0), 3), "keff", round(d["roofline"].get("kernel_efficiency", {}).get("frac", 0), 3), {a: round(b["ms"] / d["steps"], 2) for a, b in k.items() if isinstance(b, dict) and "ms" in b and b["ms"] / d["steps"] > 0.5})
PY
  done
done
if [ -n "$NCU" ]; then
  TTN_GEMM_TMA=1 timeout 600 ncu --set full --clock-control none -k regex:zgemm_grouped -s 40 -c 6 -o gpurun_out/tma/ncu_tma1 -f python bench.py --config 3 --steps 1 --warmup 3 > gpurun_out/tma/ncu1.log 2>&1
  TTN_GEMM_TMA=0 timeout 600 ncu --set full --clock-control none -k regex:zgemm_grouped -s 40 -c 6 -o gpurun_out/tma/ncu_tma0 -f python bench.py --config 3 --steps 1 --warmup 3 > gpurun_out/tma/ncu0.log 2>&1
fi
if [ -n "$FULL" ]; then
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tma/pytest_all.log 2>&1; echo "pytest all rc=$?"; tail -3 gpurun_out/tma/pytest_all.log
fi
