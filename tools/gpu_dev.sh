#!/bin/bash
# development round trip (run under gpurun): build, the selected GPU tests, optional benches
#   TESTS="tests/test_gpu_heev.py"  BENCH="3 2"  BENCH_ARGS="--steps 5 --warmup 3"
mkdir -p gpurun_out/dev
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/dev/build.log 2>&1 || { tail -30 gpurun_out/dev/build.log; exit 1; }
if [ -n "$TESTS" ]; then
  timeout ${TEST_TIMEOUT:-900} python -m pytest $TESTS -x -q ${PYTEST_ARGS} > gpurun_out/dev/pytest.log 2>&1; echo "pytest rc=$?"
  tail -${TAILN:-25} gpurun_out/dev/pytest.log
fi
for c in $BENCH; do
  timeout 600 python bench.py --config $c ${BENCH_ARGS} > gpurun_out/dev/bench_c$c.json 2> gpurun_out/dev/bench_c$c.err
  echo "bench c$c rc=$?"
  python - <<PY
import json
d = json.load(open("gpurun_out/dev/bench_c$c.json"))
k = d.get("kernels", {})
print("c$c", round(d["value"], 2), "applies/s", round(d["ms_per_step"], 2), "ms/step frac", round(d["roofline"].get("frac", 0), 3),
      {a: round(b["ms"] / d["steps"], 2) for a, b in k.items() if isinstance(b, dict) and "ms" in b},
      "e2e", (d.get("e2e") or {}).get("value"))
PY
done
