#!/bin/bash
# short bench lines of every config (development; run under gpurun after tools/gpu_tests.sh)
for c in ${CONFIGS:-3 5 2 1 4}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-showcase --no-e2e > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/bench_c{c}.json").read().strip().splitlines()[-1])
    k = d["kernels"]
    print(f"config {c}: {d['value']:.2f} applies/s, {d['ms_per_step']:.2f} ms/step, zgemm frac {d['roofline']['frac']:.3f}, "
          + ", ".join(f"{n} {v['ms']:.1f}" for n, v in k.items() if isinstance(v, dict) and 'ms' in v))
except Exception as e:
    print(f"config {c}: failed {e}"); print(open(f"gpurun_out/bench_c{c}.err").read()[-2000:])
PY
done
