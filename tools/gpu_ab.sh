#!/bin/bash
# A/B runs of bench lines under environment knobs (development)
run() {  # name, config, extra args, env...
  local name=$1 c=$2 extra=$3; shift 3
  env "$@" timeout 600 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-showcase --no-e2e $extra > gpurun_out/ab_$name.json 2> gpurun_out/ab_$name.err
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{n}.json").read().strip().splitlines()[-1])
    print(f"{n}: {d['value']:.2f} applies/s, {d['ms_per_step']:.2f} ms/step, frac {d['roofline']['frac']:.3f}")
except Exception as e:
    print(n, "failed", e, open(f"gpurun_out/ab_{n}.err").read()[-800:])
PY
}
