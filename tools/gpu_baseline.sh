#!/bin/bash
# session start: build, GPU tests, bench lines of every config (run under gpurun)
set -x
mkdir -p gpurun_out/base
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/base/build.log 2>&1 || { tail -30 gpurun_out/base/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/base/pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/base/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/base/bench_c3.json 2> gpurun_out/base/bench_c3.err
for c in ${BCONFIGS:-1 2 4 5}; do
  timeout 600 python bench.py --config $c > gpurun_out/base/bench_c$c.json 2> gpurun_out/base/bench_c$c.err
done
tail -c 600 gpurun_out/base/bench_c*.json
