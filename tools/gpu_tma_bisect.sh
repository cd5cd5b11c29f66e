#!/bin/bash
for f in "-DTCBC_TMA_FENCE" "-DTCBC_TMA_LOCKSTEP" ""; do
  echo "== flags '$f'"
  TCBC_NVCC_FLAGS="$f" python -c "import paper_2601_19650_b200._build as b; b.build(force=True)" > /tmp/b.log 2>&1 || { tail -5 /tmp/b.log; continue; }
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "config3_batch" 2>&1 | grep -E "passed|failed|AssertionError" | head -3
done
