#!/bin/bash
# ncu --set full of zgemm launches with TMA staging on / off (TTN_GEMM_TMA): raw and source-page
# CSV only, the reports are deleted on the box.  C=config SKIP=launches to skip CNT=launches
mkdir -p gpurun_out/tma
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/tma/build.log 2>&1 || { tail -30 gpurun_out/tma/build.log; exit 1; }
for t in 1 0; do
  TTN_GEMM_TMA=$t timeout 900 ncu --set full --import-source on --clock-control none -k regex:zgemm_grouped -s ${SKIP:-60} -c ${CNT:-12} -o /tmp/ncu_tma$t -f python bench.py --config ${C:-3} --steps 1 --warmup 3 > gpurun_out/tma/ncu$t.log 2>&1
  ncu -i /tmp/ncu_tma$t.ncu-rep --page raw --csv > gpurun_out/tma/ncu_c${C:-3}_tma$t.csv 2>/dev/null
  ncu -i /tmp/ncu_tma$t.ncu-rep --page source --csv --print-source sass > gpurun_out/tma/ncu_src_c${C:-3}_tma$t.csv 2>/dev/null
  gzip -f gpurun_out/tma/ncu_src_c${C:-3}_tma$t.csv
done
