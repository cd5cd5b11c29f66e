#!/bin/bash
# ncu round trip (run under gpurun): launch list of one step of config $C, full capture of the
# kernels matching $KREGEX (up to $KCOUNT launches), summaries into gpurun_out/dev/
C=${C:-3}
mkdir -p gpurun_out/dev
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/dev/build.log 2>&1 || { tail -30 gpurun_out/dev/build.log; exit 1; }
timeout 600 python tools/profile_step.py --config $C --steps 1 --skip 1 > gpurun_out/dev/pstep.log 2>&1 || { tail gpurun_out/dev/pstep.log; exit 1; }
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/dev/launches_c$C.csv \
  python tools/profile_step.py --config $C --steps 1 --skip 1 > gpurun_out/dev/ncu_c$C.log 2>&1
echo "ncu list rc=$?"
python tools/ncu_summary.py launches gpurun_out/dev/launches_c$C.csv gpurun_out/dev/launches_c$C.md > /dev/null
head -30 gpurun_out/dev/launches_c$C.md
if [ -n "$KREGEX" ]; then
  timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"$KREGEX" --launch-count ${KCOUNT:-6} -o /tmp/prof_dev -f \
    python tools/profile_step.py --config $C --steps 1 --skip 1 > gpurun_out/dev/ncu_full.log 2>&1
  echo "ncu full rc=$?"
  python tools/ncu_summary.py full /tmp/prof_dev.ncu-rep gpurun_out/dev/ncu_full.md > gpurun_out/dev/ncu_sum.log 2>&1
  ncu -i /tmp/prof_dev.ncu-rep --page raw --csv > gpurun_out/dev/full_raw.csv 2>/dev/null
  ncu -i /tmp/prof_dev.ncu-rep --page source --csv > gpurun_out/dev/full_source.csv 2>/dev/null
  ncu -i /tmp/prof_dev.ncu-rep --page source --csv --print-source cuda > gpurun_out/dev/full_cuda.csv 2>/dev/null
  gzip -f gpurun_out/dev/full_raw.csv gpurun_out/dev/full_source.csv gpurun_out/dev/full_cuda.csv
  cat gpurun_out/dev/ncu_full.md | head -60
fi
