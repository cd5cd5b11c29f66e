#!/bin/bash
# round-2 ncu evidence (run under gpurun after the programs exit 0 without ncu):
#   launch lists (time + DRAM bytes per launch) of one step of the configs, and a full capture
#   of the config-3 zgemm and tridiagonalisation kernels, summarised on the box (the raw
#   report is too big to bring back)
set -x
mkdir -p gpurun_out
for c in ${PCONFIGS:-3 2 1}; do
  timeout 600 python tools/profile_step.py --config $c --steps 1 --skip 1 > gpurun_out/pstep_c$c.log 2>&1 || { tail gpurun_out/pstep_c$c.log; continue; }
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_r02_c$c.csv \
    python tools/profile_step.py --config $c --steps 1 --skip 1 > gpurun_out/ncu_c$c.log 2>&1
  echo "ncu c$c rc=$?"
  python tools/ncu_summary.py launches gpurun_out/launches_r02_c$c.csv gpurun_out/launches_r02_c$c.md > /dev/null
  python tools/ncu_summary.py traffic gpurun_out/launches_r02_c$c.csv gpurun_out/ncu_zgemm_traffic_r02_c$c.md gpurun_out/ncu_zgemm_traffic_r02_c$c.json 1 > /dev/null
done
if [ -z "$NO_FULL" ]; then
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"zgemm_grouped|heev_tridiag" --launch-count 24 -o /tmp/prof_r02_c3 -f \
  python tools/profile_step.py --config 3 --steps 1 --skip 1 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
python tools/ncu_summary.py full /tmp/prof_r02_c3.ncu-rep gpurun_out/ncu_r02_c3_full.md > gpurun_out/ncu_sum.log 2>&1
ncu -i /tmp/prof_r02_c3.ncu-rep --page raw --csv > /tmp/raw.csv 2>/dev/null; gzip -c /tmp/raw.csv > gpurun_out/prof_r02_c3_raw.csv.gz
ls -la gpurun_out | head -40
fi
