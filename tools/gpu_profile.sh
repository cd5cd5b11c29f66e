#!/bin/bash
# round-2 ncu evidence (run under gpurun after the programs exit 0 without ncu):
#   launch lists (time + DRAM bytes per launch) of one step of configs 3 / 2 / 1, and a full
#   capture of the config-3 zgemm and tridiagonalisation kernels
set -x
mkdir -p gpurun_out
for c in ${PCONFIGS:-3 2 1}; do
  timeout 600 python tools/profile_step.py --config $c --steps 1 --skip 1 > gpurun_out/pstep_c$c.log 2>&1 || { tail gpurun_out/pstep_c$c.log; continue; }
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_r02_c$c.csv \
    python tools/profile_step.py --config $c --steps 1 --skip 1 > gpurun_out/ncu_c$c.log 2>&1
  echo "ncu c$c rc=$?"
done
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"zgemm_grouped|heev_tridiag" --launch-count 24 -o gpurun_out/prof_r02_c3 -f \
  python tools/profile_step.py --config 3 --steps 1 --skip 1 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
