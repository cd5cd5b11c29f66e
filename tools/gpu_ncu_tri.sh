mkdir -p gpurun_out
Q="python bench.py --config 3 --quick --steps 1 --warmup 1"
for r in 1 2; do TTN_TRI_ROWS=$r timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/tri_r$r.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/tri_r$r.json')); print('rows $r', d['value'], d['kernels']['heev']['ms'])"; done
TTN_TRI_ROWS=1 timeout 300 $Q > gpurun_out/quick3.log 2>&1 && \
TTN_TRI_ROWS=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:heev_tridiag -c 10 -o gpurun_out/prof_tri $Q > gpurun_out/ncu_tri.log 2>&1; echo "ncu rc=$?"
