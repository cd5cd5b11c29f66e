python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in "X=1" "TTN_GEMM_TMA=0"; do
  env $v TTN_HOST_PROF=1 timeout 300 python bench.py --config 5 --steps 1 --warmup 3 --workers 1 --no-cpu-baseline --no-showcase --no-e2e > gpurun_out/hp_$v.json 2> gpurun_out/hp_$v.err
  echo "== $v"; python -c "import json;d=json.loads(open('gpurun_out/hp_$v.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'])"
  python - "$v" <<'PY'
import sys,re,collections
acc=collections.Counter(); n=collections.Counter()
for l in open(f"gpurun_out/hp_{sys.argv[1]}.err"):
    m=re.match(r"\s*\[host\] (\S+)\s+([\d.]+) ms",l)
    if m: acc[m.group(1)]+=float(m.group(2)); n[m.group(1)]+=1
for k,v in acc.most_common(): print(f"  {k:20s} {v:10.1f} ms total over {n[k]} dumps")
PY
done
