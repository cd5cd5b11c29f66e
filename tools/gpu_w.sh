timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for w in 1 2 4; do for c in 5 3; do
timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --workers $w > gpurun_out/bw.json 2> gpurun_out/bw.err; echo "cfg $c workers $w rc=$?"; tail -2 gpurun_out/bw.err
python -c "
import json; d=json.load(open('gpurun_out/bw.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'])"
done; done
