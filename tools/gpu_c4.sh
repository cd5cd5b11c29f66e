mkdir -p gpurun_out
timeout 300 ./tools/gemm_bench 3 > gpurun_out/gemm_bench.json 2>&1; echo "gemm_bench rc=$?"
timeout 900 python -m pytest tests -x -q -m gpu -k "large_gram or config4 or config3 or small_trees" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench4 rc=$?"; tail -5 gpurun_out/bench_c4.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c4.json')); print(d['value'], d['ms_per_step'], d['fp64_tflops_end_to_end'], d['roofline']['frac']); [print(k, round(v['ms'],1), v['launches'], v['tflops']) for k,v in d['kernels'].items()]"
