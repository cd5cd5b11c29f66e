# quick GPU iteration: gemm microbench, GPU parity tests, one bench line
mkdir -p gpurun_out
timeout 300 ./tools/gemm_bench 5 > gpurun_out/gemm_bench.json 2>&1; echo "gemm_bench rc=$?"; cat gpurun_out/gemm_bench.json | cut -c1-200
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_c3.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c3.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac']); [print(k, round(v['ms'],1), v['launches'], v['tflops']) for k,v in d['kernels'].items()]"
