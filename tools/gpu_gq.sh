mkdir -p gpurun_out
./tools/gemm_bench 5 > gpurun_out/gemm_bench.json 2>&1; echo "gemm_bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/gemm_bench.json').read().split('err:')[0])
for c in d: print(c['case'][:42].ljust(42), '%.1e'%c['rel_err'], c['ms'], c['tflops'], c['cublas_tflops'])"
bash tools/gpu_quick.sh ${@:-3 4}
