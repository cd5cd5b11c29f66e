mkdir -p gpurun_out
TTN_HOST_PROF=1 timeout 600 python bench.py --config ${1:-3} --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-showcase > /dev/null 2> gpurun_out/hp$1.err; tail -16 gpurun_out/hp$1.err
