mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_partition.py -x -q -m gpu > gpurun_out/pytest_part.log 2>&1; echo "pytest part rc=$?"; tail -15 gpurun_out/pytest_part.log
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pytest_gpu.log
