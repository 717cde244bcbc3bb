set -x
timeout 900 python -m pytest tests/test_heap_big_gpu.py tests/test_heap_gpu.py -x -q > gpurun_out/pytest_big.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_big.log
tail -n 25 gpurun_out/pytest_big.log


