set -x
timeout 600 python -m pytest tests/test_bf_gpu.py -x -q > gpurun_out/pytest_bf.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_bf.log
timeout 1200 python tools/bench_suite.py c3 c2 bf > gpurun_out/suite_bf.json 2> gpurun_out/suite_bf.log
tail -n 5 gpurun_out/pytest_bf.log; tail -n 4 gpurun_out/suite_bf.log | cut -c1-400
