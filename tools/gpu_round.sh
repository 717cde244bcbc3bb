set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 2400 python tools/bench_suite.py c1 c3 c4 --c4-n 26 --c4-ds 32,1024,65536 > gpurun_out/suite.json 2> gpurun_out/suite.log
tail -n 3 gpurun_out/pytest_gpu.log; cut -c1-300 gpurun_out/suite.log
