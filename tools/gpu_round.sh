set -x
timeout 600 python -m pytest tests/test_heap_gpu.py tests/test_sssp_gpu.py -x -q > gpurun_out/pytest_hs.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_hs.log
PBH_PROF=1 timeout 600 python tools/probe_trace.py c1 fill > gpurun_out/tprof.log 2>&1
timeout 300 python tools/probe.py band_small grid_small > gpurun_out/probe.log 2>&1
tail -n 3 gpurun_out/pytest_hs.log; cat gpurun_out/tprof.log gpurun_out/probe.log | cut -c1-300
