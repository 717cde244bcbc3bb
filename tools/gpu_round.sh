timeout 900 python tools/ng_probe.py 2>&1 | tail -14
timeout 900 python -m pytest tests/test_sssp_gpu.py -x -q 2>&1 | tail -2
