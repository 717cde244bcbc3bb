timeout 900 python -m pytest tests/test_sssp_threshold_gpu.py tests/test_sssp_gpu.py tests/test_full_size_gpu.py -q -x -k "not c1 and not c4" -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/probe_sssp.py threshold grid 4096
timeout 300 python tools/probe_sssp.py threshold grid 1024
