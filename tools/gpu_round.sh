timeout 600 python -m pytest tests/test_sssp_gpu.py -x -q 2>&1 | tail -1
timeout 300 python tools/probe.py band_small band band64 grid_small 2>&1 | grep -o '"name": "[a-zA-Z0-9_^]*"\|"ns_per_round": [0-9.]*'
