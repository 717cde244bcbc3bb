for v in base p128; do echo "== $v"; cp variants/lib_$v.so paper_1908_09378_b200/libpbh_gpu.so
timeout 300 python tools/probe.py band_small grid_small 2>&1 | grep -o '"name": "[^"]*"\|"ns_per_round": [0-9.]*' | paste - -
done
timeout 900 python -m pytest tests -m gpu -x -q -k "sssp or dijkstra or smoke" 2>&1 | tail -2
