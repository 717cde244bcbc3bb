for v in lean5 sort3; do echo "== $v"; cp variants/lib_$v.so paper_1908_09378_b200/libpbh_gpu.so
PBH_PROF=1 timeout 600 python tools/probe_trace.py c1 2>&1 | tail -2 | cut -c1-250
timeout 300 python tools/probe.py grid_small 2>&1 | grep -o '"name": "[^"]*"\|"ns_per_round": [0-9.]*' | paste - -
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
