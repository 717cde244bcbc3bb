for v in base aeo; do echo "== $v"; cp variants/lib_$v.so paper_1908_09378_b200/libpbh_gpu.so
timeout 300 python tools/probe.py band_small grid_small 2>&1 | grep -o '"name": "[^"]*"\|"ns_per_round": [0-9.]*' | paste - -
timeout 600 python tools/probe_trace.py c1 2>&1 | tail -1 | cut -c1-120
done
