for v in base ipf; do echo "== $v"; cp variants/lib_$v.so paper_1908_09378_b200/libpbh_gpu.so
timeout 600 python tools/probe_trace.py c1 2>&1 | tail -1 | cut -c1-120
timeout 900 python tools/bench_suite.py c4 --c4-n 22 2>&1 >/dev/null | grep -o '"d": [0-9]*\|"us_per_batch": [0-9.]*' | paste - -
done
timeout 900 python -m pytest tests -m gpu -x -q -k "heap or trace or engine or smoke" 2>&1 | tail -2
