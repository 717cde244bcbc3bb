for ns in 64 256 1024; do echo "poll=$ns"; cp gpurun_out/lib_poll$ns.so paper_1908_09378_b200/libpbh_gpu.so
timeout 600 python tools/probe_trace.py c1 2>&1 | grep -o '"us_per_op": [0-9.]*'
timeout 900 python tools/bench_suite.py c4 --c4-n 24 --c4-ds 1024,65536 2>&1 >/dev/null | grep -o '"updates_per_s": [0-9.]*'
done
