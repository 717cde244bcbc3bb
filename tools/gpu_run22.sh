cp variants/lib_mprof.so paper_1908_09378_b200/libpbh_gpu.so
PBH_PHASES=1 timeout 300 python tools/probe_sssp.py threshold grid 1024 2>&1 | tail -3
PBH_PHASES=1 timeout 300 python tools/probe_sssp.py threshold grid 4096 2>&1 | tail -3
