for v in gf2048; do echo "== $v"; cp variants/lib_$v.so paper_1908_09378_b200/libpbh_gpu.so
PBH_PROF=1 timeout 600 python tools/probe_trace.py c1 2>&1 | tail -2 | cut -c1-200
done
