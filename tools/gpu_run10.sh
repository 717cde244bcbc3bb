PBH_PROF=1 timeout 300 python tools/probe_c4.py --ds 1024,65536 --c1 20000 2>&1 | grep "run_ops\|cfg\|C1\|jobprof"
