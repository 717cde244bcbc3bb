PBH_PROF=1 timeout 300 python tools/probe_c4.py --ds 1024,65536 2>&1 | grep "cfg\|jobprof\[run_ops"
