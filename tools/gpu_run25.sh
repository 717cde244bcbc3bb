PBH_PROF=1 timeout 300 python tools/probe_c4.py --ds 32 --c1 20000 2>&1 | grep "cfg\|run_ops\]\|run_trace\]\|jobprof\[run_ops\|jobprof\[run_trace"
