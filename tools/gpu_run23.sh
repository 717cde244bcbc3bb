timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/r02_gputest3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gputest3.log
tail -3 gpurun_out/r02_gputest3.log
PBH_PROF=1 timeout 300 python tools/probe_c4.py --ds 32,1024,65536 --c1 20000 2>&1 | grep "cfg\|jobprof\[run_ops"
timeout 300 python tools/probe_sssp.py threshold grid 4096
timeout 300 python tools/probe_sssp.py exact grid 4096
