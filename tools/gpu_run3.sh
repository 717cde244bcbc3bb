export PBH_PROF=1
timeout 600 python tools/probe_c4.py --ds 32,256,1024,8192,65536 --c1 20000 > gpurun_out/r02_prof_c4b.log 2>&1
cat gpurun_out/r02_prof_c4b.log
