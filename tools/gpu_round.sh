set -x
for gm in 256 1024 4096 16384; do PBH_GRID_MIN=$gm timeout 600 python tools/probe_trace.py c1 fill > gpurun_out/trace_gm$gm.log 2>&1; done
tail -n 5 gpurun_out/trace_gm*.log | cut -c1-200
