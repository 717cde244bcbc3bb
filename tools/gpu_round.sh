PBH_PHASES=1 timeout 300 python tools/probe.py band_small 2>&1 | grep "bank phases" | tail -4 | cut -c1-250
