# persistent single-op API: latency probe, then the whole GPU suite
export PYTHONPATH=.
timeout 600 python tools/probe_api.py --calls 2000 --pre 0,100000 2>&1 | tail -6
timeout 1500 python -m pytest -x -q -m gpu tests -p no:cacheprovider 2>&1 | tail -5
