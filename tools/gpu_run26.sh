for gm in 1024 2048 4096 8192; do
  echo "== grid_min $gm"
  PBH_GRID_MIN=$gm timeout 300 python tools/probe_c4.py --ds 256,1024,65536 --c1 20000 2>&1 | grep "cfg" | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], d.get('d'), round(d.get('us_per_batch', d.get('us_per_op', 0)),2))"
done
