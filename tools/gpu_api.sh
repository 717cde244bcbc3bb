# A/B of the grid-merge threshold (2048 vs 1280 / 4096) and the bulk-store tile minimum (1024 vs 640), interleaved
export PYTHONPATH=.
for r in 1 2; do
  for v in base gm1280 gm4096 bs640; do
    cp variants/lib_$v.so paper_1908_09378_b200/libpbh_gpu.so
    timeout 300 python tools/probe_c4.py --ds 32,1024,65536 --c1 100000 2>&1 | grep cfg | python -c "
import sys, json
out=[]
for l in sys.stdin:
    d=json.loads(l); out.append('%s=%.3f' % (d['cfg']+str(d.get('d','')), d.get('us_per_batch', d.get('us_per_op', 0))))
print('$v', ' '.join(out))"
  done
done
cp variants/lib_base.so paper_1908_09378_b200/libpbh_gpu.so
