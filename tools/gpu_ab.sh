for r in 1 2; do
  for v in 0 1 2 3 5; do
    PBH_AB_OFF=$v timeout 300 python tools/probe_c4.py --ds 1024,65536 --c1 200000 2>&1 | grep cfg | python -c "
import sys, json
out=[]
for l in sys.stdin:
    d=json.loads(l); out.append('%s=%.3f' % (d['cfg']+str(d.get('d','')), d.get('us_per_batch', d.get('us_per_op', 0))))
print('$v', ' '.join(out))"
  done
done
