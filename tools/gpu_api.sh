# A/B of the streamed-merge tile: 7 per thread, 5 per thread, 5 per thread with two staging tiles
export PYTHONPATH=.
for r in 1 2; do
  for v in vt7 vt5 vt5db; do
    cp variants/lib_$v.so paper_1908_09378_b200/libpbh_gpu.so
    timeout 300 python tools/probe_c4.py --ds 32,1024,65536 --c1 100000 2>&1 | grep cfg | python -c "
import sys, json
out=[]
for l in sys.stdin:
    d=json.loads(l); out.append('%s=%.3f' % (d['cfg']+str(d.get('d','')), d.get('us_per_batch', d.get('us_per_op', 0))))
print('$v', ' '.join(out))"
  done
done
cp variants/lib_vt5db.so paper_1908_09378_b200/libpbh_gpu.so
timeout 900 python -m pytest -x -q tests/test_heap_big_gpu.py tests/test_heap_gpu.py tests/test_persistent_gpu.py tests/test_acceptance_gpu.py 2>&1 | tail -3
