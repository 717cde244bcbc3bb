# A/B: check + classify job with two elements per thread per step (cc2) vs one (base), interleaved; then parity
export PYTHONPATH=.
cp paper_1908_09378_b200/libpbh_gpu.so variants/lib_cc2.so
for r in 1 2; do
  for v in base cc2; do
    cp variants/lib_$v.so paper_1908_09378_b200/libpbh_gpu.so
    timeout 300 python tools/probe_c4.py --ds 8192,65536 --c1 0 2>&1 | grep cfg | python -c "
import sys, json
out=[]
for l in sys.stdin:
    d=json.loads(l); out.append('%s=%.3f' % (d['cfg']+str(d.get('d','')), d.get('us_per_batch', d.get('us_per_op', 0))))
print('$v', ' '.join(out))"
  done
done
cp variants/lib_cc2.so paper_1908_09378_b200/libpbh_gpu.so
timeout 900 python -m pytest -x -q tests/test_heap_big_gpu.py tests/test_heap_gpu.py tests/test_boundary_gpu.py 2>&1 | tail -3
