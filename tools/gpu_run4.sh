for v in nw8 nw16; do
  cp variants/lib_$v.so paper_1908_09378_b200/libpbh_gpu.so
  echo "== $v"
  timeout 600 python tools/probe_c4.py --ds 32,256,1024,8192,65536 --batches 0 --c1 20000 2>&1 | grep cfg
  timeout 600 python -m pytest tests/test_heap_gpu.py tests/test_heap_big_gpu.py -q -x 2>&1 | tail -2
done
