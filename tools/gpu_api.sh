# A/B: threshold engine's B_0 capacity (6/8 of level 0 = base, 7/8, 5/8) on the grid, interleaved; then parity
export PYTHONPATH=.
cp paper_1908_09378_b200/libpbh_gpu.so variants/lib_base.so
for r in 1 2; do
  for v in base mb7 mb5; do
    cp variants/lib_$v.so paper_1908_09378_b200/libpbh_gpu.so
    timeout 300 python tools/probe_sssp.py threshold grid 2048 1 2>&1 | tail -n1 | cut -c1-160 | sed "s/^/$v /"
  done
done
for v in mb7 mb5; do
  cp variants/lib_$v.so paper_1908_09378_b200/libpbh_gpu.so
  timeout 900 python -m pytest -x -q tests/test_sssp_threshold_gpu.py 2>&1 | tail -n1 | sed "s/^/$v /"
done
cp variants/lib_base.so paper_1908_09378_b200/libpbh_gpu.so
