timeout 600 python -m pytest tests/test_gen.py -x -q 2>&1 | tail -15
timeout 300 python -c "
import sys, time; sys.path.insert(0, '.')
import torch
from paper_1908_09378_b200 import gen
g = gen.band_device(1 << 20, 256, 2); torch.cuda.synchronize()
t = time.time(); g = gen.band_device(1 << 20, 256, 2); torch.cuda.synchronize(); print('band_device C3 s', time.time() - t)
t = time.time(); gh = gen.band(1 << 20, 256, 2); print('band host C3 s', time.time() - t)
t = time.time(); g2 = gen.grid_device(4096, 4096, 1); torch.cuda.synchronize(); print('grid_device C2 s', time.time() - t)
"
