"""e2e breakdown of pbh_sssp_multi on the C5 shard (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1908_09378_b200 as P
from paper_1908_09378_b200 import gen
os.environ["PBH_E2E_PROF"] = "1"
g = gen.band(1 << 20, 256, 2)
srcs = [(i * 16384) % (1 << 20) for i in range(64)]
dist = np.zeros((64, 1 << 20), np.uint64)
parent = np.zeros((64, 1 << 20), np.uint32)
for pinned in (False, True):
    if pinned:
        P.pin(g.offsets, g.targets, g.weights, dist, parent)
    for rep in range(2):
        t = time.perf_counter()
        P.par_dijkstra_multi(g, srcs, devices=(0,), out=(dist, parent))
        print("pinned" if pinned else "pageable", "e2e s", time.perf_counter() - t, flush=True)
assert int(dist[0][(1 << 20) - 1]) == (1 << 20) - 1
