import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1908_09378_b200 as P
from paper_1908_09378_b200 import _lib
from oracle import oracle as O
for base in ["8192", "16384", "65536", "1048576"]:
    os.environ["PBH_SSSP_BASE1"] = base
    for name, g in [("complete3000", O.gen_complete(3000, 1000, 5)), ("random20k", O.gen_random(20000, 400000, 1000, 4)), ("complete1500", O.gen_complete(1500, 1000, 5)), ("random20kx100", O.gen_random(20000, 2000000, 1000, 6))]:
        l0 = _lib.lib().pbh_launch_count()
        try:
            r = P.par_dijkstra(g, 0)
            want = O.dijkstra(g, 0, 0)
            ok = np.array_equal(r.dist, want["dist"])
            print(base, name, "ok" if ok else "MISMATCH", "launches", _lib.lib().pbh_launch_count() - l0, flush=True)
        except Exception as e:
            print(base, name, "ERR", str(e)[:100], "launches", _lib.lib().pbh_launch_count() - l0, flush=True)
