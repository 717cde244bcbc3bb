"""SSSP probe (development aid / ncu target): one solve of the chosen engine
on a grid or band graph.

usage: python tools/probe_sssp.py {exact,threshold,bf} {grid,band} [size] [reps]
  grid size = side (default 1024), band size = log2 V (default 16, degree 256)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1908_09378_b200 as P  # noqa: E402
from paper_1908_09378_b200 import gen  # noqa: E402

mode, shape = sys.argv[1], sys.argv[2]
size = int(sys.argv[3]) if len(sys.argv) > 3 else (1024 if shape == "grid" else 16)
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
g = gen.grid(size, size, 1) if shape == "grid" else gen.band(1 << size, 256, 2)
for _ in range(reps):
    if mode == "bf":
        r, scanned, ms = P.bellman_ford(g, 0, with_parent=False)
        rounds = r.rounds
    else:
        ctx = P.SsspContext(g, max_sources=1, mode="threshold" if mode == "threshold" else "exact")
        ms = ctx.run([0])
        r = ctx.fetch(0, settled=False)
        rounds = r.rounds
        ctx.close()
    print(json.dumps({"mode": mode, "shape": shape, "size": size, "V": g.vertex_count,
                      "E": g.edge_count, "ms": ms, "rounds": rounds,
                      "checksum": P.distance_checksum(r.dist)}), flush=True)
