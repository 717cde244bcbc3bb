"""Quick performance probe across the BASELINE shapes (development aid)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1908_09378_b200 as P
from paper_1908_09378_b200 import gen

def t_sssp(name, g, sources, reps=1):
    ctx = P.SsspContext(g, device=0, max_sources=len(sources))
    ms = [ctx.run(sources) for _ in range(reps)]
    r = ctx.fetch(0, settled=False)
    ctx.close()
    E = g.edge_count
    res = dict(name=name, V=g.vertex_count, E=E, n_src=len(sources), ms=ms, rounds=r.rounds,
               ns_per_round=ms[-1] * 1e6 / max(r.rounds, 1),
               edges_per_s=len(sources) * E / (ms[-1] / 1e3), ops=r.ops)
    print(json.dumps(res), flush=True)

which = sys.argv[1:] or ["band_small", "band", "band64", "grid_small", "trace"]
if "band_tiny" in which:
    g = gen.band(1 << 12, 256, 2); t_sssp("band_2^12", g, [0], 1)
if "grid_tiny" in which:
    g = gen.grid(64, 64, 1); t_sssp("grid_64", g, [0], 1)
if "band_small" in which:
    g = gen.band(1 << 16, 256, 2); t_sssp("band_2^16", g, [0], 2)
if "band" in which:
    g = gen.band(1 << 20, 256, 2); t_sssp("band_C3", g, [0], 2)
    if "band64" in which:
        t_sssp("band_C5x64", g, [(i * 16384) % (1 << 20) for i in range(64)], 2)
if "grid_small" in which:
    g = gen.grid(512, 512, 1); t_sssp("grid_512", g, [0], 2)
if "grid" in which:
    g = gen.grid(4096, 4096, 1); t_sssp("grid_C2", g, [0], 1)
if "trace" in which:
    for n, k in [(20000, 1024)]:
        tr = gen.mixed_trace(n, 1 << 20, k, 1)
        eng = P.Engine(P.EngineConfig(d=k, debug_assertions=False, key_universe=1 << 20))
        t = time.time(); r = eng.run_trace(tr); w = time.time() - t
        print(json.dumps(dict(name=f"trace_{n}_{k}", n_ops=tr.n_ops, n_el=len(tr.vals), wall_ms=r.metrics.wall_ms, host_s=w,
                              us_per_op=r.metrics.wall_ms * 1e3 / tr.n_ops, upd_per_s=len(tr.vals) / (r.metrics.wall_ms / 1e3),
                              levels=len(r.metrics.resolves_per_level))), flush=True)
