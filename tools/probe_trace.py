"""Op-trace engine probe: time + per-level resolves/touches (development aid)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1908_09378_b200 as P
from paper_1908_09378_b200 import gen


def run(name, tr, d, universe):
    eng = P.Engine(P.EngineConfig(d=d, debug_assertions=False, key_universe=universe))
    r = eng.run_trace(tr)
    m = r.metrics
    n_el = len(tr.vals)
    print(json.dumps(dict(name=name, d=d, n_ops=int(tr.n_ops), n_el=n_el, wall_ms=m.wall_ms,
                          us_per_op=m.wall_ms * 1e3 / max(tr.n_ops, 1),
                          upd_per_s=n_el / max(m.wall_ms / 1e3, 1e-9),
                          resolves=list(m.resolves_per_level), touches=list(getattr(m, "touches_per_level", [])))),
          flush=True)
    eng.close()


which = sys.argv[1:] or ["c1", "fill"]
if "c1" in which:
    run("c1_20k", gen.mixed_trace(20000, 1 << 20, 1024, 1), 1024, 1 << 20)
if "fill" in which or "fill32" in which:
    for d in ((32,) if "fill32" in which else (32, 1024)):
        n = 1 << (16 if "fill32" in which else 20)
        pr = gen.sweep_prefill(n, 4)

        class T:
            pass
        t = T()
        t.kinds = np.full((n + d - 1) // d, ord("B"), np.uint8)
        t.n_ops = len(t.kinds)
        t.offsets = np.minimum(np.arange(len(t.kinds) + 1, dtype=np.uint64) * d, n)
        t.vals = np.arange(n, dtype=np.uint32)
        t.prios = pr
        run(f"prefill_2^20_d{d}", t, d, n)
