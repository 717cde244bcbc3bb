"""C4 / C1 op-engine probe (development aid): device time per batch of a
bulk_update sweep into a 2^LOG2N-key heap, and a C1 prefix; with PBH_PROF=1
the library prints the leader's cycle breakdown when each heap closes.

usage: python tools/probe_c4.py [--log2n 26] [--ds 32,1024,65536] [--batches N] [--c1 20000]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1908_09378_b200 as P  # noqa: E402
from paper_1908_09378_b200 import gen  # noqa: E402


class T:
    pass


def c4(log2n, d, batches):
    n = 1 << log2n
    pr = gen.sweep_prefill(n, 4)
    eng = P.Engine(P.EngineConfig(d=d, debug_assertions=False, key_universe=n))
    t = T()
    t.kinds = np.full((n + d - 1) // d, ord("B"), np.uint8)
    t.offsets = np.minimum(np.arange(len(t.kinds) + 1, dtype=np.uint64) * d, n)
    t.vals, t.prios = np.arange(n, dtype=np.uint32), pr.copy()
    pre = eng.run_trace(t).metrics.wall_ms
    nb = batches or max(1, (1 << 22) // d)
    v, p = gen.sweep_batches(n, d, nb, 5, pr)
    t.kinds = np.full(nb, ord("B"), np.uint8)
    t.offsets = np.arange(nb + 1, dtype=np.uint64) * d
    t.vals, t.prios = v, p
    m = eng.run_ops(t).metrics
    print(json.dumps({"cfg": "C4", "log2n": log2n, "d": d, "batches": nb, "prefill_ms": pre,
                      "ms": m.wall_ms, "us_per_batch": m.wall_ms * 1e3 / nb,
                      "updates_per_s": nb * d / (m.wall_ms / 1e3),
                      "resolves": m.resolves_per_level}), flush=True)
    eng.close()


def c1(n_ops):
    tr = gen.mixed_trace(n_ops, 1 << 20, 1024, 1)
    eng = P.Engine(P.EngineConfig(d=1024, debug_assertions=False, key_universe=1 << 20))
    m = eng.run_trace(tr).metrics
    print(json.dumps({"cfg": "C1", "n_ops": n_ops, "ms": m.wall_ms,
                      "us_per_op": m.wall_ms * 1e3 / n_ops, "resolves": m.resolves_per_level}),
          flush=True)
    eng.close()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2n", type=int, default=26)
    ap.add_argument("--ds", default="32,1024,65536")
    ap.add_argument("--batches", type=int, default=0)
    ap.add_argument("--c1", type=int, default=0)
    a = ap.parse_args()
    for d in [int(x) for x in a.ds.split(",") if x]:
        c4(a.log2n, d, a.batches)
    if a.c1:
        c1(a.c1)
