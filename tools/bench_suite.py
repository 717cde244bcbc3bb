#!/usr/bin/env python
"""Measure BASELINE configs C1-C4 on one B200 next to the reference CPU path.

Writes one JSON object (stdout) with a record per config. Device numbers use
the library's CUDA-event timing with inputs resident in HBM; the CPU numbers
run the unmodified reference (oracle/_ref) on a bounded sample, stated in
each record. Development/reporting tool — bench.py is the contract.

usage: python tools/bench_suite.py [c1 c2 c3 c4] [--c1-ops N] [--c4-n LOG2]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1908_09378_b200 as P  # noqa: E402
from paper_1908_09378_b200 import gen  # noqa: E402

PEAK = 6542.1
try:
    PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except (OSError, KeyError, ValueError):
    pass


def ref():
    from oracle import oracle as O
    return O if O.ref_available() else None


def c1(n_ops, cpu_ops):
    tr = gen.mixed_trace(n_ops, 1 << 20, 1024, 1)
    n_el = len(tr.vals)
    n_x = int(np.count_nonzero(tr.kinds == ord("E")))
    eng = P.Engine(P.EngineConfig(d=1024, debug_assertions=False, key_universe=1 << 20))
    t0 = time.time()
    r = eng.run_trace(tr)
    host_s = time.time() - t0
    ms = r.metrics.wall_ms
    rec = {"config": "C1 op trace", "n_ops": tr.n_ops, "update_elements": n_el, "extracts": n_x,
           "device_ms": ms, "host_s": host_s, "us_per_op": ms * 1e3 / tr.n_ops,
           "updates_per_s": n_el / (ms / 1e3),
           "roofline_frac": 24 * (n_el + n_x) / (ms / 1e3) / 1e9 / PEAK,
           "levels": len(r.metrics.resolves_per_level)}
    O = ref()
    if O is not None:
        # reference Engine::run_trace on the first cpu_ops ops (bounded sample)
        k = min(cpu_ops, tr.n_ops)
        sub = O.Trace(tr.kinds[:k], tr.offsets[:k + 1], tr.vals[:tr.offsets[k]],
                      tr.prios[:tr.offsets[k]])
        t0 = time.time()
        _, _, m = O.ref_run_trace(sub, 1024, workers=1, debug=False)
        s = time.time() - t0
        rec["cpu_reference"] = {"sample_ops": k, "update_elements": int(tr.offsets[k]),
                                "seconds": s, "updates_per_s": int(tr.offsets[k]) / s,
                                "us_per_op": s * 1e6 / k, "cores": 1}
        # parity on the same prefix through the device
        e2 = P.Engine(P.EngineConfig(d=1024, debug_assertions=False, key_universe=1 << 20))
        got = e2.run_trace(sub)
        want_v, want_p = O.run_oracle(sub)
        rec["parity_prefix"] = bool(np.array_equal(got.extracted_values, want_v) and
                                    np.array_equal(got.extracted_priorities, want_p))
    return rec


def sssp_rec(name, g, cpu_graph_fn):
    ctx = P.SsspContext(g, device=0, max_sources=1)
    ms = [ctx.run([0]) for _ in range(2)]
    r = ctx.fetch(0, settled=False)
    ctx.close()
    V, E = g.vertex_count, g.edge_count
    reached = int(np.count_nonzero(r.dist != np.uint64(P.K_INF_DIST)))
    alg = 8 * E + 8 * (V + 1) + 12 * reached
    rec = {"config": name, "V": V, "E": E, "device_ms": ms[-1], "rounds": r.rounds,
           "ns_per_round": ms[-1] * 1e6 / r.rounds, "edges_per_s": E / (ms[-1] / 1e3),
           "roofline_frac": alg / (ms[-1] / 1e3) / 1e9 / PEAK,
           "checksum": P.distance_checksum(r.dist)}
    O = ref()
    if O is not None and cpu_graph_fn is not None:
        sg, label = cpu_graph_fn()
        t0 = time.time()
        rr = O.ref_sssp(sg, 0, "par", debug=False)
        s = time.time() - t0
        rec["cpu_reference"] = {"sample": label, "seconds": s, "edges_per_s": sg.E / s, "cores": 1,
                                "rounds": rr["rounds"]}
    return rec


def thr_rec(name, g, heap_ms=None):
    """Threshold multi-extraction mode (extension)."""
    ctx = P.SsspContext(g, device=0, max_sources=1, mode="threshold")
    ms = [ctx.run([0]) for _ in range(2)]
    r = ctx.fetch(0, settled=False)
    ctx.close()
    V, E = g.vertex_count, g.edge_count
    rec = {"config": name, "device_ms": ms[-1], "batches": r.rounds,
           "vertices_per_batch": V / max(r.rounds, 1), "edges_per_s": E / (ms[-1] / 1e3),
           "checksum": P.distance_checksum(r.dist)}
    if heap_ms:
        rec["exact_heap_device_ms"] = heap_ms
        rec["speedup_over_exact"] = heap_ms / ms[-1]
    return rec


def bf_rec(name, g, heap_ms=None):
    """Device Bellman-Ford (frontier sweep) on the same graph as a heap config
    (heap vs sweep on dense high-diameter graphs)."""
    r, scanned, ms = P.bellman_ford(g, 0, with_parent=False)
    E = g.edge_count
    rec = {"config": name, "device_ms": ms, "frontier_iterations": r.rounds,
           "edges_scanned": scanned, "scan_over_E": scanned / max(E, 1),
           "edges_per_s": E / (ms / 1e3), "checksum": P.distance_checksum(r.dist)}
    if heap_ms:
        rec["heap_device_ms"] = heap_ms
        rec["heap_speedup_over_bf"] = ms / heap_ms
    return rec


def c4(log2n, ds, batches_per_d):
    n = 1 << log2n
    pr = gen.sweep_prefill(n, 4)
    out = []
    for d in ds:
        pr_d = pr.copy()
        vals_pre = np.arange(n, dtype=np.uint32)
        kinds = np.full((n + d - 1) // d, ord("B"), np.uint8)
        offs = np.minimum(np.arange(len(kinds) + 1, dtype=np.uint64) * d, n)
        eng = P.Engine(P.EngineConfig(d=d, debug_assertions=False, key_universe=n))

        class T:
            pass
        t = T()
        t.kinds, t.offsets, t.vals, t.prios = kinds, offs, vals_pre, pr_d
        t0 = time.time()
        eng.run_trace(t)
        pre_s = time.time() - t0
        v, p = gen.sweep_batches(n, d, batches_per_d(d), 5, pr_d)
        nb = len(v) // d
        t.kinds = np.full(nb, ord("B"), np.uint8)
        t.offsets = np.arange(nb + 1, dtype=np.uint64) * d
        t.vals, t.prios = v, p
        r = eng.run_trace(t)
        ms = r.metrics.wall_ms
        rec = {"config": "C4 bulkUpdate sweep", "heap_keys": n, "d": d, "batches": nb,
               "updates": len(v), "device_ms": ms, "updates_per_s": len(v) / (ms / 1e3),
               "us_per_batch": ms * 1e3 / max(nb, 1),  # latency metric for small d
               "roofline_frac": 24 * len(v) / (ms / 1e3) / 1e9 / PEAK, "prefill_s": pre_s,
               "levels": len(r.metrics.resolves_per_level)}
        out.append(rec)
        print(json.dumps(rec), file=sys.stderr, flush=True)
        eng.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", nargs="*", default=["c1", "c2", "c3", "c4"])
    ap.add_argument("--c1-ops", type=int, default=200_000)
    ap.add_argument("--c1-cpu-ops", type=int, default=2000)
    ap.add_argument("--c4-n", type=int, default=22)
    ap.add_argument("--c4-ds", default="32,1024,65536")
    args = ap.parse_args()
    res = {}
    if "c1" in args.which:
        res["c1"] = c1(args.c1_ops, args.c1_cpu_ops)
        print(json.dumps(res["c1"]), file=sys.stderr, flush=True)
    if "c3" in args.which:
        g = gen.band(1 << 20, 256, 2)
        res["c3"] = sssp_rec("C3 band SSSP (single source)", g, lambda: (
            __import__("oracle.oracle", fromlist=["x"]).Graph(g.vertex_count, g.offsets, g.targets, g.weights),
            "full C3 graph, 1 thread"))
        print(json.dumps(res["c3"]), file=sys.stderr, flush=True)
        del g
    if "c2" in args.which:
        g = gen.grid(4096, 4096, 1)

        def small():
            O = ref()
            return O.gen_grid(1024, 1024, 1), "1024x1024 grid (1/16 of C2), 1 thread"
        res["c2"] = sssp_rec("C2 grid SSSP", g, small)
        print(json.dumps(res["c2"]), file=sys.stderr, flush=True)
        del g
    if "thr" in args.which:
        g = gen.band(1 << 20, 256, 2)
        res["thr_c3"] = thr_rec("threshold mode on the C3 band", g,
                                res.get("c3", {}).get("device_ms"))
        print(json.dumps(res["thr_c3"]), file=sys.stderr, flush=True)
        del g
        g = gen.grid(4096, 4096, 1)
        res["thr_c2"] = thr_rec("threshold mode on the C2 grid", g,
                                res.get("c2", {}).get("device_ms"))
        print(json.dumps(res["thr_c2"]), file=sys.stderr, flush=True)
        del g
    if "bf" in args.which:
        g = gen.band(1 << 20, 256, 2)
        res["bf_c3"] = bf_rec("Bellman-Ford on the C3 band", g,
                              res.get("c3", {}).get("device_ms"))
        print(json.dumps(res["bf_c3"]), file=sys.stderr, flush=True)
        del g
        g = gen.grid(4096, 4096, 1)
        res["bf_c2"] = bf_rec("Bellman-Ford on the C2 grid", g,
                              res.get("c2", {}).get("device_ms"))
        print(json.dumps(res["bf_c2"]), file=sys.stderr, flush=True)
        del g
    if "c4" in args.which:
        ds = [int(x) for x in args.c4_ds.split(",")]
        res["c4"] = c4(args.c4_n, ds, lambda d: max(1, min((1 << 22) // d, 4096)))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
