#!/usr/bin/env python
"""Full-size goldens for BASELINE configs C1, C2, C3, C5 (SURVEY.md §8c "New
goldens needed"), computed by the UNMODIFIED reference (oracle/_ref, built
from /root/reference/proj/src by `make -C oracle ref`).

Inputs are the §8d generators as restated in oracle/pbh_oracle.c (each graph
and the C1 trace is fingerprinted here, so a consumer can prove it fed the
same bytes; tests/test_gen.py pins the product's generators to the oracle's).

  C2  grid 4096x4096 seed 1, source 0:      reference_dijkstra + par_dijkstra
  C3  band V=2^20 deg 256 seed 2, source 0: reference_dijkstra + par_dijkstra
  C5  the C3 band, sources i*16384 (i < 64): reference_dijkstra + par_dijkstra
  C1  mixed trace 10^6 ops, universe 2^20, k<=1024, seed 1: the reference's
      run_oracle (tests/oracle.hpp:55-75) extraction sequence

Per SSSP source: distance_checksum (sssp.cpp:174-183), FNV-1a of the
settled_order bytes, n_settled, rounds and metrics.ops of par_dijkstra.
C1: FNV-1a of the extracted values' bytes followed by the priorities' bytes.

usage: python tests/golden/make_full_goldens.py [c1 c2 c3 c5] [--threads N]
Writes/updates tests/golden/full_size.json (small; committed).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

OUT = os.path.join(HERE, "full_size.json")
C5_SOURCES = [i * 16384 for i in range(64)]


def graph_fp(g):
    return O.fnv1a(g.off, g.tgt, g.w)


def sssp_golden(g, sources, threads):
    rg = O.RefGraph(g)
    t0 = time.time()
    ref = rg.sssp_batch(sources, "ref", threads=threads)
    par = rg.sssp_batch(sources, "par", threads=threads)
    rg.close()
    for k in ("dist_ck", "settled_ck", "n_settled"):
        assert np.array_equal(ref[k], par[k]), f"reference_dijkstra and par_dijkstra differ on {k}"
    return {
        "sources": [int(s) for s in sources],
        "dist_checksum": [int(x) for x in ref["dist_ck"]],
        "settled_checksum": [int(x) for x in ref["settled_ck"]],
        "n_settled": [int(x) for x in ref["n_settled"]],
        "rounds": [int(x) for x in par["rounds"]],
        "ops": [int(x) for x in par["ops"]],
        "ref_seconds": {"reference_dijkstra": ref["seconds"], "par_dijkstra": par["seconds"],
                        "threads": threads},
        "wall_s": time.time() - t0,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", nargs="*", default=["c2", "c3", "c5", "c1"])
    ap.add_argument("--threads", type=int, default=len(os.sched_getaffinity(0)))
    args = ap.parse_args()
    if not O.ref_available():
        O.ref()  # builds oracle/_ref from /root/reference when present
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    out["_about"] = ("Computed by tests/golden/make_full_goldens.py from the unmodified reference "
                     "(oracle/_ref). Checksums are FNV-1a 64 (sssp.cpp:174-183's hash).")

    def save():
        # merge with what another invocation may have written meanwhile
        cur = json.load(open(OUT)) if os.path.exists(OUT) else {}
        cur.update(out)
        with open(OUT + ".tmp", "w") as f:
            json.dump(cur, f, indent=1)
        os.replace(OUT + ".tmp", OUT)

    if "c2" in args.which:
        g = O.gen_grid(4096, 4096, 1)
        rec = sssp_golden(g, [0], 2)
        rec.update(V=g.V, E=g.E, graph_fnv=graph_fp(g), gen="grid(4096,4096,seed=1)")
        out["C2"] = rec
        save()
        print("C2", rec["dist_checksum"], rec["wall_s"], flush=True)
        del g
    if "c3" in args.which or "c5" in args.which:
        g = O.gen_band(1 << 20, 256, 2)
        fp = graph_fp(g)
        if "c3" in args.which:
            rec = sssp_golden(g, [0], 2)
            rec.update(V=g.V, E=g.E, graph_fnv=fp, gen="band(2^20,256,seed=2)")
            out["C3"] = rec
            save()
            print("C3", rec["dist_checksum"], rec["wall_s"], flush=True)
        if "c5" in args.which:
            rec = sssp_golden(g, C5_SOURCES, args.threads)
            rec.update(V=g.V, E=g.E, graph_fnv=fp, gen="band(2^20,256,seed=2)")
            out["C5"] = rec
            save()
            print("C5", rec["wall_s"], flush=True)
        del g
    if "c1" in args.which:
        t0 = time.time()
        tr = O.gen_mixed_trace(1_000_000, 1 << 20, 1024, 1)
        fp = O.fnv1a(tr.kinds, tr.offsets, tr.vals, tr.prios)
        gen_s = time.time() - t0
        v, p = O.ref_run_oracle(tr)
        # the C restatement's OracleHeap must agree with the reference's
        cv, cp = O.run_oracle(tr)
        assert np.array_equal(v, cv) and np.array_equal(p, cp), "restated run_oracle differs"
        out["C1"] = {"n_ops": int(tr.n_ops), "update_elements": int(len(tr.vals)),
                     "n_extract": int(len(v)), "trace_fnv": fp,
                     "extract_checksum": O.fnv1a(v, p),
                     "prefix_2000_checksum": O.fnv1a(v[:2000], p[:2000]),
                     # the trace is generated sequentially, so the first k ops
                     # are the whole trace of a k-op run: their extractions are
                     # a prefix of the full sequence
                     "op_prefixes": {str(k): {"n_extract": int(nx),
                                              "update_elements": int(tr.offsets[k]),
                                              "extract_checksum": O.fnv1a(v[:nx], p[:nx])}
                                     for k in (20_000, 100_000, 200_000, 500_000)
                                     for nx in [int(np.count_nonzero(tr.kinds[:k] == ord("E")))]},
                     "gen": "mixed_trace(1e6 ops, universe 2^20, kmax 1024, seed 1)",
                     "gen_s": gen_s, "wall_s": time.time() - t0}
        save()
        print("C1", out["C1"], flush=True)


if __name__ == "__main__":
    main()
