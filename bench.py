#!/usr/bin/env python
"""pbh-b200 benchmark (contract: one JSON line from rank 0).

Workload (BASELINE.json configs[4], whose 1-GPU point contains configs[2]):
SSSP with the bucket-heap par_dijkstra on the dense high-diameter ring band
(V = 2^20, degree 256, weight-1 spine, seed 2), S = 64 independent sources
per GPU (weak scaling: rank r solves sources (i*16384 + 257*r) mod V).
A step = one batched solve of this rank's S sources; each source runs as one
persistent CTA of 4 warps (k_sssp_bank). value = edges relaxed by all ranks / max-over-ranks
device time. The single-source (configs[2]) latency-bound number is reported
in "single_source".

The line also carries "bulk_update": BASELINE C4 at d = 65536 into a
2^26-key heap (the other half of the metric), with its own roofline and the
reference's Engine::bulk_update timed on a sample ("cpu_baseline").

--impl reference times the reference's own CPU par_dijkstra
(oracle/_ref = /root/reference/proj/src compiled unmodified) on all host
threads for the same workload (bounded sample per step), rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

V_DEFAULT = 1 << 20
DEG_DEFAULT = 256


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="pbh", choices=["pbh", "reference"])
    ap.add_argument("--sources", type=int, default=64, help="sources per GPU")
    ap.add_argument("--v", type=int, default=V_DEFAULT)
    ap.add_argument("--deg", type=int, default=DEG_DEFAULT)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-bulk", action="store_true", help="skip the C4 bulk_update leg")
    ap.add_argument("--cpu-sample-sources", type=int, default=0,
                    help="sources in the CPU baseline sample (0 = one per host thread)")
    return ap.parse_args()


# ---------------------------------------------------------------- plumbing
class Dist:
    def __init__(self, n):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.backend = None
        self.device = self.local
        if self.world > 1:
            import torch
            import torch.distributed as dist
            n_dev = torch.cuda.device_count()
            if n_dev >= self.world:
                # one process per GPU; NCCL carries only the barrier and the
                # max-over-ranks of the timings (no collective on the data path)
                torch.cuda.set_device(self.local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
                self.backend = "nccl"
            else:
                # more ranks than GPUs (a functional check on a small box):
                # ranks share devices, timings reduce over gloo
                self.device = self.local % max(n_dev, 1)
                torch.cuda.set_device(self.device)
                dist.init_process_group("gloo")
                self.backend = "gloo"
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x):
        if not self.pg:
            return x
        import torch
        t = torch.tensor([float(x)], device="cuda" if self.backend == "nccl" else "cpu")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8 or f[0] != str(self.gpu):
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def sources_for(rank, S, V):
    return [(i * 16384 + 257 * rank) % V for i in range(S)]


def sssp_bytes(V, E_scanned, V_reached):
    """SURVEY.md §8d algorithmic bytes for one source: CSR read once
    (targets+weights 8 B/edge, offsets 8 B/vertex) + dist u64 and parent u32
    written once per reached vertex."""
    return 8 * E_scanned + 8 * (V + 1) + 12 * V_reached


def traffic_from_profiles():
    p = os.path.join(ROOT, "profiles", "ncu_k_sssp_summary.json")
    try:
        with open(p) as f:
            return json.load(f).get("dram_bytes_per_launch_per_source")
    except (OSError, ValueError):
        return None


# ------------------------------------------------------------- CPU arms
def cpu_reference_sample(g, sources, threads):
    """The reference's par_dijkstra (oracle/_ref) on host threads, one source
    per thread. Returns (seconds, edges)."""
    from oracle import oracle as O
    if not O.ref_available():
        return None
    og = O.Graph(g.vertex_count, g.offsets, g.targets, g.weights)
    t0 = time.perf_counter()
    O.ref_sssp_multi(og, sources, algo="par", threads=threads)
    return time.perf_counter() - t0


def run_reference_arm(args, D):
    if D.rank != 0:
        return
    from paper_1908_09378_b200 import gen
    g = gen.band(args.v, args.deg, 2)
    E = g.edge_count
    threads = os.cpu_count() or 1
    per_step = max(1, min(threads, args.sources))  # one source per host thread
    srcs = sources_for(0, args.sources, args.v)[:per_step]
    times = []
    for i in range(args.warmup + args.steps):
        s = cpu_reference_sample(g, srcs, per_step)
        if s is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
            return
        if i >= args.warmup:
            times.append(s)
    t = float(np.mean(times))
    value = per_step * E / t
    sample = f"{per_step} sources x full band SSSP per step on {per_step} threads"
    out = {
        "impl": "reference", "metric": "sssp_edges_relaxed_per_sec", "value": value,
        "unit": "edges/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic",
        "config": {"workload": "C5 per-GPU shard: multi-source par_dijkstra on C3 band",
                   "V": args.v, "E": E, "sources_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": per_step, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------- bulkUpdate leg
def bulk_update_leg(dev, peak, cpu=True, log2n=26, d=65536, n_batches=64):
    """BASELINE C4 at its largest batch: bulk_update batches of d distinct
    live keys (strict decreases) into a 2^26-key heap. Device time of the
    batches only (the prefill is not timed). Roofline: 24 B
    per update (key + priority read once, written once)."""
    import paper_1908_09378_b200 as P
    from paper_1908_09378_b200 import gen

    n = 1 << log2n
    pr = gen.sweep_prefill(n, 4)

    class T:
        pass
    t = T()
    t.kinds = np.full(n // d, ord("B"), np.uint8)
    t.offsets = np.arange(n // d + 1, dtype=np.uint64) * d
    t.vals = np.arange(n, dtype=np.uint32)
    t.prios = pr.copy()
    eng = P.Engine(P.EngineConfig(d=d, debug_assertions=False, key_universe=n, device=dev))
    eng.run_trace(t)  # prefill
    v, p = gen.sweep_batches(n, d, n_batches, 5, pr)
    t.kinds = np.full(n_batches, ord("B"), np.uint8)
    t.offsets = np.arange(n_batches + 1, dtype=np.uint64) * d
    t.vals, t.prios = v, p
    ms = eng.run_trace(t).metrics.wall_ms
    eng.close()
    ups = len(v) / (ms / 1e3)
    out = {"metric": "bulk_update_updates_per_sec", "value": ups, "unit": "updates/s",
           "config": {"workload": "BASELINE C4: bulk_update sweep into a 2^26-key heap",
                      "heap_keys": n, "d": d, "batches": n_batches, "updates": len(v)},
           "ms": ms,
           "roofline": {"bound": "hbm", "achieved": 24 * ups / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": 24 * ups / 1e9 / peak, "alg_bytes_per_update": 24,
                        "kernel": "k_trace_bank<4,8,4> + grid helpers (cooperative, 148 CTAs)"}}
    if cpu:
        from oracle import oracle as O
        if O.ref_available():
            # reference Engine::bulk_update on a 2^22-key sample, 16 batches
            ns = 1 << 22
            prs = gen.sweep_prefill(ns, 4)
            vs, ps = gen.sweep_batches(ns, d, 16, 5, prs.copy())
            secs = O.ref_bulk_sweep(d, np.arange(ns, dtype=np.uint32), prs, vs, ps)
            out["cpu_baseline"] = {"value": len(vs) / secs, "unit": "updates/s", "cores": 1,
                                   "kind": "reference",
                                   "sample": f"reference Engine::bulk_update, 2^22-key prefill, 16 batches of d={d}, {secs:.1f} s"}
    return out


# ------------------------------------------------------------- GPU arm
def main():
    args = parse()
    D = Dist(args.gpus)
    try:
        if args.impl == "reference":
            run_reference_arm(args, D)
            return
        run_pbh(args, D)
    finally:
        D.close()


def run_pbh(args, D):
    import paper_1908_09378_b200 as P
    from paper_1908_09378_b200 import _lib, gen

    dev = D.device
    t0 = time.time()
    g = gen.band(args.v, args.deg, 2)
    gen_s = time.time() - t0
    V, E = g.vertex_count, g.edge_count
    S = args.sources
    srcs = sources_for(D.rank, S, V)
    ctx = P.SsspContext(g, d=0, device=dev, max_sources=S)

    for _ in range(args.warmup):
        ctx.run(srcs)
    D.barrier()
    clocks = ClockSampler(dev)
    clocks.start()
    l0 = _lib.lib().pbh_launch_count()
    step_ms = []
    for _ in range(args.steps):
        D.barrier()
        step_ms.append(ctx.run(srcs))  # CUDA events on the launching stream
    D.barrier()
    launches = (_lib.lib().pbh_launch_count() - l0) // max(args.steps, 1)
    clk = clocks.stop()

    # parity spot checks on the timed output (size-independent properties)
    r0 = ctx.fetch(0, settled=False)
    reached = int(np.count_nonzero(r0.dist != np.uint64(P.K_INF_DIST)))
    ok_spine = srcs[0] != 0 or int(r0.dist[V - 1]) == V - 1
    tree = P.validate_parent_tree(g, srcs[0], r0.dist, r0.parent)
    rounds = r0.rounds
    e_scanned = E if reached == V else int(np.sum(np.diff(g.offsets)[r0.dist != np.uint64(P.K_INF_DIST)]))

    total_ms = D.max(float(np.sum(step_ms)))
    ms_per_step = total_ms / args.steps
    edges_per_step_all = D.world * S * e_scanned
    value = edges_per_step_all / (ms_per_step / 1e3)

    peak, peak_kind = peak_hbm()
    alg_bytes_launch = S * sssp_bytes(V, e_scanned, reached)
    achieved = alg_bytes_launch / (float(np.mean(step_ms)) / 1e3) / 1e9
    traffic_ps = traffic_from_profiles()

    # single source (configs[2]): latency-bound queue
    ms1 = [ctx.run(srcs[:1]) for _ in range(2)][-1]
    r1 = ctx.fetch(0, settled=False)
    single = {"edges_per_s": e_scanned / (ms1 / 1e3), "ms": ms1,
              "ns_per_round": ms1 * 1e6 / max(r1.rounds, 1), "rounds": r1.rounds,
              "roofline_frac": sssp_bytes(V, e_scanned, reached) / (ms1 / 1e3) / 1e9 / peak}

    # end-to-end through the public C-ABI with host buffers, every step: the
    # host CSR uploaded into the live context (pbh_sssp_ctx_load_graph, H2D),
    # the solve, and every source's dist + parent read back (D2H). The host
    # arrays are page-locked once outside the timed region; the context (its
    # per-source heaps) is the long-lived serving state.
    dist = np.zeros((S, V), np.uint64)
    parent = np.zeros((S, V), np.uint32)
    pinned = (g.offsets, g.targets, g.weights, dist, parent)
    P.pin(*pinned)

    def e2e_step():
        ctx.load_graph(g)
        ctx.run(srcs)
        for i in range(S):
            ctx.fetch_into(i, dist[i], parent[i])

    e2e_step()  # warm-up
    e2e_ms = []
    for _ in range(args.e2e_steps):
        D.barrier()
        t = time.perf_counter()
        e2e_step()
        e2e_ms.append((time.perf_counter() - t) * 1e3)
    P.unpin(*pinned)
    ctx.close()
    e2e_max = D.max(float(np.mean(e2e_ms)))
    e2e_ok = int(dist[0][V - 1]) == V - 1 if srcs[0] == 0 else True
    h2d = 8 * (V + 1) + 8 * E + 4 * S
    d2h = S * V * (8 + 4)

    cpu = None
    if D.rank == 0 and D.world == 1 and not args.no_cpu_baseline:
        threads = min(os.cpu_count() or 1, S)
        n_s = args.cpu_sample_sources or threads
        s = cpu_reference_sample(g, srcs[:n_s], threads)
        if s is not None:
            cpu = {"value": n_s * e_scanned / s, "unit": "edges/s", "cores": min(threads, n_s),
                   "kind": "reference",
                   "sample": f"reference par_dijkstra (oracle/_ref), {n_s} of the {S} sources, "
                             f"one per host thread, {s:.1f} s"}

    bulk = None
    if D.rank == 0 and not args.no_bulk:
        bulk = bulk_update_leg(dev, peak, cpu=(D.world == 1 and not args.no_cpu_baseline))

    if D.rank == 0:
        out = {
            "metric": "sssp_edges_relaxed_per_sec", "value": value, "unit": "edges/s",
            "n_gpus": D.world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": "BASELINE C5 shard per GPU: batched multi-source par_dijkstra, "
                                   f"{S} sources/GPU, on the C3 dense high-diameter band",
                       "V": V, "E": E, "degree": args.deg, "sources_per_gpu": S, "d": args.deg,
                       "graph_seed": 2, "l2": "inputs larger than L2 (CSR 2.15 GB)",
                       "parallelism": f"source-sharded x{D.world}, no collective on the data path"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind,
                         "traffic": (traffic_ps * S if traffic_ps else None),
                         "kernel": "k_sssp_bank<4,8,4,256> (one 128-thread CTA per source)",
                         "alg_bytes_per_launch": alg_bytes_launch},
            "cpu_baseline": cpu,
            "e2e": {"value": edges_per_step_all / (e2e_max / 1e3), "unit": "edges/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_max,
                    "api": "pbh_sssp_ctx_load_graph + pbh_sssp_ctx_run + pbh_sssp_ctx_fetch (host CSR in, host dist/parent out)"},
            "gpu_launches": int(launches),
            "clocks": clk,
            "single_source": single,
            "bulk_update": bulk,
            "parity": {"spine_dist": bool(ok_spine), "parent_tree": tree is None,
                       "reached": reached, "e2e_spine": bool(e2e_ok)},
            "gen_s": gen_s,
        }
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
