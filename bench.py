#!/usr/bin/env python
"""pbh-b200 benchmark (contract: one JSON line from rank 0).

Headline workload (BASELINE.json configs[4], "C5"): batched multi-source
par_dijkstra, the 64 sources s_i = i*16384 of SURVEY.md §8d on the C3 dense
high-diameter band (V = 2^20, degree 256, weight-1 spine, seed 2), split
contiguously over the N GPUs (64/N sources per GPU, one process per GPU).
Each source runs as one persistent 128-thread CTA (k_sssp_bank). A step =
one batched solve of every rank's shard. value = 64 * E_scanned / max over
ranks of the device time (CUDA events on the launching stream), inputs
resident in HBM (2.15 GB CSR > L2). scaling: "strong" (the 64 sources are
fixed); the weak-scaling point (64 sources per GPU) is reported as
"weak_scaling" when N > 1.

e2e: the same solve through the public C-ABI with host buffers, every step:
each rank uploads the host CSR into its live context (pbh_sssp_ctx_load_graph),
solves, and gathers its dist + parent rows into one buffer on GPU 0 over
NVLink (pbh_sssp_ctx_gather into CUDA-IPC-mapped memory, no collective);
GPU 0 then copies the gathered 64 x V results to the host. Two contexts per
rank alternate, so step i+1's upload (own stream) overlaps step i's solve;
e2e = wall time of the steps / steps (the first upload is exposed).

Also in the line (rank 0), each with parity against the reference's own
outputs (tests/golden/full_size.json, made by oracle/_ref from
/root/reference) and, where affordable, the reference CPU path timed here:
  c3   single source (configs[2]), ns per round
  c2   4096^2 grid (configs[1]), exact and threshold mode
  c1   mixed op trace (configs[0]), all 10^6 ops
  c4   bulkUpdate sweep d = 32..65536 into a 2^26-key heap (configs[3])
A parity mismatch makes the run exit non-zero after printing the line.

--impl reference times the reference's own CPU par_dijkstra (oracle/_ref =
/root/reference/proj/src compiled unmodified) on all host threads, on the
graph imported once outside the timed region, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

V_DEFAULT = 1 << 20
DEG_DEFAULT = 256
GOLDEN = os.path.join(ROOT, "tests", "golden", "full_size.json")


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="pbh", choices=["pbh", "reference"])
    ap.add_argument("--sources", type=int, default=64, help="C5 sources in total")
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--legs", default="c3,c2,c1,c4,api",
                    help="extra BASELINE configs measured on rank 0 (comma list, or 'none')")
    ap.add_argument("--c1-ops", type=int, default=1_000_000)
    ap.add_argument("--c4-ds", default="32,256,1024,8192,65536")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-sources", type=int, default=0,
                    help="sources per CPU-baseline sample (0 = one per host thread)")
    return ap.parse_args(argv)


# ---------------------------------------------------------------- plumbing
def host_info():
    cores = len(os.sched_getaffinity(0))
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "host_threads": cores}


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_spawn(args):
    """`bench.py --gpus N` outside torchrun: re-launch as N ranks (one
    process per GPU) through torch.distributed.run and return its exit code."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.backend = None
        self.device = self.local
        self.shared_devices = False
        if self.world > 1:
            import torch
            import torch.distributed as dist
            n_dev = torch.cuda.device_count()
            if n_dev >= self.world:
                # one process per GPU; NCCL carries only barriers, the IPC
                # handle of the gather buffer and the max-over-ranks timing
                torch.cuda.set_device(self.local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
                self.backend = "nccl"
            else:
                # more ranks than GPUs (a functional check on a small box):
                # ranks share devices, control traffic over gloo
                self.device = self.local % max(n_dev, 1)
                self.shared_devices = True
                if n_dev:
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

    def bcast(self, obj):
        if not self.pg:
            return obj
        box = [obj]
        self.pg.broadcast_object_list(box, src=0)
        return box[0]

    def gather_objs(self, obj):
        if not self.pg:
            return [obj]
        out = [None] * self.world
        self.pg.all_gather_object(out, obj)
        return out

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
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 7672.0, "fallback (B200_PROFILING.md nominal)"


def c5_sources(n=64):
    return [i * 16384 for i in range(n)]


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


def c4_traffic_from_profiles():
    p = os.path.join(ROOT, "profiles", "ncu_c4_summary.json")
    try:
        with open(p) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def golden():
    try:
        with open(GOLDEN) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def fnv(*arrays):
    from oracle import oracle as O  # checker only (FNV-1a, sssp.cpp:174-183's hash)
    return O.fnv1a(*arrays)


# ------------------------------------------------------------- CPU arms
def run_reference_arm(args, D):
    """The reference's par_dijkstra (oracle/_ref) on all host threads: the C5
    graph is generated with the oracle's generator and imported into the
    reference's CsrGraph ONCE; each step solves one source per host thread
    (rotating through the 64 C5 sources), timed around the solves only."""
    if D.rank != 0:
        return 0
    from oracle import oracle as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return 0
    hi = host_info()
    threads = hi["host_threads"]
    g = O.gen_band(V_DEFAULT, DEG_DEFAULT, 2)
    E = g.E
    rg = O.RefGraph(g)  # graph load: outside every timed region
    del g
    srcs = c5_sources(args.sources)
    per_step = args.cpu_sample_sources or min(threads, len(srcs))
    times, done, want = [], 0, golden().get("C5", {})
    match = True
    for i in range(args.warmup + args.steps):
        s = [srcs[(done + j) % len(srcs)] for j in range(per_step)]
        done += per_step
        r = rg.sssp_batch(s, "par", threads=threads)
        if want:
            for j, src in enumerate(s):
                k = want["sources"].index(src)
                match &= int(r["dist_ck"][j]) == want["dist_checksum"][k]
        if i >= args.warmup:
            times.append(r["seconds"])
    t = float(np.mean(times))
    value = per_step * E / t
    # the textbook CPU solver over all 64 sources once
    tb = rg.sssp_batch(srcs, "ref", threads=threads)
    rg.close()
    sample = (f"{per_step} of the {len(srcs)} C5 sources per step (rotating), one per host thread, "
              f"graph imported once outside the timed region")
    out = {
        "impl": "reference", "metric": "sssp_edges_relaxed_per_sec", "value": value,
        "unit": "edges/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic",
        "config": {"workload": "BASELINE C5: 64-source par_dijkstra on the C3 band "
                               "(reference CPU path, oracle/_ref)",
                   "V": V_DEFAULT, "E": E, "sources": len(srcs), "sources_per_step": per_step,
                   "l2": "n/a (host)"},
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": threads, "kind": "reference",
                         "sample": sample, **hi},
        "textbook_cpu_baseline": {"value": len(srcs) * E / tb["seconds"], "unit": "edges/s",
                                  "cores": threads, "kind": "reference",
                                  "sample": f"reference_dijkstra (sssp.cpp:71-97), all {len(srcs)} "
                                            f"sources, {tb['seconds']:.1f} s"},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "parity": {"C5_sample_vs_golden": bool(match) if want else None},
    }
    print(json.dumps(out), flush=True)
    return 0


# ------------------------------------------------------------- GPU legs
def leg_c3(P, g, ctx_dev, peak, want, cpu):
    """configs[2]: one source on the band (the latency-bound single queue)."""
    ctx = P.SsspContext(g, device=ctx_dev, max_sources=1)
    ms = [ctx.run([0]) for _ in range(3)]
    r = ctx.fetch(0, settled=True)
    ctx.close()
    V, E = g.vertex_count, g.edge_count
    t = float(np.median(ms))
    rec = {"edges_per_s": E / (t / 1e3), "ms": t, "rounds": r.rounds,
           "ns_per_round": t * 1e6 / max(r.rounds, 1),
           "roofline_frac": sssp_bytes(V, E, V) / (t / 1e3) / 1e9 / peak}
    if want:
        rec["parity"] = {"dist": P.distance_checksum(r.dist) == want["dist_checksum"][0],
                         "settled_order": fnv(r.settled_order) == want["settled_checksum"][0],
                         "rounds": r.rounds == want["rounds"][0], "ops": r.ops == want["ops"][0],
                         "parent_tree_optimal": P.validate_parent_tree(g, 0, r.dist, r.parent,
                                                                      optimal=True) is None}
        rec["match"] = all(rec["parity"].values())
    if cpu and want:
        rs = want.get("ref_seconds", {})
        rec["cpu_reference_container"] = {
            "note": "reference timings from the golden run (survey container), single thread",
            "par_dijkstra_s": rs.get("par_dijkstra"), "reference_dijkstra_s": rs.get("reference_dijkstra")}
    return rec


def leg_c2(P, gen, dev, peak, want, cpu):
    """configs[1]: 4096^2 grid, source 0: exact par_dijkstra, the opt-in
    threshold multi-extraction mode and the device Bellman-Ford; the textbook
    reference_dijkstra of the reference timed on one host thread."""
    g = gen.grid(4096, 4096, 1)
    V, E = g.vertex_count, g.edge_count
    ctx = P.SsspContext(g, device=dev, max_sources=1)
    ms = ctx.run([0])
    r = ctx.fetch(0, settled=True)
    rec = {"V": V, "E": E, "ms": ms, "edges_per_s": E / (ms / 1e3), "rounds": r.rounds,
           "ns_per_round": ms * 1e6 / max(r.rounds, 1),
           "roofline_frac": sssp_bytes(V, E, V) / (ms / 1e3) / 1e9 / peak}
    par = {}
    if want:
        par = {"dist": P.distance_checksum(r.dist) == want["dist_checksum"][0],
               "settled_order": fnv(r.settled_order) == want["settled_checksum"][0],
               "rounds": r.rounds == want["rounds"][0], "ops": r.ops == want["ops"][0],
               "parent_tree_optimal": P.validate_parent_tree(g, 0, r.dist, r.parent,
                                                            optimal=True) is None}
    ctx.set_mode("threshold")
    tms = ctx.run([0])
    rt = ctx.fetch(0, settled=False)
    ctx.close()
    rec["threshold_mode"] = {"ms": tms, "edges_per_s": E / (tms / 1e3), "batches": rt.rounds,
                             "speedup_over_exact": ms / tms}
    # the device Bellman-Ford frontier sweep (bellman_ford, sssp.hpp:37; the
    # reference's cross-check solver), timed on the device like the others
    rb, scanned, bms = P.bellman_ford(g, 0, device=dev, with_parent=False)
    rec["device_bellman_ford"] = {"ms": bms, "edges_scanned": scanned, "rounds": rb.rounds,
                                  "edges_per_s": E / (bms / 1e3)}
    if want:
        par["threshold_dist"] = P.distance_checksum(rt.dist) == want["dist_checksum"][0]
        par["bellman_ford_dist"] = P.distance_checksum(rb.dist) == want["dist_checksum"][0]
        rec["parity"] = par
        rec["match"] = all(par.values())
    if cpu:
        from oracle import oracle as O
        if O.ref_available():
            rg = O.RefGraph(O.Graph(V, g.offsets, g.targets, g.weights))
            tb = rg.sssp_batch([0], "ref", threads=1)
            rg.close()
            rec["cpu_textbook"] = {"value": E / tb["seconds"], "unit": "edges/s", "cores": 1,
                                   "kind": "reference", "seconds": tb["seconds"],
                                   "sample": "reference_dijkstra, full C2, 1 thread",
                                   "match": int(tb["dist_ck"][0]) == (want or {}).get("dist_checksum", [None])[0]}
            if want:
                rs = want.get("ref_seconds", {})
                rec["cpu_par_dijkstra_container_s"] = rs.get("par_dijkstra")
    return rec


def leg_c1(P, gen, dev, peak, n_ops, want, cpu):
    """configs[0]: the mixed bulkUpdate/extractMin trace (universe 2^20,
    k <= 1024, seed 1), all 10^6 ops by default (2.56e8 update elements;
    generating it takes ~70 s on the host, outside the timing), through
    run_trace (one submission + the closing drain); the extraction sequence
    is checked against the reference's run_oracle checksum."""
    tr = gen.mixed_trace(n_ops, 1 << 20, 1024, 1)
    n_el = len(tr.vals)
    n_x = int(np.count_nonzero(tr.kinds == ord("E")))
    eng = P.Engine(P.EngineConfig(d=1024, debug_assertions=False, key_universe=1 << 20, device=dev))
    r = eng.run_trace(tr)
    eng.close()
    ms = r.metrics.wall_ms
    rec = {"n_ops": n_ops, "update_elements": n_el, "extracts": n_x, "ms": ms,
           "us_per_op": ms * 1e3 / n_ops, "updates_per_s": n_el / (ms / 1e3),
           "roofline_frac": 24 * (n_el + n_x) / (ms / 1e3) / 1e9 / peak}
    want = want or {}
    pre = ({"n_extract": want["n_extract"], "extract_checksum": want["extract_checksum"]}
           if want.get("n_ops") == n_ops else want.get("op_prefixes", {}).get(str(n_ops)))
    if pre:
        rec["parity"] = {"extractions": len(r.extracted_values) == pre["n_extract"] and
                         fnv(r.extracted_values, r.extracted_priorities) == pre["extract_checksum"]}
        rec["match"] = rec["parity"]["extractions"]
    if cpu:
        from oracle import oracle as O
        if O.ref_available():
            k = 2000
            sub = O.Trace(tr.kinds[:k], tr.offsets[:k + 1], tr.vals[:tr.offsets[k]],
                          tr.prios[:tr.offsets[k]])
            t0 = time.time()
            O.ref_run_trace(sub, 1024, workers=1, debug=False)
            s = time.time() - t0
            rec["cpu_baseline"] = {"value": int(tr.offsets[k]) / s, "unit": "updates/s", "cores": 1,
                                   "kind": "reference", "us_per_op": s * 1e6 / k,
                                   "sample": f"reference Engine::run_trace, first {k} ops"}
    return rec


def leg_c4(P, gen, dev, peak, ds, cpu):
    """configs[3]: bulk_update sweep into a 2^26-key heap. Per d: prefill 2^26
    fresh keys (not timed), then >= 2^24 updates (strict decreases of random
    live keys, key-sorted batches of d), device time of the batches. Parity
    (size-independent): live_size == 2^26 and the first extractions equal the
    (priority, key) order of the priorities numpy recomputes from the batches."""
    n = 1 << 26
    pr0 = gen.sweep_prefill(n, 4)
    recs = []
    ok_all = True

    class T:
        pass
    for d in ds:
        pr = pr0.copy()
        eng = P.Engine(P.EngineConfig(d=d, debug_assertions=False, key_universe=n, device=dev))
        t = T()
        t.kinds = np.full((n + d - 1) // d, ord("B"), np.uint8)
        t.offsets = np.minimum(np.arange(len(t.kinds) + 1, dtype=np.uint64) * d, n)
        t.vals, t.prios = np.arange(n, dtype=np.uint32), pr.copy()
        t0 = time.time()
        eng.run_trace(t)
        pre_s = time.time() - t0
        nb = max(1, (1 << 24) // d)
        v, p = gen.sweep_batches(n, d, nb, 5, pr)  # pr: priorities after the batches
        t.kinds = np.full(nb, ord("B"), np.uint8)
        t.offsets = np.arange(nb + 1, dtype=np.uint64) * d
        t.vals, t.prios = v, p
        # the batches as a caller's bulk_update loop (no closing drain), like
        # the reference's timed Engine::bulk_update calls
        ms = eng.run_ops(t).metrics.wall_ms
        ups = len(v) / (ms / 1e3)
        rec = {"d": d, "batches": nb, "updates": len(v), "ms": ms, "updates_per_s": ups,
               "us_per_batch": ms * 1e3 / nb, "prefill_s": pre_s,
               "roofline": {"achieved_gbs": 24 * ups / 1e9, "frac": 24 * ups / 1e9 / peak,
                            "alg_bytes_per_update": 24}}
        tr = c4_traffic_from_profiles()
        if tr and tr.get("d") == d:
            # DRAM bytes per update from the committed ncu capture of this
            # configuration (cold caches), next to the structural cascade model
            rec["roofline"]["traffic_bytes_per_update"] = tr["dram_bytes_per_update"]
            rec["roofline"]["traffic_source"] = tr["source"]
            rec["roofline"]["structural_bytes_per_update"] = tr["structural_bytes_per_update"]
        # parity: extract a prefix and compare with numpy's (p_now, key) order
        m = 1_000_000 if d == ds[-1] else 10_000
        thr = np.partition(pr, m)[m]
        cand = np.nonzero(pr <= thr)[0]
        order = cand[np.lexsort((cand, pr[cand]))][:m]
        t.kinds = np.full(m, ord("E"), np.uint8)
        t.offsets = np.zeros(m + 1, np.uint64)
        t.vals, t.prios = np.zeros(0, np.uint32), np.zeros(0, np.uint64)
        live = eng.live_size()
        xr = eng.run_trace(t)
        ok = (live == n and np.array_equal(xr.extracted_values, order.astype(np.uint32)) and
              np.array_equal(xr.extracted_priorities, pr[order]))
        rec["parity"] = {"live_size": live == n, "extract_prefix": int(m), "match": bool(ok)}
        rec["extract_us_per_op"] = xr.metrics.wall_ms * 1e3 / m
        ok_all &= bool(ok)
        eng.close()
        recs.append(rec)
    out = {"heap_keys": n, "sweep": recs, "match": ok_all}
    if cpu:
        from oracle import oracle as O
        if O.ref_available():
            ns = 1 << 22
            cb = {}
            for d in (ds[0], ds[-1]):
                prs = gen.sweep_prefill(ns, 4)
                nb = max(1, min(16, (1 << 20) // d)) if d > 32 else 4096
                vs, ps = gen.sweep_batches(ns, d, nb, 5, prs.copy())
                secs = O.ref_bulk_sweep(d, np.arange(ns, dtype=np.uint32), prs, vs, ps)
                cb[str(d)] = {"value": len(vs) / secs, "unit": "updates/s", "seconds": secs}
            out["cpu_baseline"] = {"kind": "reference", "cores": 1, "per_d": cb,
                                   "sample": "reference Engine::bulk_update on a 2^22-key prefill "
                                             "(1/16 of the 2^26 keys; the reference's cost per "
                                             "update grows with the heap)"}
    return out


def leg_api_latency(P, dev, n_calls=2000):
    """Both single-op modes: persistent (default: a resident kernel serves
    the calls through mapped host memory) and one launch per call."""
    out = _api_latency(P, dev, n_calls, 200)
    out["one_launch_per_call"] = _api_latency(P, dev, n_calls, 0)
    cpp = _api_latency_cpp(dev, n_calls)
    if cpp:
        out["cpp"] = cpp
    return out


def _api_latency_cpp(dev, n_calls):
    """The same calls through the C++ drop-in (tools/api_latency.cpp, built
    here with g++ against libpbh_gpu.so), without the interpreter."""
    import shutil
    import subprocess
    import tempfile
    if not shutil.which("g++"):
        return None
    lib = os.path.join(ROOT, "paper_1908_09378_b200")
    exe = os.path.join(tempfile.mkdtemp(), "api_latency")
    try:
        subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tools", "api_latency.cpp"), "-L" + lib, "-lpbh_gpu",
                        "-Wl,-rpath," + lib, "-o", exe], check=True, capture_output=True, timeout=300)
        env = dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", str(dev)))
        res = {}
        for idle, key in ((200, "persistent"), (0, "one_launch_per_call")):
            r = subprocess.run([exe, str(n_calls), str(idle)], capture_output=True, text=True,
                               timeout=300, env=env)
            if r.returncode == 0:
                res[key] = json.loads(r.stdout.strip().splitlines()[-1])
        return res or None
    except (subprocess.SubprocessError, OSError, ValueError):
        return None


def _api_latency(P, dev, n_calls, idle_us):
    """Per-call cost of the single-client Engine API through the C-ABI
    (engine.cpp:90-109: update, bulk_update, extract_min, delete_value): host
    wall time per blocking call, heap of 2^20 keys at d = 32 (the latency
    regime). Calls go through the Python ctypes mirror, so each includes
    ~1-2 us of interpreter overhead."""
    import time as _t
    warm = P.Engine(P.EngineConfig(d=32, debug_assertions=False, key_universe=1 << 10, device=dev))
    for i in range(64):  # first launches (module load) outside the timing
        warm.update((i, 10 + i))
        warm.extract_min()
    warm.close()
    eng = P.Engine(P.EngineConfig(d=32, debug_assertions=False, key_universe=1 << 20, device=dev))
    eng.set_persistent(idle_us)
    rng = np.random.default_rng(3)
    keys = rng.permutation(1 << 20).astype(np.uint32)
    out = {}
    t0 = _t.perf_counter()
    for i in range(n_calls):
        eng.update((int(keys[i]), int(1000 + i)))
    out["update_us"] = (_t.perf_counter() - t0) * 1e6 / n_calls
    batches = [np.sort(keys[n_calls + 32 * i:n_calls + 32 * (i + 1)]) for i in range(n_calls)]
    pr = np.arange(32, dtype=np.uint64) + 5000
    t0 = _t.perf_counter()
    for b in batches:
        eng.bulk_update(values=b, priorities=pr)
    out["bulk_update_d32_us"] = (_t.perf_counter() - t0) * 1e6 / n_calls
    t0 = _t.perf_counter()
    for _ in range(n_calls):
        eng.extract_min()
    out["extract_min_us"] = (_t.perf_counter() - t0) * 1e6 / n_calls
    t0 = _t.perf_counter()
    for i in range(n_calls):
        eng.delete_value(int(keys[i]))
    out["delete_us"] = (_t.perf_counter() - t0) * 1e6 / n_calls
    if idle_us:
        pp = eng.persist_profile()
        out["mode"] = "persistent (idle %d us)" % idle_us
        out["kernel_us_per_call"] = {"wait": pp["wait_ns"] / 1e3 / max(pp["requests"], 1),
                                     "copy_in": pp["copy_ns"] / 1e3 / max(pp["requests"], 1),
                                     "run": pp["run_ns"] / 1e3 / max(pp["requests"], 1)}
        out["resident_launches"] = pp["launches"]
    else:
        out["mode"] = "one launch per call"
    eng.close()
    out["calls_each"] = n_calls
    return out


# ------------------------------------------------------------- GPU arm
def run_pbh(args, D):
    import paper_1908_09378_b200 as P
    from paper_1908_09378_b200 import _lib, gen
    from paper_1908_09378_b200.multi import GatherPlan, DeviceBuffer, shard

    dev = D.device
    G = golden()
    t0 = time.time()
    g = gen.band(V_DEFAULT, DEG_DEFAULT, 2)
    gen_s = time.time() - t0
    V, E = g.vertex_count, g.edge_count
    srcs_all = c5_sources(args.sources)
    b, e = shard(len(srcs_all), D.world, D.rank)
    srcs = srcs_all[b:e]
    S = len(srcs)
    ctx = P.SsspContext(g, d=0, device=dev, max_sources=max(S, 1))

    def solve():
        return ctx.run(srcs) if S else 0.0

    for _ in range(args.warmup):
        solve()
    D.barrier()
    clocks = ClockSampler(dev)
    clocks.start()
    l0 = _lib.lib().pbh_launch_count()
    step_ms = []
    for _ in range(args.steps):
        D.barrier()
        step_ms.append(solve())  # CUDA events on the launching stream
    D.barrier()
    launches = (_lib.lib().pbh_launch_count() - l0) // max(args.steps, 1)
    clk = clocks.stop()
    e_scanned = E  # every vertex of the band is reachable from every source
    total_ms = D.max(float(np.sum(step_ms)))
    ms_per_step = total_ms / args.steps
    value = len(srcs_all) * e_scanned / (ms_per_step / 1e3)
    peak, peak_kind = peak_hbm()
    alg_bytes_launch = S * sssp_bytes(V, e_scanned, V)
    achieved = alg_bytes_launch / (float(np.mean(step_ms)) / 1e3) / 1e9 if S else 0.0

    # per-source parity of the timed solves: settled order (device-computed
    # extraction order), rounds and op counts, gathered to rank 0
    mine = []
    for i in range(S):
        r = ctx.fetch(i, settled=True)
        mine.append({"src": srcs[i], "settled_ck": fnv(r.settled_order), "n": len(r.settled_order),
                     "rounds": r.rounds, "ops": r.ops})
        if srcs[i] == 0:
            tree0 = P.validate_parent_tree(g, 0, r.dist, r.parent, optimal=True)
    per_rank = D.gather_objs(mine)

    # weak scaling (N > 1): 64 sources on every GPU
    weak = None
    if D.world > 1:
        wctx = P.SsspContext(g, d=0, device=dev, max_sources=len(srcs_all))
        wsrc = [(s + 257 * D.rank) % V for s in srcs_all]
        wctx.run(wsrc)
        D.barrier()
        wms = D.max(wctx.run(wsrc))
        wctx.close()
        weak = {"value": D.world * len(srcs_all) * E / (wms / 1e3), "unit": "edges/s",
                "sources_per_gpu": len(srcs_all), "ms_per_step": wms}

    # e2e through the C-ABI with host buffers + the NVLink gather on GPU 0
    plan = GatherPlan(len(srcs_all), V, D.world)
    buf = DeviceBuffer(dev, plan.nbytes) if D.rank == 0 else None
    handle = D.bcast(buf.handle() if buf else None)
    if D.rank != 0:
        buf = DeviceBuffer.open(handle, dev, plan.nbytes)
    host_dist = host_parent = None
    pinned = [g.offsets, g.targets, g.weights]
    if D.rank == 0:
        host_dist = np.empty((len(srcs_all), V), np.uint64)
        host_parent = np.empty((len(srcs_all), V), np.uint32)
        pinned += [host_dist, host_parent]
    P.pin(*pinned)

    # two contexts per rank, used alternately: step i + 1's CSR upload (its
    # own stream, a host thread; ctypes releases the GIL) overlaps step i's
    # solve, so every step still copies its whole input from host memory
    # but only the first upload is exposed (pipeline fill)
    import threading
    ctxs = [ctx, P.SsspContext(g, d=0, device=dev, max_sources=max(S, 1))]

    def e2e_steps(k):
        ctxs[0].load_graph(g)
        for i in range(k):
            c = ctxs[i % 2]
            up = None
            if i + 1 < k:
                up = threading.Thread(target=ctxs[(i + 1) % 2].load_graph, args=(g,))
                up.start()
            if S:
                c.run(srcs)
                c.gather(0, S, buf.ptr + plan.dist_offset(D.rank), buf.ptr + plan.parent_offset(D.rank))
            if up is not None:
                up.join()
            D.barrier()
            if D.rank == 0:
                buf.copy_to_host(host_dist, 0)
                buf.copy_to_host(host_parent, plan.dist_bytes)

    e2e_steps(2)  # warm-up (both contexts)
    D.barrier()
    t = time.perf_counter()
    e2e_steps(args.e2e_steps)
    e2e_ms = [(time.perf_counter() - t) * 1e3 / args.e2e_steps]
    P.unpin(*pinned)
    e2e_max = D.max(float(np.mean(e2e_ms)))
    D.barrier()
    buf.close()
    ctxs[1].close()
    ctx.close()
    h2d = D.world * (8 * (V + 1) + 8 * E) + 4 * len(srcs_all)
    d2h = len(srcs_all) * V * (8 + 4)

    if D.rank != 0:
        return 0

    # ---- C5 parity against the reference's goldens (all 64 sources)
    parity = {}
    want = G.get("C5")
    if want and want["sources"] == srcs_all:
        rows = [x for part in per_rank for x in part]
        dist_ok = [P.distance_checksum(host_dist[i]) == want["dist_checksum"][i]
                   for i in range(len(srcs_all))]
        by_src = {x["src"]: x for x in rows}
        set_ok = [by_src[s]["settled_ck"] == want["settled_checksum"][i] and
                  by_src[s]["n"] == want["n_settled"][i] for i, s in enumerate(srcs_all)]
        rnd_ok = [by_src[s]["rounds"] == want["rounds"][i] and by_src[s]["ops"] == want["ops"][i]
                  for i, s in enumerate(srcs_all)]
        trees = [P.validate_parent_tree(g, s, host_dist[i], host_parent[i]) is None
                 for i, s in list(enumerate(srcs_all))[::8]]
        parity["C5"] = {"sources_checked": len(srcs_all),
                        "dist_checksums_equal": int(sum(dist_ok)),
                        "settled_orders_equal": int(sum(set_ok)),
                        "rounds_ops_equal": int(sum(rnd_ok)),
                        "parent_trees_valid": f"{sum(trees)}/{len(trees)} (every 8th source)",
                        "source0_optimality_certificate": tree0 is None,
                        "match": all(dist_ok) and all(set_ok) and all(rnd_ok) and all(trees) and
                        tree0 is None,
                        "against": "tests/golden/full_size.json C5 (oracle/_ref reference_dijkstra "
                                   "+ par_dijkstra)"}
    hi = host_info()
    cpu = None
    textbook = None
    run_cpu = D.world == 1 and not args.no_cpu_baseline
    if run_cpu:
        from oracle import oracle as O
        if O.ref_available():
            threads = hi["host_threads"]
            n_s = args.cpu_sample_sources or min(threads, len(srcs_all))
            rg = O.RefGraph(O.Graph(V, g.offsets, g.targets, g.weights))  # import: not timed
            rp = rg.sssp_batch(srcs_all[:n_s], "par", threads=threads)
            cpu = {"value": n_s * E / rp["seconds"], "unit": "edges/s", "cores": threads,
                   "kind": "reference", **hi,
                   "sample": f"reference par_dijkstra (oracle/_ref), {n_s} of the "
                             f"{len(srcs_all)} sources, one per host thread, {rp['seconds']:.1f} s, "
                             f"graph imported outside the timed region"}
            rt = rg.sssp_batch(srcs_all, "ref", threads=threads)
            rg.close()
            textbook = {"value": len(srcs_all) * E / rt["seconds"], "unit": "edges/s",
                        "cores": threads, "kind": "reference",
                        "sample": f"reference_dijkstra (sssp.cpp:71-97), all {len(srcs_all)} sources, "
                                  f"{rt['seconds']:.1f} s"}
            # live cross-check of the GPU results against the reference run here
            live_ok = all(P.distance_checksum(host_dist[i]) == int(rt["dist_ck"][i])
                          for i in range(len(srcs_all)))
            parity.setdefault("C5", {})["live_reference_dijkstra_equal"] = live_ok
            parity["C5"]["match"] = parity["C5"].get("match", True) and live_ok

    legs = {}
    which = [] if args.legs == "none" else [x.strip() for x in args.legs.split(",") if x.strip()]
    if "c3" in which:
        legs["c3_single_source"] = leg_c3(P, g, dev, peak, G.get("C3"), run_cpu)
    del g
    if "c2" in which:
        legs["c2_grid"] = leg_c2(P, gen, dev, peak, G.get("C2"), run_cpu)
    if "c1" in which:
        legs["c1_op_trace"] = leg_c1(P, gen, dev, peak, args.c1_ops, G.get("C1"), run_cpu)
    if "api" in which:
        legs["api_latency"] = leg_api_latency(P, dev)
    if "c4" in which:
        legs["c4_bulk_update"] = leg_c4(P, gen, dev, peak, [int(x) for x in args.c4_ds.split(",")],
                                        run_cpu)
    for k, v in legs.items():
        if "match" in v:
            parity[k] = {"match": v["match"]}
    all_match = all(v.get("match", False) for v in parity.values()) if parity else False

    traffic_ps = traffic_from_profiles()
    out = {
        "metric": "sssp_edges_relaxed_per_sec", "value": value, "unit": "edges/s",
        "n_gpus": D.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"BASELINE C5: {len(srcs_all)} sources (s_i = i*16384) of par_dijkstra "
                               f"on the C3 dense high-diameter band, split {len(srcs_all)}/{D.world} "
                               "per GPU",
                   "V": V, "E": E, "degree": DEG_DEFAULT, "sources": len(srcs_all),
                   "sources_per_gpu": S, "d": DEG_DEFAULT, "graph_seed": 2,
                   "l2": "inputs larger than L2 (CSR 2.15 GB)",
                   "parallelism": f"source-sharded x{D.world}, no collective on the data path"
                                  + (" (ranks share devices: functional run)" if D.shared_devices else "")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_kind": peak_kind,
                     "traffic": (traffic_ps * S if traffic_ps else None),
                     "kernel": "k_sssp_bank<4,8,4,256> (one 128-thread CTA per source)",
                     "alg_bytes_per_launch": alg_bytes_launch,
                     "alg_bytes_per_source": sssp_bytes(V, e_scanned, V)},
        "cpu_baseline": cpu,
        "textbook_cpu_baseline": textbook,
        "e2e": {"value": len(srcs_all) * e_scanned / (e2e_max / 1e3), "unit": "edges/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_max,
                "api": "per rank and step: pbh_sssp_ctx_load_graph (host CSR) + pbh_sssp_ctx_run + "
                       "pbh_sssp_ctx_gather into GPU 0 (CUDA IPC, NVLink); GPU 0 -> host copy of "
                       "all 64 x V dist + parent; two contexts alternate so step i+1's CSR upload "
                       "overlaps step i's solve (first upload exposed); wall time of all steps / steps",
                "steps": args.e2e_steps},
        "gpu_launches": int(launches),
        "clocks": clk,
        "weak_scaling": weak,
        "parity": {"match": all_match, **parity},
        "host": hi,
        "gen_s": gen_s,
        **legs,
    }
    print(json.dumps(out), flush=True)
    return 0 if all_match else 3


def main():
    args = parse()
    rc = maybe_spawn(args)
    if rc is not None:
        sys.exit(rc)
    D = Dist()
    rc = 0
    try:
        if args.impl == "reference":
            rc = run_reference_arm(args, D)
        else:
            rc = run_pbh(args, D)
    finally:
        D.close()
    sys.exit(rc)


if __name__ == "__main__":
    main()
