"""TEST INFRASTRUCTURE ONLY — ctypes front-end to the CPU oracle.

Two back-ends live here, both used purely as CHECKERS (tests/, smoke(),
bench.py's cpu_baseline leg and its ``--impl reference`` arm):

* ``liboracle.so``  — the plain-C restatement (oracle/pbh_oracle.c), each
  function citing the reference file:line it follows.
* ``_ref/libpbhref.so`` — the UNMODIFIED reference library compiled from
  /root/reference/proj/src by ``make -C oracle ref`` (see oracle/Makefile),
  wrapped by oracle/ref_harness.cpp.

Nothing on the product path imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
U8P, U32P, U64P = C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)


def _p(a, t):
    return a.ctypes.data_as(t)


class _Trace(C.Structure):
    _fields_ = [("n_ops", C.c_uint64), ("n_elems", C.c_uint64), ("kinds", U8P),
                ("offsets", U64P), ("vals", U32P), ("prios", U64P), ("n_extract", C.c_uint64)]


class _Graph(C.Structure):
    _fields_ = [("V", C.c_uint32), ("E", C.c_uint64), ("off", U64P), ("tgt", U32P), ("w", U32P)]


class Trace:
    """Flat op trace: kinds u8[n] in b'UBED', offsets u64[n+1], vals u32[], prios u64[]."""

    def __init__(self, kinds, offsets, vals, prios):
        self.kinds = np.ascontiguousarray(kinds, dtype=np.uint8)
        self.offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        self.vals = np.ascontiguousarray(vals, dtype=np.uint32)
        self.prios = np.ascontiguousarray(prios, dtype=np.uint64)

    @property
    def n_ops(self):
        return len(self.kinds)

    @property
    def n_extract(self):
        return int(np.count_nonzero(self.kinds == ord("E")))


class Graph:
    def __init__(self, V, off, tgt, w):
        self.V = int(V)
        self.off = np.ascontiguousarray(off, dtype=np.uint64)
        self.tgt = np.ascontiguousarray(tgt, dtype=np.uint32)
        self.w = np.ascontiguousarray(w, dtype=np.uint32)

    @property
    def E(self):
        return len(self.tgt)


# --------------------------------------------------------------------------
# C restatement
# --------------------------------------------------------------------------
_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-C", HERE, "-s"], check=True)
        L = C.CDLL(path)
        L.orc_trace_gen_legal.restype = C.POINTER(_Trace)
        L.orc_trace_gen_legal.argtypes = [C.c_uint64] * 3
        L.orc_trace_gen_mixed.restype = C.POINTER(_Trace)
        L.orc_trace_gen_mixed.argtypes = [C.c_uint64] * 4
        L.orc_trace_free.argtypes = [C.POINTER(_Trace)]
        L.orc_run_oracle.restype = C.c_int64
        L.orc_run_oracle.argtypes = [C.c_uint64, U8P, U64P, U32P, U64P, U32P, U64P]
        for name, args in [("orc_gen_random", [C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64]),
                           ("orc_gen_high_diameter", [C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64]),
                           ("orc_gen_dag", [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64]),
                           ("orc_gen_complete", [C.c_uint32, C.c_uint32, C.c_uint64]),
                           ("orc_gen_grid", [C.c_uint32, C.c_uint32, C.c_uint64]),
                           ("orc_gen_band", [C.c_uint32, C.c_uint32, C.c_uint64])]:
            f = getattr(L, name)
            f.restype = C.POINTER(_Graph)
            f.argtypes = args
        L.orc_graph_free.argtypes = [C.POINTER(_Graph)]
        L.orc_dijkstra.restype = C.c_int
        L.orc_dijkstra.argtypes = [C.c_uint32, C.c_uint64, U64P, U32P, U32P, C.c_uint32, C.c_uint64,
                                   U64P, U32P, U64P, U64P, U64P]
        L.orc_checksum.restype = C.c_uint64
        L.orc_checksum.argtypes = [U64P, C.c_uint64]
        L.orc_fnv1a.restype = C.c_uint64
        L.orc_fnv1a.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        _lib = L
    return _lib


def _take_trace(ptr):
    t = ptr.contents
    n, m = t.n_ops, t.n_elems
    out = Trace(np.ctypeslib.as_array(t.kinds, (n,)).copy() if n else np.zeros(0, np.uint8),
                np.ctypeslib.as_array(t.offsets, (n + 1,)).copy(),
                np.ctypeslib.as_array(t.vals, (m,)).copy() if m else np.zeros(0, np.uint32),
                np.ctypeslib.as_array(t.prios, (m,)).copy() if m else np.zeros(0, np.uint64))
    lib().orc_trace_free(ptr)
    return out


def gen_legal_trace(n_ops, d, seed):
    """tests/oracle.hpp:82-155 restated."""
    return _take_trace(lib().orc_trace_gen_legal(n_ops, d, seed))


def gen_mixed_trace(n_ops, universe, kmax, seed):
    """BASELINE C1 generator."""
    return _take_trace(lib().orc_trace_gen_mixed(n_ops, universe, kmax, seed))


def run_oracle(tr: Trace):
    """tests/oracle.hpp:55-75 restated. Returns (vals, prios) or raises
    IndexError(op_index) when an extract meets an empty queue."""
    nx = max(tr.n_extract, 1)
    ov = np.zeros(nx, np.uint32)
    op = np.zeros(nx, np.uint64)
    n = lib().orc_run_oracle(tr.n_ops, _p(tr.kinds, U8P), _p(tr.offsets, U64P), _p(tr.vals, U32P),
                             _p(tr.prios, U64P), _p(ov, U32P), _p(op, U64P))
    if n < 0:
        raise IndexError(-n - 1)
    return ov[:n], op[:n]


def _take_graph(ptr):
    if not ptr:
        raise ValueError("generator precondition failed")
    g = ptr.contents
    out = Graph(g.V, np.ctypeslib.as_array(g.off, (g.V + 1,)).copy(),
                np.ctypeslib.as_array(g.tgt, (max(g.E, 1),))[:g.E].copy(),
                np.ctypeslib.as_array(g.w, (max(g.E, 1),))[:g.E].copy())
    lib().orc_graph_free(ptr)
    return out


def gen_random(v, e, max_weight, seed):
    return _take_graph(lib().orc_gen_random(v, e, max_weight, seed))


def gen_high_diameter(v, e, max_weight, seed):
    return _take_graph(lib().orc_gen_high_diameter(v, e, max_weight, seed))


def gen_dag(v, out_degree, max_weight, seed):
    return _take_graph(lib().orc_gen_dag(v, out_degree, max_weight, seed))


def gen_complete(v, max_weight, seed):
    return _take_graph(lib().orc_gen_complete(v, max_weight, seed))


def gen_grid(rows, cols, seed=1):
    return _take_graph(lib().orc_gen_grid(rows, cols, seed))


def gen_band(v, degree, seed=2):
    return _take_graph(lib().orc_gen_band(v, degree, seed))


def make_graph(v, edges):
    """test_sssp.cpp:16-31: CSR from an (src, dst, w) list."""
    edges = sorted(edges)
    off = np.zeros(v + 1, np.uint64)
    for s, _, _ in edges:
        off[s + 1] += 1
    off = np.cumsum(off, dtype=np.uint64)
    return Graph(v, off, [t for _, t, _ in edges], [w for _, _, w in edges])


def dijkstra(g: Graph, source, d=0):
    """reference_dijkstra (sssp.cpp:71-97) restated; also returns par_dijkstra's op count."""
    dist = np.zeros(g.V, np.uint64)
    settled = np.zeros(g.V, np.uint32)
    ns, nr, ops = C.c_uint64(), C.c_uint64(), C.c_uint64()
    st = lib().orc_dijkstra(g.V, g.E, _p(g.off, U64P), _p(g.tgt, U32P), _p(g.w, U32P), source, d,
                            _p(dist, U64P), _p(settled, U32P), C.byref(ns), C.byref(nr), C.byref(ops))
    if st == 2:
        raise ValueError("source out of range")
    if st == 3:
        raise OverflowError("distance accumulation overflow")
    return dict(dist=dist, settled_order=settled[:ns.value], rounds=nr.value, ops=ops.value)


def checksum(dist):
    dist = np.ascontiguousarray(dist, dtype=np.uint64)
    return int(lib().orc_checksum(_p(dist, U64P), len(dist)))


FNV_BASIS = 0xcbf29ce484222325


def fnv1a(*arrays, h=FNV_BASIS):
    """FNV-1a (sssp.cpp:174-183's hash) over the raw little-endian bytes of
    the arrays in order. fnv1a(settled_order) is the settle-order checksum of
    the full-size goldens; fnv1a(vals, prios) the extraction-sequence one."""
    for a in arrays:
        a = np.ascontiguousarray(a)
        h = int(lib().orc_fnv1a(C.c_void_p(a.ctypes.data), a.nbytes, h))
    return h


def settle_order_from_dist(dist):
    """The reference's settle order recomputed from dist: reached vertices by
    (dist, vid) (SURVEY.md §8a semantic facts; test_sssp.cpp:92-100)."""
    dist = np.asarray(dist, np.uint64)
    reached = np.nonzero(dist != np.uint64(2 ** 64 - 1))[0].astype(np.uint32)
    return reached[np.lexsort((reached, dist[reached]))]


# --------------------------------------------------------------------------
# The reference itself (oracle/_ref), available where it was built
# --------------------------------------------------------------------------
_ref = None
REF_SO = os.path.join(HERE, "_ref", "libpbhref.so")


def ref_available():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            if os.path.isdir("/root/reference/proj"):
                subprocess.run(["make", "-C", HERE, "-s", "ref"], check=True)
            else:
                raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        V = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_trace_gen_legal.restype = V
        L.ref_trace_gen_legal.argtypes = [C.c_uint64] * 3
        L.ref_trace_import.restype = V
        L.ref_trace_import.argtypes = [C.c_uint64, U8P, U64P, U32P, U64P]
        L.ref_trace_sizes.argtypes = [V, U64P, U64P, U64P]
        L.ref_trace_export.argtypes = [V, U8P, U64P, U32P, U64P]
        L.ref_trace_free.argtypes = [V]
        L.ref_trace_load_text.restype = V
        L.ref_trace_load_text.argtypes = [C.c_char_p, U64P]
        L.ref_run_oracle.argtypes = [V, U32P, U64P, U64P]
        L.ref_engine_run_trace.argtypes = [V, C.c_uint64, C.c_uint64, C.c_int, U32P, U64P, U64P,
                                           U64P, U64P]
        L.ref_graph_gen.restype = V
        L.ref_graph_gen.argtypes = [C.c_int, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64]
        L.ref_graph_import.restype = V
        L.ref_graph_import.argtypes = [C.c_uint32, C.c_uint64, U64P, U32P, U32P]
        L.ref_graph_sizes.argtypes = [V, U32P, U64P]
        L.ref_graph_export.argtypes = [V, U64P, U32P, U32P]
        L.ref_graph_free.argtypes = [V]
        L.ref_sssp.argtypes = [V, C.c_int, C.c_uint32, C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                               U64P, U32P, U64P, U64P, U64P]
        L.ref_sssp_multi.argtypes = [V, C.c_int, U32P, C.c_uint64, C.c_uint64, U64P]
        L.ref_sssp_batch.argtypes = [V, C.c_int, U32P, C.c_uint64, C.c_uint64, C.c_uint64, U64P,
                                     U64P, U64P, U64P, U64P, U64P, C.POINTER(C.c_double)]
        L.ref_bulk_sweep.argtypes = [C.c_uint64, C.c_uint64, U32P, U64P, C.c_uint64, U32P, U64P,
                                     C.POINTER(C.c_double)]
        L.ref_distance_checksum.restype = C.c_uint64
        L.ref_distance_checksum.argtypes = [U64P, C.c_uint64]
        _ref = L
    return _ref


class RefError(RuntimeError):
    def __init__(self, status, msg, op_index=None):
        super().__init__(f"status {status}: {msg}")
        self.status = status
        self.op_index = op_index


def ref_gen_legal_trace(n_ops, d, seed):
    L = ref()
    h = L.ref_trace_gen_legal(n_ops, d, seed)
    n, m, x = C.c_uint64(), C.c_uint64(), C.c_uint64()
    L.ref_trace_sizes(h, C.byref(n), C.byref(m), C.byref(x))
    kinds = np.zeros(n.value, np.uint8)
    offs = np.zeros(n.value + 1, np.uint64)
    vals = np.zeros(max(m.value, 1), np.uint32)
    prios = np.zeros(max(m.value, 1), np.uint64)
    L.ref_trace_export(h, _p(kinds, U8P), _p(offs, U64P), _p(vals, U32P), _p(prios, U64P))
    L.ref_trace_free(h)
    return Trace(kinds, offs, vals[:m.value], prios[:m.value])


def ref_load_text(path):
    """The reference's load_trace (trace_format.cpp:34-98). Returns a Trace,
    or raises RefError(op_index=...) with the reference's message."""
    L = ref()
    failed = C.c_uint64()
    h = L.ref_trace_load_text(str(path).encode(), C.byref(failed))
    if not h:
        raise RefError(4, L.ref_last_error().decode(),
                       None if failed.value == 2 ** 64 - 1 else failed.value)
    n, m, x = C.c_uint64(), C.c_uint64(), C.c_uint64()
    L.ref_trace_sizes(h, C.byref(n), C.byref(m), C.byref(x))
    kinds = np.zeros(n.value, np.uint8)
    offs = np.zeros(n.value + 1, np.uint64)
    vals = np.zeros(max(m.value, 1), np.uint32)
    prios = np.zeros(max(m.value, 1), np.uint64)
    L.ref_trace_export(h, _p(kinds, U8P), _p(offs, U64P), _p(vals, U32P), _p(prios, U64P))
    L.ref_trace_free(h)
    return Trace(kinds, offs, vals[:m.value], prios[:m.value])


def _ref_trace(tr: Trace):
    return ref().ref_trace_import(tr.n_ops, _p(tr.kinds, U8P), _p(tr.offsets, U64P),
                                  _p(tr.vals, U32P), _p(tr.prios, U64P))


def ref_run_oracle(tr: Trace):
    L = ref()
    h = _ref_trace(tr)
    nx = max(tr.n_extract, 1)
    ov, op, n = np.zeros(nx, np.uint32), np.zeros(nx, np.uint64), C.c_uint64()
    st = L.ref_run_oracle(h, _p(ov, U32P), _p(op, U64P), C.byref(n))
    L.ref_trace_free(h)
    if st:
        raise RefError(st, L.ref_last_error().decode())
    return ov[:n.value], op[:n.value]


def ref_run_trace(tr: Trace, d, workers=1, debug=True):
    """pbh::Engine::run_trace on the reference bucket heap. Returns
    (vals, prios, metrics dict)."""
    L = ref()
    h = _ref_trace(tr)
    nx = max(tr.n_extract, 1)
    ov, op, n = np.zeros(nx, np.uint32), np.zeros(nx, np.uint64), C.c_uint64()
    failed = C.c_uint64()
    met = np.zeros(71, np.uint64)
    st = L.ref_engine_run_trace(h, d, workers, int(debug), _p(ov, U32P), _p(op, U64P), C.byref(n),
                                C.byref(failed), _p(met, U64P))
    L.ref_trace_free(h)
    if st:
        raise RefError(st, L.ref_last_error().decode(),
                       None if failed.value == 2 ** 64 - 1 else failed.value)
    nl = int(met[2])
    m = dict(ops=int(met[0]), wall_ms=met[1] / 1e6, resolves_per_level=met[3:3 + nl].tolist(),
             touches_per_level=met[37:37 + nl].tolist())
    return ov[:n.value], op[:n.value], m


def ref_graph(kind, v, e, max_weight, seed):
    """kind: 'random' | 'highdiam' | 'dag' | 'complete' — graphs.cpp generators."""
    L = ref()
    k = {"random": 0, "highdiam": 1, "dag": 2, "complete": 3}[kind]
    h = L.ref_graph_gen(k, v, e, max_weight, seed)
    if not h:
        raise RefError(2, L.ref_last_error().decode())
    V, E = C.c_uint32(), C.c_uint64()
    L.ref_graph_sizes(h, C.byref(V), C.byref(E))
    off = np.zeros(V.value + 1, np.uint64)
    tgt = np.zeros(max(E.value, 1), np.uint32)
    w = np.zeros(max(E.value, 1), np.uint32)
    L.ref_graph_export(h, _p(off, U64P), _p(tgt, U32P), _p(w, U32P))
    L.ref_graph_free(h)
    return Graph(V.value, off, tgt[:E.value], w[:E.value])


def _ref_graph_handle(g: Graph):
    tgt = g.tgt if g.E else np.zeros(1, np.uint32)
    w = g.w if g.E else np.zeros(1, np.uint32)
    return ref().ref_graph_import(g.V, g.E, _p(g.off, U64P), _p(tgt, U32P), _p(w, U32P))


def ref_sssp(g: Graph, source, algo="par", d=0, workers=1, debug=True, dag_mode=False):
    """algo: 'par' (par_dijkstra on the bucket heap), 'ref' (reference_dijkstra), 'bf'."""
    L = ref()
    h = _ref_graph_handle(g)
    dist = np.zeros(g.V, np.uint64)
    settled = np.zeros(g.V, np.uint32)
    ns, nr, ops = C.c_uint64(), C.c_uint64(), C.c_uint64()
    st = L.ref_sssp(h, {"par": 0, "ref": 1, "bf": 2}[algo], source, d, workers, int(debug),
                    int(dag_mode), _p(dist, U64P), _p(settled, U32P), C.byref(ns), C.byref(nr),
                    C.byref(ops))
    L.ref_graph_free(h)
    if st:
        raise RefError(st, L.ref_last_error().decode())
    return dict(dist=dist, settled_order=settled[:ns.value], rounds=nr.value, ops=ops.value)


def ref_sssp_multi(g: Graph, sources, algo="par", threads=None):
    L = ref()
    h = _ref_graph_handle(g)
    src = np.ascontiguousarray(sources, dtype=np.uint32)
    dist = np.zeros(len(src) * g.V, np.uint64)
    st = L.ref_sssp_multi(h, 0 if algo == "par" else 1, _p(src, U32P), len(src),
                          threads or os.cpu_count(), _p(dist, U64P))
    L.ref_graph_free(h)
    if st:
        raise RefError(st, L.ref_last_error().decode())
    return dist.reshape(len(src), g.V)


class RefGraph:
    """A CSR imported into the reference's CsrGraph ONCE (graph load is not
    part of any timed CPU solve)."""

    def __init__(self, g: Graph):
        self.V, self.E = g.V, g.E
        self._h = _ref_graph_handle(g)

    def sssp_batch(self, sources, algo="par", threads=1, d=0, want_dist=False):
        """ref_sssp_batch: independent sources on `threads` host threads.
        Returns dict of per-source arrays (dist_ck, settled_ck, n_settled,
        rounds, ops[, dist]) and the solve-only wall seconds."""
        L = ref()
        src = np.ascontiguousarray(sources, dtype=np.uint32)
        n = len(src)
        out = {k: np.zeros(n, np.uint64) for k in ("dist_ck", "settled_ck", "n_settled", "rounds", "ops")}
        dist = np.zeros(n * self.V, np.uint64) if want_dist else None
        secs = C.c_double()
        st = L.ref_sssp_batch(self._h, {"par": 0, "ref": 1}[algo], _p(src, U32P), n, threads, d,
                              _p(out["dist_ck"], U64P), _p(out["settled_ck"], U64P),
                              _p(out["n_settled"], U64P), _p(out["rounds"], U64P),
                              _p(out["ops"], U64P), _p(dist, U64P) if want_dist else None,
                              C.byref(secs))
        if st:
            raise RefError(st, L.ref_last_error().decode())
        if want_dist:
            out["dist"] = dist.reshape(n, self.V)
        out["seconds"] = secs.value
        return out

    def close(self):
        if getattr(self, "_h", None):
            ref().ref_graph_free(self._h)
            self._h = None

    __del__ = close


def ref_bulk_sweep(d, pre_v, pre_p, v, p):
    """Reference Engine::bulk_update timing: prefill then time len(v)//d batches."""
    L = ref()
    pre_v = np.ascontiguousarray(pre_v, np.uint32)
    pre_p = np.ascontiguousarray(pre_p, np.uint64)
    v = np.ascontiguousarray(v, np.uint32)
    p = np.ascontiguousarray(p, np.uint64)
    secs = C.c_double()
    st = L.ref_bulk_sweep(d, len(pre_v), _p(pre_v, U32P), _p(pre_p, U64P), len(v) // d, _p(v, U32P),
                          _p(p, U64P), C.byref(secs))
    if st:
        raise RefError(st, L.ref_last_error().decode())
    return secs.value
