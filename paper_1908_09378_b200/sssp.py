"""Host-side mirror of the reference SSSP API (/root/reference/proj/include/pbh/sssp.hpp:13-48)
over the pbh-b200 C-ABI: ``par_dijkstra`` runs as one persistent CTA per
source on the B200; ``par_dijkstra_multi`` shards independent sources.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import raise_for

K_INF_DIST = (1 << 64) - 1  # sssp.hpp:16


@dataclass
class CsrGraph:
    """graphs.hpp:11-20: offsets u64[V+1], targets u32[E], weights u32[E]."""
    vertex_count: int
    offsets: np.ndarray
    targets: np.ndarray
    weights: np.ndarray

    @property
    def edge_count(self):
        return len(self.targets)

    @staticmethod
    def of(g):
        """Adopt any object with V/off/tgt/w or vertex_count/offsets/targets/weights."""
        if isinstance(g, CsrGraph):
            return g
        if hasattr(g, "off"):
            return CsrGraph(int(g.V), g.off, g.tgt, g.w)
        return CsrGraph(int(g.vertex_count), g.offsets, g.targets, g.weights)

    def c_struct(self):
        self._off = np.ascontiguousarray(self.offsets, dtype=np.uint64)
        self._tgt = np.ascontiguousarray(self.targets if len(self.targets) else [0], dtype=np.uint32)
        self._w = np.ascontiguousarray(self.weights if len(self.weights) else [1], dtype=np.uint32)
        return _lib.Csr(self.vertex_count, len(self.targets),
                        self._off.ctypes.data_as(_lib.U64P), self._tgt.ctypes.data_as(_lib.U32P),
                        self._w.ctypes.data_as(_lib.U32P))


@dataclass
class SsspResult:
    """sssp.hpp:18-23 plus ``parent`` (shortest-path tree; extension)."""
    dist: np.ndarray
    settled_order: np.ndarray
    rounds: int
    ops: int
    parent: np.ndarray | None = None


def par_dijkstra(g, source: int, d: int = 0, dag_mode: bool = False, device: int = 0) -> SsspResult:
    """par_dijkstra (sssp.hpp:28-29; sssp.cpp:21-69). ``d == 0`` selects the
    maximum out-degree (sssp.cpp:24-26)."""
    g = CsrGraph.of(g)
    cs = g.c_struct()
    V = g.vertex_count
    dist = np.zeros(max(V, 1), np.uint64)
    parent = np.zeros(max(V, 1), np.uint32)
    settled = np.zeros(max(V, 1), np.uint32)
    ns, nr, ops = C.c_uint64(), C.c_uint64(), C.c_uint64()
    raise_for(_lib.lib().pbh_sssp(C.byref(cs), int(source), int(d), int(dag_mode), device,
                                  dist.ctypes.data_as(_lib.U64P), parent.ctypes.data_as(_lib.U32P),
                                  settled.ctypes.data_as(_lib.U32P), C.byref(ns), C.byref(nr),
                                  C.byref(ops)))
    return SsspResult(dist[:V], settled[:ns.value], nr.value, ops.value, parent[:V])


def threshold_sssp(g, source: int, device: int = 0) -> SsspResult:
    """Threshold multi-extraction SSSP (extension):
    exact distances and a valid parent tree; ``rounds`` counts batches and
    ``settled_order`` is reported as the reference's settle order, i.e. the
    reached vertices sorted by (dist, vid)."""
    ctx = SsspContext(g, device=device, max_sources=1, mode="threshold")
    try:
        ctx.run([source])
        r = ctx.fetch(0, settled=True)
    finally:
        ctx.close()
    order = r.settled_order[np.lexsort((r.settled_order, r.dist[r.settled_order]))]
    return SsspResult(r.dist, order, r.rounds, r.ops, r.parent)


def bellman_ford(g, source: int, device: int = 0, with_parent: bool = True):
    """bellman_ford (sssp.hpp:37; sssp.cpp:99-129) as a device frontier sweep.
    Returns (SsspResult with settled_order = reached vertices by (dist, vid),
    edges_scanned, device_ms); ``rounds`` counts frontier iterations."""
    g = CsrGraph.of(g)
    cs = g.c_struct()
    V = g.vertex_count
    dist = np.zeros(max(V, 1), np.uint64)
    parent = np.zeros(max(V, 1), np.uint32) if with_parent else None
    nr, ne, ms = C.c_uint64(), C.c_uint64(), C.c_double()
    raise_for(_lib.lib().pbh_bellman_ford(
        C.byref(cs), int(source), device, dist.ctypes.data_as(_lib.U64P),
        parent.ctypes.data_as(_lib.U32P) if with_parent else None, C.byref(nr), C.byref(ne),
        C.byref(ms)))
    d = dist[:V]
    reached = np.nonzero(d != K_INF_DIST)[0].astype(np.uint32)
    order = reached[np.lexsort((reached, d[reached]))]
    return (SsspResult(d, order, nr.value, 0, parent[:V] if with_parent else None),
            ne.value, ms.value)


def par_dijkstra_multi(g, sources, d: int = 0, devices=(0,), out=None):
    """Independent sources dealt contiguously over ``devices`` (BASELINE C5).
    Returns (dist[n_sources, V], parent[n_sources, V]); ``out`` may supply
    those two arrays (e.g. page-locked with :func:`pin`)."""
    g = CsrGraph.of(g)
    cs = g.c_struct()
    src = np.ascontiguousarray(sources, dtype=np.uint32)
    devs = (C.c_int * len(devices))(*devices)
    if out is None:
        dist = np.zeros((len(src), g.vertex_count), np.uint64)
        parent = np.zeros((len(src), g.vertex_count), np.uint32)
    else:
        dist, parent = out
        assert dist.shape == (len(src), g.vertex_count) and dist.dtype == np.uint64
        assert parent.shape == (len(src), g.vertex_count) and parent.dtype == np.uint32
    raise_for(_lib.lib().pbh_sssp_multi(C.byref(cs), src.ctypes.data_as(_lib.U32P), len(src), d,
                                        devs, len(devices), dist.ctypes.data_as(_lib.U64P),
                                        parent.ctypes.data_as(_lib.U32P)))
    return dist, parent


class SsspContext:
    """Device-resident CSR for repeated solves (bench: inputs already in HBM)."""

    def __init__(self, g, d: int = 0, device: int = 0, max_sources: int = 1,
                 mode: str = "exact"):
        # a DeviceCsr (gen.band_device / grid_device) is copied device-to-device
        self.g = g if hasattr(g, "data_ptr") or type(g).__name__ == "DeviceCsr" else CsrGraph.of(g)
        cs = self.g.c_struct()
        h = C.c_void_p()
        raise_for(_lib.lib().pbh_sssp_ctx_create(C.byref(cs), d, device, max_sources, C.byref(h)))
        self._h = h
        self.mode = mode
        if mode != "exact":
            self.set_mode(mode)

    def set_mode(self, mode: str):
        """'exact' = par_dijkstra (one extraction per round); 'threshold' =
        multi-extraction by the Crauser IN/OUT criteria (extension)."""
        raise_for(_lib.lib().pbh_sssp_ctx_set_mode(self._h, {"exact": 0, "threshold": 1}[mode]))
        self.mode = mode

    def load_graph(self, g):
        """Re-upload a same-shape CSR (host arrays: H2D; a DeviceCsr: D2D)
        into this context (pbh_sssp_ctx_load_graph)."""
        g = g if hasattr(g, "data_ptr") or type(g).__name__ == "DeviceCsr" else CsrGraph.of(g)
        cs = g.c_struct()
        raise_for(_lib.lib().pbh_sssp_ctx_load_graph(self._h, C.byref(cs)))
        self.g = g

    def gather(self, first_slot: int, n_slots: int, dist_addr: int, parent_addr: int = 0):
        """pbh_sssp_ctx_gather: copy the dist / parent rows of slots
        [first_slot, first_slot + n_slots) to raw addresses (host, this
        device, a peer device or an IPC-mapped buffer of another process)."""
        raise_for(_lib.lib().pbh_sssp_ctx_gather(self._h, first_slot, n_slots,
                                                 C.c_void_p(dist_addr or None),
                                                 C.c_void_p(parent_addr or None)))

    def fetch_into(self, slot, dist, parent=None):
        """D2H of one source's dist (u64[V]) and parent (u32[V]) into
        caller-owned (e.g. page-locked) arrays."""
        raise_for(_lib.lib().pbh_sssp_ctx_fetch(
            self._h, slot, dist.ctypes.data_as(_lib.U64P),
            parent.ctypes.data_as(_lib.U32P) if parent is not None else None, None, None, None,
            None))

    def run(self, sources, dag_mode=False) -> float:
        src = np.ascontiguousarray(sources, dtype=np.uint32)
        ms = C.c_double()
        raise_for(_lib.lib().pbh_sssp_ctx_run(self._h, src.ctypes.data_as(_lib.U32P), len(src),
                                              int(dag_mode), C.byref(ms)))
        return ms.value

    def fetch(self, slot=0, settled=True) -> SsspResult:
        V = self.g.vertex_count
        dist = np.zeros(max(V, 1), np.uint64)
        parent = np.zeros(max(V, 1), np.uint32)
        st = np.zeros(max(V, 1), np.uint32) if settled else None
        ns, nr, ops = C.c_uint64(), C.c_uint64(), C.c_uint64()
        raise_for(_lib.lib().pbh_sssp_ctx_fetch(
            self._h, slot, dist.ctypes.data_as(_lib.U64P), parent.ctypes.data_as(_lib.U32P),
            st.ctypes.data_as(_lib.U32P) if settled else None, C.byref(ns), C.byref(nr),
            C.byref(ops)))
        return SsspResult(dist[:V], st[:ns.value] if settled else None, nr.value, ops.value,
                          parent[:V])

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().pbh_sssp_ctx_destroy(self._h)
            self._h = None

    __del__ = close


def validate_graph(g, device: int = 0):
    """validate_graph (graphs.hpp:23; graphs.cpp:55-72) as one device pass:
    raises InvariantError with the reference's message."""
    g = g if type(g).__name__ == "DeviceCsr" else CsrGraph.of(g)
    cs = g.c_struct()
    raise_for(_lib.lib().pbh_validate_graph(C.byref(cs), device))


def max_out_degree(g, device: int = 0) -> int:
    """CsrGraph::max_out_degree (graphs.hpp:18; graphs.cpp:47-53)."""
    g = g if type(g).__name__ == "DeviceCsr" else CsrGraph.of(g)
    cs = g.c_struct()
    out = C.c_uint32()
    raise_for(_lib.lib().pbh_csr_max_out_degree(C.byref(cs), device, C.byref(out)))
    return out.value


def distance_checksum(dist) -> int:
    """sssp.cpp:174-183."""
    d = np.ascontiguousarray(dist, dtype=np.uint64)
    return int(_lib.lib().pbh_distance_checksum(d.ctypes.data_as(_lib.U64P), len(d)))


def distances_to_csv(dist) -> str:
    """sssp.cpp:159-172."""
    out = ["vertex,dist"]
    for v, x in enumerate(np.asarray(dist, dtype=np.uint64).tolist()):
        out.append(f"{v},{'inf' if x == K_INF_DIST else x}")
    return "\n".join(out) + "\n"


def certify_distances(g, source, dist, chunk=1 << 24) -> str | None:
    """Optimality certificate for ``dist`` (independent of any solver): the
    source is at 0 and no edge can still relax, i.e. for every edge (u, v, w)
    with dist[u] finite, dist[u] + w >= dist[v] (and dist[v] finite). With a
    valid parent tree (every reached vertex at the end of a tight edge path
    from the source) this proves dist is the exact shortest-path distance.
    Returns None when it holds, else a message. Chunked over edges."""
    g = CsrGraph.of(g)
    off = np.asarray(g.offsets, np.uint64)
    tgt = np.asarray(g.targets, np.uint32)
    w = np.asarray(g.weights, np.uint64)
    dist = np.asarray(dist, np.uint64)
    V = g.vertex_count
    if dist[source] != 0:
        return "dist[source] != 0"
    inf = np.uint64(K_INF_DIST)
    deg = np.diff(off).astype(np.int64)
    E = len(tgt)
    for b in range(0, E, chunk):
        e = min(E, b + chunk)
        # source vertex of each edge in [b, e)
        u0 = int(np.searchsorted(off, b, side="right")) - 1
        u1 = int(np.searchsorted(off, e - 1, side="right")) - 1
        us = np.repeat(np.arange(u0, u1 + 1, dtype=np.int64), deg[u0:u1 + 1])
        first = b - int(off[u0])
        us = us[first:first + (e - b)]
        du = dist[us]
        fin = du != inf
        dv = dist[tgt[b:e]]
        # fin & (dv == inf): a reachable target never reached
        if np.any(fin & (dv == inf)):
            return "reachable vertex left at infinity"
        cand = du[fin] + w[b:e][fin]
        if np.any(cand < du[fin]):
            return "distance overflow"
        if np.any(cand < dv[fin]):
            i = int(np.nonzero(cand < dv[fin])[0][0])
            return f"edge can still relax (edge {b + int(np.nonzero(fin)[0][i])})"
    del V
    return None


def validate_parent_tree(g, source, dist, parent, optimal=False) -> str | None:
    """Shortest-path-tree validator: for every reached v != s,
    parent[v] has an edge to v with dist[v] == dist[parent] + w; the source is
    its own parent; unreachable vertices have no parent. With ``optimal``,
    also the certificate of :func:`certify_distances` (no edge can relax), so
    a consistent-but-wrong dist vector fails. Returns None when valid, else a
    message."""
    g = CsrGraph.of(g)
    off = np.asarray(g.offsets, np.uint64)
    tgt = np.asarray(g.targets, np.uint32)
    w = np.asarray(g.weights, np.uint64)
    dist = np.asarray(dist, np.uint64)
    parent = np.asarray(parent, np.uint32)
    V = g.vertex_count
    if parent[source] != source or dist[source] != 0:
        return "source is not the tree root"
    reached = dist != np.uint64(K_INF_DIST)
    if np.any(parent[~reached] != 0xFFFFFFFF):
        return "unreachable vertex has a parent"
    vs = np.nonzero(reached)[0]
    vs = vs[vs != source]
    if len(vs) == 0:
        return None
    par = parent[vs].astype(np.int64)
    if np.any(par >= V) or np.any(~reached[par]):
        return "parent out of range or unreached"
    # locate edge par -> v in the target-sorted row of par
    lo = off[par].astype(np.int64)
    hi = off[par + 1].astype(np.int64)
    # vectorised binary search per row
    a, b = lo.copy(), hi.copy()
    for _ in range(64):
        m = (a + b) // 2
        go = (a < b) & (tgt[np.minimum(m, len(tgt) - 1)] < vs)
        a = np.where(go, m + 1, a)
        b = np.where(go | (a >= b), b, m)
        if not np.any(a < b):
            break
    ok = (a < hi) & (tgt[np.minimum(a, len(tgt) - 1)] == vs)
    if not np.all(ok):
        return "parent edge missing"
    if not np.all(dist[par] + w[a] == dist[vs]):
        return "dist[v] != dist[parent] + w"
    if optimal:
        return certify_distances(g, source, dist)
    return None


def par_dijkstra_multi_device(g, sources, dist_dev0: int, parent_dev0: int = 0, d: int = 0,
                              devices=(0,)) -> float:
    """pbh_sssp_multi_device: results gathered on devices[0] over NVLink into
    the device buffers at the given addresses (e.g. torch ``data_ptr()``).
    Returns the max-over-devices solve time in ms."""
    g = CsrGraph.of(g)
    cs = g.c_struct()
    src = np.ascontiguousarray(sources, dtype=np.uint32)
    devs = (C.c_int * len(devices))(*devices)
    ms = C.c_double()
    raise_for(_lib.lib().pbh_sssp_multi_device(
        C.byref(cs), src.ctypes.data_as(_lib.U32P), len(src), d, devs, len(devices),
        C.c_void_p(dist_dev0), C.c_void_p(parent_dev0 or None), C.byref(ms)))
    return ms.value


def pin(*arrays):
    """Page-lock numpy arrays for fast host<->device copies (pbh_host_register)."""
    for a in arrays:
        raise_for(_lib.lib().pbh_host_register(C.c_void_p(a.ctypes.data), a.nbytes))


def unpin(*arrays):
    for a in arrays:
        raise_for(_lib.lib().pbh_host_unregister(C.c_void_p(a.ctypes.data)))
