"""Op-trace files (include/pbh_trace_io.h): the reference's text format
(trace_format.cpp:34-126) and the packed binary form with a streaming chunk
reader, in the flat layout of Engine.run_trace."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import TraceError

U8P, U32P, U64P = _lib.U8P, _lib.U32P, _lib.U64P
U64R = C.POINTER(C.c_uint64)

IO_SIGNATURES = {
    "pbh_trace_load_text": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p), U64R]),
    "pbh_trace_buf_sizes": (None, [C.c_void_p, U64R, U64R]),
    "pbh_trace_buf_export": (None, [C.c_void_p, U8P, U64P, U32P, U64P]),
    "pbh_trace_buf_free": (None, [C.c_void_p]),
    "pbh_trace_save_text": (C.c_int, [C.c_char_p, C.c_uint64, U8P, U64P, U32P, U64P]),
    "pbh_trace_save_binary": (C.c_int, [C.c_char_p, C.c_uint64, U8P, U64P, U32P, U64P]),
    "pbh_trace_open_binary": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p), U64R, U64R]),
    "pbh_trace_chunk_elems": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, U64R]),
    "pbh_trace_read_chunk": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, U8P, U64P, U32P,
                                       U64P]),
    "pbh_trace_close": (None, [C.c_void_p]),
    "pbh_trace_last_error": (C.c_char_p, []),
}

_bound = False


def _L():
    global _bound
    L = _lib.lib()
    if not _bound:
        for name, (res, args) in IO_SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _bound = True
    return L


def _err():
    return _L().pbh_trace_last_error().decode()


@dataclass
class FlatTrace:
    kinds: np.ndarray    # u8 'U','B','E','D'
    offsets: np.ndarray  # u64[n_ops + 1]
    vals: np.ndarray     # u32
    prios: np.ndarray    # u64

    @property
    def n_ops(self):
        return len(self.kinds)


def _flat(tr):
    return (np.ascontiguousarray(tr.kinds, np.uint8), np.ascontiguousarray(tr.offsets, np.uint64),
            np.ascontiguousarray(tr.vals if len(tr.vals) else [0], np.uint32),
            np.ascontiguousarray(tr.prios if len(tr.prios) else [0], np.uint64))


def load_text(path) -> FlatTrace:
    """load_trace (trace_format.cpp:92-96); raises TraceError(op_index)."""
    L = _L()
    h = C.c_void_p()
    failed = C.c_uint64()
    st = L.pbh_trace_load_text(str(path).encode(), C.byref(h), C.byref(failed))
    if st:
        raise TraceError(failed.value, _err())
    try:
        no, ne = C.c_uint64(), C.c_uint64()
        L.pbh_trace_buf_sizes(h, C.byref(no), C.byref(ne))
        t = FlatTrace(np.zeros(max(no.value, 1), np.uint8), np.zeros(no.value + 1, np.uint64),
                      np.zeros(max(ne.value, 1), np.uint32), np.zeros(max(ne.value, 1), np.uint64))
        L.pbh_trace_buf_export(h, t.kinds.ctypes.data_as(U8P), t.offsets.ctypes.data_as(U64P),
                               t.vals.ctypes.data_as(U32P), t.prios.ctypes.data_as(U64P))
    finally:
        L.pbh_trace_buf_free(h)
    return FlatTrace(t.kinds[:no.value], t.offsets, t.vals[:ne.value], t.prios[:ne.value])


def save_text(tr, path):
    """save_trace (trace_format.cpp:121-126)."""
    k, o, v, p = _flat(tr)
    st = _L().pbh_trace_save_text(str(path).encode(), len(tr.kinds), k.ctypes.data_as(U8P),
                                  o.ctypes.data_as(U64P), v.ctypes.data_as(U32P),
                                  p.ctypes.data_as(U64P))
    if st:
        raise TraceError(0, _err())


def save_binary(tr, path):
    k, o, v, p = _flat(tr)
    st = _L().pbh_trace_save_binary(str(path).encode(), len(tr.kinds), k.ctypes.data_as(U8P),
                                    o.ctypes.data_as(U64P), v.ctypes.data_as(U32P),
                                    p.ctypes.data_as(U64P))
    if st:
        raise TraceError(0, _err())


class BinaryTraceReader:
    """Streams op ranges of a packed binary trace."""

    def __init__(self, path):
        h = C.c_void_p()
        no, ne = C.c_uint64(), C.c_uint64()
        if _L().pbh_trace_open_binary(str(path).encode(), C.byref(h), C.byref(no), C.byref(ne)):
            raise TraceError(0, _err())
        self._h, self.n_ops, self.n_elems = h, no.value, ne.value

    def read(self, op0, n) -> FlatTrace:
        L = _L()
        ne = C.c_uint64()
        if L.pbh_trace_chunk_elems(self._h, op0, n, C.byref(ne)):
            raise TraceError(op0, _err())
        t = FlatTrace(np.zeros(max(n, 1), np.uint8), np.zeros(n + 1, np.uint64),
                      np.zeros(max(ne.value, 1), np.uint32), np.zeros(max(ne.value, 1), np.uint64))
        if L.pbh_trace_read_chunk(self._h, op0, n, t.kinds.ctypes.data_as(U8P),
                                  t.offsets.ctypes.data_as(U64P), t.vals.ctypes.data_as(U32P),
                                  t.prios.ctypes.data_as(U64P)):
            raise TraceError(op0, _err())
        return FlatTrace(t.kinds[:n], t.offsets, t.vals[:ne.value], t.prios[:ne.value])

    def chunks(self, chunk_ops):
        for op0 in range(0, self.n_ops, chunk_ops):
            yield op0, self.read(op0, min(chunk_ops, self.n_ops - op0))

    def close(self):
        if getattr(self, "_h", None):
            _L().pbh_trace_close(self._h)
            self._h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def run_trace_file(engine, path, chunk_ops=1 << 16):
    """Replay a binary trace through ``engine`` chunk by chunk (the heap state
    stays in HBM between chunks). Returns (extracted values, priorities,
    total device ms). A failing op raises TraceError with its global index."""
    vs, ps, ms = [], [], 0.0
    with BinaryTraceReader(path) as r:
        for op0, ch in r.chunks(chunk_ops):
            try:
                res = engine.run_trace(ch)
            except TraceError as e:
                raise TraceError(op0 + (e.op_index or 0), str(e)) from None
            vs.append(res.extracted_values)
            ps.append(res.extracted_priorities)
            ms += res.metrics.wall_ms
    cat = (lambda xs, dt: np.concatenate(xs) if xs else np.zeros(0, dt))
    return cat(vs, np.uint32), cat(ps, np.uint64), ms
