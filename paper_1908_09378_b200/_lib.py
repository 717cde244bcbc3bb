"""Loader for the in-tree C-ABI library ``libpbh_gpu.so`` (include/pbh_gpu.h).

There is no CPU fallback: if the shared library is missing or fails to load,
every entry point raises. Build it with ``python -c "import __graft_entry__ as
g; g.build()"`` (or ``make -C paper_1908_09378_b200``).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libpbh_gpu.so")

U8P, U32P, U64P, I64P = (C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                         C.POINTER(C.c_int64))
DBLP = C.POINTER(C.c_double)

# pbh_status
OK, EMPTY, PRECONDITION, INVARIANT, TRACE, CUDA, OOM = range(7)
MAX_LEVELS = 24


class Csr(C.Structure):
    _fields_ = [("vertex_count", C.c_uint32), ("edge_count", C.c_uint64),
                ("offsets", U64P), ("targets", U32P), ("weights", U32P)]


# name -> (restype, argtypes); mirrors include/pbh_gpu.h exactly
SIGNATURES = {
    "pbh_last_error": (C.c_char_p, []),
    "pbh_version": (C.c_char_p, []),
    "pbh_launch_count": (C.c_uint64, []),
    "pbh_heap_create": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "pbh_heap_destroy": (C.c_int, [C.c_void_p]),
    "pbh_heap_update": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint64]),
    "pbh_heap_bulk_update": (C.c_int, [C.c_void_p, U32P, U64P, C.c_uint64]),
    "pbh_heap_extract_min": (C.c_int, [C.c_void_p, U32P, U64P]),
    "pbh_heap_find_min": (C.c_int, [C.c_void_p, U32P, U64P]),
    "pbh_heap_delete": (C.c_int, [C.c_void_p, C.c_uint32]),
    "pbh_heap_set_persistent": (C.c_int, [C.c_void_p, C.c_uint64]),
    "pbh_heap_persist_profile": (C.c_int, [C.c_void_p, U64P]),
    "pbh_heap_live_size": (C.c_int, [C.c_void_p, I64P]),
    "pbh_heap_drain": (C.c_int, [C.c_void_p]),
    "pbh_heap_metrics": (C.c_int, [C.c_void_p, U64P, U64P, U64P, U32P]),
    "pbh_heap_stats": (C.c_int, [C.c_void_p, U64P, U64P]),
    "pbh_heap_check_invariants": (C.c_int, [C.c_void_p, U64P]),
    "pbh_heap_run_trace": (C.c_int, [C.c_void_p, C.c_uint64, U8P, U64P, U32P, U64P, U32P, U64P,
                                     U64P, U64P, DBLP]),
    "pbh_heap_run_ops": (C.c_int, [C.c_void_p, C.c_uint64, U8P, U64P, U32P, U64P, U32P, U64P,
                                   U64P, U64P, DBLP]),
    "pbh_heap_run_trace_device": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, U64P,
                                            U64P, DBLP]),
    "pbh_sssp": (C.c_int, [C.POINTER(Csr), C.c_uint32, C.c_uint64, C.c_int, C.c_int, U64P, U32P,
                           U32P, U64P, U64P, U64P]),
    "pbh_sssp_multi": (C.c_int, [C.POINTER(Csr), U32P, C.c_uint64, C.c_uint64,
                                 C.POINTER(C.c_int), C.c_int, U64P, U32P]),
    "pbh_sssp_ctx_create": (C.c_int, [C.POINTER(Csr), C.c_uint64, C.c_int, C.c_uint64,
                                      C.POINTER(C.c_void_p)]),
    "pbh_sssp_ctx_run": (C.c_int, [C.c_void_p, U32P, C.c_uint64, C.c_int, DBLP]),
    "pbh_sssp_ctx_fetch": (C.c_int, [C.c_void_p, C.c_uint64, U64P, U32P, U32P, U64P, U64P, U64P]),
    "pbh_sssp_ctx_destroy": (C.c_int, [C.c_void_p]),
    "pbh_distance_checksum": (C.c_uint64, [U64P, C.c_uint64]),
    "pbh_host_register": (C.c_int, [C.c_void_p, C.c_uint64]),
    "pbh_sssp_ctx_set_mode": (C.c_int, [C.c_void_p, C.c_int]),
    "pbh_sssp_ctx_load_graph": (C.c_int, [C.c_void_p, C.c_void_p]),
    "pbh_sssp_multi_device": (C.c_int, [C.POINTER(Csr), U32P, C.c_uint64, C.c_uint64,
                                        C.POINTER(C.c_int), C.c_int, C.c_void_p, C.c_void_p,
                                        C.POINTER(C.c_double)]),
    "pbh_bellman_ford": (C.c_int, [C.POINTER(Csr), C.c_uint32, C.c_int, U64P, U32P,
                                   C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                   C.POINTER(C.c_double)]),
    "pbh_host_unregister": (C.c_int, [C.c_void_p]),
    "pbh_validate_graph": (C.c_int, [C.POINTER(Csr), C.c_int]),
    "pbh_csr_max_out_degree": (C.c_int, [C.POINTER(Csr), C.c_int, U32P]),
    "pbh_sssp_ctx_gather": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p]),
    "pbh_device_alloc": (C.c_int, [C.c_int, C.c_uint64, C.POINTER(C.c_void_p)]),
    "pbh_device_free": (C.c_int, [C.c_int, C.c_void_p]),
    "pbh_ipc_export": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8)]),
    "pbh_ipc_open": (C.c_int, [C.POINTER(C.c_uint8), C.c_int, C.POINTER(C.c_void_p)]),
    "pbh_ipc_close": (C.c_int, [C.c_int, C.c_void_p]),
    "pbh_copy": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
}

_lib = None


def lib():
    """The loaded C-ABI library. Raises if it is not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(f"pbh-b200 CUDA library not built: {SO_PATH} is missing "
                              "(run __graft_entry__.build())")
        L = C.CDLL(SO_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().pbh_last_error().decode(errors="replace")
