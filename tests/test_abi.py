"""C-ABI boundary checks that need no GPU: the library loads and exports every
symbol include/pbh_gpu.h declares, and the Python mirror binds them all."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols(header="pbh_gpu.h"):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pbh_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1908_09378_b200 import _lib
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_python_mirror_binds_every_symbol():
    from paper_1908_09378_b200 import _lib, gen
    assert set(declared_symbols()) == set(_lib.SIGNATURES)
    assert set(declared_symbols("pbh_gen.h")) == set(gen.GEN_SIGNATURES)
    from paper_1908_09378_b200 import trace_io
    assert set(declared_symbols("pbh_trace_io.h")) == set(trace_io.IO_SIGNATURES)
    L = _lib.lib()
    assert all(hasattr(L, s) for s in gen.GEN_SIGNATURES)
    assert all(hasattr(L, s) for s in trace_io.IO_SIGNATURES)


def test_version_and_error_without_gpu():
    from paper_1908_09378_b200 import _lib
    assert b"sm_100a" in _lib.lib().pbh_version()
    # d == 0 is rejected before any device call (bucket_heap.cpp:13)
    import ctypes as C
    h = C.c_void_p()
    st = _lib.lib().pbh_heap_create(0, 0, 0, 1, C.byref(h))
    assert st == _lib.PRECONDITION
    assert "d must be positive" in _lib.last_error()


def test_checksum_matches_oracle():
    import numpy as np
    from paper_1908_09378_b200 import distance_checksum
    from oracle import oracle as O
    d = np.array([0, 4, 2 ** 64 - 1, 123456789], np.uint64)
    assert distance_checksum(d) == O.checksum(d)
