"""Exception types of the reference (/root/reference/proj/include/pbh/error.hpp:9-30).

The C-ABI returns a pbh_status; ``raise_for`` maps it back onto the same four
types the reference throws, so callers (and the parity tests) catch the same
errors they would catch from ``pbh::Engine``.
"""
from __future__ import annotations

from . import _lib


class PbhError(RuntimeError):
    pass


class EmptyHeapError(PbhError):
    """error.hpp:9-12 — extract_min / find_min on a heap with no live value."""


class PreconditionError(PbhError):
    """error.hpp:14-18 — bad arguments, malformed batch, illegal trace."""


class InvariantError(PbhError):
    """error.hpp:20-24 — internal invariant failure."""


class TraceError(PbhError):
    """error.hpp:26-30 — replay failure carrying the offending op index."""

    def __init__(self, op_index, msg):
        super().__init__(msg)
        self.op_index = op_index


class DeviceError(PbhError):
    """CUDA failure or device allocation failure (PBH_CUDA / PBH_OOM)."""


def raise_for(status: int, op_index=None):
    if status == _lib.OK:
        return
    msg = _lib.last_error()
    if status == _lib.EMPTY:
        raise EmptyHeapError(msg)
    if status == _lib.PRECONDITION:
        raise PreconditionError(msg)
    if status == _lib.INVARIANT:
        raise InvariantError(msg)
    if status == _lib.TRACE:
        raise TraceError(op_index, msg)
    raise DeviceError(f"status {status}: {msg}")
