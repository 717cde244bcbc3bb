"""Multi-source SSSP across GPUs, one process per GPU (BASELINE C5,
SURVEY.md §8e): independent sources sharded contiguously over ranks, each
rank solving its shard with one persistent CTA per source on its own replica
of the CSR, the results gathered into one buffer on GPU 0 over NVLink by
peer copies into CUDA-IPC-mapped memory. No collective touches the data
path; torch.distributed only carries the IPC handle, barriers and the
max-over-ranks timing.

The per-source unit is the reference's ``par_dijkstra``
(/root/reference/proj/src/sssp.cpp:21-69).
"""
from __future__ import annotations

import ctypes as C

from . import _lib
from .errors import raise_for

C5_SOURCES = tuple(i * 16384 for i in range(64))  # s_i = i * 16384


def shard(n_sources: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous source range [b, e) of ``rank``: the first n % world ranks
    take one extra source. Ranks beyond n_sources get an empty range."""
    base, extra = divmod(n_sources, world)
    b = rank * base + min(rank, extra)
    return b, b + base + (1 if rank < extra else 0)


class DeviceBuffer:
    """A raw device allocation (pbh_device_alloc) that other processes can map
    (pbh_ipc_export / pbh_ipc_open)."""

    def __init__(self, device: int, nbytes: int, *, _ptr: int | None = None, _mapped=False):
        self.device, self.nbytes, self.mapped = device, nbytes, _mapped
        if _ptr is None:
            p = C.c_void_p()
            raise_for(_lib.lib().pbh_device_alloc(device, nbytes, C.byref(p)))
            _ptr = p.value
        self.ptr = _ptr

    def handle(self) -> bytes:
        """The 64-byte CUDA IPC handle of this allocation."""
        h = (C.c_uint8 * 64)()
        raise_for(_lib.lib().pbh_ipc_export(C.c_void_p(self.ptr), h))
        return bytes(h)

    @classmethod
    def open(cls, handle: bytes, device: int, nbytes: int) -> "DeviceBuffer":
        """Map another process's allocation into this one (peer access is
        enabled lazily, so copies into it run over NVLink)."""
        h = (C.c_uint8 * 64).from_buffer_copy(handle)
        p = C.c_void_p()
        raise_for(_lib.lib().pbh_ipc_open(h, device, C.byref(p)))
        return cls(device, nbytes, _ptr=p.value, _mapped=True)

    def copy_to_host(self, arr, offset: int = 0):
        """Blocking D2H of arr.nbytes bytes starting at byte ``offset``."""
        assert offset + arr.nbytes <= self.nbytes
        raise_for(_lib.lib().pbh_copy(C.c_void_p(arr.ctypes.data), C.c_void_p(self.ptr + offset),
                                      arr.nbytes))

    def close(self):
        if getattr(self, "ptr", None):
            if self.mapped:
                _lib.lib().pbh_ipc_close(self.device, C.c_void_p(self.ptr))
            else:
                _lib.lib().pbh_device_free(self.device, C.c_void_p(self.ptr))
            self.ptr = None

    __del__ = close


class GatherPlan:
    """Where rank r's source rows land in the gathered, source-major result
    on GPU 0: dist (u64) rows first, then parent (u32) rows."""

    def __init__(self, n_sources: int, V: int, world: int):
        self.n, self.V, self.world = n_sources, V, world
        self.dist_bytes = n_sources * V * 8
        self.parent_bytes = n_sources * V * 4
        self.nbytes = self.dist_bytes + self.parent_bytes

    def rows(self, rank: int) -> tuple[int, int]:
        return shard(self.n, self.world, rank)

    def dist_offset(self, rank: int) -> int:
        return self.rows(rank)[0] * self.V * 8

    def parent_offset(self, rank: int) -> int:
        return self.dist_bytes + self.rows(rank)[0] * self.V * 4
