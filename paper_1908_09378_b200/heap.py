"""Host-side mirror of ``pbh::Engine`` (/root/reference/proj/include/pbh/engine.hpp:47-103)
over the pbh-b200 C-ABI. Same method names, argument meaning and exceptions;
every operation executes on the B200 (no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import raise_for

U32P, U64P = _lib.U32P, _lib.U64P


def _ptr(a, t):
    return a.ctypes.data_as(t)


@dataclass
class Element:
    """element.hpp:16-27 (live elements only; DEL signals do not exist here)."""
    value: int
    priority: int

    def __iter__(self):
        return iter((self.value, self.priority))


@dataclass
class EngineConfig:
    """engine.hpp:17-21. ``workers`` is accepted for API parity: the device
    engine runs every resolve inside the owning CTA, so it has no effect on
    results (test_engine.cpp:107-119 pins worker-count independence)."""
    d: int = 1
    workers: int = 1
    debug_assertions: bool = True
    key_universe: int = 0  # extension: initial position-index size (0 = default)
    device: int = 0


@dataclass
class Metrics:
    """engine.hpp:23-31; schema pbh.metrics.v1 (engine.cpp:12-20)."""
    ops: int = 0
    resolves_per_level: list = field(default_factory=list)
    touches_per_level: list = field(default_factory=list)
    wall_ms: float = 0.0

    def to_json(self) -> str:
        return json.dumps({"schema": "pbh.metrics.v1", "ops": self.ops,
                           "resolves_per_level": self.resolves_per_level,
                           "touches_per_level": self.touches_per_level, "wall_ms": self.wall_ms})


@dataclass
class RunResult:
    extracted_values: np.ndarray
    extracted_priorities: np.ndarray
    metrics: Metrics

    @property
    def extracted(self):
        return [Element(int(v), int(p)) for v, p in zip(self.extracted_values,
                                                        self.extracted_priorities)]


class Engine:
    """pbh::Engine on the device. Single-client and blocking, like the reference."""

    def __init__(self, cfg: EngineConfig | None = None, **kw):
        cfg = cfg or EngineConfig(**kw)
        if cfg.workers == 0:
            from .errors import PreconditionError
            raise PreconditionError("engine: workers must be >= 1")  # engine.cpp:26
        self.cfg = cfg
        h = C.c_void_p()
        raise_for(_lib.lib().pbh_heap_create(cfg.d, cfg.key_universe, cfg.device,
                                             int(cfg.debug_assertions), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().pbh_heap_destroy(self._h)
            self._h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- ops (engine.hpp:56-61)
    def update(self, e):
        v, p = e
        raise_for(_lib.lib().pbh_heap_update(self._h, int(v), int(p)))

    def bulk_update(self, batch=None, *, values=None, priorities=None):
        """Engine::bulk_update (engine.cpp:95-98). ``batch`` is a sequence of
        Elements or (value, priority) pairs; columnar input is given by
        keyword (``values=``, ``priorities=``) or as a pair of numpy arrays."""
        if values is not None or priorities is not None:
            if batch is not None or values is None or priorities is None:
                raise TypeError("bulk_update: pass either a batch or values= and priorities=")
            vals, prios = values, priorities
        elif (isinstance(batch, tuple) and len(batch) == 2 and isinstance(batch[0], np.ndarray)
              and isinstance(batch[1], np.ndarray)):
            vals, prios = batch
        else:
            pairs = [tuple(e) for e in batch]  # Element or (value, priority)
            vals = [e[0] for e in pairs]
            prios = [e[1] for e in pairs]
        v = np.ascontiguousarray(vals, dtype=np.uint32)
        p = np.ascontiguousarray(prios, dtype=np.uint64)
        raise_for(_lib.lib().pbh_heap_bulk_update(self._h, _ptr(v, U32P), _ptr(p, U64P), len(v)))

    def extract_min(self) -> Element:
        v, p = C.c_uint32(), C.c_uint64()
        raise_for(_lib.lib().pbh_heap_extract_min(self._h, C.byref(v), C.byref(p)))
        return Element(v.value, p.value)

    def find_min(self) -> Element:
        v, p = C.c_uint32(), C.c_uint64()
        raise_for(_lib.lib().pbh_heap_find_min(self._h, C.byref(v), C.byref(p)))
        return Element(v.value, p.value)

    def delete_value(self, value: int):
        raise_for(_lib.lib().pbh_heap_delete(self._h, int(value)))

    def set_persistent(self, idle_us: int = 200):
        """Latency mode of the single ops (pbh_heap_set_persistent): a
        resident kernel serves them through mapped host memory until idle
        for ``idle_us``; 0 launches one kernel per op."""
        raise_for(_lib.lib().pbh_heap_set_persistent(self._h, int(idle_us)))

    def persist_profile(self) -> dict:
        """pbh_heap_persist_profile: requests served by resident kernels,
        launches, and the resident kernel's wait / copy-in / run time (ns)."""
        o = np.zeros(5, np.uint64)
        raise_for(_lib.lib().pbh_heap_persist_profile(self._h, _ptr(o, U64P)))
        return dict(zip(["requests", "launches", "wait_ns", "copy_ns", "run_ns"], map(int, o)))

    def live_size(self) -> int:
        n = C.c_int64()
        raise_for(_lib.lib().pbh_heap_live_size(self._h, C.byref(n)))
        return n.value

    def drain(self):
        raise_for(_lib.lib().pbh_heap_drain(self._h))

    def snapshot_metrics(self) -> Metrics:
        ops = C.c_uint64()
        res = np.zeros(_lib.MAX_LEVELS, np.uint64)
        tch = np.zeros(_lib.MAX_LEVELS, np.uint64)
        nl = C.c_uint32()
        raise_for(_lib.lib().pbh_heap_metrics(self._h, C.byref(ops), _ptr(res, U64P),
                                              _ptr(tch, U64P), C.byref(nl)))
        n = nl.value
        return Metrics(ops.value, [int(x) for x in res[:n]], [int(x) for x in tch[:n]])

    def stats(self) -> dict:
        """pbh_heap_stats: entries stored below level 0 and stale entries
        dropped by the filtered deep merges (extension)."""
        st, dr = C.c_uint64(), C.c_uint64()
        raise_for(_lib.lib().pbh_heap_stats(self._h, C.byref(st), C.byref(dr)))
        return {"stored_deep": st.value, "stale_dropped": dr.value}

    def check_invariants(self) -> list:
        n = C.c_uint64()
        raise_for(_lib.lib().pbh_heap_check_invariants(self._h, C.byref(n)))
        return [_lib.last_error()] * int(n.value > 0) if n.value else []

    def run_trace(self, trace) -> RunResult:
        """Engine::run_trace (engine.cpp:207-226): the whole trace in one
        device submission, then drain. ``trace`` is any object with flat
        ``kinds``/``offsets``/``vals``/``prios`` arrays."""
        return self._run(trace, _lib.lib().pbh_heap_run_trace)

    def run_ops(self, trace) -> RunResult:
        """The trace's ops as the equivalent sequence of single-client calls
        (update / bulk_update / extract_min / delete_value) in one device
        submission, without run_trace's closing drain (pbh_heap_run_ops)."""
        return self._run(trace, _lib.lib().pbh_heap_run_ops)

    def _run(self, trace, fn) -> RunResult:
        kinds = np.ascontiguousarray(trace.kinds, dtype=np.uint8)
        offs = np.ascontiguousarray(trace.offsets, dtype=np.uint64)
        vals = np.ascontiguousarray(trace.vals, dtype=np.uint32)
        prios = np.ascontiguousarray(trace.prios, dtype=np.uint64)
        n_ops = len(kinds)
        nx = max(int(np.count_nonzero(kinds == ord("E"))), 1)
        ov = np.zeros(nx, np.uint32)
        op = np.zeros(nx, np.uint64)
        n_out, failed = C.c_uint64(), C.c_uint64()
        wall = C.c_double()
        if len(vals) == 0:
            vals = np.zeros(1, np.uint32)
            prios = np.zeros(1, np.uint64)
        if n_ops == 0:
            kinds = np.zeros(1, np.uint8)
        st = fn(self._h, n_ops, _ptr(kinds, _lib.U8P), _ptr(offs, U64P), _ptr(vals, U32P),
                _ptr(prios, U64P), _ptr(ov, U32P), _ptr(op, U64P), C.byref(n_out),
                C.byref(failed), C.byref(wall))
        raise_for(st, op_index=failed.value)
        m = self.snapshot_metrics()
        m.wall_ms = wall.value
        return RunResult(ov[:n_out.value].copy(), op[:n_out.value].copy(), m)
