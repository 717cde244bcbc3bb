"""pbh-b200: a B200-native parBucketHeap (arXiv 1908.09378) hot path.

The product is the C-ABI library ``libpbh_gpu.so`` (include/pbh_gpu.h) built
from ``csrc/`` for sm_100a; this package is the host-side mirror of the
reference's C++ interface used by tests and the benchmark.
"""
from .errors import (DeviceError, EmptyHeapError, InvariantError, PreconditionError,  # noqa: F401
                     TraceError)
from .heap import Element, Engine, EngineConfig, Metrics, RunResult  # noqa: F401
from .sssp import (K_INF_DIST, CsrGraph, bellman_ford, SsspContext, SsspResult, distance_checksum,  # noqa: F401
                   certify_distances, distances_to_csv, max_out_degree, par_dijkstra,
                   par_dijkstra_multi, par_dijkstra_multi_device, pin, threshold_sssp, unpin,
                   validate_graph, validate_parent_tree)
