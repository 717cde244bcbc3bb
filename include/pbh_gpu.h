/* pbh-b200 — C-ABI of the B200-native parBucketHeap hot path.
 *
 * Drop-in boundary for the reference's priority-queue + SSSP API
 * (/root/reference/proj/include/pbh/ headers). Plain pointers and sizes only;
 * no torch or CUDA types. Every entry point returns a pbh_status; the message
 * of the last failure on the calling thread is pbh_last_error().
 *
 * Status codes map one-to-one onto the reference's exception types
 * (/root/reference/proj/include/pbh/error.hpp:9-30):
 *   PBH_EMPTY        -> pbh::EmptyHeapError      (error.hpp:9-12)
 *   PBH_PRECONDITION -> pbh::PreconditionError   (error.hpp:14-18)
 *   PBH_INVARIANT    -> pbh::InvariantError      (error.hpp:20-24)
 *   PBH_TRACE        -> pbh::TraceError{op_index}(error.hpp:26-30)
 * plus PBH_CUDA / PBH_OOM for device failures (no reference equivalent).
 *
 * Threading: a handle owns one CUDA stream and is not thread-safe; distinct
 * handles may be used concurrently ("externally a single-client, blocking
 * interface"). Host pointers are copied; *_device variants take
 * device pointers already resident in HBM on the handle's device.
 */
#ifndef PBH_GPU_H
#define PBH_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PBH_OK = 0,
  PBH_EMPTY = 1,
  PBH_PRECONDITION = 2,
  PBH_INVARIANT = 3,
  PBH_TRACE = 4,
  PBH_CUDA = 5,
  PBH_OOM = 6
} pbh_status;

typedef struct pbh_heap pbh_heap;

/* Message of the last non-OK status returned on this thread. */
const char* pbh_last_error(void);

/* Library version string. */
const char* pbh_version(void);

/* Number of CUDA kernels this library has launched in the process so far
 * (benchmark accounting of gpu_launches). */
uint64_t pbh_launch_count(void);

/* ---- heap lifecycle ---------------------------------------------------
 * Replaces pbh::Engine::Engine(EngineConfig{d, workers, debug_assertions})
 * (engine.hpp:49, engine.cpp:22-30) and BucketHeap(HeapConfig)
 * (bucket_heap.cpp:11-15): d must be in [1, 2^40] else PBH_PRECONDITION.
 * key_universe: initial size of the per-key position index (keys are
 * u32 values); 0 picks a default. The index grows on demand for update
 * keys beyond it; deletes of keys beyond it are no-ops (absent values) that
 * are remembered, so a later insert of such a value is PBH_PRECONDITION
 * like any re-insertion. key_universe > 2^32 -> PBH_PRECONDITION.
 * debug_checks mirrors EngineConfig::debug_assertions with workers == 1
 * (trace_checks, engine.cpp:23-24): priority increases are rejected. */
pbh_status pbh_heap_create(uint64_t d, uint64_t key_universe, int device, int debug_checks,
                           pbh_heap** out);
pbh_status pbh_heap_destroy(pbh_heap* h);

/* ---- single-client ops (engine.hpp:56-61) ------------------------------ */
/* Engine::update(Element) (engine.cpp:90-93; bucket_heap.cpp:101-111):
 * insert-if-absent / decrease-key. Re-inserting an extracted or deleted
 * value -> PBH_PRECONDITION (bucket_heap.cpp:55-58). */
pbh_status pbh_heap_update(pbh_heap* h, uint32_t value, uint64_t priority);
/* Engine::bulk_update(span) (engine.cpp:95-98; bucket_heap.cpp:127-146):
 * 1 <= n <= d, values strictly increasing, else PBH_PRECONDITION. Batches
 * above 2^26 elements (the device batch buffers) are PBH_PRECONDITION too. */
pbh_status pbh_heap_bulk_update(pbh_heap* h, const uint32_t* values, const uint64_t* priorities,
                                uint64_t n);
/* Engine::extract_min() (engine.cpp:100-104): PBH_EMPTY when no live value. */
pbh_status pbh_heap_extract_min(pbh_heap* h, uint32_t* value, uint64_t* priority);
/* BucketHeap::find_min() (bucket_heap.cpp:66-77). */
pbh_status pbh_heap_find_min(pbh_heap* h, uint32_t* value, uint64_t* priority);
/* Engine::delete_value(Value) (engine.cpp:106-109): absent -> no-op. */
pbh_status pbh_heap_delete(pbh_heap* h, uint32_t value);
/* Latency mode of the single ops above (no reference counterpart; the
 * reference runs them on the calling thread, engine.cpp:90-109). With
 * idle_us > 0 (default 200) the first single op leaves one k_trace_bank
 * resident on the heap's stream: later single ops are posted to it through
 * mapped host memory (no launch, no level-0 reload) until it has been idle
 * for idle_us, when it saves its state and exits. Every other call on the
 * heap stops it first. idle_us = 0: one launch per single op. idle_us above
 * 10^7 -> PBH_PRECONDITION. */
pbh_status pbh_heap_set_persistent(pbh_heap* h, uint64_t idle_us);
/* Latency profile of persistent mode: out[0] requests served by resident
 * kernels, out[1] resident kernels launched, out[2..4] nanoseconds the
 * resident kernels spent waiting for requests, copying them in and running
 * them (cumulative; out[2..4] are current once the heap has been stopped by
 * any non-single-op call or the kernel's idle exit). */
pbh_status pbh_heap_persist_profile(pbh_heap* h, uint64_t out[5]);
/* Engine::live_size() (engine.hpp:61). */
pbh_status pbh_heap_live_size(pbh_heap* h, int64_t* n);
/* Engine::drain() (engine.cpp:138-150): flush all signal buffers. */
pbh_status pbh_heap_drain(pbh_heap* h);

/* Engine::snapshot_metrics() (engine.cpp:152-163), schema pbh.metrics.v1:
 * ops, resolves/touches per level for levels [0, *n_levels). Arrays must
 * hold PBH_GPU_MAX_LEVELS entries. */
#define PBH_GPU_MAX_LEVELS 24
pbh_status pbh_heap_metrics(pbh_heap* h, uint64_t* ops, uint64_t* resolves_per_level,
                            uint64_t* touches_per_level, uint32_t* n_levels);

/* Storage counters (no reference counterpart): entries stored below level 0
 * (live copies plus stale ones not yet dropped) and the stale entries the
 * filtered grid / streamed merges have dropped so far (drop_stale_duplicates,
 * primitives.cpp:103-120, done through the position index). */
pbh_status pbh_heap_stats(pbh_heap* h, uint64_t* stored_deep, uint64_t* stale_dropped);

/* Structural audit (BucketHeap::check_invariants, bucket_heap.cpp:302-409)
 * restated for the (priority, value)-sorted SoA levels: sortedness, splitter
 * separation, capacity, live count. Returns the number of violations in
 * *n_violations (0 = clean). Blocking; copies the levels to the host. */
pbh_status pbh_heap_check_invariants(pbh_heap* h, uint64_t* n_violations);

/* ---- op traces (trace_format.hpp:16-33; engine.cpp:207-226) -------------
 * Flat trace: op i has kind kinds[i] in {'U','B','E','D'} and owns elements
 * [offsets[i], offsets[i+1]) of values/priorities (D: one value, E: none).
 * Engine::run_trace: replays the whole trace in ONE device submission, then
 * drains. out_values/out_priorities receive the extracted elements in order
 * (capacity = number of 'E' ops); *n_out their count. On an op failure the
 * status is PBH_TRACE and *failed_op the op index (TraceError::op_index);
 * out arrays then hold the extractions before it. wall_ms (nullable) is the
 * device-timed replay, like Metrics::wall_ms. */
pbh_status pbh_heap_run_trace(pbh_heap* h, uint64_t n_ops, const uint8_t* kinds,
                              const uint64_t* offsets, const uint32_t* values,
                              const uint64_t* priorities, uint32_t* out_values,
                              uint64_t* out_priorities, uint64_t* n_out, uint64_t* failed_op,
                              double* wall_ms);
/* The op sequence of a trace executed exactly as the same sequence of
 * single-client calls (Engine::update / bulk_update / extract_min /
 * delete_value, engine.cpp:90-109) would execute it, in ONE device
 * submission, WITHOUT run_trace's closing drain: the device form of a
 * caller's loop over bulk_update (the C4 sweep is timed through it, like the
 * reference's bulk_update batches). Same arguments and errors as
 * pbh_heap_run_trace (a failing op -> PBH_TRACE with *failed_op). */
pbh_status pbh_heap_run_ops(pbh_heap* h, uint64_t n_ops, const uint8_t* kinds,
                            const uint64_t* offsets, const uint32_t* values,
                            const uint64_t* priorities, uint32_t* out_values,
                            uint64_t* out_priorities, uint64_t* n_out, uint64_t* failed_op,
                            double* wall_ms);
/* Same with every pointer in device memory (inputs resident in HBM). */
pbh_status pbh_heap_run_trace_device(pbh_heap* h, uint64_t n_ops, const uint8_t* d_kinds,
                                     const uint64_t* d_offsets, const uint32_t* d_values,
                                     const uint64_t* d_priorities, uint32_t* d_out_values,
                                     uint64_t* d_out_priorities, uint64_t* n_out,
                                     uint64_t* failed_op, double* wall_ms);

/* ---- SSSP (sssp.hpp:13-29) ----------------------------------------------
 * par_dijkstra(g, source, EngineConfig{d}, dag_mode) (sssp.cpp:21-69) as
 * ONE persistent CTA per source. CSR: offsets u64[V+1], targets u32[E],
 * weights u32[E] (graphs.hpp:11-20). d == 0 selects max(1, max out-degree).
 * Outputs (caller-allocated, nullable except dist): dist u64[V] (kInfDist =
 * ~0 where unreachable), parent u32[V] (predecessor on a shortest-path tree;
 * source -> source, unreachable -> 0xFFFFFFFF; an extension: SsspResult has
 * no parent field), settled u32[V] (extraction order), *n_settled, *rounds,
 * *ops (Metrics::ops). debug_checks as in pbh_heap_create. */
typedef struct {
  uint32_t vertex_count;
  uint64_t edge_count;
  const uint64_t* offsets;
  const uint32_t* targets;
  const uint32_t* weights;
} pbh_csr;

pbh_status pbh_sssp(const pbh_csr* g, uint32_t source, uint64_t d, int dag_mode, int device,
                    uint64_t* dist, uint32_t* parent, uint32_t* settled, uint64_t* n_settled,
                    uint64_t* rounds, uint64_t* ops);

/* Multi-source batch (BASELINE config 5): n_sources independent
 * par_dijkstra runs. Sources are dealt contiguously over `n_devices`
 * devices; each device holds a replica of the CSR and runs its sources as
 * concurrent persistent CTAs; results are gathered to the host. dist is
 * n_sources x V (row-major), parent likewise (nullable). */
pbh_status pbh_sssp_multi(const pbh_csr* g, const uint32_t* sources, uint64_t n_sources,
                          uint64_t d, const int* devices, int n_devices, uint64_t* dist,
                          uint32_t* parent);

/* Device-resident SSSP context for timing with inputs already in HBM:
 * the CSR is uploaded once; each pbh_sssp_ctx_run solves n_sources sources
 * on this device and leaves dist/parent in device memory. */
typedef struct pbh_sssp_ctx pbh_sssp_ctx;
pbh_status pbh_sssp_ctx_create(const pbh_csr* g, uint64_t d, int device, uint64_t max_sources,
                               pbh_sssp_ctx** out);
pbh_status pbh_sssp_ctx_run(pbh_sssp_ctx* c, const uint32_t* sources, uint64_t n_sources,
                            int dag_mode, double* device_ms);
pbh_status pbh_sssp_ctx_fetch(pbh_sssp_ctx* c, uint64_t source_slot, uint64_t* dist,
                              uint32_t* parent, uint32_t* settled, uint64_t* n_settled,
                              uint64_t* rounds, uint64_t* ops);
/* Extension: mode 1 = threshold multi-extraction.
 * Each round settles every level-0 vertex whose distance is final by the
 * Crauser IN/OUT criteria; distances and parents are exact/valid, `rounds`
 * counts batches, `settled` lists vertices in batch order (sort by
 * (dist, vid) for the reference's settle order). mode 0 = par_dijkstra. */
pbh_status pbh_sssp_ctx_set_mode(pbh_sssp_ctx* c, int mode);
/* Re-upload a CSR of the same shape (vertex_count, edge_count and max
 * out-degree) into a live context (host or device arrays), e.g. a serving
 * loop that receives a new graph per request without re-allocating the
 * per-source heaps. PRECONDITION if the shape differs. */
pbh_status pbh_sssp_ctx_load_graph(pbh_sssp_ctx* c, const pbh_csr* g);
pbh_status pbh_sssp_ctx_destroy(pbh_sssp_ctx* c);

/* The multi-source batch of pbh_sssp_multi with the results gathered on
 * devices[0] over NVLink (peer copies, no collective): dist_dev0 /
 * parent_dev0 (may be NULL) are device pointers on devices[0] holding
 * n_sources * V entries, source-major. device_ms = max over devices of the
 * solve time. */
pbh_status pbh_sssp_multi_device(const pbh_csr* g, const uint32_t* sources, uint64_t n_sources,
                                 uint64_t d, const int* devices, int n_devices,
                                 uint64_t* dist_dev0, uint32_t* parent_dev0, double* device_ms);

/* bellman_ford (sssp.hpp:37, sssp.cpp:99-129) on the device: a frontier
 * label-correcting sweep (one cooperative grid, 64-bit atomicMin), the
 * baseline the bucket heap is compared with. Distances are
 * the exact shortest-path distances; parent (optional) is a valid
 * shortest-path tree recovered from tight edges, parent[source] = source;
 * rounds = frontier iterations (the reference counts full sweeps). */
pbh_status pbh_bellman_ford(const pbh_csr* g, uint32_t source, int device, uint64_t* dist,
                            uint32_t* parent, uint64_t* rounds, uint64_t* edges_scanned,
                            double* device_ms);

/* Page-lock a caller-owned host range (cudaHostRegister, portable) so the
 * CSR uploads and result downloads of pbh_sssp / pbh_sssp_multi run at DMA
 * speed; no reference counterpart (the reference is host-only). */
pbh_status pbh_host_register(void* ptr, uint64_t bytes);
pbh_status pbh_host_unregister(void* ptr);

/* ---- CSR input contract (graphs.hpp:11-23) -------------------------------
 * validate_graph (graphs.hpp:23, graphs.cpp:55-72) as one device pass over
 * host or device arrays: PBH_INVARIANT with the reference's message for the
 * violation its sequential loop would report first ("graph: inconsistent
 * array sizes", "graph: offsets not monotone", "graph: target out of range",
 * "graph: self-loop", "graph: row not sorted or parallel edge",
 * "graph: zero weight"). The SSSP entry points (pbh_sssp*, pbh_sssp_ctx_create,
 * pbh_sssp_ctx_load_graph, pbh_bellman_ford) run the same pass and return
 * PBH_PRECONDITION for the violations that would make a kernel read out of
 * bounds (sizes, offsets, targets >= V). */
pbh_status pbh_validate_graph(const pbh_csr* g, int device);
/* CsrGraph::max_out_degree() (graphs.hpp:18, graphs.cpp:47-53): on the host
 * for host offsets, on `device` for device arrays. */
pbh_status pbh_csr_max_out_degree(const pbh_csr* g, int device, uint32_t* out);

/* ---- multi-source gather (BASELINE C5) --------------------
 * Copy the dist / parent rows of source slots [first_slot, first_slot +
 * n_slots) of the last pbh_sssp_ctx_run into dist_dst (n_slots x V u64) /
 * parent_dst (n_slots x V u32), either nullable. The destination may be host
 * memory, this device, a peer device (NVLink peer copy) or a buffer of
 * another process mapped with pbh_ipc_open: one process per GPU gathers into
 * GPU 0 without a collective. Blocking. */
pbh_status pbh_sssp_ctx_gather(pbh_sssp_ctx* c, uint64_t first_slot, uint64_t n_slots,
                               uint64_t* dist_dst, uint32_t* parent_dst);

/* Device buffers shareable across processes (CUDA IPC): pbh_device_alloc on
 * the gathering GPU, pbh_ipc_export its 64-byte handle, pbh_ipc_open it in
 * each peer process (peer access enabled lazily), pbh_ipc_close when done.
 * pbh_copy is a blocking copy between any two of host / device / peer /
 * IPC-mapped memory. No reference counterpart (the reference is host-only). */
pbh_status pbh_device_alloc(int device, uint64_t bytes, void** ptr);
pbh_status pbh_device_free(int device, void* ptr);
pbh_status pbh_ipc_export(void* dev_ptr, uint8_t handle[64]);
pbh_status pbh_ipc_open(const uint8_t handle[64], int device, void** ptr);
pbh_status pbh_ipc_close(int device, void* ptr);
pbh_status pbh_copy(void* dst, const void* src, uint64_t bytes);

/* distance_checksum (sssp.cpp:174-183): FNV-1a over the distance bytes. */
uint64_t pbh_distance_checksum(const uint64_t* dist, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif
