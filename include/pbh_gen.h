/* pbh-b200 — synthetic workload generators for the BASELINE configs
 * (SURVEY.md §8d). Host C++ (no device work); they produce the inputs the
 * benchmark feeds through include/pbh_gpu.h. The CPU oracle restates each
 * one independently (oracle/pbh_oracle.c) and tests/test_gen.py requires
 * both to agree draw for draw (std::mt19937_64 with rng() % n, as in
 * /root/reference/proj/src/graphs.cpp:15-17).
 */
#ifndef PBH_GEN_H
#define PBH_GEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* C2: rows x cols 4-neighbour grid; offsets u64[V+1], targets/weights u32[E]
 * with E = pbh_gen_grid_edges(rows, cols). Weights 1 + rng()%(2^32-1). */
uint64_t pbh_gen_grid_edges(uint32_t rows, uint32_t cols);
void pbh_gen_grid(uint32_t rows, uint32_t cols, uint64_t seed, uint64_t* offsets,
                  uint32_t* targets, uint32_t* weights);

/* C3: ring band, row u -> (u + j) mod V, j = 1..degree, target-sorted; spine
 * weight 1 on u -> u+1 (u + 1 < V), others V + rng()%1000. E = V * degree. */
void pbh_gen_band(uint32_t v, uint32_t degree, uint64_t seed, uint64_t* offsets,
                  uint32_t* targets, uint32_t* weights);

/* C1: mixed bulkUpdate / extractMin trace (definition in
 * oracle/pbh_oracle.c:orc_trace_gen_mixed). Handle-based: generate, query
 * sizes, export into caller arrays, free. */
typedef struct pbh_gen_trace pbh_gen_trace;
pbh_gen_trace* pbh_gen_mixed_trace(uint64_t n_ops, uint64_t universe, uint64_t kmax,
                                   uint64_t seed);
void pbh_gen_trace_sizes(const pbh_gen_trace* t, uint64_t* n_ops, uint64_t* n_elems,
                         uint64_t* n_extract);
void pbh_gen_trace_export(const pbh_gen_trace* t, uint8_t* kinds, uint64_t* offsets,
                          uint32_t* values, uint64_t* priorities);
void pbh_gen_trace_free(pbh_gen_trace* t);

/* C4: prefill keys [0, n) with priorities uniform in [2^39, 2^40) (seed),
 * then n_batches batches of d distinct live keys, value-sorted, each a
 * strict decrease p -= 1 + rng()%1024. prios_now (u64[n]) carries the
 * current priorities between calls; call prefill once, batches repeatedly. */
void pbh_gen_sweep_prefill(uint64_t n, uint64_t seed, uint64_t* prios_now);
void pbh_gen_sweep_batches(uint64_t n, uint64_t d, uint64_t n_batches, uint64_t seed,
                           uint64_t* prios_now, uint32_t* values, uint64_t* priorities);

/* Device versions: the same C2 grid / C3 band built
 * directly in device memory (pointers on `device`), bit-identical to the host
 * generators; one CTA replays std::mt19937_64 twist by twist. Return a
 * pbh_status (0 = ok). The CSR may then be passed to pbh_sssp_ctx_create as
 * device pointers (copied device-to-device). */
int pbh_gen_grid_device(uint32_t rows, uint32_t cols, uint64_t seed, int device,
                        uint64_t* offsets, uint32_t* targets, uint32_t* weights);
int pbh_gen_band_device(uint32_t v, uint32_t degree, uint64_t seed, int device,
                        uint64_t* offsets, uint32_t* targets, uint32_t* weights);

#ifdef __cplusplus
}
#endif
#endif
