/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the pbh-b200 hot path.
 *
 * A plain-C restatement of the reference's algorithms, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the CHECKER.
 * Nothing on the product path links or calls this. Each function cites the
 * reference file:line it restates (paths relative to /root/reference/proj).
 *
 * Parity of this restatement is pinned against the reference itself: the
 * golden fixtures in tests/golden/ were produced by the unmodified reference
 * library (oracle/_ref, built by `make -C oracle ref`), see
 * tests/golden/make_golden.py and tests/test_oracle.py.
 */
#ifndef PBH_ORACLE_H
#define PBH_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- std::mt19937_64 (graphs.cpp:15-17 draws rng() % n) -------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_mt64;
void orc_mt64_seed(orc_mt64* r, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* r);

/* ---- op traces (trace_format.hpp:16-33), flat layout ------------------ *
 * kinds[i] in {'U','B','E','D'}; op i owns elements [offsets[i], offsets[i+1]). */
typedef struct {
  uint64_t n_ops, n_elems;
  uint8_t* kinds;
  uint64_t* offsets;
  uint32_t* vals;
  uint64_t* prios;
  uint64_t n_extract;
} orc_trace;

/* gen_legal_trace (tests/oracle.hpp:82-155). */
orc_trace* orc_trace_gen_legal(uint64_t n_ops, uint64_t d, uint64_t seed);
/* BASELINE config C1 mixed bulk/extract trace (no reference
 * generator exists — the spec is restated in pbh_oracle.c). */
orc_trace* orc_trace_gen_mixed(uint64_t n_ops, uint64_t universe, uint64_t kmax, uint64_t seed);
void orc_trace_free(orc_trace* t);

/* run_oracle (tests/oracle.hpp:55-75) over a flat trace. Returns the number
 * of extracted elements, or -(1 + op_index) when an extract hits an empty
 * queue (the reference raises EmptyHeapError -> TraceError(op_index)). */
int64_t orc_run_oracle(uint64_t n_ops, const uint8_t* kinds, const uint64_t* offsets,
                       const uint32_t* vals, const uint64_t* prios, uint32_t* out_v,
                       uint64_t* out_p);

/* ---- CSR graphs (graphs.hpp:11-20) ------------------------------------ */
typedef struct {
  uint32_t V;
  uint64_t E;
  uint64_t* off;
  uint32_t* tgt;
  uint32_t* w;
} orc_graph;

orc_graph* orc_gen_random(uint32_t v, uint64_t e, uint32_t max_weight, uint64_t seed);        /* graphs.cpp:74-110 */
orc_graph* orc_gen_high_diameter(uint32_t v, uint64_t e, uint32_t max_weight, uint64_t seed); /* graphs.cpp:112-140 */
orc_graph* orc_gen_dag(uint32_t v, uint32_t out_degree, uint32_t max_weight, uint64_t seed);  /* graphs.cpp:142-169 */
orc_graph* orc_gen_complete(uint32_t v, uint32_t max_weight, uint64_t seed);                  /* graphs.cpp:171-186 */
/* BASELINE C2 / C3 shapes. */
orc_graph* orc_gen_grid(uint32_t rows, uint32_t cols, uint64_t seed);
orc_graph* orc_gen_band(uint32_t v, uint32_t degree, uint64_t seed);
void orc_graph_free(orc_graph* g);

/* reference_dijkstra (sssp.cpp:71-97): binary heap, lazy deletion, (dist,
 * vertex) order. Also reports the op count par_dijkstra (sssp.cpp:21-69)
 * would log with batch bound d: 1 seed + one extract per settled vertex +
 * ceil(improving relaxations / d) per round. Returns 0, 2 (source out of
 * range) or 3 (distance overflow). */
int orc_dijkstra(uint32_t V, uint64_t E, const uint64_t* off, const uint32_t* tgt,
                 const uint32_t* w, uint32_t source, uint64_t d, uint64_t* dist,
                 uint32_t* settled, uint64_t* n_settled, uint64_t* rounds, uint64_t* ops);

/* distance_checksum (sssp.cpp:174-183): FNV-1a over the distance bytes. */
uint64_t orc_checksum(const uint64_t* dist, uint64_t n);

/* FNV-1a over n raw bytes continued from h; start from ORC_FNV_BASIS. */
#define ORC_FNV_BASIS 0xcbf29ce484222325ULL
uint64_t orc_fnv1a(const void* p, uint64_t n, uint64_t h);

#ifdef __cplusplus
}
#endif
#endif
