// Device-resident heap layout shared by the kernels and the host runtime.
// Plain C layout (no torch types): everything below lives in HBM.
#pragma once
#include <stdint.h>

#define PBH_MAX_LEVELS 24

// Per-key position index entry (16 B, one sector-aligned load):
//   prio   current priority of the key's single valid copy
//   state  PBH_ST_ABSENT (never inserted), PBH_ST_LIVE, PBH_ST_DEAD
//   parent SSSP predecessor (unused by the plain heap)
// A memset to 0xFF is the initial state (absent, prio = kInfDist).
#define PBH_ST_ABSENT 0xFFFFFFFFu
#define PBH_ST_LIVE 1u
#define PBH_ST_DEAD 2u
// The low two bits of `state` hold the state (absent reads as 3); the fast
// SSSP path keeps the key's level-0 location in the upper 30 bits:
// loc = slot (S_0), PBH_LOC_B | slot (B_0), PBH_LOC_DEEP (an HBM level).
#define PBH_ST(x) ((x) & 3u)
#define PBH_LOC_B 0x20000000u
#define PBH_LOC_DEEP 0x3FFFFFFFu

typedef struct __attribute__((aligned(16))) {
  uint64_t prio;
  uint32_t state;
  uint32_t parent;
} pbh_idx_entry;

// Mutable per-level state. B_i = bucket run bk/bp[b_sel][b_head, b_head+b_size),
// S_i = signal run sk/sp[s_sel][s_head, s_head+s_size). Both (prio, key)-sorted.
typedef struct {
  uint32_t b_sel, s_sel;
  uint32_t b_head, b_size;
  uint32_t s_head, s_size;
  uint32_t spl_inf, spl_k;
  uint64_t spl_p;
} pbh_level_state;

// Immutable per-level buffers (ping-pong pairs).
typedef struct {
  uint32_t* bk[2];
  uint64_t* bp[2];
  uint32_t* sk[2];
  uint64_t* sp[2];
  uint32_t cap_b;  // bucket capacity (elements)
  uint32_t buf_s;  // signal buffer capacity (elements, 2x the signal capacity)
  uint32_t pad[2];
} pbh_level_bufs;

typedef struct {
  pbh_level_bufs lv[PBH_MAX_LEVELS];
  pbh_level_state st[PBH_MAX_LEVELS];
  pbh_idx_entry* idx;
  uint64_t universe;
  uint32_t n_levels;  // allocated levels
  uint32_t d;         // batch bound
  uint32_t cap0;      // B_0 capacity
  uint32_t debug_checks;
  int64_t live;
  uint64_t ops;
  uint64_t resolves[PBH_MAX_LEVELS];
  uint64_t touches[PBH_MAX_LEVELS];
  // level-0 scratch in HBM (used when B_0 does not fit in shared memory):
  // batch keys/prios (d), push list (d), B_0 removal flags (cap0)
  uint32_t* g_bk;
  uint64_t* g_bp;
  uint32_t* g_pk;
  uint64_t* g_pp;
  uint8_t* g_rm;
  // SSSP relaxation collection (d + 1024 entries)
  uint32_t* g_ck;
  uint64_t* g_cp;
  uint64_t* g_co;
  uint32_t* g_cs;
  // deletes of values beyond the index (absent values: no-ops) remembered so
  // that a later index growth marks them DEAD, as the reference's
  // shadow_dead_ set does (bucket_heap.cpp:55-58,113-125)
  uint32_t* oor_del;
  uint32_t oor_n, oor_cap;
  // stale entries dropped by the filtered grid / streamed merges (the
  // CTA-local tile merges near level 0 always filter and are not counted)
  uint64_t stale_dropped;
} pbh_heap_dev;

// Op stream (trace_format.hpp:16-33) in device memory.
typedef struct {
  const uint8_t* kinds;     // 'U','B','E','D'
  const uint64_t* offsets;  // n_ops + 1
  const uint32_t* vals;
  const uint64_t* prios;
} pbh_trace_dev;

// Single-op channel of the Engine's per-call API (engine.cpp:90-109), in
// mapped pinned host memory. One-shot launches read the op from the plain
// fields and write the extraction back to them. In persistent mode one
// resident k_trace_bank serves op after op through flagged words (request
// number << 32 | 32-bit payload; a word is current iff it carries the
// expected number, so neither side needs a fence):
//   rq[0] kind | n << 8, rq[1] value, rq[2..3] priority (lo, hi) of a
//   single-element op; rv / rplo / rphi the elements of a larger one;
//   rs[0] n_out (0xFFFFFFFF: the op failed, see the status block),
//   rs[1] extracted value, rs[2..3] its priority.
// The kernel exits (saving its level-0 image) on `stop`, on a failed op, or
// after `idle_ns` without a request.
#define PBH_INLINE_OP_MAX 256
typedef struct {
  uint8_t kinds[16];
  uint64_t off[2];
  uint32_t vals[PBH_INLINE_OP_MAX];
  uint64_t prios[PBH_INLINE_OP_MAX];
  uint32_t out_v[2];
  uint64_t out_p[1];
  uint64_t idle_ns;
  uint64_t tprof[3];  // kernel: ns spent waiting for / copying in / running requests
  volatile uint64_t rq[4];
  uint64_t pad1[4];
  volatile uint64_t rs[4];
  uint64_t pad2[4];
  volatile uint64_t stop;
  uint64_t pad3[7];
  volatile uint64_t rv[PBH_INLINE_OP_MAX];
  volatile uint64_t rplo[PBH_INLINE_OP_MAX];
  volatile uint64_t rphi[PBH_INLINE_OP_MAX];
} pbh_op_channel;

// Kernel status block (device memory, read back by the host).
typedef struct {
  uint32_t status;      // pbh_status
  uint32_t detail;      // PBH_ERR_*
  uint64_t ops_done;    // ops fully applied in this launch
  uint64_t n_out;       // extracted elements written (cumulative)
  uint64_t failed_op;   // op index of the failure
  uint64_t aux;         // detail payload (value, level, ...)
  uint64_t pad[3];
} pbh_kstatus;

// error details (mapped to the reference's messages on the host)
#define PBH_ERR_NONE 0
#define PBH_ERR_EMPTY_HEAP 1       // bucket_heap.cpp:68-69
#define PBH_ERR_EMPTY_BATCH 2      // bucket_heap.cpp:129
#define PBH_ERR_BATCH_TOO_BIG 3    // bucket_heap.cpp:130
#define PBH_ERR_UNSORTED 4         // bucket_heap.cpp:133-135
#define PBH_ERR_REINSERT 5         // bucket_heap.cpp:55-58
#define PBH_ERR_INCREASE 6         // bucket_heap.cpp:60-62
#define PBH_ERR_NEED_GROW 7        // internal: allocate a deeper level and resume
#define PBH_ERR_INVARIANT 8        // internal invariant broken
#define PBH_ERR_OVERFLOW 9         // sssp.cpp:13-17 distance overflow
#define PBH_ERR_KEY_RANGE 10       // key >= universe (host grows the index first)
#define PBH_ERR_BAD_OP 11          // unknown op kind
