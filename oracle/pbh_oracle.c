/* TEST INFRASTRUCTURE ONLY — CPU oracle restating the reference algorithms.
 * See pbh_oracle.h for the contract. Paths are relative to
 * /root/reference/proj. Product code never links this file. */
#include "pbh_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ===================================================================== */
/* std::mt19937_64                                                        */
/* ===================================================================== */
#define MT_N 312
#define MT_M 156
void orc_mt64_seed(orc_mt64* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = MT_N;
}

uint64_t orc_mt64_next(orc_mt64* r) {
  static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (r->idx >= MT_N) {
    int i;
    uint64_t x;
    for (i = 0; i < MT_N - MT_M; ++i) {
      x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + MT_M] ^ (x >> 1) ^ mag[x & 1ULL];
    }
    for (; i < MT_N - 1; ++i) {
      x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + (MT_M - MT_N)] ^ (x >> 1) ^ mag[x & 1ULL];
    }
    x = (r->mt[MT_N - 1] & UM) | (r->mt[0] & LM);
    r->mt[MT_N - 1] = r->mt[MT_M - 1] ^ (x >> 1) ^ mag[x & 1ULL];
    r->idx = 0;
  }
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* ===================================================================== */
/* u32 -> u32 open-addressing map (linear probe, backward-shift delete)   */
/* ===================================================================== */
typedef struct {
  uint32_t* keys;
  uint32_t* vals;
  uint8_t* used;
  uint64_t cap, n;
} u32map;

static uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

static void u32map_init(u32map* m, uint64_t cap) {
  uint64_t c = 16;
  while (c < cap * 2) c <<= 1;
  m->cap = c;
  m->n = 0;
  m->keys = (uint32_t*)malloc(c * sizeof(uint32_t));
  m->vals = (uint32_t*)malloc(c * sizeof(uint32_t));
  m->used = (uint8_t*)calloc(c, 1);
}
static void u32map_free(u32map* m) {
  free(m->keys);
  free(m->vals);
  free(m->used);
}
static int u32map_get(const u32map* m, uint32_t k, uint32_t* out) {
  uint64_t i = mix64(k) & (m->cap - 1);
  while (m->used[i]) {
    if (m->keys[i] == k) {
      *out = m->vals[i];
      return 1;
    }
    i = (i + 1) & (m->cap - 1);
  }
  return 0;
}
static void u32map_grow(u32map* m);
static void u32map_put(u32map* m, uint32_t k, uint32_t v) {
  if ((m->n + 1) * 2 > m->cap) u32map_grow(m);
  uint64_t i = mix64(k) & (m->cap - 1);
  while (m->used[i]) {
    if (m->keys[i] == k) {
      m->vals[i] = v;
      return;
    }
    i = (i + 1) & (m->cap - 1);
  }
  m->used[i] = 1;
  m->keys[i] = k;
  m->vals[i] = v;
  m->n++;
}
static void u32map_grow(u32map* m) {
  u32map nm;
  u32map_init(&nm, m->cap);
  for (uint64_t i = 0; i < m->cap; ++i)
    if (m->used[i]) u32map_put(&nm, m->keys[i], m->vals[i]);
  u32map_free(m);
  *m = nm;
}
static void u32map_del(u32map* m, uint32_t k) {
  uint64_t mask = m->cap - 1, i = mix64(k) & mask;
  while (m->used[i] && m->keys[i] != k) i = (i + 1) & mask;
  if (!m->used[i]) return;
  m->used[i] = 0;
  m->n--;
  uint64_t j = i;
  for (;;) {
    j = (j + 1) & mask;
    if (!m->used[j]) break;
    uint64_t h = mix64(m->keys[j]) & mask;
    /* can the entry at j move to the hole at i? (h cyclically outside (i, j]) */
    int move = (i <= j) ? (h <= i || h > j) : (h <= i && h > j);
    if (move) {
      m->keys[i] = m->keys[j];
      m->vals[i] = m->vals[j];
      m->used[i] = 1;
      m->used[j] = 0;
      i = j;
    }
  }
}

/* ===================================================================== */
/* OracleHeap (tests/oracle.hpp:19-51): (priority, value) ordered PQ with  */
/* replace-priority update and erase. Restated as an indexed binary heap:  */
/* the extraction order is a pure function of the (p, v) total order.      */
/* ===================================================================== */
typedef struct {
  uint64_t p;
  uint32_t v;
} ent;
typedef struct {
  ent* h;
  uint64_t n, cap;
  u32map pos;      /* general value -> heap slot map */
  uint32_t* apos;  /* dense fast path when every value < alen (slot+1, 0 = absent) */
  uint64_t alen;
} oheap;

static int pos_get(const oheap* q, uint32_t v, uint32_t* out) {
  if (q->apos) {
    if (v >= q->alen || q->apos[v] == 0) return 0;
    *out = q->apos[v] - 1;
    return 1;
  }
  return u32map_get(&q->pos, v, out);
}
static void pos_put(oheap* q, uint32_t v, uint32_t i) {
  if (q->apos) q->apos[v] = i + 1;
  else u32map_put(&q->pos, v, i);
}
static void pos_del(oheap* q, uint32_t v) {
  if (q->apos) q->apos[v] = 0;
  else u32map_del(&q->pos, v);
}

static int ent_less(ent a, ent b) { return a.p != b.p ? a.p < b.p : a.v < b.v; }

static void oh_init_dense(oheap* q, uint64_t alen) {
  q->cap = 1024;
  q->n = 0;
  q->h = (ent*)malloc(q->cap * sizeof(ent));
  q->alen = alen;
  q->apos = alen ? (uint32_t*)calloc(alen, sizeof(uint32_t)) : NULL;
  u32map_init(&q->pos, alen ? 1 : 1024);
}
static void oh_init(oheap* q) { oh_init_dense(q, 0); }
static void oh_free(oheap* q) {
  free(q->h);
  free(q->apos);
  u32map_free(&q->pos);
}
static void oh_set(oheap* q, uint64_t i, ent e) {
  q->h[i] = e;
  pos_put(q, e.v, (uint32_t)i);
}
static void oh_up(oheap* q, uint64_t i) {
  ent e = q->h[i];
  while (i > 0) {
    uint64_t par = (i - 1) / 2;
    if (!ent_less(e, q->h[par])) break;
    oh_set(q, i, q->h[par]);
    i = par;
  }
  oh_set(q, i, e);
}
static void oh_down(oheap* q, uint64_t i) {
  ent e = q->h[i];
  for (;;) {
    uint64_t c = 2 * i + 1;
    if (c >= q->n) break;
    if (c + 1 < q->n && ent_less(q->h[c + 1], q->h[c])) ++c;
    if (!ent_less(q->h[c], e)) break;
    oh_set(q, i, q->h[c]);
    i = c;
  }
  oh_set(q, i, e);
}
/* OracleHeap::update (oracle.hpp:21-30): replace or insert. */
static void oh_update(oheap* q, uint32_t v, uint64_t p) {
  uint32_t i;
  if (pos_get(q, v, &i)) {
    q->h[i].p = p;
    oh_up(q, i);
    pos_get(q, v, &i); /* position may have moved up */
    oh_down(q, i);
    return;
  }
  if (q->n == q->cap) {
    q->cap *= 2;
    q->h = (ent*)realloc(q->h, q->cap * sizeof(ent));
  }
  ent e = {p, v};
  q->h[q->n] = e;
  pos_put(q, v, (uint32_t)q->n);
  q->n++;
  oh_up(q, q->n - 1);
}
static void oh_remove_at(oheap* q, uint64_t i) {
  pos_del(q, q->h[i].v);
  q->n--;
  if (i == q->n) return;
  const uint32_t moved = q->h[q->n].v;
  oh_set(q, i, q->h[q->n]);
  oh_up(q, i);
  uint32_t j = 0;
  pos_get(q, moved, &j); /* the moved entry may have gone up */
  oh_down(q, j);
}
/* OracleHeap::erase (oracle.hpp:32-37): absent values are a no-op. */
static void oh_erase(oheap* q, uint32_t v) {
  uint32_t i;
  if (pos_get(q, v, &i)) oh_remove_at(q, i);
}
/* OracleHeap::extract_min (oracle.hpp:39-44). */
static ent oh_extract(oheap* q) {
  ent e = q->h[0];
  oh_remove_at(q, 0);
  return e;
}
static uint64_t oh_prio(oheap* q, uint32_t v) {
  uint32_t i = 0;
  pos_get(q, v, &i);
  return q->h[i].p;
}

/* ===================================================================== */
/* flat traces                                                            */
/* ===================================================================== */
typedef struct {
  orc_trace t;
  uint64_t cap_ops, cap_el;
} tbuild;

static void tb_init(tbuild* b) {
  memset(b, 0, sizeof *b);
  b->cap_ops = 1024;
  b->cap_el = 1024;
  b->t.kinds = (uint8_t*)malloc(b->cap_ops);
  b->t.offsets = (uint64_t*)malloc((b->cap_ops + 1) * sizeof(uint64_t));
  b->t.vals = (uint32_t*)malloc(b->cap_el * sizeof(uint32_t));
  b->t.prios = (uint64_t*)malloc(b->cap_el * sizeof(uint64_t));
  b->t.offsets[0] = 0;
}
static void tb_op(tbuild* b, char kind) {
  if (b->t.n_ops == b->cap_ops) {
    b->cap_ops *= 2;
    b->t.kinds = (uint8_t*)realloc(b->t.kinds, b->cap_ops);
    b->t.offsets = (uint64_t*)realloc(b->t.offsets, (b->cap_ops + 1) * sizeof(uint64_t));
  }
  b->t.kinds[b->t.n_ops++] = (uint8_t)kind;
  b->t.offsets[b->t.n_ops] = b->t.n_elems;
  if (kind == 'E') b->t.n_extract++;
}
static void tb_el(tbuild* b, uint32_t v, uint64_t p) {
  if (b->t.n_elems == b->cap_el) {
    b->cap_el *= 2;
    b->t.vals = (uint32_t*)realloc(b->t.vals, b->cap_el * sizeof(uint32_t));
    b->t.prios = (uint64_t*)realloc(b->t.prios, b->cap_el * sizeof(uint64_t));
  }
  b->t.vals[b->t.n_elems] = v;
  b->t.prios[b->t.n_elems] = p;
  b->t.n_elems++;
}
static orc_trace* tb_finish(tbuild* b) {
  orc_trace* t = (orc_trace*)malloc(sizeof(orc_trace));
  *t = b->t;
  return t;
}

void orc_trace_free(orc_trace* t) {
  if (!t) return;
  free(t->kinds);
  free(t->offsets);
  free(t->vals);
  free(t->prios);
  free(t);
}

/* live-set mirror with O(1) uniform pick (oracle.hpp:86-99): `live` vector
 * plus value -> index map; removal swaps with the back. */
typedef struct {
  uint32_t* a;
  uint64_t n, cap;
  u32map pos;
} liveset;
static void ls_init(liveset* s) {
  s->cap = 1024;
  s->n = 0;
  s->a = (uint32_t*)malloc(s->cap * sizeof(uint32_t));
  u32map_init(&s->pos, 1024);
}
static void ls_free(liveset* s) {
  free(s->a);
  u32map_free(&s->pos);
}
static void ls_add(liveset* s, uint32_t v) {
  if (s->n == s->cap) {
    s->cap *= 2;
    s->a = (uint32_t*)realloc(s->a, s->cap * sizeof(uint32_t));
  }
  u32map_put(&s->pos, v, (uint32_t)s->n);
  s->a[s->n++] = v;
}
static void ls_remove(liveset* s, uint32_t v) {
  uint32_t i;
  u32map_get(&s->pos, v, &i);
  uint32_t back = s->a[s->n - 1];
  u32map_put(&s->pos, back, i); /* pos[live.back()] = i */
  s->a[i] = back;               /* swap(live[i], live.back()) */
  s->a[s->n - 1] = v;
  s->n--;       /* live.pop_back() */
  u32map_del(&s->pos, v); /* pos.erase(v) */
}

/* gen_legal_trace (tests/oracle.hpp:82-155), draw for draw. */
orc_trace* orc_trace_gen_legal(uint64_t n_ops, uint64_t d, uint64_t seed) {
  orc_mt64 rng;
  orc_mt64_seed(&rng, seed);
  tbuild b;
  tb_init(&b);
  oheap model;
  oh_init(&model);
  liveset live;
  ls_init(&live);
  uint32_t next_fresh = 0, next_absent = 0x80000000u;

#define FRESH_UPDATE()                                  \
  do {                                                  \
    uint32_t v_ = next_fresh++;                         \
    uint64_t p_ = 1 + orc_mt64_next(&rng) % 1000000ULL; \
    oh_update(&model, v_, p_);                          \
    ls_add(&live, v_);                                  \
    tb_el(&b, v_, p_);                                  \
    tb_op(&b, 'U');                                     \
  } while (0)

  for (uint64_t i = 0; i < n_ops; ++i) {
    uint64_t r = orc_mt64_next(&rng) % 100;
    if (model.n == 0 || r < 60) {
      if (live.n == 0 || r < 40) {
        FRESH_UPDATE();
      } else {
        uint32_t v = live.a[orc_mt64_next(&rng) % live.n];
        uint64_t cur = oh_prio(&model, v);
        if (cur <= 1) {
          FRESH_UPDATE();
        } else {
          uint64_t p = 1 + orc_mt64_next(&rng) % (cur - 1);
          oh_update(&model, v, p);
          tb_el(&b, v, p);
          tb_op(&b, 'U');
        }
      }
    } else if (r < 85) {
      ent e = oh_extract(&model);
      ls_remove(&live, e.v);
      tb_op(&b, 'E');
    } else if (r < 95) {
      if (r < 94 && live.n > 0) {
        uint32_t v = live.a[orc_mt64_next(&rng) % live.n];
        oh_erase(&model, v);
        ls_remove(&live, v);
        tb_el(&b, v, 0);
        tb_op(&b, 'D');
      } else {
        tb_el(&b, next_absent++, 0);
        tb_op(&b, 'D');
      }
    } else {
      uint64_t k = 1 + orc_mt64_next(&rng) % d;
      for (uint64_t j = 0; j < k; ++j) {
        uint32_t v = next_fresh++;
        uint64_t p = 1 + orc_mt64_next(&rng) % 1000000ULL;
        tb_el(&b, v, p);
        oh_update(&model, v, p);
        ls_add(&live, v);
      }
      tb_op(&b, 'B');
    }
  }
#undef FRESH_UPDATE
  oh_free(&model);
  ls_free(&live);
  return tb_finish(&b);
}

/* BASELINE C1 trace (SURVEY.md §8d "C1, op trace"). No reference generator
 * exists, so this restatement IS the definition; the package's generator
 * (paper_1908_09378_b200/csrc/pbh_gen.cpp) must reproduce it draw for draw.
 *   per op: bulk when nothing is live or rng()%2 == 0, else extract;
 *   bulk:   k = 1 + rng()%kmax slots; a slot is a fresh key (next unused)
 *           when keys remain and (nothing live or rng()%2 == 0), priority
 *           1 + rng()%(2^31-2); otherwise a strict decrease of a random live
 *           key not already in this batch: p' = p - 1 - rng()%min(p-1, 65536),
 *           skipped when p <= 1 or the key is already in the batch.
 *           Batches are emitted value-sorted; an all-skipped batch becomes an
 *           extract. Generation stops early once keys are exhausted and
 *           nothing is live. */
static int cmp_vp(const void* a, const void* b) {
  const ent* x = (const ent*)a;
  const ent* y = (const ent*)b;
  return x->v < y->v ? -1 : x->v > y->v;
}

orc_trace* orc_trace_gen_mixed(uint64_t n_ops, uint64_t universe, uint64_t kmax, uint64_t seed) {
  orc_mt64 rng;
  orc_mt64_seed(&rng, seed);
  tbuild b;
  tb_init(&b);
  oheap model;
  oh_init_dense(&model, universe);
  uint64_t* cur = (uint64_t*)calloc(universe, sizeof(uint64_t));
  uint64_t* mark = (uint64_t*)malloc(universe * sizeof(uint64_t));
  memset(mark, 0xff, universe * sizeof(uint64_t));
  uint32_t* live = (uint32_t*)malloc(universe * sizeof(uint32_t));
  uint32_t* lpos = (uint32_t*)malloc(universe * sizeof(uint32_t));
  ent* batch = (ent*)malloc(kmax * sizeof(ent));
  uint64_t live_n = 0, next_fresh = 0;

  for (uint64_t op = 0; op < n_ops; ++op) {
    if (live_n == 0 && next_fresh >= universe) break;
    int bulk = live_n == 0 || orc_mt64_next(&rng) % 2 == 0;
    uint64_t nb = 0;
    if (bulk) {
      uint64_t k = 1 + orc_mt64_next(&rng) % kmax;
      for (uint64_t j = 0; j < k; ++j) {
        int fresh_ok = next_fresh < universe;
        if (fresh_ok && (live_n == 0 || orc_mt64_next(&rng) % 2 == 0)) {
          uint32_t v = (uint32_t)next_fresh++;
          uint64_t p = 1 + orc_mt64_next(&rng) % 2147483646ULL;
          cur[v] = p;
          mark[v] = op;
          lpos[v] = (uint32_t)live_n;
          live[live_n++] = v;
          oh_update(&model, v, p);
          batch[nb].v = v;
          batch[nb].p = p;
          nb++;
        } else if (live_n > 0) {
          uint32_t v = live[orc_mt64_next(&rng) % live_n];
          if (mark[v] == op) continue;
          uint64_t p = cur[v];
          if (p <= 1) continue;
          uint64_t m = p - 1 < 65536 ? p - 1 : 65536;
          uint64_t np = p - 1 - orc_mt64_next(&rng) % m;
          cur[v] = np;
          mark[v] = op;
          oh_update(&model, v, np);
          batch[nb].v = v;
          batch[nb].p = np;
          nb++;
        }
      }
    }
    if (nb > 0) {
      qsort(batch, nb, sizeof(ent), cmp_vp);
      for (uint64_t j = 0; j < nb; ++j) tb_el(&b, batch[j].v, batch[j].p);
      tb_op(&b, 'B');
    } else {
      ent e = oh_extract(&model);
      uint32_t i = lpos[e.v];
      uint32_t back = live[live_n - 1];
      live[i] = back;
      lpos[back] = i;
      live_n--;
      tb_op(&b, 'E');
    }
  }
  free(cur);
  free(mark);
  free(live);
  free(lpos);
  free(batch);
  oh_free(&model);
  return tb_finish(&b);
}

/* run_oracle (tests/oracle.hpp:55-75). */
int64_t orc_run_oracle(uint64_t n_ops, const uint8_t* kinds, const uint64_t* offsets,
                       const uint32_t* vals, const uint64_t* prios, uint32_t* out_v,
                       uint64_t* out_p) {
  uint32_t vmax = 0;
  for (uint64_t j = 0; j < offsets[n_ops]; ++j)
    if (vals[j] > vmax) vmax = vals[j];
  oheap h;
  oh_init_dense(&h, vmax < (1u << 28) ? (uint64_t)vmax + 1 : 0);
  int64_t n = 0;
  for (uint64_t i = 0; i < n_ops; ++i) {
    switch (kinds[i]) {
      case 'U':
      case 'B':
        for (uint64_t j = offsets[i]; j < offsets[i + 1]; ++j) oh_update(&h, vals[j], prios[j]);
        break;
      case 'E': {
        if (h.n == 0) {
          oh_free(&h);
          return -(int64_t)(1 + i);
        }
        ent e = oh_extract(&h);
        out_v[n] = e.v;
        out_p[n] = e.p;
        ++n;
        break;
      }
      case 'D':
        oh_erase(&h, vals[offsets[i]]);
        break;
      default:
        break;
    }
  }
  oh_free(&h);
  return n;
}

/* ===================================================================== */
/* graphs                                                                 */
/* ===================================================================== */
/* u64 set for edge dedup (graphs.cpp uses std::unordered_set: only the
 * membership answers matter, so the RNG draw sequence is reproduced). */
typedef struct {
  uint64_t* k;
  uint8_t* used;
  uint64_t cap, n;
} u64set;
static void s64_init(u64set* s, uint64_t want) {
  uint64_t c = 16;
  while (c < want * 2) c <<= 1;
  s->cap = c;
  s->n = 0;
  s->k = (uint64_t*)malloc(c * sizeof(uint64_t));
  s->used = (uint8_t*)calloc(c, 1);
}
static void s64_free(u64set* s) {
  free(s->k);
  free(s->used);
}
static int s64_insert(u64set* s, uint64_t key);
static void s64_grow(u64set* s) {
  u64set ns;
  s64_init(&ns, s->cap);
  for (uint64_t i = 0; i < s->cap; ++i)
    if (s->used[i]) s64_insert(&ns, s->k[i]);
  s64_free(s);
  *s = ns;
}
static int s64_insert(u64set* s, uint64_t key) {
  if ((s->n + 1) * 2 > s->cap) s64_grow(s);
  uint64_t i = mix64(key) & (s->cap - 1);
  while (s->used[i]) {
    if (s->k[i] == key) return 0;
    i = (i + 1) & (s->cap - 1);
  }
  s->used[i] = 1;
  s->k[i] = key;
  s->n++;
  return 1;
}

typedef struct {
  uint64_t code; /* (src << 32) | dst */
  uint32_t w;
} cedge;
static int cmp_cedge(const void* a, const void* b) {
  const cedge* x = (const cedge*)a;
  const cedge* y = (const cedge*)b;
  if (x->code != y->code) return x->code < y->code ? -1 : 1;
  return x->w < y->w ? -1 : x->w > y->w;
}

static orc_graph* galloc(uint32_t v, uint64_t e) {
  orc_graph* g = (orc_graph*)malloc(sizeof(orc_graph));
  g->V = v;
  g->E = e;
  g->off = (uint64_t*)calloc((uint64_t)v + 1, sizeof(uint64_t));
  g->tgt = (uint32_t*)malloc((e ? e : 1) * sizeof(uint32_t));
  g->w = (uint32_t*)malloc((e ? e : 1) * sizeof(uint32_t));
  return g;
}

/* from_edges (graphs.cpp:27-43): sort by (src, dst) and build CSR. */
static orc_graph* from_edges(uint32_t v, cedge* c, uint64_t e) {
  qsort(c, e, sizeof(cedge), cmp_cedge);
  orc_graph* g = galloc(v, e);
  for (uint64_t i = 0; i < e; ++i) {
    g->off[(c[i].code >> 32) + 1]++;
    g->tgt[i] = (uint32_t)(c[i].code & 0xffffffffu);
    g->w[i] = c[i].w;
  }
  for (uint64_t i = 1; i <= v; ++i) g->off[i] += g->off[i - 1];
  free(c);
  return g;
}

static uint64_t pair_code(uint32_t u, uint32_t t) { return ((uint64_t)u << 32) | t; }

orc_graph* orc_gen_random(uint32_t v, uint64_t e, uint32_t max_weight, uint64_t seed) {
  if (v == 0 || max_weight == 0) return NULL;
  uint64_t all = (uint64_t)v * (v - 1);
  if (e > all) return NULL;
  orc_mt64 rng;
  orc_mt64_seed(&rng, seed);
  cedge* c = (cedge*)malloc((e ? e : 1) * sizeof(cedge));
  if (e > all / 2) {
    uint64_t* codes = (uint64_t*)malloc(all * sizeof(uint64_t));
    uint64_t n = 0;
    for (uint32_t u = 0; u < v; ++u)
      for (uint32_t t = 0; t < v; ++t)
        if (u != t) codes[n++] = pair_code(u, t);
    for (uint64_t i = 0; i < e; ++i) {
      uint64_t j = i + orc_mt64_next(&rng) % (all - i);
      uint64_t tmp = codes[i];
      codes[i] = codes[j];
      codes[j] = tmp;
    }
    for (uint64_t i = 0; i < e; ++i) {
      c[i].code = codes[i];
      c[i].w = 1 + (uint32_t)(orc_mt64_next(&rng) % max_weight);
    }
    free(codes);
  } else {
    u64set seen;
    s64_init(&seen, e);
    uint64_t n = 0;
    while (seen.n < e) {
      uint32_t u = (uint32_t)(orc_mt64_next(&rng) % v);
      uint32_t t = (uint32_t)(orc_mt64_next(&rng) % v);
      if (u == t) continue;
      if (s64_insert(&seen, pair_code(u, t))) {
        c[n].code = pair_code(u, t);
        c[n].w = 1 + (uint32_t)(orc_mt64_next(&rng) % max_weight);
        n++;
      }
    }
    s64_free(&seen);
  }
  return from_edges(v, c, e);
}

orc_graph* orc_gen_high_diameter(uint32_t v, uint64_t e, uint32_t max_weight, uint64_t seed) {
  if (v < 2 || max_weight == 0 || e < (uint64_t)v - 1) return NULL;
  uint64_t all = (uint64_t)v * (v - 1);
  if (e > all) return NULL;
  orc_mt64 rng;
  orc_mt64_seed(&rng, seed);
  cedge* c = (cedge*)malloc(e * sizeof(cedge));
  u64set seen;
  s64_init(&seen, e);
  uint64_t n = 0;
  for (uint32_t u = 0; u + 1 < v; ++u) {
    s64_insert(&seen, pair_code(u, u + 1));
    c[n].code = pair_code(u, u + 1);
    c[n].w = 1;
    n++;
  }
  while (seen.n < e) {
    uint32_t u = (uint32_t)(orc_mt64_next(&rng) % v);
    uint32_t t = (uint32_t)(orc_mt64_next(&rng) % v);
    if (u == t) continue;
    if (s64_insert(&seen, pair_code(u, t))) {
      c[n].code = pair_code(u, t);
      c[n].w = v + (uint32_t)(orc_mt64_next(&rng) % max_weight);
      n++;
    }
  }
  s64_free(&seen);
  return from_edges(v, c, e);
}

orc_graph* orc_gen_dag(uint32_t v, uint32_t out_degree, uint32_t max_weight, uint64_t seed) {
  if (v == 0 || out_degree >= v || max_weight == 0) return NULL;
  orc_mt64 rng;
  orc_mt64_seed(&rng, seed);
  uint64_t capn = (uint64_t)v * out_degree + 1, n = 0;
  cedge* c = (cedge*)malloc(capn * sizeof(cedge));
  for (uint32_t u = 0; u + 1 < v; ++u) {
    uint32_t room = v - 1 - u;
    uint32_t deg = out_degree < room ? out_degree : room;
    if (deg == room) {
      for (uint32_t t = u + 1; t < v; ++t) {
        c[n].code = pair_code(u, t);
        c[n].w = 1 + (uint32_t)(orc_mt64_next(&rng) % max_weight);
        n++;
      }
      continue;
    }
    u64set row;
    s64_init(&row, deg);
    while (row.n < deg) {
      uint32_t t = u + 1 + (uint32_t)(orc_mt64_next(&rng) % room);
      if (s64_insert(&row, t)) {
        c[n].code = pair_code(u, t);
        c[n].w = 1 + (uint32_t)(orc_mt64_next(&rng) % max_weight);
        n++;
      }
    }
    s64_free(&row);
  }
  return from_edges(v, c, n);
}

orc_graph* orc_gen_complete(uint32_t v, uint32_t max_weight, uint64_t seed) {
  if (v < 2 || v > 8192 || max_weight == 0) return NULL;
  orc_mt64 rng;
  orc_mt64_seed(&rng, seed);
  uint64_t e = (uint64_t)v * (v - 1), n = 0;
  cedge* c = (cedge*)malloc(e * sizeof(cedge));
  for (uint32_t u = 0; u < v; ++u)
    for (uint32_t t = u + 1; t < v; ++t) {
      uint32_t w = 1 + (uint32_t)(orc_mt64_next(&rng) % max_weight);
      c[n].code = pair_code(u, t);
      c[n].w = w;
      n++;
      c[n].code = pair_code(t, u);
      c[n].w = w;
      n++;
    }
  return from_edges(v, c, e);
}

/* C2: rows x cols 4-neighbour grid, vid = r*cols + c, row order up, left,
 * right, down (ascending vid); weights 1 + rng()%(2^32-1) in CSR order. */
orc_graph* orc_gen_grid(uint32_t rows, uint32_t cols, uint64_t seed) {
  uint64_t V = (uint64_t)rows * cols;
  uint64_t E = 2 * ((uint64_t)rows * (cols - 1) + (uint64_t)cols * (rows - 1));
  orc_graph* g = galloc((uint32_t)V, E);
  orc_mt64 rng;
  orc_mt64_seed(&rng, seed);
  uint64_t n = 0;
  for (uint32_t r = 0; r < rows; ++r)
    for (uint32_t c = 0; c < cols; ++c) {
      uint64_t u = (uint64_t)r * cols + c;
      g->off[u] = n;
      if (r > 0) g->tgt[n++] = (uint32_t)(u - cols);
      if (c > 0) g->tgt[n++] = (uint32_t)(u - 1);
      if (c + 1 < cols) g->tgt[n++] = (uint32_t)(u + 1);
      if (r + 1 < rows) g->tgt[n++] = (uint32_t)(u + cols);
    }
  g->off[V] = n;
  for (uint64_t i = 0; i < n; ++i) g->w[i] = 1 + (uint32_t)(orc_mt64_next(&rng) % 4294967295ULL);
  return g;
}

/* C3: ring band, row u -> (u + j) mod V for j = 1..degree, sorted; spine
 * w(u, u+1) = 1 for u + 1 < V; every other edge V + rng()%1000 in CSR order. */
orc_graph* orc_gen_band(uint32_t v, uint32_t degree, uint64_t seed) {
  if (degree >= v) return NULL;
  uint64_t E = (uint64_t)v * degree;
  orc_graph* g = galloc(v, E);
  orc_mt64 rng;
  orc_mt64_seed(&rng, seed);
  uint64_t n = 0;
  for (uint32_t u = 0; u < v; ++u) {
    g->off[u] = n;
    /* wrapped targets (< u) first, ascending, then the forward run */
    uint64_t end = (uint64_t)u + degree;
    if (end >= v) {
      uint32_t wrap = (uint32_t)(end - v + 1); /* targets 0 .. wrap-1 */
      for (uint32_t t = 0; t < wrap; ++t) g->tgt[n++] = t;
      for (uint64_t t = (uint64_t)u + 1; t < v; ++t) g->tgt[n++] = (uint32_t)t;
    } else {
      for (uint64_t t = (uint64_t)u + 1; t <= end; ++t) g->tgt[n++] = (uint32_t)t;
    }
  }
  g->off[v] = n;
  for (uint32_t u = 0; u < v; ++u)
    for (uint64_t i = g->off[u]; i < g->off[u + 1]; ++i)
      g->w[i] = ((uint64_t)g->tgt[i] == (uint64_t)u + 1) ? 1u
                                                           : v + (uint32_t)(orc_mt64_next(&rng) % 1000);
  return g;
}

void orc_graph_free(orc_graph* g) {
  if (!g) return;
  free(g->off);
  free(g->tgt);
  free(g->w);
  free(g);
}

/* ===================================================================== */
/* reference_dijkstra (sssp.cpp:71-97)                                     */
/* ===================================================================== */
int orc_dijkstra(uint32_t V, uint64_t E, const uint64_t* off, const uint32_t* tgt,
                 const uint32_t* w, uint32_t source, uint64_t d, uint64_t* dist,
                 uint32_t* settled, uint64_t* n_settled, uint64_t* rounds, uint64_t* ops) {
  (void)E;
  if (source >= V) return 2;
  if (d == 0) { /* sssp.cpp:24-26: d = max(1, max out-degree) */
    uint64_t best = 0;
    for (uint32_t u = 0; u < V; ++u)
      if (off[u + 1] - off[u] > best) best = off[u + 1] - off[u];
    d = best ? best : 1;
  }
  for (uint32_t i = 0; i < V; ++i) dist[i] = ~0ULL;
  uint8_t* done = (uint8_t*)calloc(V, 1);
  /* plain binary heap of (dist, vertex) with duplicates (lazy deletion) */
  uint64_t cap = 1024, n = 0;
  ent* h = (ent*)malloc(cap * sizeof(ent));
  uint64_t ns = 0, nr = 0, nops = 1;
  int status = 0;
  dist[source] = 0;
  h[n++] = (ent){0, source};
  while (n > 0) {
    ent top = h[0];
    ent last = h[--n];
    if (n > 0) { /* sift last down from the root */
      uint64_t i = 0;
      for (;;) {
        uint64_t c = 2 * i + 1;
        if (c >= n) break;
        if (c + 1 < n && ent_less(h[c + 1], h[c])) ++c;
        if (!ent_less(h[c], last)) break;
        h[i] = h[c];
        i = c;
      }
      h[i] = last;
    }
    uint32_t v = top.v;
    if (done[v]) continue;
    done[v] = 1;
    if (settled) settled[ns] = v;
    ns++;
    nr++;
    nops++; /* par_dijkstra's extract */
    uint64_t improving = 0;
    for (uint64_t i = off[v]; i < off[v + 1]; ++i) {
      uint32_t u = tgt[i];
      uint64_t cand = top.p + w[i];
      if (cand < top.p) { /* checked_add (sssp.cpp:13-17) */
        status = 3;
        goto out;
      }
      if (cand < dist[u]) {
        if (!done[u]) ++improving; /* par_dijkstra skips settled targets */
        dist[u] = cand;
        if (n == cap) {
          cap *= 2;
          h = (ent*)realloc(h, cap * sizeof(ent));
        }
        uint64_t j = n++;
        ent e = {cand, u};
        while (j > 0 && ent_less(e, h[(j - 1) / 2])) {
          h[j] = h[(j - 1) / 2];
          j = (j - 1) / 2;
        }
        h[j] = e;
      }
    }
    nops += (improving + d - 1) / d;
  }
out:
  free(h);
  free(done);
  *n_settled = ns;
  *rounds = nr;
  *ops = nops;
  return status;
}

uint64_t orc_checksum(const uint64_t* dist, uint64_t n) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (uint64_t i = 0; i < n; ++i)
    for (int b = 0; b < 8; ++b) {
      h ^= (dist[i] >> (8 * b)) & 0xff;
      h *= 0x100000001b3ULL;
    }
  return h;
}

/* FNV-1a (the hash of distance_checksum, sssp.cpp:174-183) over raw bytes,
 * continued from h (start with PBH_FNV_BASIS). Used to fingerprint settle
 * orders and extraction sequences for the full-size goldens. */
uint64_t orc_fnv1a(const void* p, uint64_t n, uint64_t h) {
  const unsigned char* b = (const unsigned char*)p;
  for (uint64_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}
