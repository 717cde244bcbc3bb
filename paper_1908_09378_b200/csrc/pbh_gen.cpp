// Synthetic workload generators for the BASELINE configs (include/pbh_gen.h).
// Host C++; the sequences are defined in SURVEY.md §8d and restated
// independently by the oracle (oracle/pbh_oracle.c).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

#include "../../include/pbh_gen.h"

namespace {

using u32 = uint32_t;
using u64 = uint64_t;

// Indexed binary min-heap over (priority, value) for values < universe; the
// generator needs it only to know which key each extract removes.
struct IndexedHeap {
  std::vector<u64> hp;
  std::vector<u32> hv;
  std::vector<u32> pos;  // slot + 1, 0 = absent
  explicit IndexedHeap(u64 universe) : pos(universe, 0) {}
  static bool less(u64 pa, u32 va, u64 pb, u32 vb) { return pa != pb ? pa < pb : va < vb; }
  void place(size_t i, u64 p, u32 v) {
    hp[i] = p;
    hv[i] = v;
    pos[v] = (u32)i + 1;
  }
  void up(size_t i) {
    const u64 p = hp[i];
    const u32 v = hv[i];
    while (i > 0) {
      const size_t par = (i - 1) / 2;
      if (!less(p, v, hp[par], hv[par])) break;
      place(i, hp[par], hv[par]);
      i = par;
    }
    place(i, p, v);
  }
  void down(size_t i) {
    const u64 p = hp[i];
    const u32 v = hv[i];
    const size_t n = hp.size();
    for (;;) {
      size_t c = 2 * i + 1;
      if (c >= n) break;
      if (c + 1 < n && less(hp[c + 1], hv[c + 1], hp[c], hv[c])) ++c;
      if (!less(hp[c], hv[c], p, v)) break;
      place(i, hp[c], hv[c]);
      i = c;
    }
    place(i, p, v);
  }
  void update(u32 v, u64 p) {
    if (pos[v]) {
      const size_t i = pos[v] - 1;
      hp[i] = p;
      up(i);
      down(pos[v] - 1);
      return;
    }
    hp.push_back(p);
    hv.push_back(v);
    pos[v] = (u32)hp.size();
    up(hp.size() - 1);
  }
  u32 extract() {
    const u32 v = hv[0];
    pos[v] = 0;
    const u64 lp = hp.back();
    const u32 lv = hv.back();
    hp.pop_back();
    hv.pop_back();
    if (!hp.empty()) {
      place(0, lp, lv);
      down(0);
    }
    return v;
  }
};

}  // namespace

struct pbh_gen_trace {
  std::vector<uint8_t> kinds;
  std::vector<u64> offsets{0};
  std::vector<u32> vals;
  std::vector<u64> prios;
  u64 n_extract = 0;
};

extern "C" {

uint64_t pbh_gen_grid_edges(uint32_t rows, uint32_t cols) {
  return 2ull * ((u64)rows * (cols - 1) + (u64)cols * (rows - 1));
}

void pbh_gen_grid(uint32_t rows, uint32_t cols, uint64_t seed, uint64_t* off, uint32_t* tgt,
                  uint32_t* w) {
  u64 n = 0;
  for (u32 r = 0; r < rows; ++r)
    for (u32 c = 0; c < cols; ++c) {
      const u64 u = (u64)r * cols + c;
      off[u] = n;
      if (r > 0) tgt[n++] = (u32)(u - cols);
      if (c > 0) tgt[n++] = (u32)(u - 1);
      if (c + 1 < cols) tgt[n++] = (u32)(u + 1);
      if (r + 1 < rows) tgt[n++] = (u32)(u + cols);
    }
  off[(u64)rows * cols] = n;
  std::mt19937_64 rng(seed);
  for (u64 i = 0; i < n; ++i) w[i] = 1 + (u32)(rng() % 4294967295ull);
}

void pbh_gen_band(uint32_t v, uint32_t degree, uint64_t seed, uint64_t* off, uint32_t* tgt,
                  uint32_t* w) {
  u64 n = 0;
  for (u32 u = 0; u < v; ++u) {
    off[u] = n;
    const u64 end = (u64)u + degree;
    if (end >= v) {
      const u32 wrap = (u32)(end - v + 1);
      for (u32 t = 0; t < wrap; ++t) tgt[n++] = t;
      for (u64 t = (u64)u + 1; t < v; ++t) tgt[n++] = (u32)t;
    } else {
      for (u64 t = (u64)u + 1; t <= end; ++t) tgt[n++] = (u32)t;
    }
  }
  off[v] = n;
  std::mt19937_64 rng(seed);
  for (u32 u = 0; u < v; ++u)
    for (u64 i = off[u]; i < off[u + 1]; ++i)
      w[i] = ((u64)tgt[i] == (u64)u + 1) ? 1u : v + (u32)(rng() % 1000);
}

pbh_gen_trace* pbh_gen_mixed_trace(uint64_t n_ops, uint64_t universe, uint64_t kmax,
                                   uint64_t seed) {
  auto* t = new pbh_gen_trace();
  std::mt19937_64 rng(seed);
  IndexedHeap model(universe);
  std::vector<u64> cur(universe, 0), mark(universe, ~0ull);
  std::vector<u32> live(universe), lpos(universe);
  std::vector<std::pair<u32, u64>> batch;
  batch.reserve(kmax);
  u64 live_n = 0, next_fresh = 0;
  for (u64 op = 0; op < n_ops; ++op) {
    if (live_n == 0 && next_fresh >= universe) break;
    const bool bulk = live_n == 0 || rng() % 2 == 0;
    batch.clear();
    if (bulk) {
      const u64 k = 1 + rng() % kmax;
      for (u64 j = 0; j < k; ++j) {
        const bool fresh_ok = next_fresh < universe;
        if (fresh_ok && (live_n == 0 || rng() % 2 == 0)) {
          const u32 v = (u32)next_fresh++;
          const u64 p = 1 + rng() % 2147483646ull;
          cur[v] = p;
          mark[v] = op;
          lpos[v] = (u32)live_n;
          live[live_n++] = v;
          model.update(v, p);
          batch.emplace_back(v, p);
        } else if (live_n > 0) {
          const u32 v = live[rng() % live_n];
          if (mark[v] == op) continue;
          const u64 p = cur[v];
          if (p <= 1) continue;
          const u64 m = std::min<u64>(p - 1, 65536);
          const u64 np = p - 1 - rng() % m;
          cur[v] = np;
          mark[v] = op;
          model.update(v, np);
          batch.emplace_back(v, np);
        }
      }
    }
    if (!batch.empty()) {
      std::sort(batch.begin(), batch.end());
      for (auto& [v, p] : batch) {
        t->vals.push_back(v);
        t->prios.push_back(p);
      }
      t->kinds.push_back('B');
    } else {
      const u32 v = model.extract();
      const u32 i = lpos[v];
      const u32 back = live[live_n - 1];
      live[i] = back;
      lpos[back] = i;
      --live_n;
      t->kinds.push_back('E');
      ++t->n_extract;
    }
    t->offsets.push_back(t->vals.size());
  }
  return t;
}

void pbh_gen_trace_sizes(const pbh_gen_trace* t, uint64_t* n_ops, uint64_t* n_elems,
                         uint64_t* n_extract) {
  *n_ops = t->kinds.size();
  *n_elems = t->vals.size();
  *n_extract = t->n_extract;
}

void pbh_gen_trace_export(const pbh_gen_trace* t, uint8_t* kinds, uint64_t* offsets,
                          uint32_t* values, uint64_t* priorities) {
  std::memcpy(kinds, t->kinds.data(), t->kinds.size());
  std::memcpy(offsets, t->offsets.data(), t->offsets.size() * 8);
  std::memcpy(values, t->vals.data(), t->vals.size() * 4);
  std::memcpy(priorities, t->prios.data(), t->prios.size() * 8);
}

void pbh_gen_trace_free(pbh_gen_trace* t) { delete t; }

void pbh_gen_sweep_prefill(uint64_t n, uint64_t seed, uint64_t* prios_now) {
  std::mt19937_64 rng(seed);
  for (u64 v = 0; v < n; ++v) prios_now[v] = (1ull << 39) + rng() % (1ull << 39);
}

void pbh_gen_sweep_batches(uint64_t n, uint64_t d, uint64_t n_batches, uint64_t seed,
                           uint64_t* prios_now, uint32_t* values, uint64_t* priorities) {
  std::mt19937_64 rng(seed);
  std::vector<u32> keys;
  keys.reserve(d);
  for (u64 b = 0; b < n_batches; ++b) {
    keys.clear();
    while (keys.size() < d) {
      keys.push_back((u32)(rng() % n));
      if (keys.size() == d) {
        std::sort(keys.begin(), keys.end());
        keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
      }
    }
    for (u64 j = 0; j < d; ++j) {
      const u32 k = keys[j];
      prios_now[k] -= 1 + rng() % 1024;
      values[b * d + j] = k;
      priorities[b * d + j] = prios_now[k];
    }
  }
}

}  // extern "C"
