// pbh-b200 device engine: a bucket heap (Iacono, Karsin, Sitchinava,
// arXiv 1908.09378) re-designed for one Blackwell CTA per queue.
//
// Reference semantics restated here (paths relative to /root/reference/proj):
//   * element order (priority, value) lexicographic   element.hpp:30-33
//   * splitter admits / infinity                       element.hpp:46-72
//   * level capacities B_i = 2d*4^i, S_i = d*4^i        bucket_heap.hpp:54-55
//   * op on level 0 followed by resolve(0)             engine.cpp:41-68
//   * resolve(i) after every 4th resolve(i-1)          scheduler.cpp:11-20
//   * resolve phase 1 (absorb S_i, cut, push down)     bucket_heap.cpp:196-224
//   * resolve phase 2 (refill B_i from level i+1)      bucket_heap.cpp:228-271
//   * delete_duplicates keep-min / DEL annihilation    primitives.cpp:25-57
//   * drop_stale_duplicates                            primitives.cpp:103-120
//
// What changes on B200:
//   * Levels are structure-of-arrays runs (u32 key[], u64 prio[]) in HBM,
//     kept sorted by (priority, value) instead of by value, so a splitter
//     cut is a prefix and a refill is a merge-path pull from two run heads.
//   * A per-key position index idx[key] = {prio, state, parent} (16 B)
//     replaces DEL signals and duplicate annihilation: an entry (k, p) is
//     valid iff idx[k].state == LIVE && idx[k].prio == p. Stale copies are
//     dropped inside every merge (fused filter) and never resurrect because
//     priorities only decrease.
//   * Level 0 (B_0) lives in shared memory and is kept clean eagerly:
//     a decrease or delete whose old copy is <= splitter_0 removes it from
//     B_0 by binary search, so extract_min is B_0[head] with no index read.
//   * Every primitive is CTA-wide: warp-shuffle scans, k-ary merge-path
//     searches, shared-memory tile merges with VT outputs per thread.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "pbh_types.h"

namespace pbh_dev {

using u8 = uint8_t;
using u32 = uint32_t;
using u64 = uint64_t;
using i64 = int64_t;

#define DEV __device__ __forceinline__
#define NOINL __device__ __noinline__

DEV bool less_pk(u64 pa, u32 ka, u64 pb, u32 kb) { return pa < pb || (pa == pb && ka < kb); }

// Splitter::admits (element.hpp:55-59): key <= splitter, infinity admits all.
DEV bool admits(const pbh_level_state& s, u64 p, u32 k) {
  return s.spl_inf || p < s.spl_p || (p == s.spl_p && k <= s.spl_k);
}

DEV bool entry_valid(const pbh_idx_entry* idx, u32 k, u64 p) {
  const ulonglong2 e = __ldcg(reinterpret_cast<const ulonglong2*>(idx + k));
  return PBH_ST((u32)e.y) == PBH_ST_LIVE && e.x == p;
}

// 4-byte global -> shared copy that bypasses registers (zero-fill when !pred).
DEV void cp_async4(void* smem, const void* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(pred ? 4 : 0)
               : "memory");
}
// Warp-cooperative L2 prefetch of the first 2 KB of two 4-byte arrays over
// [i0, i1): lanes 0-15 take the lines of a, lanes 16-31 those of b, one
// prefetch.global.L2 each (no uniform operands, so no divergent waterfall).
DEV void l2_prefetch_rows(const u32* a, const u32* b, u64 i0, u64 i1, u32 lane) {
  const u32* arr = lane < 16 ? a : b;
  const u64 lo = reinterpret_cast<u64>(arr + i0), hi = reinterpret_cast<u64>(arr + i1);
  const u64 line = (lo & ~127ull) + (u64)(lane & 15) * 128;
  if (line < hi) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(line));
}
// Bulk L2 prefetch of the 4-byte array range [a[i0], a[i1]) (16-byte granular).
DEV void l2_prefetch_range(const u32* a, u64 i0, u64 i1) {
  const u64 b0 = (reinterpret_cast<u64>(a + i0)) & ~15ull;
  const u64 b1 = (reinterpret_cast<u64>(a + i1) + 15) & ~15ull;
  if (b1 > b0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(b0), "r"((u32)(b1 - b0))
                 : "memory");
}
// 8-byte global -> shared copy (both 8-byte aligned).
DEV void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// --------------------------------------------------------------------------
// CTA primitives
// --------------------------------------------------------------------------
template <int NT>
struct Blk {
  static constexpr int NW = NT / 32;
  DEV static void sync() {
    if constexpr (NT == 32) {
      __syncwarp();
    } else {
      __syncthreads();
    }
  }
  // Exclusive scan over the CTA. scratch: u32[NW + 1] in smem.
  DEV static u32 scan_excl(u32 x, u32& total, u32* scratch) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    u32 v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      u32 y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    if constexpr (NW == 1) {
      total = __shfl_sync(0xffffffffu, v, 31);
      return v - x;
    } else {
      if (lane == 31) scratch[w] = v;
      __syncthreads();
      if (w == 0) {
        u32 s = lane < NW ? scratch[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          u32 y = __shfl_up_sync(0xffffffffu, s, o);
          if (lane >= o) s += y;
        }
        if (lane < NW) scratch[lane] = s;
      }
      __syncthreads();
      const u32 base = w ? scratch[w - 1] : 0;
      total = scratch[NW - 1];
      __syncthreads();
      return base + v - x;
    }
  }
  DEV static u32 sum(u32 x, u32* scratch) {
    u32 t;
    scan_excl(x, t, scratch);
    return t;
  }
  DEV static bool any(bool p, u32* scratch) {
    if constexpr (NW == 1) {
      return __any_sync(0xffffffffu, p);
    } else {
      return __syncthreads_or(p) != 0;
    }
  }
};

// Smallest a in [lo, hi] with !pred(a), for pred monotone (true..false) on
// [lo, hi); pred(hi) is never evaluated. k-ary: each round every thread
// tests one probe, so a span of NT^r resolves in r rounds of one load each.
template <int NT, class Pred>
DEV u32 kary_search(u32 lo, u32 hi, Pred pred, u32* scratch) {
  using B = Blk<NT>;
  while (lo < hi) {
    const u32 span = hi - lo;
    if (span <= (u32)NT) {
      const bool t = threadIdx.x < span && pred(lo + threadIdx.x);
      return lo + B::sum(t ? 1u : 0u, scratch);
    }
    // probes m_t = lo + floor(span * (t+1) / (NT+1)), t = 0..NT-1
    const u32 m = lo + (u32)(((u64)span * (threadIdx.x + 1)) / (NT + 1));
    const bool t = pred(m);
    const u32 ntrue = B::sum(t ? 1u : 0u, scratch);
    // probes are nondecreasing in t; pred true on a prefix of them
    const u32 new_lo = ntrue ? lo + (u32)(((u64)span * ntrue) / (NT + 1)) + 1 : lo;
    const u32 new_hi = ntrue < (u32)NT ? lo + (u32)(((u64)span * (ntrue + 1)) / (NT + 1)) : hi;
    lo = new_lo;
    hi = new_hi;
  }
  return lo;
}

// --------------------------------------------------------------------------
// Runs and sinks
// --------------------------------------------------------------------------
struct Run {
  const u32* k;
  const u64* p;
  u32 n;
};

// Output stream: position pos < lim goes to (k1, p1)[pos], the rest to
// (k2, p2)[pos - lim].
struct Sink {
  u32* k1;
  u64* p1;
  u32 lim;
  u32* k2;
  u64* p2;
  DEV void put(u32 pos, u32 k, u64 p) const {
    if (pos < lim) {
      k1[pos] = k;
      p1[pos] = p;
    } else {
      k2[pos - lim] = k;
      p2[pos - lim] = p;
    }
  }
};

// Merge-path split: number of A elements among the first c outputs of
// merge(A, B) (A first on ties; keys are distinct so ties do not occur).
template <int NT>
DEV u32 merge_split(const Run& A, const Run& B, u32 c, u32* scratch) {
  const u32 lo = c > B.n ? c - B.n : 0;
  const u32 hi = c < A.n ? c : A.n;
  return kary_search<NT>(
      lo, hi, [&](u32 a) { return less_pk(A.p[a], A.k[a], B.p[c - 1 - a], B.k[c - 1 - a]); },
      scratch);
}

// Both merge-path splits of one output range [c0, c1) at once: each half
// of the CTA runs a k-ary search with NT/2 probes per round, so the two
// HBM-latency-bound searches overlap instead of running back to back.
// scratch: u32[NT/32 + 2].
template <int NT>
DEV u32 merge_split(const Run& A, const Run& B, u32 c, u32* scratch);

template <int NT>
DEV void merge_split2(const Run& A, const Run& B, u32 c0, u32 c1, u32* scratch, u32& a0, u32& a1) {
  if constexpr (NT < 64) {  // one warp: the two searches in sequence
    a0 = merge_split<NT>(A, B, c0, scratch);
    a1 = merge_split<NT>(A, B, c1, scratch);
    return;
  } else {
  constexpr u32 H = NT / 2;
  const u32 half = threadIdx.x >= H, t = threadIdx.x - half * H;
  const u32 lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const u32 c = half ? c1 : c0;
  u32 lo = c > B.n ? c - B.n : 0, hi = c < A.n ? c : A.n;
  auto pred = [&](u32 a) { return less_pk(A.p[a], A.k[a], B.p[c - 1 - a], B.k[c - 1 - a]); };
  for (;;) {
    const bool active = lo < hi;
    if (!__syncthreads_or(active)) break;
    const u32 span = hi - lo;
    bool pt = false;
    if (active) {
      if (span <= H) {
        pt = t < span && pred(lo + t);
      } else {
        pt = pred(lo + (u32)(((u64)span * (t + 1)) / (H + 1)));
      }
    }
    const u32 cnt = __popc(__ballot_sync(0xffffffffu, pt));
    if (lane == 0) scratch[w] = cnt;
    __syncthreads();
    u32 ntrue = 0;
#pragma unroll
    for (u32 i = 0; i < H / 32; ++i) ntrue += scratch[half * (H / 32) + i];
    __syncthreads();
    if (active) {
      if (span <= H) {
        lo += ntrue;
        hi = lo;
      } else {
        const u32 nl = ntrue ? lo + (u32)(((u64)span * ntrue) / (H + 1)) + 1 : lo;
        const u32 nh = ntrue < H ? lo + (u32)(((u64)span * (ntrue + 1)) / (H + 1)) : hi;
        lo = nl;
        hi = nh;
      }
    }
  }
  if (t == 0) scratch[half] = lo;
  __syncthreads();
  a0 = scratch[0];
  a1 = scratch[1];
  __syncthreads();
  }
}

// ---- 1-D TMA (cp.async.bulk) staging with an mbarrier --------------------
DEV u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
DEV void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// Arm the barrier for `bytes` of async-proxy transfers (one arrival).
DEV void mbar_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
DEV void mbar_wait(u64* bar, u32 parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Order this thread's earlier generic-proxy shared-memory accesses before
// later async-proxy (TMA) writes to the same buffers.
DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// Bulk copy of `bytes` (multiple of 16, both addresses 16-byte aligned)
// from global memory into this CTA's shared memory, completing on `bar`.
DEV void tma_load_1d(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Bulk store of `bytes` (multiple of 16, both addresses 16-byte aligned)
// from this CTA's shared memory to global memory, in the thread's bulk group.
DEV void tma_store_1d(void* dst, const void* src, u32 bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// The committed bulk stores have read their shared-memory sources.
DEV void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
// The committed bulk stores are complete (their writes visible).
DEV void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

// A 16-byte aligned window covering elements [i, i + n) of an array of
// E-byte elements: source address, element offset of i inside the window,
// and the copy size.
template <int E>
struct Window {
  const void* src = nullptr;
  u32 off = 0, bytes = 0;
  Window() = default;
  DEV Window(const void* base, u32 i, u32 n) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(base) + (uintptr_t)i * E;
    const uintptr_t a0 = a & ~uintptr_t(15);
    src = reinterpret_cast<const void*>(a0);
    off = (u32)((a - a0) / E);
    bytes = (u32)(((a - a0) + (uintptr_t)n * E + 15) & ~uintptr_t(15));
  }
};

// Shared-memory scratch needed by the merge machinery.
template <int NT, int VT>
struct TileSmem {
  static constexpr int T = NT * VT;
  u32 k[T];
  u64 p[T];
};

// Merge exactly ca elements of A (from a0) with cb elements of B (from b0)
// — one merge-path tile, ca + cb <= NT*VT — optionally dropping entries that
// fail the index check, and stream the survivors to `sink` from out_base.
// Returns the number written. If last_k/last_p are non-null, thread 0 stores
// the last element of the tile in merged order (valid or not).
template <int NT, int VT>
NOINL u32 merge_tile(const Run& A, u32 a0, u32 ca, const Run& B, u32 b0, u32 cb, bool filter,
                   const pbh_idx_entry* idx, const Sink& sink, u32 out_base,
                   TileSmem<NT, VT>& ts, u32* scratch) {
  using Bk = Blk<NT>;
  const u32 c = ca + cb;
  for (u32 i = threadIdx.x; i < c; i += NT) {
    if (i < ca) {
      ts.k[i] = A.k[a0 + i];
      ts.p[i] = A.p[a0 + i];
    } else {
      ts.k[i] = B.k[b0 + i - ca];
      ts.p[i] = B.p[b0 + i - ca];
    }
  }
  Bk::sync();
  // per-thread diagonal
  const u32 d0 = min((u32)threadIdx.x * VT, c);
  const u32 d1 = min(d0 + VT, c);
  u32 lo = d0 > cb ? d0 - cb : 0, hi = d0 < ca ? d0 : ca;
  while (lo < hi) {
    const u32 m = (lo + hi) >> 1;
    const u32 j = ca + (d0 - 1 - m);
    if (less_pk(ts.p[m], ts.k[m], ts.p[j], ts.k[j]))
      lo = m + 1;
    else
      hi = m;
  }
  u32 ia = lo, ib = d0 - lo;  // ib indexes B-part (offset ca in ts)
  u32 ok[VT];
  u64 op[VT];
  u32 nv = 0;
  bool keep[VT];
#pragma unroll
  for (int v = 0; v < VT; ++v) {
    keep[v] = false;
    if (d0 + v < d1) {
      bool takeA;
      if (ia >= ca)
        takeA = false;
      else if (ib >= cb)
        takeA = true;
      else
        takeA = less_pk(ts.p[ia], ts.k[ia], ts.p[ca + ib], ts.k[ca + ib]);
      const u32 s = takeA ? ia++ : ca + ib++;
      ok[v] = ts.k[s];
      op[v] = ts.p[s];
      keep[v] = true;
    }
  }
  if (filter) {
#pragma unroll
    for (int v = 0; v < VT; ++v)
      if (keep[v]) keep[v] = entry_valid(idx, ok[v], op[v]);
  }
#pragma unroll
  for (int v = 0; v < VT; ++v) nv += keep[v];
  u32 total;
  u32 pos = out_base + Bk::scan_excl(nv, total, scratch);
#pragma unroll
  for (int v = 0; v < VT; ++v)
    if (keep[v]) sink.put(pos++, ok[v], op[v]);
  Bk::sync();
  return total;
}

// Full merge of A[0..na) and B[0..nb) into sink (filtered or not).
template <int NT, int VT>
NOINL u32 merge_runs(const Run& A, const Run& B, bool filter, const pbh_idx_entry* idx,
                   const Sink& sink, u32 out_base, TileSmem<NT, VT>& ts, u32* scratch) {
  constexpr u32 T = NT * VT;
  const u32 total = A.n + B.n;
  u32 a_prev = 0, written = 0;
  for (u32 t0 = 0; t0 < total; t0 += T) {
    const u32 t1 = min(t0 + T, total);
    const u32 a1 = merge_split<NT>(A, B, t1, scratch);
    const u32 b_prev = t0 - a_prev, b1 = t1 - a1;
    written += merge_tile<NT, VT>(A, a_prev, a1 - a_prev, B, b_prev, b1 - b_prev, filter, idx,
                                  sink, out_base + written, ts, scratch);
    a_prev = a1;
  }
  return written;
}

// Copy a run (optionally filtered) into sink at out_base.
template <int NT, int VT>
NOINL u32 copy_run(const Run& A, bool filter, const pbh_idx_entry* idx, const Sink& sink,
                 u32 out_base, u32* scratch) {
  using Bk = Blk<NT>;
  u32 written = 0;
  for (u32 t0 = 0; t0 < A.n; t0 += NT * VT) {
    u32 nv = 0;
    u32 kk[VT];
    u64 pp[VT];
    bool keep[VT];
#pragma unroll
    for (int v = 0; v < VT; ++v) {
      const u32 i = t0 + threadIdx.x * VT + v;
      keep[v] = i < A.n;
      if (keep[v]) {
        kk[v] = A.k[i];
        pp[v] = A.p[i];
      }
    }
    if (filter) {
#pragma unroll
      for (int v = 0; v < VT; ++v)
        if (keep[v]) keep[v] = entry_valid(idx, kk[v], pp[v]);
    }
#pragma unroll
    for (int v = 0; v < VT; ++v) nv += keep[v];
    u32 total;
    u32 pos = out_base + written + Bk::scan_excl(nv, total, scratch);
#pragma unroll
    for (int v = 0; v < VT; ++v)
      if (keep[v]) sink.put(pos++, kk[v], pp[v]);
    written += total;
  }
  Bk::sync();
  return written;
}

// Number of run elements admitted by a splitter (an upper bound: runs are
// (p, k)-sorted so the admitted ones form a prefix).
template <int NT>
DEV u32 count_admitted(const Run& A, const pbh_level_state& s, u32* scratch) {
  if (s.spl_inf) return A.n;
  return kary_search<NT>(0, A.n, [&](u32 i) { return admits(s, A.p[i], A.k[i]); }, scratch);
}

// Bitonic sort of n <= cap (pow2) elements in shared memory by (p, k).
// Padding slots hold (~0, ~0); a real (~0, ~0) is indistinguishable from
// padding and sorts identically, so the first n outputs are exact.
template <int NT>
NOINL void bitonic_sort(u32* k, u64* p, u32 n) {
  using Bk = Blk<NT>;
  if (n <= 1) return;
  u32 m = 1;
  while (m < n) m <<= 1;
  for (u32 i = n + threadIdx.x; i < m; i += NT) {
    k[i] = 0xffffffffu;
    p[i] = ~0ull;
  }
  Bk::sync();
  for (u32 size = 2; size <= m; size <<= 1) {
    for (u32 stride = size >> 1; stride > 0; stride >>= 1) {
      for (u32 t = threadIdx.x; t < (m >> 1); t += NT) {
        const u32 i = 2 * t - (t & (stride - 1));
        const u32 j = i + stride;
        const bool up = (i & size) == 0;
        const bool sw = less_pk(p[j], k[j], p[i], k[i]) == up;
        if (sw) {
          const u32 tk = k[i];
          k[i] = k[j];
          k[j] = tk;
          const u64 tp = p[i];
          p[i] = p[j];
          p[j] = tp;
        }
      }
      Bk::sync();
    }
  }
}

}  // namespace pbh_dev
