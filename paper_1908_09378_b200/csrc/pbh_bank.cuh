// Banked level 0 for par_dijkstra (sssp.cpp:21-69): the default SSSP engine.
//
// One CTA of NW warps (B = 32*NW threads) owns one source's bucket heap.
// Level 0 (everything <= splitter_0, bucket_heap.hpp:37-41) is an UNSORTED
// slot array in shared memory, banked by thread: slot s = i*B + t belongs to
// thread t, which keeps its bank's occupancy mask and minimum in registers.
//   extract_min   = a CTA argmin of the B bank minima (three redux.sync per
//                   warp, one barrier), then the owner rescans its bank;
//   insert        = the relaxing thread takes a free slot of its own bank;
//   decrease-key  = in place: the position index records the slot, the
//                   relaxing thread overwrites the priority and flags the
//                   owner, which rescans its bank in the next pass.
// Each slot carries its vertex's CSR row (begin, degree), captured from the
// offsets gathered with the index entry at relax time, so the extracted
// vertex's row needs no dependent offsets load.
//
// A round relaxes the extracted vertex's row in passes of 256 edges (256/B
// per thread, thread t taking the edges j with (j - round) mod B == t so the
// new slots spread over the banks). Every pass ends with ONE barrier that
// exchanges each warp's best offer (its bank minima and its applied admitted
// candidates) and its counters. After the last pass that argmin IS the next
// extraction: a decreased slot's stale bank minimum is larger than the
// candidate that replaced it, and that candidate is offered by its writer.
// So the next row's first pass is loaded before the round's bookkeeping and
// the owners' rescans, which run under its latency.
//
// Deeper levels are the CTA engine of pbh_heap.cuh in HBM (cold path):
//   * candidates beyond splitter_0 collect in a push buffer, sorted and
//     merged into S_1 (push_down) in batches;
//   * when a bank runs out of room for a pass, level 0 is sorted, the largest
//     half is pushed into S_1 and the splitter lowered (the capacity cut of
//     bucket_heap.cpp:205-219); the kept half is redistributed round-robin;
//   * when level 0 empties, fill0() refills it with the smallest cap0
//     entries of the deeper levels (bucket_heap.cpp:228-271);
//   * resolve(i) runs after every 4^i-th push (scheduler.cpp:11-20).
// Stale copies below level 0 are dropped by the index filter of every merge.
#pragma once

#include "pbh_kernels.cuh"
#include "pbh_grid.cuh"

namespace pbh_dev {

constexpr int kBankQ = 4096;    // push-buffer capacity (entries beyond the splitter)
constexpr int kBankPass = 256;  // edges relaxed per pass
constexpr u32 kGridFlushMin = 1024;  // push-buffer flushes at least this large sort on the grid

// The part of the shared-memory image that survives a NEED_GROW relaunch.
template <int B, int KI, bool MW = false>
struct BankL0 {
  static constexpr int C0 = B * KI;
  u64 lp[C0];    // slot priority
  u64 lrb[C0];   // slot vertex's CSR row begin
  u32 lk[C0];    // slot key (vertex)
  u32 ldeg[C0];  // slot vertex's out-degree
  u64 qp[kBankQ];
  u32 qk[kBankQ];
  u32 occ[B];    // per-thread occupancy masks (bit i = slot i*B + t)
  u64 spl_p;
  u32 spl_k, spl_inf, qn, pad;
  u64 pushes;    // push_down count (drives the 4-to-1 resolve schedule)
  // multi-extraction mode: the slot vertex's minimum out / in edge weight
  u32 lmo[MW ? C0 : 1];
  u32 lmi[MW ? C0 : 1];
};

// One warp's offer and counters for the per-pass exchange.
struct BankOffer {
  u64 p, rb;
  u64 t;  // multi-extraction: min over offers of (p + min out weight)
  u32 k, slot, deg, has;
  u32 fresh, nimp, nq, flags;  // flags: 1 evict due, 2 bad slot, 4 overflow
};

// A warp's offer in the SSSP rounds' exchange: (p, k) = (~0, ~0) is "none";
// the winner's row is read from its slot after the barrier.
struct __align__(16) LeanOffer {
  u64 p;
  u32 k, slot;
  u32 c0, c1, pad0, pad1;
};

#ifndef PBH_MULTI_B0_EIGHTHS
#define PBH_MULTI_B0_EIGHTHS 6  // threshold engine's B_0: 3/4 of level 0
#endif
// 5/8 measured equal on the 2048² grid; 7/8 leaves a refill no free slot
// (invariant site 0xE5), so the bound is 3/4
static_assert(PBH_MULTI_B0_EIGHTHS >= 1 && PBH_MULTI_B0_EIGHTHS <= 6, "threshold B_0 above 3/4 of level 0");
template <int NW, int KI, int VT, bool MW = false>
struct BankSmem {
  static constexpr int B = 32 * NW;
  static constexpr int C0 = B * KI;
  BankL0<B, KI, MW> l0;
  // cold-engine B_0 ping-pong; as one array (>= C0 entries) it is also the
  // sort scratch of evict(). A refill pulls up to its capacity: C0/2, or
  // 3/4 of C0 for the threshold engine (its batches drain level 0 fast;
  // fewer, larger refills)
  static constexpr int B0CAP = MW ? (C0 * PBH_MULTI_B0_EIGHTHS) / 8 : C0 / 2;
  u32 bk[2][B0CAP];
  u64 bp[2][B0CAP];
  u32 sk[kBankQ];  // sort scratch of the push-buffer flush
  u64 sp[kBankQ];
  u32 pf_t[kBankPass];  // next row's first pass, prefetched by cp.async
  u32 pf_w[kBankPass];
  BankOffer ex[2][NW];  // per-pass exchange (parity double-buffered)
  LeanOffer lx[2][NW];  // the SSSP rounds' lean exchange
  u8 dirty[2][B];       // decreased-bank flags (parity double-buffered)
  u64 fr_lo[NW], fr_hi[NW];  // grid flush: per-warp priority range
  u32 fr_nb;
  HeapSmem<B, VT> hs;
#ifdef PBH_XPROF
  long long xarr[2][NW];  // per-warp barrier arrival clocks (diagnostics)
  long long xph[2][NW][8];  // per-warp phase cycles of this pass (PBH_PROF_BUILD)
#endif
};

template <int NW, int KI, int VT, bool MW = false>
DEV BankSmem<NW, KI, VT, MW>& bank_smem() {
  extern __shared__ __align__(16) unsigned char dyn[];
  return *reinterpret_cast<BankSmem<NW, KI, VT, MW>*>(dyn);
}

// ceil(a / b) out of line: the integer division stays off the hot path
// (ptxas otherwise if-converts it into every round)
__device__ __noinline__ u32 ceil_div_cold(u32 a, u32 b) { return (a + b - 1) / b; }

// warp argmin of (p, k) over lanes with `has`; returns the winning lane.
DEV u32 warp_argmin(bool& has, u64& p, u32& k) {
  const u32 hi = has ? (u32)(p >> 32) : 0xffffffffu;
  const u32 mhi = __reduce_min_sync(0xffffffffu, hi);
  const bool c1 = has && hi == mhi;
  const u32 lo = c1 ? (u32)p : 0xffffffffu;
  const u32 mlo = __reduce_min_sync(0xffffffffu, lo);
  const bool c2 = c1 && (u32)p == mlo;
  const u32 mk = __reduce_min_sync(0xffffffffu, c2 ? k : 0xffffffffu);
  const u32 win = __ballot_sync(0xffffffffu, c2 && k == mk);
  has = win != 0;
  p = ((u64)mhi << 32) | mlo;
  k = mk;
  return win ? __ffs(win) - 1 : 0;
}

// This thread's bank minimum (inline on kernel locals so they stay in registers).
template <int B, int KI, bool MW>
DEV void bank_rescan(const BankL0<B, KI, MW>& L, u32 tid, u32 occm, bool& lhas, u64& lmin_p,
                     u32& lmin_k, u32& lmin_s) {
  lhas = false;
  u32 m = occm;
  while (m) {
    const u32 i = __ffs(m) - 1;
    m &= m - 1;
    const u32 s = i * B + tid;
    const u64 p = L.lp[s];
    const u32 k = L.lk[s];
    if (!lhas || less_pk(p, k, lmin_p, lmin_k)) {
      lhas = true;
      lmin_p = p;
      lmin_k = k;
      lmin_s = s;
    }
  }
}


// Per-pass exchange: CTA argmin of the offers (has, p, k) with their slot
// and row, and the sums of the counters. One barrier. Counters are packed
// 9 bits each (every one is <= 256 per pass): c0 = fresh | nimp << 9 |
// ovf << 18, c1 = nq | evict << 9 | bad << 18 (the last two per-thread flags).
__device__ unsigned long long g_xprof[16];
__device__ unsigned long long g_xprof2[8];  // PBH_PHASES: exchange breakdown (thread 0, block 0)

template <int NW, int KI, int VT, bool MW = false>
DEV BankOffer bank_exchange(u32 par, bool has, u64 p, u32 k, u32 slot, u64 rb, u32 deg, u32 c0,
                            u32 c1, u64 t = ~0ull) {
  BankSmem<NW, KI, VT, MW>& S = bank_smem<NW, KI, VT, MW>();
  const u32 tid = threadIdx.x;
  const u32 lane = tid & 31, w = tid >> 5;
#ifdef PBH_XPROF
  auto clk = []() {
    long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
    return c;
  };
  const long long xa = clk();
#endif
  bool h = has;
  u64 wp = p;
  u32 wk = k;
  const u32 wl = warp_argmin(h, wp, wk);
  const u32 s0 = __reduce_add_sync(0xffffffffu, c0);
  const u32 s1 = __reduce_add_sync(0xffffffffu, c1);
  u64 wt_ = ~0ull;
  if constexpr (MW) {  // warp min of t (u64) in two 32-bit reductions
    const u32 thi = __reduce_min_sync(0xffffffffu, (u32)(t >> 32));
    const u32 tlo = __reduce_min_sync(0xffffffffu, (u32)(t >> 32) == thi ? (u32)t : 0xffffffffu);
    wt_ = ((u64)thi << 32) | tlo;
  }
  if (lane == wl) {
    BankOffer& o = S.ex[par][w];
    o.t = wt_;
    o.p = wp;
    o.k = wk;
    o.has = h;
    o.slot = slot;
    o.rb = rb;
    o.deg = deg;
    o.fresh = s0;
    o.nq = s1;
  }
  if constexpr (NW == 1) {
    __syncwarp();
    BankOffer r;
    r.p = wp;
    r.k = wk;
    r.has = h;
    r.slot = __shfl_sync(0xffffffffu, slot, wl);
    r.rb = __shfl_sync(0xffffffffu, rb, wl);
    r.deg = __shfl_sync(0xffffffffu, deg, wl);
    r.t = wt_;
    r.fresh = s0 & 511u;
    r.nimp = (s0 >> 9) & 511u;
    r.nq = s1 & 511u;
    r.flags = ((s1 >> 9) & 511u ? 1u : 0u) | ((s1 >> 18) & 511u ? 2u : 0u) | ((s0 >> 18) & 511u ? 4u : 0u);
    return r;
  } else {
#ifdef PBH_XPROF
    const long long xb = clk();
    if (lane == 0) S.xarr[par][w] = xb;
#endif
    __syncthreads();
#ifdef PBH_XPROF
    const long long xc = clk();
#endif
    // tree argmin over the NW warp winners (index only), then one read
    u32 bi = 0;
    bool bh = S.ex[par][0].has;
    u64 bp = S.ex[par][0].p;
    u32 bk = S.ex[par][0].k;
    u32 t0 = S.ex[par][0].fresh, t1 = S.ex[par][0].nq;
    u64 tm = S.ex[par][0].t;
#pragma unroll
    for (int i = 1; i < NW; ++i) {
      const bool xh = S.ex[par][i].has;
      const u64 xp = S.ex[par][i].p;
      const u32 xk = S.ex[par][i].k;
      t0 += S.ex[par][i].fresh;
      t1 += S.ex[par][i].nq;
      if constexpr (MW) tm = min(tm, S.ex[par][i].t);
      if (xh && (!bh || less_pk(xp, xk, bp, bk))) {
        bh = true;
        bp = xp;
        bk = xk;
        bi = i;
      }
    }
    BankOffer r;
    r.p = bp;
    r.k = bk;
    r.has = bh;
    r.slot = S.ex[par][bi].slot;
    r.rb = S.ex[par][bi].rb;
    r.deg = S.ex[par][bi].deg;
    r.t = tm;
    r.fresh = t0 & 511u;
    r.nimp = (t0 >> 9) & 511u;
    r.nq = t1 & 511u;
    r.flags = ((t1 >> 9) & 511u ? 1u : 0u) | ((t1 >> 18) & 511u ? 2u : 0u) | ((t0 >> 18) & 511u ? 4u : 0u);
#ifdef PBH_XPROF
    if (blockIdx.x == 0 && (tid & 31) == 0) {
      const long long xd = clock64();
      atomicAdd(&g_xprof[0], (unsigned long long)(xb - xa));
      atomicAdd(&g_xprof[1], (unsigned long long)(xc - xb));
      atomicAdd(&g_xprof[2], (unsigned long long)(xd - xc));
      atomicAdd(&g_xprof[3], 1ull);
      if (tid == 0) {  // skew: last - first arrival, release latency, which warp was last
        long long mx = S.xarr[par][0], mn = mx;
        int lw = 0;
        for (int i = 1; i < NW; ++i) {
          const long long a = S.xarr[par][i];
          if (a > mx) mx = a, lw = i;
          mn = a < mn ? a : mn;
        }
        atomicAdd(&g_xprof[4], (unsigned long long)(mx - mn));
        atomicAdd(&g_xprof[5], (unsigned long long)(xc - mx));
        atomicAdd(&g_xprof[6], 1ull);
        atomicAdd(&g_xprof[8 + lw], 1ull);
        if (mx - mn > 1000) atomicAdd(&g_xprof[7], 1ull);
        // phase excess of the last warp over the mean of the others
        for (int ph = 0; ph < 8; ++ph) {
          long long o = 0;
          for (int i = 0; i < NW; ++i)
            if (i != lw) o += S.xph[par][i][ph];
          atomicAdd(&g_xprof2[ph], (unsigned long long)(S.xph[par][lw][ph] - o / (NW - 1)));
        }
      }
    }
#endif
    return r;
  }
}

// Lean per-pass exchange of the SSSP rounds: CTA argmin of (p, k) with the
// offering slot, plus the packed counter sums (see bank_exchange). Absent
// offers are (~0, ~0). Branch-free combine of the NW warp winners.
struct LeanRes {
  u64 p;
  u32 k, slot;
  bool has;
  u32 fresh, nimp, nq, flags;
};
template <int NW, int KI, int VT>
DEV LeanRes lean_exchange(u32 par, u64 p, u32 k, u32 slot, u32 c0, u32 c1) {
  BankSmem<NW, KI, VT>& S = bank_smem<NW, KI, VT>();
  const u32 lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const u32 hi = (u32)(p >> 32);
  const u32 mhi = __reduce_min_sync(0xffffffffu, hi);
  const bool e1 = hi == mhi;
  const u32 mlo = __reduce_min_sync(0xffffffffu, e1 ? (u32)p : 0xffffffffu);
  const bool e2 = e1 && (u32)p == mlo;
  const u32 mk = __reduce_min_sync(0xffffffffu, e2 ? k : 0xffffffffu);
  const u32 win = __ballot_sync(0xffffffffu, e2 && k == mk);
  const u32 s0 = __reduce_add_sync(0xffffffffu, c0);
  const u32 s1 = __reduce_add_sync(0xffffffffu, c1);
  if (lane == (u32)(__ffs(win) - 1)) {
    LeanOffer o;
    o.p = ((u64)mhi << 32) | mlo;
    o.k = mk;
    o.slot = slot;
    o.c0 = s0;
    o.c1 = s1;
    o.pad0 = o.pad1 = 0;
    S.lx[par][w] = o;
  }
  __syncthreads();
  LeanOffer b = S.lx[par][0];
  u32 t0 = b.c0, t1 = b.c1;
#pragma unroll
  for (int i = 1; i < NW; ++i) {
    const LeanOffer x = S.lx[par][i];
    t0 += x.c0;
    t1 += x.c1;
    const bool lt = x.p < b.p || (x.p == b.p && x.k < b.k);
    b.p = lt ? x.p : b.p;
    b.k = lt ? x.k : b.k;
    b.slot = lt ? x.slot : b.slot;
  }
  LeanRes r;
  r.p = b.p;
  r.k = b.k;
  r.slot = b.slot;
  r.has = !(b.p == ~0ull && b.k == 0xffffffffu);
  r.fresh = t0 & 511u;
  r.nimp = (t0 >> 9) & 511u;
  r.nq = t1 & 511u;
  r.flags = ((t1 >> 9) & 511u ? 1u : 0u) | ((t1 >> 18) & 511u ? 2u : 0u) | ((t0 >> 18) & 511u ? 4u : 0u);
  return r;
}

template <int NW, int KI, int VT, bool MW = false>
struct BankHeap {
  static constexpr int B = 32 * NW;
  static constexpr int C0 = B * KI;
  static constexpr u32 PE = kBankPass / B;  // edges per thread per pass
  static_assert(KI <= 32, "occupancy mask is 32 bits");
  static_assert(KI >= (int)PE, "a bank must hold one pass of inserts");
  using HC = HeapCta<B, VT>;
  using Bk = Blk<B>;
  using SM = BankSmem<NW, KI, VT, MW>;
  HC& hc;
  SM& S;
  BankL0<B, KI, MW>& L;
  pbh_idx_entry* idx;
  const u64* off;
  const u32* mwo = nullptr;  // multi-extraction: per-vertex min out / in weight
  const u32* mwi = nullptr;
  const u32 tid;
  // per-thread
  u32 occm;
  bool lhas;
  u64 lmin_p;
  u32 lmin_k, lmin_s;
  // replicated
  i64 live;
  u64 pushes;
  u64 deep_n;
  u32 n_l0;
  u32 qn;  // push-buffer fill (mirrors L.qn at pass boundaries)
  unsigned long long* prof = nullptr;  // PBH_PROF counters 8.. (cold-path breakdown)
  BatchJob* bj = nullptr;  // grid sort buffers (trace interpreter with helpers)
  DEV void pr(int i, long long& t) {
    if (prof && tid == 0) {
      const long long t1 = clock64();
      atomicAdd(prof + i, (unsigned long long)(t1 - t));
      t = t1;
    }
  }

  DEV BankHeap(HC& h, SM& s, pbh_idx_entry* ix, const u64* of)
      : hc(h), S(s), L(s.l0), idx(ix), off(of), tid(threadIdx.x) {}

  DEV bool adm(u64 p, u32 k) const {
    return L.spl_inf || p < L.spl_p || (p == L.spl_p && k <= L.spl_k);
  }

  // Recompute this thread's bank minimum.
  DEV void rescan() {
    lhas = false;
    u32 m = occm;
    while (m) {
      const u32 i = __ffs(m) - 1;
      m &= m - 1;
      const u32 s = i * B + tid;
      const u64 p = L.lp[s];
      const u32 k = L.lk[s];
      if (!lhas || less_pk(p, k, lmin_p, lmin_k)) {
        lhas = true;
        lmin_p = p;
        lmin_k = k;
        lmin_s = s;
      }
    }
  }

  // ------------------------------------------------------------ cold glue
  DEV void to_cold() {
    Bk::sync();
    if (tid == 0) {
      pbh_level_state& t = hc.s.st[0];
      t.b_head = 0;
      t.b_size = 0;
      t.spl_p = L.spl_p;
      t.spl_k = L.spl_k;
      t.spl_inf = L.spl_inf;
      hc.s.live = live;
    }
    Bk::sync();
  }
  DEV void after_cold() { deep_n = hc.content_from(1); }

  // Merge the sorted run (K, P)[0, n) into S_1 and run the 4-to-1 schedule.
  NOINL void push_run(const u32* K, const u64* P, u32 n) {
    if (n == 0) return;
    long long t = clock64();
    to_cold();
    if (__isShared(K) && n <= kBankQ) {
      // stage the run in HBM (g_pk/g_pp hold kBankQ entries) so the merge
      // into S_1 can stream through cp.async windows or run on the grid
      for (u32 i = tid; i < n; i += B) {
        hc.pk[i] = K[i];
        hc.pp[i] = P[i];
      }
      __threadfence_block();
      Bk::sync();
      K = hc.pk;
      P = hc.pp;
    }
    hc.template push_down<true>(0, Run{K, P, n});
    pr(9, t);
    ++pushes;
    for (u32 i = 1; i < hc.s.n_levels && i < 31 && !hc.failed(); ++i) {
      if (pushes & ((1ull << (2 * i)) - 1)) break;  // resolve(i) every 4^i pushes
      hc.resolve(i);
      pr(9 + (i < 6 ? i : 6), t);
    }
    after_cold();
  }

  NOINL void flush_q() {
    Bk::sync();
    const u32 n = qn;
    if (n == 0) return;
    long long t = clock64();
    if (bj && hc.gj && n >= kGridFlushMin &&
        (grid_flush_merge(n, t) || grid_flush_union(n, t))) {
      // sorted and merged into S_1 by one grid job, resolves done
    } else if (bj && hc.gj && n >= kGridFlushMin && grid_flush_sort(n)) {
      pr(8, t);
      push_run(bj->sk[1], bj->sp[1], n);
    } else {
      // through bank_smem() (not the member references) so the inlined sort
      // sees the shared address space and uses LDS/STS
      auto& SS = bank_smem<NW, KI, VT, MW>();
      cta_sort<NW>(SS.l0.qk, SS.l0.qp, n, SS.sk, SS.sp);
      pr(8, t);
      push_run(L.qk, L.qp, n);
    }
    if (tid == 0) L.qn = 0;
    qn = 0;
    Bk::sync();
  }

  // The push buffer merged into S_1 by ONE grid job (job 9: bucket by S_1
  // chunks, sort each bucket, merge it with its chunk), then the 4-to-1
  // resolve schedule. False (nothing changed) when the fused path does not
  // apply: no level 1 yet, S_1 too small to bucket by or without room, a
  // stale share that wants the filtered merge, or a bucket over the tile.
  NOINL bool grid_flush_merge(u32 n, long long& t) {
    if (!grid_push_fits(n)) return false;
    u32* const dk = bj->sk[0];
    u64* const dp = bj->sp[0];
    for (u32 i = tid; i < n; i += B) {
      dk[i] = L.qk[i];
      dp[i] = L.qp[i];
    }
    return grid_push_unsorted(n, false, t);
  }

  // Whether job 9 can take a push of n entries into S_1 now (level 1
  // exists, S_1 is large enough to bucket by and has room, and no filtered
  // merge is due). Writes the level-0 state to the cold engine.
  NOINL bool grid_push_fits(u32 n) {
    if (hc.s.n_levels < 2) return false;
    const pbh_level_state& st1 = hc.s.st[1];
    if (st1.s_size < 4 * hc.gsz || (u64)st1.s_size + n > hc.s.lv[1].buf_s) return false;
    to_cold();
    return !hc.stale_share_above(kGridFilterNum, kGridFilterDen);
  }

  // Job 9 over the unsorted run staged in bj->sk/sp[0][0, n), then the
  // 4-to-1 resolve schedule (push_run's tail). write_idx: publish each
  // entry's index entry {p, LIVE, deep} (a staged big batch). False when a
  // bucket overflowed (S_1 unchanged; the caller sorts and pushes).
  NOINL bool grid_push_unsorted(u32 n, bool write_idx, long long& t) {
    const pbh_level_state st1 = hc.s.st[1];
    const u32 G = hc.gsz;
    for (u32 i = tid; i < G; i += B) bj->bcnt[i] = 0;
    const Run S1 = hc.signal(1);
    const u32 ns = 1 - st1.s_sel;
    if (tid == 0) {
      bj->stg_n = n;
      bj->mk = S1.k;
      bj->mp = S1.p;
      bj->mn = S1.n;
      bj->ok = hc.s.lv[1].sk[ns];
      bj->op = hc.s.lv[1].sp[ns];
      bj->bovf = 0;
      bj->write_idx = write_idx ? 1u : 0u;
    }
    __threadfence();
    Bk::sync();
    grid_run<B>(hc.gj, G, 9, Run{}, Run{}, 0, Sink{}, 0, *hc.gs, hc.gs->scr);
    if (*(volatile u32*)&bj->bovf) return false;
    if (tid == 0) {
      pbh_level_state& s1 = hc.s.st[1];
      s1.s_sel = ns;
      s1.s_head = 0;
      s1.s_size = S1.n + n;
      hc.s.touches[0] += 2ull * (S1.n + n);
    }
    Bk::sync();
    pr(9, t);
    ++pushes;
    for (u32 i = 1; i < hc.s.n_levels && i < 31 && !hc.failed(); ++i) {
      if (pushes & ((1ull << (2 * i)) - 1)) break;  // resolve(i) every 4^i pushes
      hc.resolve(i);
      pr(9 + (i < 6 ? i : 6), t);
    }
    after_cold();
    return true;
  }

  // The push buffer sorted by the whole grid: staged to HBM (bj->sk/sp[0])
  // with its priority range, bucket-sorted into bj->sk/sp[1] (grid job 7,
  // index untouched). False when a bucket overflowed (the caller sorts in
  // the CTA; the push buffer is still intact).
  NOINL bool grid_flush_sort(u32 n) { return grid_flush_bucket(n, nullptr); }

  // S_1 too small for job 9 to bucket by: the push buffer and S_1 sorted
  // together by job 7 straight into S_1's other buffer (no merge job), then
  // the resolve schedule. False (nothing changed) when it does not apply.
  NOINL bool grid_flush_union(u32 n, long long& t) {
    if (hc.s.n_levels < 2) return false;
    const pbh_level_state st1 = hc.s.st[1];
    if (st1.s_size >= 4 * hc.gsz || (u64)st1.s_size + n > hc.s.lv[1].buf_s) return false;
    to_cold();
    if (hc.stale_share_above(kGridFilterNum, kGridFilterDen)) return false;
    const Run S1 = hc.signal(1);
    const u32 ns = 1 - st1.s_sel;
    if (!grid_flush_bucket(n, &S1, hc.s.lv[1].sk[ns], hc.s.lv[1].sp[ns])) return false;
    if (tid == 0) {
      pbh_level_state& s1 = hc.s.st[1];
      s1.s_sel = ns;
      s1.s_head = 0;
      s1.s_size = S1.n + n;
      hc.s.touches[0] += 2ull * (S1.n + n);
    }
    Bk::sync();
    pr(9, t);
    ++pushes;
    for (u32 i = 1; i < hc.s.n_levels && i < 31 && !hc.failed(); ++i) {
      if (pushes & ((1ull << (2 * i)) - 1)) break;  // resolve(i) every 4^i pushes
      hc.resolve(i);
      pr(9 + (i < 6 ? i : 6), t);
    }
    after_cold();
    return true;
  }

  // Job 7 over the push buffer (plus, when `also`, a sorted run folded in),
  // into bj->sk/sp[1] or, when given, (ok, op).
  NOINL bool grid_flush_bucket(u32 n, const Run* also, u32* ok = nullptr, u64* op = nullptr) {
    u64 lo = ~0ull, hi = 0;
    u32* const dk = bj->sk[0];
    u64* const dp = bj->sp[0];
    for (u32 i = tid; i < n; i += B) {
      const u64 p = L.qp[i];
      dk[i] = L.qk[i];
      dp[i] = p;
      lo = min(lo, p);
      hi = max(hi, p);
    }
    const u32 m = also ? also->n : 0u;
    for (u32 i = tid; i < m; i += B) {
      const u64 p = also->p[i];
      dk[n + i] = also->k[i];
      dp[n + i] = p;
      lo = min(lo, p);
      hi = max(hi, p);
    }
    for (int s = 16; s; s >>= 1) {
      lo = min(lo, (u64)__shfl_xor_sync(0xffffffffu, (unsigned long long)lo, s));
      hi = max(hi, (u64)__shfl_xor_sync(0xffffffffu, (unsigned long long)hi, s));
    }
    if ((tid & 31) == 0) {
      S.fr_lo[tid >> 5] = lo;
      S.fr_hi[tid >> 5] = hi;
    }
    Bk::sync();
    const u32 G = hc.gsz;
    if (tid == 0) {
      u64 a = ~0ull, b = 0;
      for (int w = 0; w < NW; ++w) {
        a = min(a, S.fr_lo[w]);
        b = max(b, S.fr_hi[w]);
      }
      const u64 range = b - a;
      u32 nb = G;
      if (range < (u64)nb - 1) nb = (u32)range + 1;
      bj->stg_n = n + m;
      bj->pmin = a;
      bj->pmax = b;
      bj->nbkt = nb;
      bj->bwidth = range / nb + 1;
      bj->bovf = 0;
      bj->write_idx = 0;
      bj->ok = ok;
      bj->op = op;
      S.fr_nb = nb;
    }
    Bk::sync();
    for (u32 i = tid; i < S.fr_nb; i += B) bj->bcnt[i] = 0;
    __threadfence();
    Bk::sync();
    grid_run<B>(hc.gj, G, 7, Run{}, Run{}, 0, Sink{}, 0, *hc.gs, hc.gs->scr);
    return *(volatile u32*)&bj->bovf == 0;
  }

  // Rebuild level 0 from the sorted run (K, P)[0, n), n <= C0: entry j goes
  // to slot j (round-robin over the banks), rows reloaded from the offsets.
  NOINL void rebuild(const u32* K, const u64* P, u32 n) {
    Bk::sync();
    occm = 0;
    for (u32 j = tid; j < n; j += B) {
      const u32 k = K[j];
      const u64 rb = off ? __ldg(off + k) : 0, re = off ? __ldg(off + k + 1) : 0;
      L.lk[j] = k;
      L.lp[j] = P[j];
      L.lrb[j] = rb;
      L.ldeg[j] = (u32)(re - rb);
      if constexpr (MW) {
        L.lmo[j] = __ldg(mwo + k);
        L.lmi[j] = __ldg(mwi + k);
      }
      idx[k].state = PBH_ST_LIVE | (j << 2);
      occm |= 1u << (j / B);
    }
    lhas = tid < n;
    if (lhas) {
      lmin_p = P[tid];
      lmin_k = K[tid];
      lmin_s = tid;
    }
    n_l0 = n;
    Bk::sync();
  }

  // A bank lacks room for one pass: sort level 0, keep the smallest C0/2
  // (splitter lowered to the last kept one), push the rest down.
  NOINL void evict() {
    u32* SK = &S.bk[0][0];
    u64* SP = &S.bp[0][0];
    Bk::sync();
    u32 n = 0;
    for (u32 i = 0; i < (u32)KI; ++i) {
      const bool f = (occm >> i) & 1u;
      u32 tot;
      const u32 pos = n + Bk::scan_excl(f ? 1u : 0u, tot, hc.scr());
      if (f) {
        const u32 s = i * B + tid;
        SK[pos] = L.lk[s];
        SP[pos] = L.lp[s];
      }
      n += tot;
    }
    Bk::sync();
    {
      auto& SS = bank_smem<NW, KI, VT, MW>();  // LDS-addressed sort (see flush_q)
      cta_sort<NW>(&SS.bk[0][0], &SS.bp[0][0], n, SS.sk, SS.sp);
    }
    const u32 keep = n < (u32)C0 / 2 ? n : (u32)C0 / 2;
    if (n > keep) {
      if (tid == 0) {
        L.spl_inf = 0;
        L.spl_p = SP[keep - 1];
        L.spl_k = SK[keep - 1];
      }
      for (u32 j = keep + tid; j < n; j += B) idx[SK[j]].state = PBH_ST_LIVE | (PBH_LOC_DEEP << 2);
    }
    rebuild(SK, SP, keep);
    push_run(SK + keep, SP + keep, n - keep);
  }

  // Level 0 is empty: refill it from the deeper levels (cold fill0).
  NOINL void refill() {
    flush_q();
    if (hc.failed()) return;
    to_cold();
    hc.fill0();
    if (hc.failed()) return;
    const Run b = hc.bucket(0);
    if (tid == 0) {
      const pbh_level_state& t = hc.s.st[0];
      L.spl_inf = t.spl_inf;
      L.spl_p = t.spl_p;
      L.spl_k = t.spl_k;
    }
    rebuild(b.k, b.p, b.n);
    if (tid == 0) {
      hc.s.st[0].b_head = 0;
      hc.s.st[0].b_size = 0;
    }
    Bk::sync();
    after_cold();
  }

};

// par_dijkstra with one CTA (NW warps) per source and a banked level 0.
// The hot loop keeps all state in locals (registers); the BankHeap object is
// only the hand-off to the cold-path methods.
template <int NW, int KI, int VT, int PASS = kBankPass>
__global__ void __launch_bounds__(32 * NW, 1)
    k_sssp_bank(pbh_heap_dev* heaps, const u64* __restrict__ off, const u32* __restrict__ tgt,
                const u32* __restrict__ wt, u32 V, const u32* sources, u64* dist, u32* settled,
                SsspState* sst, BankL0<32 * NW, KI>* save, u32 dag_mode, u32 max_deg, u32 d,
                unsigned long long* prof) {
  using BH = BankHeap<NW, KI, VT>;
  using HC = typename BH::HC;
  using Bk = Blk<BH::B>;
  constexpr u32 B = BH::B;
  constexpr u32 C0 = BH::C0;
  // edges per thread per pass: PASS = 256 for dense rows; the low-degree
  // variant (grids) uses one warp and PASS = 32 (one edge per lane)
  constexpr u32 PE = PASS / B;
  static_assert(PE >= 1 && PE * B == PASS && KI >= (int)PE, "pass shape");
  BankSmem<NW, KI, VT>& S = bank_smem<NW, KI, VT>();
  SsspState* my = sst + blockIdx.x;
  if (my->status != 0 && my->status != 7) return;
  pbh_heap_dev* g = heaps + blockIdx.x;
  typename HC::Sm& sm = S.hs;
  HC hc{sm};
  hc.load(g, S.bk[0], S.bp[0], S.bk[1], S.bp[1], true);
  hc.bk = g->g_bk;
  hc.bp = g->g_bp;
  hc.pk = g->g_pk;
  hc.pp = g->g_pp;
  hc.rm = g->g_rm;
  hc.bo = nullptr;
  const u32 tid = threadIdx.x;
  BankL0<B, KI>& L = S.l0;
  BH H(hc, S, g->idx, off);
  pbh_idx_entry* const idx = g->idx;
  u64* my_dist = dist + (u64)blockIdx.x * V;
  u32* my_settled = settled + (u64)blockIdx.x * V;
  u64 n_settled = my->n_settled, rounds = my->rounds, ops = my->ops;
  H.live = hc.s.live;
  H.pushes = sm.ops;  // persisted push counter (this engine reuses the ops slot)
  H.after_cold();
  for (u32 i = tid; i < 2 * B; i += B) (&S.dirty[0][0])[i] = 0;

  if (!my->started) {
    if (tid == 0) {
      L.qn = 0;
      L.spl_inf = 1;
      L.spl_p = 0;
      L.spl_k = 0;
      const u32 s = sources[blockIdx.x];
      pbh_idx_entry e;
      e.prio = 0;
      e.state = PBH_ST_LIVE;
      e.parent = s;
      idx[s] = e;
      S.bk[0][0] = s;
      S.bp[0][0] = 0;
    }
    H.rebuild(S.bk[0], S.bp[0], 1);  // eng.update({s, 0}) (sssp.cpp:36)
    H.live = 1;
    ops = 1;
  } else {
    // resume after NEED_GROW: reload the level-0 image
    const u32* src = reinterpret_cast<const u32*>(save + blockIdx.x);
    u32* dst = reinterpret_cast<u32*>(&L);
    for (u32 i = tid; i < sizeof(BankL0<B, KI>) / 4; i += B) dst[i] = src[i];
    Bk::sync();
    H.occm = L.occ[tid];
    H.rescan();
  }
  H.qn = L.qn;
  Bk::sync();

  // ---- hot state in registers
  u32 occm = H.occm;
  bool lhas = H.lhas;
  u64 lmin_p = H.lmin_p;
  u32 lmin_k = H.lmin_k, lmin_s = H.lmin_s;
  i64 live = H.live;
  u32 qn = H.qn;
  u64 deep_n = H.deep_n;
#define BANK_TO_H()     \
  H.occm = occm;        \
  H.lhas = lhas;        \
  H.lmin_p = lmin_p;    \
  H.lmin_k = lmin_k;    \
  H.lmin_s = lmin_s;    \
  H.live = live;        \
  H.qn = qn;            \
  H.deep_n = deep_n;
#define BANK_FROM_H()   \
  occm = H.occm;        \
  lhas = H.lhas;        \
  lmin_p = H.lmin_p;    \
  lmin_k = H.lmin_k;    \
  lmin_s = H.lmin_s;    \
  live = H.live;        \
  qn = H.qn;            \
  deep_n = H.deep_n;

  bool need_grow = false;
  const u32 Lnl = sm.n_levels;
  const u64 cap_last = Lnl == 1 ? (u64)sm.cap0 : sm.lv[Lnl - 1].cap_b;
  const u64 grow_at = cap_last - ((u64)2 * C0 + max_deg + kBankQ);  // NEED_GROW threshold
  const bool grow_ok = cap_last > (u64)2 * C0 + max_deg + kBankQ;
  u32 par = 0;                // exchange parity
  bool rescan_due = false;    // this thread's bank minimum is stale
  // replicated: some bank lacks room for a pass (also after a resume)
  bool evict_due = Bk::any(__popc(occm) > (int)(KI - PE), hc.scr());
  bool nx = false;            // the next extraction is known (cur)
  struct {
    u64 p, rb;
    u32 k, slot, deg;
  } cur{};
  // Take the exchange winner as the next extraction: its row from its slot
  // (written before the exchange barrier). free_cur(): the owner frees the
  // slot and rescans its bank — at the round start, or for dense rows early,
  // under the next row's copy (`freed`; a NEED_GROW exit before the vertex is
  // settled re-occupies the slot).
  auto take = [&](const LeanRes& r) {
    cur.p = r.p;
    cur.k = r.k;
    cur.slot = r.slot;
    cur.rb = L.lrb[r.slot];
    cur.deg = L.ldeg[r.slot];
  };
  bool freed = false;  // the taken extraction's slot is already freed
  auto free_cur = [&]() {
    if (!freed && cur.slot % B == tid) {
      occm &= ~(1u << (cur.slot / B));
      rescan_due = true;
    }
    freed = false;
  };
  bool fail_bad = false, fail_ovf = false;
  // round-phase breakdown per warp (build with -DPBH_PROF_BUILD, run with
  // PBH_PHASES=1); compiled out otherwise (it costs ~7 % of a round)
  u64 pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#ifdef PBH_PROF_BUILD
  long long pt = clock64();
#define SPROF(i)                          \
  if (prof) {                             \
    const long long t1_ = clock64();      \
    pc[i] += (u64)(t1_ - pt);             \
    pt = t1_;                             \
  }
#else
#define SPROF(i)
  prof = nullptr;
#endif
#if defined(PBH_XPROF) && defined(PBH_PROF_BUILD)
  u64 xsnap[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  // One pass over the edges (uu, ww)[t], t < PE, of the extracted vertex v
  // (priority p): gather the index entries, run the deferred rescans, apply
  // the improving candidates in place / into a new slot / into the push
  // buffer, and exchange the offers. Shared by the steady-state loop and the
  // general round below.
  bool pf_has = false;  // a first-sighted vertex's row to pull into L2
  u64 pf_b = 0, pf_e = 0;
  const bool dag = dag_mode != 0;
  auto relax_pass = [&](const u32 (&uu)[PE], const u32 (&ww)[PE], u32 rem, u32 te, u64 p,
                        u32 v) -> LeanRes {
    ulonglong2 ee[PE];
    u64 ob[PE], oe[PE];
#pragma unroll
    for (u32 t = 0; t < PE; ++t) {
      ee[t] = make_ulonglong2(0ull, PBH_ST_DEAD);  // no edge: never improves (c < 0)
      ob[t] = oe[t] = 0;
      if (te + B * t < rem) {
        ee[t] = __ldca(reinterpret_cast<const ulonglong2*>(idx + uu[t]));  // L1: sole writer is this CTA
        ob[t] = __ldg(off + uu[t]);
        oe[t] = __ldg(off + uu[t] + 1);
      }
    }
    asm volatile("" ::: "memory");  // issue the gathers before the rescans' shared loads
#ifdef PBH_XPROF
    if (prof) {  // split: gather latency (idx + off) | rescans
      u32 sink = 0;
#pragma unroll
      for (u32 t = 0; t < PE; ++t) sink += (u32)ee[t].y + (u32)ob[t] + (u32)oe[t];
      asm volatile("" ::"r"(sink));
    }
    SPROF(3);
#endif
    // deferred rescans (extraction owner, decreased banks) under the gathers
    if (rescan_due) bank_rescan<B, KI>(L, tid, occm, lhas, lmin_p, lmin_k, lmin_s);
    rescan_due = false;
#ifdef PBH_PROF_BUILD
    if (prof) {
      u32 sink = 0;
#pragma unroll
      for (u32 t = 0; t < PE; ++t) sink += (u32)ee[t].y;
      asm volatile("" ::"r"(sink));
    }
#endif
#ifdef PBH_XPROF
    SPROF(7);
#else
    SPROF(3);
#endif
    // ---- candidates, applied by the relaxing thread
    u32 fresh = 0, nimp = 0, nq = 0;
    bool ovf = false, bad = false;
    pf_has = false;
    // this thread's offer: min(bank minimum, best admitted candidate)
    u64 op = lhas ? lmin_p : ~0ull;
    u32 ok = lhas ? lmin_k : 0xffffffffu, os = lmin_s;
#pragma unroll
    for (u32 t = 0; t < PE; ++t) {
      // (an absent edge has w = 0 and entry (0, DEAD): c = p, no overflow, no improvement)
      const u32 st = (u32)ee[t].y;
      const u64 c = p + ww[t];
      const bool open = dag | (PBH_ST(st) != PBH_ST_DEAD);
      ovf |= open & (c < p);
      if (!(open & (c < ee[t].x))) continue;
      const u32 u = uu[t];
      ++nimp;
      fresh += PBH_ST(st) != PBH_ST_LIVE;
      const u32 loc = st >> 2;
      u32 nst, sl = 0;
      bool admitted = true;
      if (PBH_ST(st) == PBH_ST_LIVE && loc < C0) {
        // decrease in place; the owner rescans next pass
        bad |= !(L.lk[loc] == u && L.lp[loc] == ee[t].x);
        L.lp[loc] = c;
        S.dirty[par][loc % B] = 1;
        nst = st;
        sl = loc;
      } else if (L.spl_inf || c < L.spl_p || (c == L.spl_p && u <= L.spl_k)) {
        const u32 i = __ffs(~occm) - 1;
        sl = i * B + tid;
        occm |= 1u << i;
        L.lk[sl] = u;
        L.lp[sl] = c;
        L.lrb[sl] = ob[t];
        L.ldeg[sl] = (u32)(oe[t] - ob[t]);
        if (!lhas || less_pk(c, u, lmin_p, lmin_k)) {
          lhas = true;
          lmin_p = c;
          lmin_k = u;
          lmin_s = sl;
        }
        nst = PBH_ST_LIVE | (sl << 2);
        if (PBH_ST(st) != PBH_ST_LIVE) {
          // first sighting of a vertex that may be extracted soon: its row is
          // pulled into L2 after the exchange (warp-cooperatively; a second
          // fresh row in the same pass falls back to the bulk prefetch)
          if (pf_has) {
            l2_prefetch_range(tgt, pf_b, pf_e);
            l2_prefetch_range(wt, pf_b, pf_e);
          }
          pf_has = true;
          pf_b = ob[t];
          pf_e = oe[t];
        }
      } else {
        const u32 qp_ = atomicAdd(&L.qn, 1u);
        L.qk[qp_] = u;
        L.qp[qp_] = c;
        ++nq;
        admitted = false;
        nst = PBH_ST_LIVE | (PBH_LOC_DEEP << 2);
      }
      if (admitted && less_pk(c, u, op, ok)) {
        op = c;
        ok = u;
        os = sl;
      }
      pbh_idx_entry e;
      e.prio = c;
      e.state = nst;
      e.parent = v;
      __stwb(reinterpret_cast<ulonglong2*>(idx) + u, *reinterpret_cast<const ulonglong2*>(&e));
    }
    SPROF(4);
#if defined(PBH_XPROF) && defined(PBH_PROF_BUILD)
    if ((tid & 31) == 0)
      for (int i = 0; i < 8; ++i) {
        S.xph[par][tid >> 5][i] = (long long)(pc[i] - xsnap[i]);
        xsnap[i] = pc[i];
      }
#endif
    const u32 ev = (u32)__popc(occm) > (u32)KI - PE ? 1u : 0u;
    const LeanRes r = lean_exchange<NW, KI, VT>(par, op, ok, os,
                                                fresh | (nimp << 9) | ((ovf ? 1u : 0u) << 18),
                                                nq | (ev << 9) | ((bad ? 1u : 0u) << 18));
    if (S.dirty[par][tid]) {
      S.dirty[par][tid] = 0;
      rescan_due = true;
    }
    par ^= 1;
    live += r.fresh;
    qn += r.nq;
    evict_due = (r.flags & 1u) != 0;
    return r;
  };
  // The next extraction is known: copy its row's first pass into S.pf (the
  // edge j -> thread (j - rot') mod B mapping of the next round), then issue
  // the L2 prefetches of this pass's first sightings under that copy.
  auto next_row = [&](u32 rot) {
    const u32 te2 = (tid + rot + 1) & (B - 1);
#pragma unroll
    for (u32 t = 0; t < PE; ++t) {
      const u32 j = te2 + B * t;
      const bool in = j < cur.deg;
      cp_async4(&S.pf_t[t * B + tid], in ? tgt + cur.rb + j : tgt, in);
      cp_async4(&S.pf_w[t * B + tid], in ? wt + cur.rb + j : wt, in);
    }
    cp_async_commit();
  };
  auto fresh_rows_l2 = [&]() {
    for (u32 fm = __ballot_sync(0xffffffffu, pf_has); fm; fm &= fm - 1) {
      const u32 src = __ffs(fm) - 1;
      const u64 b = __shfl_sync(0xffffffffu, pf_b, src), e = __shfl_sync(0xffffffffu, pf_e, src);
      l2_prefetch_rows(tgt, wt, b, e, tid & 31);
    }
    pf_has = false;
  };
  auto settle = [&](u64 p, u32 v) {
    if (tid == 0) {
      idx[v].state = PBH_ST_DEAD;
      my_dist[v] = p;
      my_settled[n_settled] = v;
    }
    ++n_settled;
    ++rounds;
    ++ops;
    --live;
  };

  u32 fail_v = 0;
  while (live > 0) {
    // ---- steady state (most rounds): the next extraction is known, its row
    // fits one pass (already in S.pf) and no cold work is due
    // (qn + deep_n <= grow_at and qn <= kBankQ - PASS as one bound; deep_n
    // only changes on the cold path)
    const bool steady_ok = grow_ok && deep_n <= grow_at;
    const u32 qn_cap = (u32)min((u64)(kBankQ - PASS), steady_ok ? grow_at - deep_n : (u64)0);
    while (steady_ok && nx && cur.deg <= PASS && !evict_due && qn <= qn_cap) {
      const u64 p = cur.p;
      const u32 v = cur.k;
      free_cur();
      const u32 rot = (u32)n_settled & (B - 1);
      const u32 te = (tid + rot) & (B - 1);
      settle(p, v);
      SPROF(0);
      u32 uu[PE], ww[PE];
      cp_async_wait_all();
#pragma unroll
      for (u32 t = 0; t < PE; ++t) {
        uu[t] = S.pf_t[t * B + tid];
        ww[t] = S.pf_w[t * B + tid];
      }
      SPROF(2);
      const LeanRes r = relax_pass(uu, ww, cur.deg, te, p, v);
      if (r.flags & 6u) {
        fail_bad = (r.flags & 2u) != 0;
        fail_ovf = (r.flags & 4u) != 0;
        fail_v = v;
        break;
      }
      SPROF(5);
      nx = r.has;
      if (r.has) {
        take(r);
        next_row(rot);
      }
      // the extraction owner's and the decreased banks' rescans: under the
      // next row's copy when the row is dense (its index gathers then hit L1),
      // else under the gathers (sparse rows' gathers miss L1)
      if (r.has && cur.deg >= 64) {
        free_cur();
        freed = true;
        if (rescan_due) bank_rescan<B, KI>(L, tid, occm, lhas, lmin_p, lmin_k, lmin_s);
        rescan_due = false;
      }
      fresh_rows_l2();
      if (r.nimp) ops += r.nimp <= d ? 1u : ceil_div_cold(r.nimp, d);
      SPROF(6);
    }
    if (fail_bad || fail_ovf || live <= 0) break;
    // ---- general round
    if (!grow_ok || (u64)qn + deep_n > grow_at) {
      need_grow = true;
      // the taken extraction is not settled: its slot stays occupied (the
      // relaunch rescans and extracts it again)
      if (nx && freed && cur.slot % B == tid) occm |= 1u << (cur.slot / B);
      break;
    }
    const bool hit = nx;
    if (!nx) {
      // ---- extract_min: CTA argmin of the bank minima
      if (rescan_due) bank_rescan<B, KI>(L, tid, occm, lhas, lmin_p, lmin_k, lmin_s);
      rescan_due = false;
      const LeanRes x = lean_exchange<NW, KI, VT>(par, lhas ? lmin_p : ~0ull,
                                                  lhas ? lmin_k : 0xffffffffu, lmin_s, 0, 0);
      par ^= 1;
      if (x.has) take(x);
      if (!x.has) {
        BANK_TO_H();
        H.refill();
        BANK_FROM_H();
        if (hc.failed()) break;
        if (H.n_l0 == 0) {
          hc.fail(PBH_ERR_INVARIANT, 0xE5);
          break;
        }
        evict_due = false;
        continue;
      }
    }
    nx = false;
    SPROF(0);
    const u64 p = cur.p;
    const u32 v = cur.k;
    free_cur();
    const u32 rot = (u32)n_settled & (B - 1);  // edge j of a pass -> thread (j - rot) mod B
    settle(p, v);
    // ---- relax the row in passes of 256 edges (sssp.cpp:49-57)
    u32 n_imp = 0;
    const u64 rb = cur.rb;
    const u32 deg = cur.deg;
    const u32 te = (tid + rot) & (B - 1);  // this thread's edge offset within a group of B
    bool cold_fail = false;
    for (u32 done = 0; done < deg; done += PASS) {
      const bool last = done + PASS >= deg;
      const u32 rem = deg - done;
      const u64 base = rb + done;
      if (evict_due || qn > (u32)(kBankQ - PASS)) {
        BANK_TO_H();
        if (evict_due) H.evict();
        if (!hc.failed() && H.qn > (u32)(kBankQ - PASS)) H.flush_q();
        BANK_FROM_H();
        if (evict_due) rescan_due = false;
        evict_due = false;
        if (hc.failed()) {
          cold_fail = true;
          break;
        }
      }
      u32 uu[PE], ww[PE];
      SPROF(1);
      if (hit && done == 0) {
        cp_async_wait_all();
#pragma unroll
        for (u32 t = 0; t < PE; ++t) {
          uu[t] = S.pf_t[t * B + tid];
          ww[t] = S.pf_w[t * B + tid];
        }
      } else {
#pragma unroll
        for (u32 t = 0; t < PE; ++t) {
          const bool in = te + B * t < rem;
          uu[t] = in ? __ldg(tgt + base + te + B * t) : 0;
          ww[t] = in ? __ldg(wt + base + te + B * t) : 0;
        }
      }
#ifdef PBH_PROF_BUILD
      if (prof) {  // make the row load visible in its own bucket
        u32 sink = 0;
#pragma unroll
        for (u32 t = 0; t < PE; ++t) sink += uu[t];
        asm volatile("" ::"r"(sink));
      }
#endif
      SPROF(2);
      const LeanRes r = relax_pass(uu, ww, rem, te, p, v);
      n_imp += r.nimp;
      if (r.flags & 6u) {
        fail_bad = (r.flags & 2u) != 0;
        fail_ovf = (r.flags & 4u) != 0;
        fail_v = v;
        break;
      }
      SPROF(5);
      if (last && r.has) {
        // the next extraction: load its row's first pass now
        nx = true;
        take(r);
        next_row(rot);
      }
      fresh_rows_l2();
    }
    SPROF(6);
    if (cold_fail || fail_bad || fail_ovf) break;
    // bulk_update batches of <= d (sssp.cpp:59-64)
    if (n_imp) ops += n_imp <= d ? 1u : ceil_div_cold(n_imp, d);
  }
  cp_async_wait_all();
#undef SPROF
  if (prof && (threadIdx.x & 31) == 0 && blockIdx.x == 0)
    for (int i = 0; i < 8; ++i) atomicAdd(prof + (threadIdx.x >> 5) * 8 + i, (unsigned long long)pc[i]);
  BANK_TO_H();
#undef BANK_TO_H
#undef BANK_FROM_H
  if (fail_bad && !hc.failed()) hc.fail(PBH_ERR_INVARIANT, 0xD1);
  if (fail_ovf && !hc.failed()) hc.fail(PBH_ERR_OVERFLOW, fail_v);
  // persist the level-0 image (a NEED_GROW relaunch resumes from it)
  Bk::sync();
  L.occ[tid] = H.occm;
  if (tid == 0) L.qn = H.qn;
  Bk::sync();
  {
    const u32* src = reinterpret_cast<const u32*>(&L);
    u32* dst = reinterpret_cast<u32*>(save + blockIdx.x);
    for (u32 i = tid; i < sizeof(BankL0<B, KI>) / 4; i += B) dst[i] = src[i];
  }
  H.to_cold();
  if (tid == 0) sm.ops = H.pushes;
  Bk::sync();
  hc.store();
  if (tid == 0) {
    my->n_settled = n_settled;
    my->rounds = rounds;
    my->started = 1;
    my->ops = ops;
    if (need_grow && !hc.failed()) {
      my->status = 7;
    } else {
      my->status = sm.status;
      my->detail = sm.detail;
      my->aux = sm.aux;
    }
  }
}


// ---------------------------------------------------------------------------
// Op-trace interpreter on the banked level 0: Engine::run_trace
// (engine.cpp:207-226) with update / bulk_update / extract_min / delete
// (bucket_heap.cpp:79-146). CTA 0 replays the ops; CTAs 1..G-1 are the grid
// helpers of the deep merges (pbh_grid.cuh). A bulk batch is validated in one
// pass (no mutation before every precondition holds, bucket_heap.cpp:127-136)
// and applied in passes of B elements, one per thread, with the SSSP engine's
// three outcomes: decrease in place, new level-0 slot, push buffer.
// ---------------------------------------------------------------------------
template <int NW, int KI, int VT>
struct TraceBankSmem {
  BankSmem<NW, KI, VT> b;  // first: bank_smem() aliases it
  GridSmem<32 * NW> g;
};

// Level-0 image transfer of the op-trace engine (shared memory <-> HBM):
// everything except the SSSP row fields, and only the filled prefix of the
// push buffer. `to_smem`: the image is the source (its qn is read first).
template <int B, int KI>
DEV void trace_image_copy(BankL0<B, KI>& dst, const BankL0<B, KI>& src, bool to_smem) {
  constexpr u32 C0 = B * KI;
  const u32 tid = threadIdx.x;
  for (u32 i = tid; i < C0; i += B) {
    dst.lp[i] = src.lp[i];
    dst.lk[i] = src.lk[i];
  }
  dst.occ[tid] = src.occ[tid];
  if (tid == 0) {
    dst.spl_p = src.spl_p;
    dst.spl_k = src.spl_k;
    dst.spl_inf = src.spl_inf;
    dst.qn = src.qn;
    dst.pad = src.pad;
    dst.pushes = src.pushes;
  }
  __syncthreads();
  const u32 qn = to_smem ? dst.qn : src.qn;
  for (u32 i = tid; i < qn; i += B) {
    dst.qk[i] = src.qk[i];
    dst.qp[i] = src.qp[i];
  }
  __syncthreads();
}

template <int NW, int KI, int VT>
__global__ void __launch_bounds__(32 * NW, 1)
    k_trace_bank(pbh_heap_dev* g, pbh_trace_dev tr, u64 op_begin, u64 op_end, u32* out_v,
                 u64* out_p, pbh_kstatus* ks, BankL0<32 * NW, KI>* save, u32 allow_internal,
                 GridJob* gj, u32 grid_min, unsigned long long* prof, BatchJob* bj,
                 pbh_op_channel* pm) {
  using BH = BankHeap<NW, KI, VT>;
  using HC = typename BH::HC;
  using Bk = Blk<BH::B>;
  constexpr u32 B = BH::B;
  constexpr u32 C0 = BH::C0;
  extern __shared__ __align__(16) unsigned char dyn[];
  TraceBankSmem<NW, KI, VT>& T = *reinterpret_cast<TraceBankSmem<NW, KI, VT>*>(dyn);
  if (blockIdx.x > 0) {  // helper CTA: deep merges of the leader's heap
    grid_helper_loop<B>(gj, T.g, T.g.scr);
    return;
  }
  BankSmem<NW, KI, VT>& S = T.b;
  typename HC::Sm& sm = S.hs;
  HC hc{sm};
  hc.load(g, S.bk[0], S.bp[0], S.bk[1], S.bp[1], true);
  hc.bk = g->g_bk;
  hc.bp = g->g_bp;
  hc.pk = g->g_pk;
  hc.pp = g->g_pp;
  hc.rm = g->g_rm;
  hc.bo = nullptr;
  hc.gs = &T.g;  // streamed CTA-local merges
  grid_smem_init<B>(T.g);
  if (gridDim.x > 1) {
    hc.gj = gj;
    hc.gsz = gridDim.x;
    hc.gmin = grid_min;
    grid_leader_init<B>(T.g);
  }
  const u32 tid = threadIdx.x;
  BankL0<B, KI>& L = S.l0;
  BH H(hc, S, g->idx, nullptr);
  H.prof = prof;
  if (tid == 0) {
    T.g.job.ext = nullptr;
    T.g.job.idx = g->idx;
  }
  if (gridDim.x > 1 && bj) {
    H.bj = bj;
    if (tid == 0) T.g.job.ext = bj;
  }
  Bk::sync();
  pbh_idx_entry* const idx = g->idx;
  const u64 universe = g->universe;
  // batches beyond the large-batch buffers (2^26 entries) are rejected, not split
  const u32 dmax = min(sm.d, kMaxBatch);
  const bool debug = sm.debug != 0;
  // restore the level-0 image: the parts this engine uses (slot keys and
  // priorities, bank masks, splitter, counters, the filled push-buffer
  // prefix; the SSSP-only row fields stay behind), which keeps a single-op
  // launch short
  trace_image_copy<B, KI>(L, *save, true);
  for (u32 i = tid; i < 2 * B; i += B) (&S.dirty[0][0])[i] = 0;
  Bk::sync();
  H.occm = L.occ[tid];
  H.rescan();
  H.qn = L.qn;
  H.live = hc.s.live;
  H.pushes = L.pushes;
  H.after_cold();
  Bk::sync();
  u32 occm = H.occm;
  bool lhas = H.lhas;
  u64 lmin_p = H.lmin_p;
  u32 lmin_k = H.lmin_k, lmin_s = H.lmin_s;
  i64 live = H.live;
  u32 qn = H.qn;
  u64 deep_n = H.deep_n;
#define BANK_TO_H()     \
  H.occm = occm;        \
  H.lhas = lhas;        \
  H.lmin_p = lmin_p;    \
  H.lmin_k = lmin_k;    \
  H.lmin_s = lmin_s;    \
  H.live = live;        \
  H.qn = qn;            \
  H.deep_n = deep_n;
#define BANK_FROM_H()   \
  occm = H.occm;        \
  lhas = H.lhas;        \
  lmin_p = H.lmin_p;    \
  lmin_k = H.lmin_k;    \
  lmin_s = H.lmin_s;    \
  live = H.live;        \
  qn = H.qn;            \
  deep_n = H.deep_n;
  const u32 Lnl = sm.n_levels;
  const u64 cap_last = Lnl == 1 ? (u64)sm.cap0 : sm.lv[Lnl - 1].cap_b;
  u32 par = 0;
  bool rescan_due = false;
  // a bank may be full already (the image of the previous launch)
  bool evict_due = __syncthreads_or(__popc(occm) > KI - 1) != 0;
  u64 n_out = ks->n_out;
  u64 op = op_begin;
  // PBH_PROF: leader-side cycle breakdown (thread 0), categories below
  long long pt0 = clock64();
  u64 pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define TPROF(i)                          \
  if (prof) {                             \
    const long long t1_ = clock64();      \
    pc[i] += (u64)(t1_ - pt0);            \
    pt0 = t1_;                            \
  }
  // op headers run ahead: (kind, end) of op and op+1 are in registers when op
  // starts and op+2's load during op, so op+1's exact element range is known
  // and pulled into L2 (bulk prefetch) while op runs: an op's first loads no
  // longer wait behind a dependent header load and an HBM miss
  u64 hs_ = op < op_end ? tr.offsets[op] : 0;
  u8 ka = op < op_end ? tr.kinds[op] : 0;
  u64 ea = op < op_end ? tr.offsets[op + 1] : 0;
  u8 kb = op + 1 < op_end ? tr.kinds[op + 1] : 0;
  u64 eb = op + 1 < op_end ? tr.offsets[op + 2] : 0;
  // persistent mode (pm != null): requests are served one after another from
  // the mapped channel. Every channel word is a flagged word (request number
  // in the high 32 bits, payload in the low 32), so a word is valid exactly
  // when it carries the expected number: no fences on either side, one PCIe
  // round trip to read a single-element request, none to publish a result.
  u32 seq = pm ? (u32)(pm->rs[0] >> 32) : 0;  // last request served
  __shared__ u32 s_ctl, s_hdr, s_v;  // leader's wait verdict and the request header
  __shared__ u64 s_p;
  bool in_req = false;  // a request is being served (its result is still owed)
  // thread 0: wait / copy / run (ns), cumulative over the heap's resident kernels
  u64 tw = 0, tc = 0, tx = 0, t_seen = 0, t_cop = 0;
  if (pm && tid == 0) {
    tw = pm->tprof[0];
    tc = pm->tprof[1];
    tx = pm->tprof[2];
  }
  for (;; ++op) {
    if (op >= op_end) {
      if (!pm) break;
      if (in_req && tid == 0) {
        // the finished request's result record
        const u64 sq = (u64)seq << 32;
        const u32 ov = n_out ? out_v[0] : 0;
        const u64 opr = n_out ? out_p[0] : 0;
        u64 t2;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
        tc += t_cop - t_seen;
        tx += t2 - t_cop;
        asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(&pm->rs[0]),
                     "l"(sq | (u32)n_out), "l"(sq | ov) : "memory");
        asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(&pm->rs[2]),
                     "l"(sq | (u32)opr), "l"(sq | (u32)(opr >> 32)) : "memory");
        pm->tprof[0] = tw;
        pm->tprof[1] = tc;
        pm->tprof[2] = tx;
      }
      in_req = false;
      if (tid == 0) {
        u64 t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        const u64 idle = pm->idle_ns;
        const u32 want = seq + 1;
        u32 cmd = 0;
        for (;;) {
          u64 a0, a1, a2, a3, stp;
          asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a0), "=l"(a1) : "l"(&pm->rq[0]));
          asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a2), "=l"(a3) : "l"(&pm->rq[2]));
          stp = pm->stop;
          if (stp) break;
          if ((u32)(a0 >> 32) == want && (u32)(a1 >> 32) == want && (u32)(a2 >> 32) == want &&
              (u32)(a3 >> 32) == want) {
            cmd = 1;
            s_hdr = (u32)a0;
            s_v = (u32)a1;
            s_p = (u64)(u32)a2 | (a3 << 32);
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_seen));
            tw += t_seen - t0;
            break;
          }
          u64 t1;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
          if (t1 - t0 > idle) break;
        }
        s_ctl = cmd;
      }
      Bk::sync();
      if (s_ctl == 0) break;
      // the op into device staging (the engine reads staging written by
      // this CTA); a multi-element payload is read until every word carries
      // the request number
      ++seq;
      const u32 hdr = s_hdr;
      const u32 n = hdr >> 8;
      u32* sv = const_cast<u32*>(tr.vals);
      u64* sp = const_cast<u64*>(tr.prios);
      if (n == 1) {
        if (tid == 0) {
          sv[0] = s_v;
          sp[0] = s_p;
        }
      } else if (n > 1) {
        for (;;) {
          bool ok = true;
          for (u32 i = tid; i < n; i += B) {
            const u64 w0 = pm->rv[i], w1 = pm->rplo[i], w2 = pm->rphi[i];
            ok &= (u32)(w0 >> 32) == seq && (u32)(w1 >> 32) == seq && (u32)(w2 >> 32) == seq;
            sv[i] = (u32)w0;
            sp[i] = (u64)(u32)w1 | (w2 << 32);
          }
          if (__syncthreads_and(ok)) break;
        }
      }
      if (tid == 0) {
        const_cast<u8*>(tr.kinds)[0] = (u8)hdr;
        const_cast<u64*>(tr.offsets)[0] = 0;
        const_cast<u64*>(tr.offsets)[1] = n;
      }
      __threadfence_block();
      Bk::sync();
      if (tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_cop));
      in_req = true;
      n_out = 0;
      op = 0;
      op_end = 1;
      hs_ = 0;
      ka = (u8)hdr;
      ea = n;
      kb = 0;
      eb = 0;
    }
    const u8 kind = ka;
    const u64 ob = hs_, oe = ea;
    if (tid == 0 && op + 1 < op_end && eb > ea) {
      l2_prefetch_range(tr.vals, ea, eb);
      l2_prefetch_range(reinterpret_cast<const u32*>(tr.prios), 2 * ea, 2 * eb);
    }
    hs_ = ea;
    ka = kb;
    ea = eb;
    if (op + 2 < op_end) {
      kb = tr.kinds[op + 2];
      eb = tr.offsets[op + 3];
    }
    // a small next bulk op (<= 128 keys): its index entries into L2. The last
    // warp loads the keys (already L2-resident) and prefetches their lines,
    // overlapping this op's own gather latency (larger batches: the detour
    // costs the warp more than the next op's gathers save)
    if (tid >= B - 32 && op + 1 < op_end && (ka == 'U' || ka == 'B') && ea - hs_ <= 128) {
      const u32 nn = (u32)(ea - hs_);
      const u32 l = tid - (B - 32);
      u32 kq[4];
#pragma unroll
      for (u32 q = 0; q < 4; ++q) kq[q] = l + 32 * q < nn ? tr.vals[hs_ + l + 32 * q] : 0xffffffffu;
#pragma unroll
      for (u32 q = 0; q < 4; ++q)
        if (kq[q] < universe) asm volatile("prefetch.global.L2 [%0];" ::"l"(idx + kq[q]));
    }
    if (kind == 'U' || kind == 'B') {
      // ------------------------------------------------ bulk_update / update
      const u32* vals = tr.vals + ob;
      const u64* prios = tr.prios + ob;
      const u64 n64 = oe - ob;
      const bool check = kind == 'B';
      if (check && n64 == 0) {
        hc.fail(PBH_ERR_EMPTY_BATCH);
        break;
      }
      if (check && n64 > dmax) {
        hc.fail(PBH_ERR_BATCH_TOO_BIG, n64);
        break;
      }
      const u32 n = (u32)n64;
      if ((u64)2 * C0 + qn + deep_n + n + kBankQ > cap_last) {
        hc.fail(PBH_ERR_NEED_GROW, Lnl);
        break;
      }
      // a large batch is validated and classified by the whole grid: only
      // the elements that touch level 0 stay with this CTA (list `lst`)
      const bool big = bj != nullptr && gridDim.x > 1 && n >= kBigBatch;
      u32 m_apply = n, stg_n = 0, big_src = 0;
      const u32* lst = nullptr;
      if (big) {
        if (tid == 0) {
          bj->vals = vals;
          bj->prios = prios;
          bj->idx = idx;
          bj->universe = universe;
          bj->spl_p = L.spl_p;
          bj->spl_k = L.spl_k;
          bj->spl_inf = L.spl_inf;
          bj->n = n;
          bj->check = check ? 1u : 0u;
          bj->debug = debug ? 1u : 0u;
          bj->c0 = C0;
          bj->stg_n = bj->ll_n = bj->fresh = bj->errs = 0;
          bj->pmin = ~0ull;
          bj->pmax = 0;
          T.g.job.ext = bj;
        }
        __threadfence();
        Bk::sync();
        // one pass: every precondition checked and every element routed,
        // nothing mutated (the index is published by the sort job below)
        grid_run<B>(gj, gridDim.x, 6, Run{}, Run{}, 0, Sink{}, 0, T.g, T.g.scr);
        const u32 errs = *(volatile u32*)&bj->errs;
        if (errs) {
          hc.fail(errs & 1 ? PBH_ERR_UNSORTED : errs & 2 ? PBH_ERR_KEY_RANGE
                  : errs & 4 ? PBH_ERR_REINSERT : PBH_ERR_INCREASE);
          break;
        }
        m_apply = *(volatile u32*)&bj->ll_n;
        stg_n = *(volatile u32*)&bj->stg_n;
        live += *(volatile u32*)&bj->fresh;
        lst = bj->ll;
        TPROF(6);
        bool big_pushed = false;
        if (stg_n) {
          // the staged part straight into S_1 (job 9: bucket by S_1 chunks,
          // sort, merge, publish the index entries) when S_1 allows it
          BANK_TO_H();
          long long tj = clock64();
          if (H.grid_push_fits(stg_n) && H.grid_push_unsorted(stg_n, true, tj)) big_pushed = true;
          BANK_FROM_H();
          if (hc.failed()) break;
          TPROF(8 - 1);
        }
        if (stg_n && !big_pushed) {
          // the HBM-bound part of the batch, sorted by (p, k) on the grid:
          // a bucket sort (one job) when the buckets fit the CTA tiles,
          // else CTA-sorted chunks + merge passes; both publish the staged
          // elements' index entries before the leader applies its own part
          const u32 G = gridDim.x;
          u32 nb = G * ((stg_n + G * 1024u - 1) / (G * 1024u));
          const bool bucketed = nb <= kBucketMax;
          if (bucketed) {
            const u64 pmin = *(volatile u64*)&bj->pmin, pmax = *(volatile u64*)&bj->pmax;
            const u64 range = pmax - pmin;  // bucket q: priorities pmin + [q, q + 1) * width
            if (range < (u64)nb - 1) nb = (u32)range + 1;
            for (u32 i = tid; i < nb; i += B) bj->bcnt[i] = 0;
            if (tid == 0) {
              bj->nbkt = nb;
              bj->bwidth = range / nb + 1;
              bj->bovf = 0;
              bj->write_idx = 1;
              bj->ok = nullptr;
              bj->op = nullptr;
            }
            __threadfence();
            Bk::sync();
            grid_run<B>(gj, G, 7, Run{}, Run{}, 0, Sink{}, 0, T.g, T.g.scr);
            big_src = 1;
          }
          if (!bucketed || *(volatile u32*)&bj->bovf) {
            if (tid == 0) {
              bj->sort_n = stg_n;
              bj->src = bucketed ? 1u : 0u;
              bj->write_idx = bucketed ? 0u : 1u;
            }
            __threadfence();
            Bk::sync();
            grid_run<B>(gj, G, 4, Run{}, Run{}, 0, Sink{}, 0, T.g, T.g.scr);
            big_src = bucketed ? 1u : 0u;
            for (u32 w = kSortChunk; w < stg_n; w <<= 1) {
              if (tid == 0) {
                bj->width = w;
                bj->src = big_src;
              }
              __threadfence();
              Bk::sync();
              grid_run<B>(gj, G, 5, Run{}, Run{}, 0, Sink{}, 0, T.g, T.g.scr);
              big_src ^= 1;
            }
          }
          TPROF(8 - 1);
          // one push_down of the sorted staged run into S_1, before the
          // leader's own part: the push-buffer flushes of that part reuse
          // the grid sort buffers (the order of pushes into S_1 does not
          // matter: it is a set, and the staged elements lie beyond
          // splitter_0, which the leader's part can only lower)
          BANK_TO_H();
          H.push_run(bj->sk[big_src], bj->sp[big_src], stg_n);
          BANK_FROM_H();
          if (hc.failed()) break;
          TPROF(2);
        }
      }
      // pass 1: validate (no mutation)
      bool bad_sort = false, bad_key = false, bad_dead = false, bad_inc = false;
      // 4 elements per thread per step: their loads are all in flight at once
      // the first pass's element, index entry and priority are kept for
      // pass 2 (no mutation in between)
      u32 v_first = 0;
      u64 p_first = 0;
      ulonglong2 e_first = make_ulonglong2(0, 0);
      for (u32 j0 = tid; !big && j0 < n; j0 += 4 * B) {
        u32 kk[4], kp[4];
        ulonglong2 e[4];
        if (j0 == tid) p_first = prios[tid];
#pragma unroll
        for (u32 t = 0; t < 4; ++t) {
          const u32 j = j0 + t * B;
          kk[t] = j < n ? vals[j] : 0;
          kp[t] = j < n && j > 0 ? vals[j - 1] : 0;
        }
#pragma unroll
        for (u32 t = 0; t < 4; ++t) {
          const u32 j = j0 + t * B;
          e[t] = j < n && kk[t] < universe
                     ? __ldcg(reinterpret_cast<const ulonglong2*>(idx + kk[t]))
                     : make_ulonglong2(0, 0);
        }
#pragma unroll
        for (u32 t = 0; t < 4; ++t) {
          const u32 j = j0 + t * B;
          if (j >= n) continue;
          if (check && j > 0 && kp[t] >= kk[t]) bad_sort = true;
          if (kk[t] >= universe) {
            bad_key = true;
            continue;
          }
          if (PBH_ST((u32)e[t].y) == PBH_ST_DEAD) bad_dead = true;
          if (debug && PBH_ST((u32)e[t].y) == PBH_ST_LIVE && prios[j] > e[t].x) bad_inc = true;
        }
        if (j0 == tid) {
          v_first = kk[0];
          e_first = e[0];
        }
      }
      if (!big) TPROF(6);
      const u32 bad = (u32)__syncthreads_or(bad_sort) | ((u32)__syncthreads_or(bad_key) << 1) |
                      ((u32)__syncthreads_or(bad_dead) << 2) | ((u32)__syncthreads_or(bad_inc) << 3);
      if (bad) {
        hc.fail(bad & 1 ? PBH_ERR_UNSORTED : bad & 2 ? PBH_ERR_KEY_RANGE
                : bad & 4 ? PBH_ERR_REINSERT : PBH_ERR_INCREASE);
        break;
      }
      // pass 2: apply, one element per thread per pass
      TPROF(0);
      bool cold_fail = false;
      u32 nx_u = 0;
      u64 nx_c = 0;
      ulonglong2 nx_e = make_ulonglong2(0, 0);
      if (tid < m_apply) {
        if (big) {
          const u32 jj = lst[tid];
          nx_u = vals[jj];
          nx_c = prios[jj];
          nx_e = __ldcg(reinterpret_cast<const ulonglong2*>(idx + nx_u));
        } else {
          nx_u = v_first;
          nx_c = p_first;
          nx_e = e_first;
        }
      }
      for (u32 base = 0; base < m_apply; base += B) {
        const bool cold_now = evict_due || qn > (u32)(kBankQ - B);
        if (cold_now) {
          TPROF(1);
          BANK_TO_H();
          if (evict_due) H.evict();
          if (!hc.failed() && H.qn > (u32)(kBankQ - B)) H.flush_q();
          BANK_FROM_H();
          if (evict_due) rescan_due = false;
          evict_due = false;
          TPROF(2);
          if (hc.failed()) {
            cold_fail = true;
            break;
          }
        }
        const u32 j = base + tid;
        bool fresh = false, pushed = false;
        // this pass's element came with the previous pass (prefetch below);
        // a cold op just now (evict) may have moved its slot: re-read then
        const u32 u = nx_u;
        const u64 c = nx_c;
        const ulonglong2 e = cold_now && j < m_apply
                                 ? __ldcg(reinterpret_cast<const ulonglong2*>(idx + u))
                                 : nx_e;
        {
          const u32 jn = j + B;  // next pass (distinct keys: no conflict)
          if (jn < m_apply) {
            const u32 jj = lst ? lst[jn] : jn;
            nx_u = vals[jj];
            nx_c = prios[jj];
            nx_e = __ldcg(reinterpret_cast<const ulonglong2*>(idx + nx_u));
          }
        }
        if (j < m_apply) {
          const u32 st = (u32)e.y;
          fresh = PBH_ST(st) != PBH_ST_LIVE;
          if (fresh || c < e.x) {
            const u32 loc = st >> 2;
            u32 nst;
            if (!fresh && loc < C0) {
              L.lp[loc] = c;  // decrease in place; the owner rescans
              S.dirty[par][loc % B] = 1;
              nst = st;
            } else if (L.spl_inf || c < L.spl_p || (c == L.spl_p && u <= L.spl_k)) {
              const u32 i = __ffs(~occm) - 1;
              const u32 sl = i * B + tid;
              occm |= 1u << i;
              L.lk[sl] = u;
              L.lp[sl] = c;
              if (!lhas || less_pk(c, u, lmin_p, lmin_k)) {
                lhas = true;
                lmin_p = c;
                lmin_k = u;
                lmin_s = sl;
              }
              nst = PBH_ST_LIVE | (sl << 2);
            } else {
              const u32 qp_ = atomicAdd(&L.qn, 1u);
              L.qk[qp_] = u;
              L.qp[qp_] = c;
              pushed = true;
              nst = PBH_ST_LIVE | (PBH_LOC_DEEP << 2);
            }
            pbh_idx_entry ne;
            ne.prio = c;
            ne.state = nst;
            ne.parent = 0;
            reinterpret_cast<ulonglong2*>(idx)[u] = *reinterpret_cast<const ulonglong2*>(&ne);
          }
        }
        live += __syncthreads_count(fresh);
        qn += __syncthreads_count(pushed);
        evict_due = __syncthreads_or(__popc(occm) > KI - 1) != 0;
        if (S.dirty[par][tid]) {
          S.dirty[par][tid] = 0;
          rescan_due = true;
        }
        par ^= 1;
      }
      if (cold_fail) break;
      TPROF(1);

      if (tid == 0) sm.touches[0] += 2ull * n;
    } else if (kind == 'E' || (kind == kOpFind && allow_internal)) {
      // ------------------------------------------------ extract_min / find_min
      if (live <= 0) {
        hc.fail(PBH_ERR_EMPTY_HEAP);
        break;
      }
      BankOffer r{};
      bool cold_fail = false;
      for (int guard = 0; guard < 64; ++guard) {
        if (rescan_due) bank_rescan<B, KI>(L, tid, occm, lhas, lmin_p, lmin_k, lmin_s);
        rescan_due = false;
        r = bank_exchange<NW, KI, VT>(par, lhas, lmin_p, lmin_k, lmin_s, 0, 0, 0, 0);
        par ^= 1;
        if (r.has) break;
        TPROF(3);
        BANK_TO_H();
        H.refill();
        BANK_FROM_H();
        TPROF(4);
        rescan_due = false;
        evict_due = false;
        if (hc.failed()) {
          cold_fail = true;
          break;
        }
      }
      if (cold_fail) break;
      if (!r.has) {
        hc.fail(PBH_ERR_INVARIANT, 0xE0);
        break;
      }
      if (tid == 0) {
        out_v[n_out] = r.k;
        out_p[n_out] = r.p;
      }
      ++n_out;
      if (kind == 'E') {
        if (r.slot % B == tid) {
          occm &= ~(1u << (r.slot / B));
          rescan_due = true;
        }
        if (tid == 0) idx[r.k].state = PBH_ST_DEAD;
        --live;
      }
      TPROF(3);
    } else if (kind == 'D') {
      // ------------------------------------------------ delete_value
      const u32 k = tr.vals[ob];
      if (k < universe) {
        const ulonglong2 e = __ldcg(reinterpret_cast<const ulonglong2*>(idx + k));
        const u32 st = (u32)e.y;
        Bk::sync();  // every thread has read the entry before it changes
        if (PBH_ST(st) == PBH_ST_LIVE) {
          const u32 loc = st >> 2;
          if (loc < C0 && loc % B == tid) {
            occm &= ~(1u << (loc / B));
            rescan_due = true;
          }
          --live;
        }
        if (tid == 0) idx[k].state = PBH_ST_DEAD;  // deeper copies are now stale
        Bk::sync();
      } else {
        // beyond the index: an absent value (no-op), remembered so that the
        // index growth that later covers it marks it DEAD; a full list makes
        // the host grow the index now
        const u32 on = *(volatile u32*)&g->oor_n;
        if (on >= g->oor_cap) {
          hc.fail(PBH_ERR_KEY_RANGE, k);
          break;
        }
        if (tid == 0) {
          g->oor_del[on] = k;
          *(volatile u32*)&g->oor_n = on + 1;
        }
        Bk::sync();
      }
    } else if (kind == kOpDrain && allow_internal) {
      BANK_TO_H();
      H.flush_q();
      if (!hc.failed()) {
        H.to_cold();
        hc.drain();
        H.after_cold();
      }
      BANK_FROM_H();
      if (hc.failed()) break;
    } else {
      hc.fail(PBH_ERR_BAD_OP, kind);
      break;
    }
    if (kind != kOpFind && kind != kOpDrain && tid == 0) {
      sm.ops += 1;
      sm.resolves[0] += 1;
    }
  }
  TPROF(5);
#undef TPROF
  if (prof && tid == 0)
    for (int i = 0; i < 8; ++i) atomicAdd(prof + i, (unsigned long long)pc[i]);
  if (gridDim.x > 1) grid_run<B>(gj, gridDim.x, 1, Run{}, Run{}, 0, Sink{}, 0, T.g, T.g.scr);
  BANK_TO_H();
#undef BANK_TO_H
#undef BANK_FROM_H
  // persist the level-0 image
  Bk::sync();
  L.occ[tid] = H.occm;
  if (tid == 0) {
    L.qn = H.qn;
    L.pushes = H.pushes;
  }
  Bk::sync();
  trace_image_copy<B, KI>(*save, L, false);
  H.to_cold();
  hc.store();
  if (tid == 0 && (!pm || in_req)) {
    ks->status = sm.status;
    ks->detail = sm.detail;
    ks->aux = sm.aux;
    ks->ops_done = op - op_begin;
    ks->n_out = n_out;
    ks->failed_op = op;
    if (pm) {
      // a failed request: its result record says so; the host resolves it
      // (index growth, error) from the status block after this launch ends
      pm->rs[0] = ((u64)seq << 32) | 0xFFFFFFFFu;
    }
  }
}

}  // namespace pbh_dev
