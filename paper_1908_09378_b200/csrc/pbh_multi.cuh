// Threshold multi-extraction SSSP (opt-in, the
// Crauser et al. IN/OUT criteria of the paper's related work, PAPER.md:100,
// 123-131), on the banked level 0 of pbh_bank.cuh.
//
// A round settles EVERY level-0 vertex v whose tentative distance is already
// final by one of two criteria, with L = the minimum tentative distance and
// T = min over queued u of (tent(u) + minout(u)):
//   OUT: tent(v) <= T        (any path through a queued vertex costs >= T)
//   IN:  tent(v) - minin(v) <= L  (v's cheapest in-edge leaves a vertex at >= L)
// Entries below level 0 (push buffer, HBM levels) are > splitter_0, so they
// contribute at least splitter_0 + 1 to T (weights >= 1); L is level 0's
// minimum. The settled batch's rows are flattened into passes of 256 edges;
// a target relaxed from two batch vertices in one pass is resolved with a
// 64-bit atomicMin on its index priority followed by a CAS on its parent word
// (one winner applies the slot update). Distances are exact; the parent tree
// is valid; `rounds` counts batches and `settled` lists vertices in batch
// order (the reference's one-per-round settle order is the (dist, vid) sort
// of the reached vertices, sssp.cpp:39-47).
#pragma once

#include "pbh_bank.cuh"

namespace pbh_dev {

// Per-vertex minimum out-edge weight (row minimum) and minimum in-edge weight
// (atomicMin over targets); 0xFFFFFFFF = none.
__global__ void k_min_weights(const u64* __restrict__ off, const u32* __restrict__ tgt,
                              const u32* __restrict__ wt, u32 V, u32* mwo, u32* mwi) {
  const u32 lane = threadIdx.x & 31;
  const u64 gw = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const u64 nw = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 v = gw; v < V; v += nw) {
    u32 m = 0xffffffffu;
    for (u64 j = off[v] + lane; j < off[v + 1]; j += 32) {
      const u32 w = wt[j];
      m = min(m, w);
      atomicMin(mwi + tgt[j], w);
    }
    m = __reduce_min_sync(0xffffffffu, m);
    if (lane == 0) mwo[v] = m;
  }
}

template <int NW, int KI>
struct MultiBatch {
  static constexpr int C0 = 32 * NW * KI;
  u64 p[C0];
  u64 rb[C0];
  u32 k[C0];
  u32 deg[C0];
  u32 pre[C0 + 1];  // exclusive prefix of deg (edge offset of each batch row)
};

template <int NW, int KI, int VT>
struct MultiSmem {
  BankSmem<NW, KI, VT, true> b;  // first: bank_smem<..., true>() aliases it
  MultiBatch<NW, KI> m;
};

// bank minimum (p, k, slot) and min over the bank of p + minout (saturating)
template <int B, int KI>
DEV void multi_rescan(const BankL0<B, KI, true>& L, u32 tid, u32 occm, bool& lhas, u64& lmin_p,
                      u32& lmin_k, u32& lmin_s, u64& tmin) {
  lhas = false;
  tmin = ~0ull;
  u32 m = occm;
  while (m) {
    const u32 i = __ffs(m) - 1;
    m &= m - 1;
    const u32 s = i * B + tid;
    const u64 p = L.lp[s];
    const u32 k = L.lk[s];
    const u32 mo = L.lmo[s];
    const u64 t = mo == 0xffffffffu ? ~0ull : p + mo;
    tmin = min(tmin, (u64)(t < p ? ~0ull : t));
    if (!lhas || less_pk(p, k, lmin_p, lmin_k)) {
      lhas = true;
      lmin_p = p;
      lmin_k = k;
      lmin_s = s;
    }
  }
}

template <int NW, int KI, int VT>
__global__ void __launch_bounds__(32 * NW, 1)
    k_sssp_multi(pbh_heap_dev* heaps, const u64* __restrict__ off, const u32* __restrict__ tgt,
                 const u32* __restrict__ wt, const u32* __restrict__ mwo,
                 const u32* __restrict__ mwi, u32 V, const u32* sources, u64* dist, u32* settled,
                 SsspState* sst, BankL0<32 * NW, KI, true>* save, u32 max_deg, u32 d) {
  using BH = BankHeap<NW, KI, VT, true>;
  using HC = typename BH::HC;
  using Bk = Blk<BH::B>;
  constexpr u32 B = BH::B;
  constexpr u32 C0 = BH::C0;
  constexpr u32 PE = BH::PE;
  extern __shared__ __align__(16) unsigned char dyn[];
  MultiSmem<NW, KI, VT>& MS = *reinterpret_cast<MultiSmem<NW, KI, VT>*>(dyn);
  BankSmem<NW, KI, VT, true>& S = MS.b;
  MultiBatch<NW, KI>& M = MS.m;
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
  BankL0<B, KI, true>& L = S.l0;
  BH H(hc, S, g->idx, off);
  H.mwo = mwo;
  H.mwi = mwi;
  pbh_idx_entry* const idx = g->idx;
  u64* my_dist = dist + (u64)blockIdx.x * V;
  u32* my_settled = settled + (u64)blockIdx.x * V;
  u64 n_settled = my->n_settled, rounds = my->rounds, ops = my->ops;
  H.live = hc.s.live;
  H.pushes = sm.ops;
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
    H.rebuild(S.bk[0], S.bp[0], 1);
    H.live = 1;
    ops = 1;
  } else {
    const u32* src = reinterpret_cast<const u32*>(save + blockIdx.x);
    u32* dst = reinterpret_cast<u32*>(&L);
    for (u32 i = tid; i < sizeof(BankL0<B, KI, true>) / 4; i += B) dst[i] = src[i];
    Bk::sync();
    H.occm = L.occ[tid];
  }
  H.qn = L.qn;
  Bk::sync();
  u32 occm = H.occm;
  bool lhas = false;
  u64 lmin_p = 0, tmin = ~0ull;
  u32 lmin_k = 0, lmin_s = 0;
  multi_rescan<B, KI>(L, tid, occm, lhas, lmin_p, lmin_k, lmin_s, tmin);
  i64 live = H.live;
  u32 qn = H.qn;
  u64 deep_n = H.deep_n;
#define MULTI_TO_H() \
  H.occm = occm;     \
  H.live = live;     \
  H.qn = qn;         \
  H.deep_n = deep_n;
#define MULTI_FROM_H() \
  occm = H.occm;       \
  live = H.live;       \
  qn = H.qn;           \
  deep_n = H.deep_n;
  bool need_grow = false;
  const u32 Lnl = sm.n_levels;
  const u64 cap_last = Lnl == 1 ? (u64)sm.cap0 : sm.lv[Lnl - 1].cap_b;
  const bool grow_ok = cap_last > (u64)2 * C0 + max_deg + kBankQ;
  const u64 grow_at = grow_ok ? cap_last - ((u64)2 * C0 + max_deg + kBankQ) : 0;
  u32 par = 0;
  bool rescan_due = false;
  bool evict_due = Bk::any(__popc(occm) > (int)(KI - PE), hc.scr());
  bool fail_bad = false, fail_ovf = false, cold_fail = false;
  u32 pass_id = 0;
  u64 mph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long mpt = clock64();
#ifdef PBH_PROF_BUILD
#define MPROF(i)                     \
  {                                  \
    const long long t1_ = clock64(); \
    mph[i] += (u64)(t1_ - mpt);      \
    mpt = t1_;                       \
  }
#else
#define MPROF(i)
#endif
  while (live > 0) {
    if (!grow_ok || (u64)qn + deep_n > grow_at) {
      need_grow = true;
      break;
    }
    MPROF(7);
    // ---- the thresholds: L (level-0 minimum) and T (min of p + minout)
    if (rescan_due) multi_rescan<B, KI>(L, tid, occm, lhas, lmin_p, lmin_k, lmin_s, tmin);
    rescan_due = false;
    const BankOffer x = bank_exchange<NW, KI, VT, true>(par, lhas, lmin_p, lmin_k, lmin_s, 0, 0,
                                                        0, 0, tmin);
    par ^= 1;
    if (!x.has) {
      MULTI_TO_H();
      H.refill();
      MULTI_FROM_H();
      rescan_due = true;
      evict_due = false;
      if (hc.failed() || H.n_l0 == 0) {
        if (!hc.failed()) hc.fail(PBH_ERR_INVARIANT, 0xE5);
        cold_fail = true;
        break;
      }
      continue;
    }
    u64 T = x.t;
    if (!L.spl_inf) T = min(T, L.spl_p + 1);
    const u64 Lp = x.p;
    MPROF(0);
    // ---- select this bank's settled slots (OUT or IN criterion)
    u32 sel = 0;
    {
      u32 m = occm;
      while (m) {
        const u32 i = __ffs(m) - 1;
        m &= m - 1;
        const u32 s = i * B + tid;
        const u64 p = L.lp[s];
        const u32 mi = L.lmi[s];
        if (p <= T || (mi != 0xffffffffu && p - Lp <= (u64)mi)) sel |= 1u << i;
      }
    }
    u32 nb;
    const u32 pos0 = Bk::scan_excl((u32)__popc(sel), nb, hc.scr());
    {
      u32 pos = pos0;
      u32 m = sel;
      while (m) {
        const u32 i = __ffs(m) - 1;
        m &= m - 1;
        const u32 s = i * B + tid;
        M.k[pos] = L.lk[s];
        M.p[pos] = L.lp[s];
        M.rb[pos] = L.lrb[s];
        M.deg[pos] = L.ldeg[s];
        ++pos;
      }
    }
    Bk::sync();
    MPROF(1);
    // ---- edge offsets of the batch rows
    u32 te;
    {
      u32 run = 0;
      for (u32 j0 = 0; j0 < nb; j0 += B) {
        const u32 j = j0 + tid;
        const u32 dg = j < nb ? M.deg[j] : 0;
        u32 tot;
        const u32 ex = Bk::scan_excl(dg, tot, hc.scr());
        if (j < nb) M.pre[j] = run + ex;
        run += tot;
      }
      if (tid == 0) M.pre[nb] = run;
      te = run;
    }
    Bk::sync();
    // the round may push up to te entries: grow first (nothing changed yet)
    if ((u64)qn + deep_n + te > grow_at) {
      need_grow = true;
      break;
    }
    // ---- commit the batch: settle (sssp.cpp:41-47)
    for (u32 j = tid; j < nb; j += B) {
      const u32 k = M.k[j];
      idx[k].state = PBH_ST_DEAD;
      my_dist[k] = M.p[j];
      my_settled[n_settled + j] = k;
    }
    if (sel) {
      occm &= ~sel;
      rescan_due = true;
    }
    Bk::sync();
    n_settled += nb;
    ++rounds;
    ops += nb;
    live -= nb;
    MPROF(2);
    // ---- relax the flattened rows in passes of 256 edges
    u32 n_imp = 0;
    for (u32 base = 0; base < te; base += kBankPass) {
      if (evict_due || qn > (u32)(kBankQ - kBankPass)) {
        MULTI_TO_H();
        if (evict_due) H.evict();
        if (!hc.failed() && H.qn > (u32)(kBankQ - kBankPass)) H.flush_q();
        MULTI_FROM_H();
        rescan_due = true;
        evict_due = false;
        if (hc.failed()) {
          cold_fail = true;
          break;
        }
      }
      MPROF(3);
      u32 uu[PE], ww[PE], vv[PE];
      u64 pv[PE];
      bool in[PE];
#pragma unroll
      for (u32 t = 0; t < PE; ++t) {
        const u32 e = base + tid + B * t;
        in[t] = e < te;
        uu[t] = ww[t] = vv[t] = 0;
        pv[t] = 0;
        if (in[t]) {
          u32 lo = 0, hi = nb;  // last row with pre <= e
          while (hi - lo > 1) {
            const u32 mid = (lo + hi) >> 1;
            if (M.pre[mid] <= e)
              lo = mid;
            else
              hi = mid;
          }
          const u64 j = M.rb[lo] + (e - M.pre[lo]);
          vv[t] = M.k[lo];
          pv[t] = M.p[lo];
          uu[t] = __ldg(tgt + j);
          ww[t] = __ldg(wt + j);
        }
      }
      ulonglong2 ee[PE];
      u64 ob[PE], oe[PE];
      u32 mo[PE], mi[PE];
#pragma unroll
      for (u32 t = 0; t < PE; ++t) {
        ee[t] = make_ulonglong2(~0ull, PBH_ST_DEAD);
        ob[t] = oe[t] = 0;
        mo[t] = mi[t] = 0xffffffffu;
        if (in[t]) {
          ee[t] = __ldcg(reinterpret_cast<const ulonglong2*>(idx + uu[t]));
          ob[t] = __ldg(off + uu[t]);
          oe[t] = __ldg(off + uu[t] + 1);
          mo[t] = __ldg(mwo + uu[t]);
          mi[t] = __ldg(mwi + uu[t]);
        }
      }
      asm volatile("" ::: "memory");
      if (rescan_due) multi_rescan<B, KI>(L, tid, occm, lhas, lmin_p, lmin_k, lmin_s, tmin);
      rescan_due = false;
      MPROF(4);
      // phase A: candidates lower the index priority (64-bit atomicMin)
      bool imp[PE];
      u64 cand[PE];
      bool ovf = false;
#pragma unroll
      for (u32 t = 0; t < PE; ++t) {
        cand[t] = pv[t] + ww[t];
        imp[t] = false;
        if (!in[t] || PBH_ST((u32)ee[t].y) == PBH_ST_DEAD) continue;
        ovf |= cand[t] < pv[t];
        if (cand[t] < ee[t].x) {
          const u64 old = atomicMin(reinterpret_cast<unsigned long long*>(&idx[uu[t]].prio),
                                    (unsigned long long)cand[t]);
          imp[t] = cand[t] <= old;
        }
      }
      Bk::sync();
      // phase B: the relaxation that holds the final minimum claims the
      // target through its parent word and applies the slot update
      u32 fresh = 0, nimp = 0, nq = 0;
      bool bad = false;
#pragma unroll
      for (u32 t = 0; t < PE; ++t) {
        if (!imp[t]) continue;
        const u32 u = uu[t];
        const u64 c = cand[t];
        if (__ldcg(reinterpret_cast<const unsigned long long*>(&idx[u].prio)) != c) continue;
        const u32 old_parent = (u32)(ee[t].y >> 32);
        if (atomicCAS(&idx[u].parent, old_parent, vv[t]) != old_parent) continue;
        ++nimp;
        const u32 st = (u32)ee[t].y;
        fresh += PBH_ST(st) != PBH_ST_LIVE;
        const u32 loc = st >> 2;
        u32 nst;
        if (PBH_ST(st) == PBH_ST_LIVE && loc < C0) {
          // (a gather may already see another relaxation's phase-A
          // priority, so only the key is checked here)
          bad |= L.lk[loc] != u;
          L.lp[loc] = c;
          S.dirty[par][loc % B] = 1;
          nst = st;
        } else if (L.spl_inf || c < L.spl_p || (c == L.spl_p && u <= L.spl_k)) {
          const u32 i = __ffs(~occm) - 1;
          const u32 sl = i * B + tid;
          occm |= 1u << i;
          L.lk[sl] = u;
          L.lp[sl] = c;
          L.lrb[sl] = ob[t];
          L.ldeg[sl] = (u32)(oe[t] - ob[t]);
          L.lmo[sl] = mo[t];
          L.lmi[sl] = mi[t];
          if (!lhas || less_pk(c, u, lmin_p, lmin_k)) {
            lhas = true;
            lmin_p = c;
            lmin_k = u;
            lmin_s = sl;
          }
          const u64 tt = mo[t] == 0xffffffffu ? ~0ull : c + mo[t];
          tmin = min(tmin, (u64)(tt < c ? ~0ull : tt));
          nst = PBH_ST_LIVE | (sl << 2);
        } else {
          const u32 qp_ = atomicAdd(&L.qn, 1u);
          L.qk[qp_] = u;
          L.qp[qp_] = c;
          ++nq;
          nst = PBH_ST_LIVE | (PBH_LOC_DEEP << 2);
        }
        idx[u].state = nst;
      }
      MPROF(5);
      ++pass_id;
      const u32 ev = (u32)__popc(occm) > (u32)KI - PE ? 1u : 0u;
      const BankOffer r = bank_exchange<NW, KI, VT, true>(
          par, false, 0, 0, 0, 0, 0, fresh | (nimp << 9) | ((ovf ? 1u : 0u) << 18),
          nq | (ev << 9) | ((bad ? 1u : 0u) << 18));
      if (S.dirty[par][tid]) {
        S.dirty[par][tid] = 0;
        rescan_due = true;
      }
      par ^= 1;
      n_imp += r.nimp;
      live += r.fresh;
      qn += r.nq;
      evict_due = (r.flags & 1u) != 0;
      if (r.flags & 6u) {
        fail_bad = (r.flags & 2u) != 0;
        fail_ovf = (r.flags & 4u) != 0;
        break;
      }
    }
    MPROF(6);
    if (cold_fail || fail_bad || fail_ovf) break;
    if (n_imp) ops += n_imp <= d ? 1u : ceil_div_cold(n_imp, d);
  }
  H.occm = occm;
  H.live = live;
  H.qn = qn;
  H.deep_n = deep_n;
#undef MULTI_TO_H
#undef MULTI_FROM_H
  if (fail_bad && !hc.failed()) hc.fail(PBH_ERR_INVARIANT, 0xD1);
  if (fail_ovf && !hc.failed()) hc.fail(PBH_ERR_OVERFLOW, 0);
  Bk::sync();
  L.occ[tid] = H.occm;
  if (tid == 0) L.qn = H.qn;
  Bk::sync();
  {
    const u32* src = reinterpret_cast<const u32*>(&L);
    u32* dst = reinterpret_cast<u32*>(save + blockIdx.x);
    for (u32 i = tid; i < sizeof(BankL0<B, KI, true>) / 4; i += B) dst[i] = src[i];
  }
  H.to_cold();
  if (tid == 0) sm.ops = H.pushes;
  Bk::sync();
  hc.store();
#undef MPROF
  (void)mpt;
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) my->phase[i] += mph[i];
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

}  // namespace pbh_dev
