// Warp-synchronous fast path for par_dijkstra (sssp.cpp:21-69).
//
// One warp owns one source's bucket heap. The hot level lives in shared
// memory as two (priority, value)-sorted runs:
//   B_0  the bucket (capacity cap0), everything <= splitter_0
//   S_0  a small insertion buffer (capacity S0CAP) — the paper's signal
//        buffer S_0, resolved into B_0 when full ("resolve(0)")
// Both carry tombstone flags: a decrease-key or extraction of a copy held in
// B_0/S_0 is removed eagerly by binary search, so the minimum is always the
// smaller live head of the two runs — no position-index read on extract.
// Deeper levels (HBM) are handled by the CTA engine of pbh_heap.cuh (cold
// path): overflow of B_0 is pushed into S_1, and resolve(i >= 1) runs after
// every 4th push into level i (the 4-to-1 rule, scheduler.cpp:11-20).
// Scalar state is kept in registers, replicated across the 32 lanes.
#pragma once

#include "pbh_kernels.cuh"

namespace pbh_dev {

constexpr int kFastS0 = 64;    // S_0 slots (2 per lane)
constexpr int kChunk = 256;    // edges relaxed per pass (8 per lane)

// Static shared-memory image of one fast-path heap (CAP0 = B_0 capacity).
template <int CAP0, int VT>
struct FastSmem {
  u64 bp[2][CAP0];
  u32 bk[2][CAP0];
  u8 bt[2][CAP0];
  u64 sp[kFastS0];
  u64 tp[kFastS0];
  u64 pp[2 * kFastS0];
  u64 cp[kChunk];
  u64 co[kChunk];
  u32 sk[kFastS0];
  u32 tk[kFastS0];
  u32 pk[2 * kFastS0];
  u32 cpos[CAP0 + 64];
  u32 ck[kChunk];
  u32 cs[kChunk];
  u8 sv[kFastS0];
  u8 kf[kChunk];
  u32 sh[2 * kFastS0];  // key -> S_0 slot + 1 (open addressing; 0 = empty)
  HeapSmem<32, VT> hs;
};

// The one shared-memory image per CTA (a function-scope __shared__ is static).
template <int CAP0, int VT>
DEV FastSmem<CAP0, VT>& fast_smem() {
  __shared__ __align__(16) FastSmem<CAP0, VT> S;
  return S;
}

struct FastLayout {
  u32 off_hs;                  // HeapSmem<32, VT> (cold path)
  u32 off_bk[2], off_bp[2];    // B_0 ping-pong runs (cap0)
  u32 off_bt[2];               // B_0 tombstones (cap0 bytes each)
  u32 off_sk, off_sp, off_sv;  // S_0 slots (unsorted) + valid flags
  u32 off_tk, off_tp;          // S_0 sort scratch (kFastS0)
  u32 off_pk, off_pp;          // push list (2 * kFastS0)
  u32 off_cpos;                // prefix counts (max(cap0, S0) + 64)
  u32 off_ck, off_cp, off_co, off_cs, off_kf;  // one chunk's improving relaxations
  u32 total;
};

template <int CAP0, int VT>
struct FastSssp {
  using HC = HeapCta<32, VT>;
  HC& hc;
  const u32 lane;
  pbh_idx_entry* idx;
  static constexpr u32 cap0 = CAP0;

  DEV FastSssp(HC& h, u32 ln, pbh_idx_entry* ix) : hc(h), lane(ln), idx(ix) {}

  DEV void set_loc(u32 k, u32 loc) { idx[k].state = PBH_ST_LIVE | (loc << 2); }
  // Relabel every B_0 entry with its slot (after B_0 was rebuilt elsewhere).
  DEV void relabel_b0() {
    for (u32 i = bh + lane; i < be; i += 32)
      if (!bt(bsel)[i]) set_loc(bk(bsel)[i], PBH_LOC_B | i);
    __syncwarp();
  }
  // replicated scalar state
  u32 bsel, bh, be;    // B_0 = bk[bsel][bh, be)
  u32 b_live;
  u32 s0n, s_live;     // S_0 slots used / live
  u64 smin_p;          // minimum live S_0 entry (valid when s_live > 0)
  u32 smin_k, smin_slot;
  u64 spl_p;
  u32 spl_k, spl_inf;
  i64 live;
  u64 pushes;
  bool deep;
  u64 deep_n;  // entries stored below level 0
  u32 xp_ = 0;  // ablation switches (timing experiments only)
  u64 t_flush = 0, n_flush = 0, t_smin = 0;

  DEV static FastSmem<CAP0, VT>& Sm() { return fast_smem<CAP0, VT>(); }
  DEV u32* bk(u32 s) const { return Sm().bk[s]; }
  DEV u64* bp(u32 s) const { return Sm().bp[s]; }
  DEV u8* bt(u32 s) const { return Sm().bt[s]; }
  DEV u32* sk() const { return Sm().sk; }
  DEV u64* sp() const { return Sm().sp; }
  DEV u8* sv() const { return Sm().sv; }
  DEV u32* tk() const { return Sm().tk; }
  DEV u64* tp() const { return Sm().tp; }
  DEV u32* pk() const { return Sm().pk; }
  DEV u64* pp() const { return Sm().pp; }
  DEV u32* cpos() const { return Sm().cpos; }
  DEV u32* sh() const { return Sm().sh; }
  DEV static u32 hslot(u32 k) { return (k * 2654435761u) >> (32 - 7); }  // 128 buckets

  DEV bool adm0(u64 p, u32 k) const { return spl_inf || p < spl_p || (p == spl_p && k <= spl_k); }

  DEV static u32 wscan(bool f, u32& tot) {
    const u32 m = __ballot_sync(0xffffffffu, f);
    tot = __popc(m);
    return __popc(m & ((1u << (threadIdx.x & 31)) - 1));
  }

  // warp argmin of (p, k, tag) over lanes with `has`: three redux.sync
  // minimum reductions (high word, low word, key) instead of a shuffle tree.
  DEV static void wmin(bool& has, u64& p, u32& k, u32& tag) {
    const u32 hi = has ? (u32)(p >> 32) : 0xffffffffu;
    const u32 mhi = __reduce_min_sync(0xffffffffu, hi);
    const bool c1 = has && hi == mhi;
    const u32 lo = c1 ? (u32)p : 0xffffffffu;
    const u32 mlo = __reduce_min_sync(0xffffffffu, lo);
    const bool c2 = c1 && (u32)p == mlo;
    const u32 mk = __reduce_min_sync(0xffffffffu, c2 ? k : 0xffffffffu);
    const u32 win = __ballot_sync(0xffffffffu, c2 && k == mk);
    const bool any = __any_sync(0xffffffffu, has);
    tag = __shfl_sync(0xffffffffu, tag, win ? __ffs(win) - 1 : 0);
    p = ((u64)mhi << 32) | mlo;
    k = mk;
    has = any;
  }

  // ---------------------------------------------------------- state sync
  DEV void from_cold() {
    const pbh_level_state& t = hc.s.st[0];
    bsel = t.b_sel;
    bh = t.b_head;
    be = t.b_head + t.b_size;
    b_live = t.b_size;
    spl_p = t.spl_p;
    spl_k = t.spl_k;
    spl_inf = t.spl_inf;
    live = hc.s.live;
    deep_n = hc.content_from(1);
    deep = deep_n > 0;
    u8* f = bt(bsel);
    for (u32 i = bh + lane; i < be; i += 32) f[i] = 0;
    __syncwarp();
  }
  DEV void to_cold() {
    // requires S_0 empty and B_0 compact (flush() guarantees both)
    if (lane == 0) {
      pbh_level_state& t = hc.s.st[0];
      t.b_sel = bsel;
      t.b_head = bh;
      t.b_size = be - bh;
      t.spl_p = spl_p;
      t.spl_k = spl_k;
      t.spl_inf = spl_inf;
      hc.s.live = live;
    }
    __syncwarp();
  }

  DEV static u32 lbound(const u32* k, const u64* p, u32 lo, u32 hi, u64 pq, u32 kq) {
    while (lo < hi) {
      const u32 m = (lo + hi) >> 1;
      const u64 pm = p[m];
      if (pm < pq || (pm == pq && k[m] < kq))
        lo = m + 1;
      else
        hi = m;
    }
    return lo;
  }

  // ---------------------------------------------------------------- S_0
  DEV void smin_recompute() {
    bool has = false;
    u64 p = 0;
    u32 k = 0, tag = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const u32 i = lane + 32 * h;
      if (i < s0n && sv()[i]) {
        const u64 pi = sp()[i];
        const u32 ki = sk()[i];
        if (!has || less_pk(pi, ki, p, k)) {
          p = pi;
          k = ki;
          tag = i;
          has = true;
        }
      }
    }
    wmin(has, p, k, tag);
    smin_p = p;
    smin_k = k;
    smin_slot = tag;
  }

  // ------------------------------------------------------- resolve(0)
  // Sort the live S_0 entries, merge the admitted ones into B_0, cut at
  // cap0, push the overflow and the non-admitted ones down into S_1.
  // Leaves S_0 empty and B_0 compact in the other buffer.
  DEV void flush() {
    const long long f0 = clock64();
    flush_body();
    t_flush += (u64)(clock64() - f0);
    ++n_flush;
  }
  DEV void flush_body() {
    // 1) compact live S_0 slots into the sort scratch
    u32 n_s = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const u32 i = lane + 32 * h;
      const bool f = i < s0n && sv()[i];
      u32 tot;
      const u32 pos = n_s + wscan(f, tot);
      if (f) {
        tk()[pos] = sk()[i];
        tp()[pos] = sp()[i];
      }
      n_s += tot;
    }
    __syncwarp();
    // 2) bitonic sort of n_s <= 64 entries (pad with +inf)
    u32* SK = tk();
    u64* SP = tp();
    u32 m = 1;
    while (m < n_s) m <<= 1;
    for (u32 i = n_s + lane; i < m; i += 32) {
      SK[i] = 0xffffffffu;
      SP[i] = ~0ull;
    }
    __syncwarp();
    for (u32 size = 2; size <= m; size <<= 1)
      for (u32 stride = size >> 1; stride > 0; stride >>= 1) {
        for (u32 t = lane; t < (m >> 1); t += 32) {
          const u32 i = 2 * t - (t & (stride - 1)), j = i + stride;
          const bool up = (i & size) == 0;
          const u64 pi = SP[i], pj = SP[j];
          const u32 ki = SK[i], kj = SK[j];
          if (less_pk(pj, kj, pi, ki) == up) {
            SP[i] = pj;
            SP[j] = pi;
            SK[i] = kj;
            SK[j] = ki;
          }
        }
        __syncwarp();
      }
    // admitted prefix
    u32 adm = n_s;
    if (!spl_inf) {
      u32 lo = 0, hi = n_s;
      while (lo < hi) {
        const u32 mm = (lo + hi) >> 1;
        if (adm0(SP[mm], SK[mm]))
          lo = mm + 1;
        else
          hi = mm;
      }
      adm = lo;
    }
    // 3) live-prefix counts of B_0
    const u32* BK = bk(bsel);
    const u64* BP = bp(bsel);
    const u8* BT = bt(bsel);
    u32* cp = cpos();
    u32 n_b = 0;
    for (u32 b = bh; b < be; b += 32) {
      const u32 i = b + lane;
      const bool f = i < be && !BT[i];
      u32 tot;
      const u32 pre = wscan(f, tot);
      if (i < be) cp[i - bh] = n_b + pre;
      n_b += tot;
    }
    if (lane == 0) cp[be - bh] = n_b;
    __syncwarp();
    // 4) rank merge into the other B buffer; positions >= cap0 -> push list
    const u32 nb = 1 - bsel;
    u32* OK = bk(nb);
    u64* OP = bp(nb);
    u32* PK = pk();
    u64* PP = pp();
    const u32 total = n_b + adm;
    auto put = [&](u32 pos, u32 k, u64 p) {
      if (pos < cap0) {
        OK[pos] = k;
        OP[pos] = p;
        set_loc(k, PBH_LOC_B | pos);
      } else {
        PK[pos - cap0] = k;
        PP[pos - cap0] = p;
        set_loc(k, PBH_LOC_DEEP);
      }
    };
    for (u32 b = bh; b < be; b += 32) {
      const u32 i = b + lane;
      if (i < be && !BT[i]) {
        const u32 r = lbound(SK, SP, 0, adm, BP[i], BK[i]);
        put(cp[i - bh] + r, BK[i], BP[i]);
      }
    }
    for (u32 j = lane; j < adm; j += 32) {
      const u32 r = lbound(BK, BP, bh, be, SP[j], SK[j]);
      put(j + cp[r - bh], SK[j], SP[j]);
    }
    __syncwarp();
    const u32 keep = total < cap0 ? total : cap0;
    u32 n_push = total - keep;
    if (total > cap0) {
      spl_inf = 0;
      spl_p = OP[cap0 - 1];
      spl_k = OK[cap0 - 1];
    }
    for (u32 j = adm + lane; j < n_s; j += 32) {
      PK[n_push + j - adm] = SK[j];
      PP[n_push + j - adm] = SP[j];
      set_loc(SK[j], PBH_LOC_DEEP);
    }
    n_push += n_s - adm;
    u8* NT = bt(nb);
    for (u32 i = lane; i < keep; i += 32) NT[i] = 0;
    __syncwarp();
    bsel = nb;
    bh = 0;
    be = keep;
    b_live = keep;
    s0n = 0;
    s_live = 0;
    if (n_push) push(n_push);
  }

  // Push pk/pp[0, n) into S_1 and run the 4-to-1 schedule (cold path).
  DEV void push(u32 n) {
    to_cold();
    hc.template push_down<true>(0, Run{pk(), pp(), n});
    ++pushes;
    for (u32 i = 1; i < hc.s.n_levels && i < 31 && !hc.failed(); ++i) {
      if (pushes & ((1ull << (2 * i)) - 1)) break;  // resolve(i) every 4^i pushes
      hc.resolve(i);
    }
    from_cold();
  }

  // Refill B_0 from level 1 (and below) — cold path; requires flush first.
  DEV void refill() {
    to_cold();
    if (be == bh)
      hc.fill0();
    else
      hc.refill(0);
    from_cold();
    relabel_b0();
  }

  DEV void skip_b() {
    while (bh < be && bt(bsel)[bh]) ++bh;
  }

  // ------------------------------------------------------------ extract
  DEV bool extract(u32& v, u64& p) {
    for (int guard = 0; guard < 4; ++guard) {
      skip_b();
      const bool hb = bh < be, hs = s_live > 0;
      if (!hb && deep) {
        flush();
        if (hc.failed()) return false;
        refill();
        if (hc.failed()) return false;
        continue;
      }
      if (!hb && !hs) return false;
      bool take_b = hb;
      if (hb && hs) take_b = less_pk(bp(bsel)[bh], bk(bsel)[bh], smin_p, smin_k);
      if (take_b) {
        v = bk(bsel)[bh];
        p = bp(bsel)[bh];
        ++bh;
        --b_live;
      } else {
        v = smin_k;
        p = smin_p;
        if (lane == 0) sv()[smin_slot] = 0;
        __syncwarp();
        --s_live;
        const long long s0 = clock64();
        if (s_live && !(xp_ & 4)) smin_recompute();
        t_smin += (u64)(clock64() - s0);
      }
      --live;
      return true;
    }
    return false;
  }

  // --------------------------------------------------------- kill/insert
  // Eagerly remove the old copies of the decreased keys among the n
  // candidates (ck/co/cs in smem). The old index entry read at relax time
  // carries the copy's level-0 location (S_0 slot or B_0 slot), so a kill is
  // one verified O(1) tombstone; copies in HBM levels are dropped lazily by
  // the merge filters. A binary-search fallback guards a stale location.
  DEV void kill(const u32* ck, const u64* co, const u32* cs, u32 n) {
    bool smin_hit = false;
    u32 ks = 0, kb = 0;
    for (u32 j = lane; j < n; j += 32) {
      const u32 sw = cs[j];
      if (PBH_ST(sw) != PBH_ST_LIVE) continue;
      const u32 loc = sw >> 2;
      if (loc == PBH_LOC_DEEP) continue;
      const u32 k = ck[j];
      const u64 po = co[j];
      // 1) the recorded S_0 slot (or a scan when the slot is stale)
      bool found = false;
      if (!(loc & PBH_LOC_B) && s0n) {
        u32 i = loc;
        if (!(i < s0n && sk()[i] == k && sp()[i] == po))
          for (i = 0; i < s0n && !(sk()[i] == k && sp()[i] == po && sv()[i]); ++i) {
          }
        if (i < s0n && sv()[i]) {
          sv()[i] = 0;
          ++ks;
          smin_hit |= i == smin_slot;
          found = true;
        }
      }
      // 2) the recorded B_0 slot (or a binary search when it is stale)
      if (!found && adm0(po, k)) {
        const u32* K = bk(bsel);
        const u64* P = bp(bsel);
        u32 i = loc & ~PBH_LOC_B;
        if (!((loc & PBH_LOC_B) && i >= bh && i < be && K[i] == k && P[i] == po))
          i = lbound(K, P, bh, be, po, k);
        if (i < be && K[i] == k && P[i] == po && !bt(bsel)[i]) {
          bt(bsel)[i] = 1;
          ++kb;
        }
      }
    }
    s_live -= __reduce_add_sync(0xffffffffu, ks);
    b_live -= __reduce_add_sync(0xffffffffu, kb);
    __syncwarp();
    if (__any_sync(0xffffffffu, smin_hit) && s_live) smin_recompute();
  }

  // Append the n candidates (ck/cp) to S_0; (gm_p, gm_k, gm_j) is their
  // minimum and its list index.
  DEV void append(const u32* ck, const u64* cp, u32 n, u64 gm_p, u32 gm_k, u32 gm_j, u32 par) {
    u32 done = 0;
    while (done < n) {
      if (s0n >= (u32)kFastS0) {
        flush();
        if (hc.failed()) return;
      }
      const u32 m = min(n - done, (u32)kFastS0 - s0n);
      for (u32 j = lane; j < m; j += 32) {
        const u32 k = ck[done + j];
        const u64 pk_ = cp[done + j];
        sk()[s0n + j] = k;
        sp()[s0n + j] = pk_;
        sv()[s0n + j] = 1;
        pbh_idx_entry e;
        e.prio = pk_;
        e.state = PBH_ST_LIVE | ((s0n + j) << 2);
        e.parent = par;
        reinterpret_cast<ulonglong2*>(idx)[k] = *reinterpret_cast<const ulonglong2*>(&e);
      }
      __syncwarp();
      if (done == 0 && m == n) {
        // whole group in one piece: the known minimum is at slot s0n + gm_j
        if (!s_live || less_pk(gm_p, gm_k, smin_p, smin_k)) {
          smin_p = gm_p;
          smin_k = gm_k;
          smin_slot = s0n + gm_j;
        }
        s0n += m;
        s_live += m;
      } else {
        s0n += m;
        s_live += m;
        smin_recompute();
      }
      done += m;
    }
  }
};

// par_dijkstra with one warp per source (blockDim = 32, one source per CTA).
template <int CAP0, int VT>
__global__ void __launch_bounds__(32, 1)
    k_sssp_fast(pbh_heap_dev* heaps, const u64* __restrict__ off, const u32* __restrict__ tgt,
                const u32* __restrict__ wt, u32 V, const u32* sources, u64* dist, u32* settled,
                SsspState* sst, u32 dag_mode, u32 max_deg, u32 d, FastLayout FL, u32 xp) {
  FastSmem<CAP0, VT>& S = fast_smem<CAP0, VT>();
  using HC = HeapCta<32, VT>;
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
  FastSssp<CAP0, VT> F(hc, threadIdx.x, g->idx);
  F.xp_ = xp;
  F.s0n = 0;
  F.s_live = 0;
  F.pushes = sm.ops;  // persisted push counter (fast path reuses the ops slot)
  F.from_cold();
  F.relabel_b0();  // B_0 was reloaded at offset 0
  pbh_idx_entry* idx = g->idx;
  u64* my_dist = dist + (u64)blockIdx.x * V;
  u32* my_settled = settled + (u64)blockIdx.x * V;
  u64 n_settled = my->n_settled, rounds = my->rounds;
  u64 ops = my->ops;  // Metrics::ops of the reference loop
  const u32 lane = threadIdx.x;
  u32* ck = S.ck;
  u64* cpv = S.cp;
  u64* cov = S.co;
  u32* csv = S.cs;
  u8* kf = S.kf;

  if (!my->started) {
    const u32 s = sources[blockIdx.x];
    if (lane == 0) {
      ck[0] = s;
      cpv[0] = 0;
    }
    __syncwarp();
    F.append(ck, cpv, 1, 0, s, 0, s);
    F.live = 1;
    ops = 1;  // eng.update({s, 0}) (sssp.cpp:36)
  }

  bool need_grow = false, overflow = false;
  const u32 Lnl = sm.n_levels;
  const u64 cap_last = Lnl == 1 ? (u64)CAP0 : sm.lv[Lnl - 1].cap_b;
  const bool tm = (xp & 16) != 0;
  u64 ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tA = clock64(), tB;
#define PH(i)                   \
  if (tm) {                     \
    tB = clock64();             \
    ph[i] += (u64)(tB - tA);    \
    tA = tB;                    \
  }
  // Exact next-vertex prefetch: after the candidates of round r are known,
  // the next extraction is min(live heads, new entries); its offsets load
  // under the kill phase and its first row chunk under append + extract.
  bool pf = false;
  u32 pf_v = 0;
  u64 pf_rb = 0, pf_re = 0;
  u32 pu[8], pw[8];
  while (!hc.failed() && F.live > 0) {
    if ((u64)(F.be - F.bh) + F.s0n + F.deep_n + max_deg + kFastS0 > cap_last) {
      need_grow = true;
      break;
    }
    u32 v;
    u64 p;
    if (!F.extract(v, p)) {
      if (!hc.failed()) hc.fail(PBH_ERR_INVARIANT, 0xE5);
      break;
    }
    if (lane == 0) {
      idx[v].state = PBH_ST_DEAD;
      my_dist[v] = p;
      my_settled[n_settled] = v;
    }
    ++n_settled;
    ++rounds;
    ++ops;
    PH(0);
    const bool hit = pf && pf_v == v;
    if (tm && hit) ph[7] += 1;
    u64 rb, re;
    if (hit) {
      rb = pf_rb;
      re = pf_re;
    } else {
      rb = off[v];
      re = off[v + 1];
    }
    pf = false;
    u32 n_imp = 0;
    for (u64 base = rb; base < re; base += kChunk) {
      const bool last_chunk = base + kChunk >= re;
      u32 uu[8], ww[8];
      ulonglong2 ee[8];
      if (hit && base == rb) {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          uu[t] = pu[t];
          ww[t] = pw[t];
        }
      } else {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const u64 j = base + lane + 32 * t;
          uu[t] = j < re ? __ldg(tgt + j) : 0;
          ww[t] = j < re ? __ldg(wt + j) : 0;
        }
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const u64 j = base + lane + 32 * t;
        if (j < re) ee[t] = __ldcg(reinterpret_cast<const ulonglong2*>(idx + uu[t]));
      }
      u32 mask = 0, nfresh = 0;
      u64 cand[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const u64 j = base + lane + 32 * t;
        cand[t] = 0;
        if (j < re && (dag_mode || PBH_ST((u32)ee[t].y) != PBH_ST_DEAD)) {
          cand[t] = p + ww[t];
          overflow |= cand[t] < p;
          if (cand[t] < ee[t].x) mask |= 1u << t;
        }
      }
      const u32 cnt = __popc(mask);
      u32 pos = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, pos, o);
        if (lane >= (u32)o) pos += y;
      }
      const u32 tot = __shfl_sync(0xffffffffu, pos, 31);
      pos -= cnt;
      bool bany = false;
      u64 bp_ = 0;
      u32 bk_ = 0, bj_ = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        if (mask & (1u << t)) {
          nfresh += PBH_ST((u32)ee[t].y) != PBH_ST_LIVE;
          ck[pos] = uu[t];
          cpv[pos] = cand[t];
          cov[pos] = ee[t].x;
          csv[pos] = (u32)ee[t].y;
          if (!bany || less_pk(cand[t], uu[t], bp_, bk_)) {
            bp_ = cand[t];
            bk_ = uu[t];
            bj_ = pos;
            bany = true;
          }
          ++pos;
        }
      }
      __syncwarp();
      F.live += __reduce_add_sync(0xffffffffu, nfresh);
      n_imp += tot;
      if (tot) FastSssp<CAP0, VT>::wmin(bany, bp_, bk_, bj_);
      if (last_chunk) {
        F.skip_b();
        const bool hb = F.bh < F.be;
        bool nh = bany;
        u32 nv = bk_;
        u64 np_ = bp_;
        if (hb && (!nh || less_pk(F.bp(F.bsel)[F.bh], F.bk(F.bsel)[F.bh], np_, nv))) {
          nv = F.bk(F.bsel)[F.bh];
          np_ = F.bp(F.bsel)[F.bh];
          nh = true;
        }
        if (F.s_live && (!nh || less_pk(F.smin_p, F.smin_k, np_, nv))) {
          nv = F.smin_k;
          nh = true;
        }
        if (nh && !(xp & 8)) {
          pf = true;
          pf_v = nv;
          pf_rb = off[pf_v];
          pf_re = off[pf_v + 1];
        }
      }
      PH(1);
      if (tot && !(xp & 1)) F.kill(ck, cov, csv, tot);
      PH(2);
      if (tot && !(xp & 2)) F.append(ck, cpv, tot, bp_, bk_, bj_, v);
      PH(3);
      if (hc.failed()) break;
    }
    if (hc.failed()) break;
    if (pf) {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const u64 j = pf_rb + lane + 32 * t;
        pu[t] = j < pf_re ? __ldg(tgt + j) : 0;
        pw[t] = j < pf_re ? __ldg(wt + j) : 0;
      }
    }
    if (__any_sync(0xffffffffu, overflow)) {
      hc.fail(PBH_ERR_OVERFLOW, v);
      break;
    }
    ops += (n_imp + d - 1) / d;
    PH(4);
  }
#undef PH
  // persist: flush S_0 so the HBM image is a plain bucket heap
  if (!hc.failed()) F.flush();
  F.to_cold();
  if (lane == 0) sm.ops = F.pushes;
  __syncwarp();
  hc.store();
  if (lane == 0) {
    my->n_settled = n_settled;
    my->rounds = rounds;
    my->started = 1;
    my->ops = ops;
    ph[5] += F.t_flush;
    ph[6] += F.t_smin;
    for (int i = 0; i < 8; ++i) my->phase[i] += ph[i];
    my->pad2 += F.n_flush;
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
