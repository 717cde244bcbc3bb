// CTA-resident bucket-heap engine (see pbh_engine.cuh header comment).
//
// One CTA owns one heap. All threads run the same control flow; scalar level
// state lives in shared memory and is written by thread 0 between barriers.
#pragma once

#include "pbh_grid.cuh"

namespace pbh_dev {

constexpr u32 kInfCount = 0xffffffffu;
// Stale shares of the deep content above which the grid (two gather passes)
// and the streamed (one pass) merges drop stale entries. Measured on the
// full C1 trace (10^6 ops): 7/8 6.28, 3/4 6.30, 1/2 6.40, never 7.10 µs/op
// (the carried stale entries add two levels); on short runs and on C4 the
// stale share stays lower and a lower gate only costs gathers.
constexpr u32 kGridFilterNum = 7, kGridFilterDen = 8;
constexpr u32 kStreamFilterNum = 7, kStreamFilterDen = 8;

template <int NT, int VT>
struct HeapSmem {
  pbh_level_state st[PBH_MAX_LEVELS];
  pbh_level_bufs lv[PBH_MAX_LEVELS];
  TileSmem<NT, VT> tile;
  u32 scratch[NT / 32 + 2];
  i64 live;
  u64 ops;
  u64 stale_dropped;
  u64 resolves[PBH_MAX_LEVELS];
  u64 touches[PBH_MAX_LEVELS];
  u32 n_levels, d, cap0, debug;
  u32 status, detail;
  u64 aux;
  u32 bc[8];
  u64 bc64[4];
};

template <int NT, int VT>
struct HeapCta {
  using Bk = Blk<NT>;
  using Sm = HeapSmem<NT, VT>;
  static constexpr u32 T = NT * VT;

  Sm& s;
  pbh_heap_dev* g;
  pbh_idx_entry* idx;
  // level-0 working buffers (shared or global memory; generic pointers)
  u32* bk;  // batch keys   (d + NT)
  u64* bp;  // batch prios
  u64* bo;  // batch old priorities (SSSP path)
  u32* pk;  // push list keys (d + cap0)
  u64* pp;
  u8* rm;   // B_0 removal flags (cap0)
  u32* b0k_global[2];
  u64* b0p_global[2];
  bool b0_in_smem;
  // grid helpers for deep merges (trace interpreter only; null = CTA-local)
  GridJob* gj = nullptr;
  u32 gsz = 1;
  u32 gmin = kGridMin;  // smallest merge sent to the grid
  GridSmem<NT>* gs = nullptr;

  // Merge / copy dispatch: a big merge runs on the whole grid (unfiltered,
  // see pbh_grid.cuh), anything else in this CTA with the index filter.
  // helpers cannot see this CTA's shared memory: grid jobs take HBM runs only
  DEV static bool hbm(const void* p) { return p == nullptr || !__isShared(p); }
  DEV static bool hbm_sink(const Sink& k) { return hbm(k.k1) && (k.lim == kInfCount || hbm(k.k2)); }
  // This CTA alone streams the merge through the GridSmem windows
  // (unfiltered; cp.async window loads).
  // Returns the entries written (fewer than A.n + B.n when filtering).
  NOINL u32 stream_local(const Run& A, const Run& B, const Sink& snk, u32 out_base,
                         bool filter = false) {
    Bk::sync();
    if (threadIdx.x == 0) {
      GridJob& J = gs->job;
      J.ak = A.k;
      J.ap = A.p;
      J.bk = B.k;
      J.bp = B.p;
      J.na = A.n;
      J.nb = B.n;
      J.c = A.n + B.n;
      J.sink = snk;
      J.filter = filter ? 1u : 0u;
      J.idx = idx;
    }
    Bk::sync();
    const u32 n = grid_stream<NT>(gs->job, 0, A.n, 0, B.n, out_base, *gs);
    Bk::sync();
    return n;
  }
  // A filtered merge on the grid (job 8: count, prefix, compacting streams)
  // needs the job block of the grid sorts for its barrier and counts.
  DEV bool grid_filter_ok() const { return gs->job.ext != nullptr; }
  // Stale-entry filtering costs one index gather (a 32-byte sector) per
  // entry, per pass, and saves the stale entries' traffic through the
  // deeper merges; it pays only when a good part of the deep content is
  // stale. The heap's own counters estimate that share with no memory
  // traffic: entries stored below level 0 minus live values (an
  // underestimate while level 0 holds live values). True above num/den.
  DEV u32 dropped(u32 in, u32 out) {
    if (t0()) s.stale_dropped += in - out;
    return out;
  }
  DEV bool stale_share_above(u32 num, u32 den) const {
    const u64 stored = content_from(1);
    const u64 lv = s.live > 0 ? (u64)s.live : 0ull;
    const u64 stale = stored > lv ? stored - lv : 0ull;
    return stale * den > (u64)num * stored;
  }
  NOINL u32 mrg(const Run& A, const Run& B, bool filter, const Sink& snk, u32 out_base) {
    const u32 tot = A.n + B.n;
    const bool mem = gs && hbm(A.k) && hbm(B.k) && hbm_sink(snk);
    if (mem && gj && tot >= gmin) {
      // two gather passes (count, then compacting stream): at least half stale
      if (filter && grid_filter_ok() && stale_share_above(kGridFilterNum, kGridFilterDen)) {
        grid_run<NT>(gj, gsz, 8, A, B, tot, snk, out_base, *gs, gs->scr);
        return dropped(tot, *(volatile u32*)&gs->job.ext->merge_total);
      }
      grid_run<NT>(gj, gsz, 0, A, B, tot, snk, out_base, *gs, gs->scr);
      return tot;
    }
    if (mem && tot >= kStreamMin) {
      const bool f = filter && stale_share_above(kStreamFilterNum, kStreamFilterDen);
      return dropped(tot, stream_local(A, B, snk, out_base, f));
    }
    return merge_runs<NT, VT>(A, B, filter, idx, snk, out_base, s.tile, scr());
  }
  NOINL u32 cpy(const Run& A, bool filter, const Sink& snk, u32 out_base) {
    const Run E{A.k, A.p, 0};
    const bool mem = gs && hbm(A.k) && hbm_sink(snk);
    if (mem && gj && A.n >= gmin) {
      if (filter && grid_filter_ok() && stale_share_above(kGridFilterNum, kGridFilterDen)) {
        grid_run<NT>(gj, gsz, 8, A, E, A.n, snk, out_base, *gs, gs->scr);
        return dropped(A.n, *(volatile u32*)&gs->job.ext->merge_total);
      }
      grid_run<NT>(gj, gsz, 0, A, E, A.n, snk, out_base, *gs, gs->scr);
      return A.n;
    }
    if (mem && A.n >= kStreamMin) {
      const bool f = filter && stale_share_above(kStreamFilterNum, kStreamFilterDen);
      return dropped(A.n, stream_local(A, E, snk, out_base, f));
    }
    return copy_run<NT, VT>(A, filter, idx, snk, out_base, scr());
  }

  DEV bool t0() const { return threadIdx.x == 0; }
  DEV u32* scr() { return s.scratch; }

  DEV Run bucket(u32 i) const {
    const pbh_level_state& t = s.st[i];
    return Run{s.lv[i].bk[t.b_sel] + t.b_head, s.lv[i].bp[t.b_sel] + t.b_head, t.b_size};
  }
  DEV Run signal(u32 i) const {
    const pbh_level_state& t = s.st[i];
    return Run{s.lv[i].sk[t.s_sel] + t.s_head, s.lv[i].sp[t.s_sel] + t.s_head, t.s_size};
  }
  DEV u64 content(u32 i) const { return (u64)s.st[i].b_size + s.st[i].s_size; }
  DEV u64 content_from(u32 j) const {
    u64 c = 0;
    for (u32 m = j; m < s.n_levels; ++m) c += content(m);
    return c;
  }
  DEV void fail(u32 detail, u64 aux = 0) {
    if (t0() && s.status == 0) {
      s.status = detail == PBH_ERR_EMPTY_HEAP         ? 1u
                 : (detail == PBH_ERR_INVARIANT || detail == PBH_ERR_OVERFLOW) ? 3u
                 : detail == PBH_ERR_NEED_GROW ? 7u
                                               : 2u;
      s.detail = detail;
      s.aux = aux;
    }
    Bk::sync();
  }
  DEV bool failed() const { return s.status != 0; }

  // ---------------------------------------------------------------- setup
  // Load the heap header into shared memory; B_0 optionally into smem.
  NOINL void load(pbh_heap_dev* gh, u32* sm_b0k0, u64* sm_b0p0, u32* sm_b0k1, u64* sm_b0p1,
                bool use_smem_b0) {
    g = gh;
    idx = gh->idx;
    for (u32 i = threadIdx.x; i < PBH_MAX_LEVELS; i += NT) {
      s.st[i] = gh->st[i];
      s.lv[i] = gh->lv[i];
      s.resolves[i] = gh->resolves[i];
      s.touches[i] = gh->touches[i];
    }
    if (t0()) {
      s.live = gh->live;
      s.ops = gh->ops;
      s.stale_dropped = gh->stale_dropped;
      s.n_levels = gh->n_levels;
      s.d = gh->d;
      s.cap0 = gh->cap0;
      s.debug = gh->debug_checks;
      s.status = 0;
      s.detail = 0;
      s.aux = 0;
    }
    Bk::sync();
    b0k_global[0] = s.lv[0].bk[0];
    b0k_global[1] = s.lv[0].bk[1];
    b0p_global[0] = s.lv[0].bp[0];
    b0p_global[1] = s.lv[0].bp[1];
    b0_in_smem = use_smem_b0;
    if (use_smem_b0) {
      // copy the current B_0 run to smem buffer 0 at offset 0
      const Run b = bucket(0);
      for (u32 i = threadIdx.x; i < b.n; i += NT) {
        sm_b0k0[i] = b.k[i];
        sm_b0p0[i] = b.p[i];
      }
      Bk::sync();
      if (t0()) {
        s.lv[0].bk[0] = sm_b0k0;
        s.lv[0].bp[0] = sm_b0p0;
        s.lv[0].bk[1] = sm_b0k1;
        s.lv[0].bp[1] = sm_b0p1;
        s.st[0].b_sel = 0;
        s.st[0].b_head = 0;
      }
      Bk::sync();
    }
  }

  // Write the header (and B_0) back to global memory.
  NOINL void store() {
    Bk::sync();
    if (b0_in_smem) {
      const Run b = bucket(0);
      for (u32 i = threadIdx.x; i < b.n; i += NT) {
        b0k_global[0][i] = b.k[i];
        b0p_global[0][i] = b.p[i];
      }
      Bk::sync();
      if (t0()) {
        s.lv[0].bk[0] = b0k_global[0];
        s.lv[0].bk[1] = b0k_global[1];
        s.lv[0].bp[0] = b0p_global[0];
        s.lv[0].bp[1] = b0p_global[1];
        s.st[0].b_sel = 0;
        s.st[0].b_head = 0;
      }
      Bk::sync();
    }
    for (u32 i = threadIdx.x; i < PBH_MAX_LEVELS; i += NT) {
      g->st[i] = s.st[i];
      g->resolves[i] = s.resolves[i];
      g->touches[i] = s.touches[i];
    }
    if (t0()) {
      g->live = s.live;
      g->ops = s.ops;
      g->stale_dropped = s.stale_dropped;
    }
    Bk::sync();
  }

  // ------------------------------------------------------------ push down
  // Merge run X (level i's push list) into S_{i+1}. Without the valve the
  // caller guarantees room.
  template <bool Valve>
  NOINL void push_down(u32 i, Run X) {
    const u32 j = i + 1;
    if (X.n == 0) return;
    if (j >= s.n_levels) {
      fail(PBH_ERR_NEED_GROW, j);
      return;
    }
    if ((u64)s.st[j].s_size + X.n > s.lv[j].buf_s) {
      if constexpr (Valve) {
        make_room(j);
        if (failed()) return;
      }
      if ((u64)s.st[j].s_size + X.n > s.lv[j].buf_s) {
        fail(PBH_ERR_INVARIANT, j);
        return;
      }
    }
    const Run Sj = signal(j);
    const u32 ns = 1 - s.st[j].s_sel;
    const Sink snk{s.lv[j].sk[ns], s.lv[j].sp[ns], kInfCount, nullptr, nullptr};
    const u32 n = mrg(Sj, X, true, snk, 0);
    if (t0()) {
      s.st[j].s_sel = ns;
      s.st[j].s_head = 0;
      s.st[j].s_size = n;
      s.touches[i] += 2ull * (Sj.n + X.n);
    }
    Bk::sync();
  }

  // Phase 1 of resolve(i), i >= 1 (bucket_heap.cpp:196-224): absorb the
  // admitted prefix of S_i into B_i (dropping stale entries), cut B_i at its
  // capacity, and push the overflow plus the non-admitted suffix of S_i
  // down into S_{i+1}.
  template <bool Valve>
  NOINL void phase1(u32 i) {
    const Run Sr = signal(i);
    if (Sr.n == 0) return;
    const Run Br = bucket(i);
    const u32 adm = count_admitted<NT>(Sr, s.st[i], scr());
    const Run Sa{Sr.k, Sr.p, adm};
    const Run Sb{Sr.k + adm, Sr.p + adm, Sr.n - adm};
    const pbh_level_bufs& L = s.lv[i];
    const u32 nb = 1 - s.st[i].b_sel, ns = 1 - s.st[i].s_sel;
    const Sink snk{L.bk[nb], L.bp[nb], L.cap_b, L.sk[ns], L.sp[ns]};
    const u32 n = mrg(Br, Sa, true, snk, 0);
    const u32 keep = n < L.cap_b ? n : L.cap_b;
    const u32 over = n - keep;
    const Sink snk2{L.sk[ns], L.sp[ns], kInfCount, nullptr, nullptr};
    const u32 nr = cpy(Sb, true, snk2, over);
    if (t0()) {
      pbh_level_state& t = s.st[i];
      t.b_sel = nb;
      t.b_head = 0;
      t.b_size = keep;
      if (over > 0) {
        t.spl_inf = 0;
        t.spl_p = L.bp[nb][L.cap_b - 1];
        t.spl_k = L.bk[nb][L.cap_b - 1];
      }
      t.s_sel = ns;
      t.s_head = 0;
      t.s_size = 0;
      s.resolves[i] += 1;
      s.touches[i] += 2ull * (Br.n + Sr.n);
    }
    Bk::sync();
    push_down<Valve>(i, Run{L.sk[ns], L.sp[ns], over + nr});
  }

  // Empty S_m for every m >= j, deepest first, so that S_j has room.
  NOINL void make_room(u32 j) {
    for (int m = (int)s.n_levels - 1; m >= (int)j; --m) {
      if (s.st[m].s_size) phase1<false>((u32)m);
      if (failed()) return;
    }
  }

  // Phase 2 of resolve(i) (bucket_heap.cpp:228-271): refill B_i up to its
  // capacity with the smallest valid entries of level i+1's candidates
  // (B_{i+1} and the admitted prefix of S_{i+1}); both are run heads, so the
  // pull is a merge-path walk that never rewrites level i+1.
  NOINL void refill(u32 i) {
    const u32 j = i + 1;
    if (j >= s.n_levels) return;
    const pbh_level_bufs& L = s.lv[i];
    const u32 cap = i == 0 ? s.cap0 : L.cap_b;
    if (content(j) == 0) {
      if (content_from(j) == 0 && t0()) s.st[i].spl_inf = 1;
      Bk::sync();
      return;
    }
    const Run Bi = bucket(i);
    const u32 nb = 1 - s.st[i].b_sel;
    const Sink dst{L.bk[nb], L.bp[nb], kInfCount, nullptr, nullptr};
    u32 n = cpy(Bi, i > 0, dst, 0);
    const Run Bj = bucket(j);
    const Run Sj = signal(j);
    const u32 adm = count_admitted<NT>(Sj, s.st[j], scr());
    u32 ha = 0, hb = 0;
    u64 last_p = 0;
    u32 last_k = 0;
    while (n < cap && (ha < Bj.n || hb < adm)) {
      const u32 need = cap - n;
      const u32 avail = (Bj.n - ha) + (adm - hb);
      u32 c = need < avail ? need : avail;
      // deep refills pull a whole prefix on the grid (unfiltered); level 0
      // is always refilled here, tile by tile, through the index filter
      const Run A{Bj.k + ha, Bj.p + ha, Bj.n - ha};
      const Run B{Sj.k + hb, Sj.p + hb, adm - hb};
      const bool mem = gs && i > 0 && hbm(A.k) && hbm(B.k) && hbm_sink(dst);
      const bool on_grid = mem && gj && c >= gmin;
      const bool streamed = mem && !on_grid && c >= kStreamMin;
      if (!on_grid && !streamed && c > T) c = T;
      const u32 a = merge_split<NT>(A, B, c, scr());
      // last element of the tile in merged order
      {
        const bool ha_ok = a > 0, hb_ok = c - a > 0;
        u64 pa = ha_ok ? A.p[a - 1] : 0, pb = hb_ok ? B.p[c - a - 1] : 0;
        u32 ka = ha_ok ? A.k[a - 1] : 0, kb = hb_ok ? B.k[c - a - 1] : 0;
        if (!hb_ok || (ha_ok && less_pk(pb, kb, pa, ka))) {
          last_p = pa;
          last_k = ka;
        } else {
          last_p = pb;
          last_k = kb;
        }
      }
      if (on_grid) {
        grid_run<NT>(gj, gsz, 0, A, B, c, dst, n, *gs, gs->scr);
        n += c;
      } else if (streamed) {
        const u32 a_c = a;  // first c outputs = A[0, a) + B[0, c - a)
        stream_local(Run{A.k, A.p, a_c}, Run{B.k, B.p, c - a_c}, dst, n);
        n += c;
      } else {
        n += merge_tile<NT, VT>(A, 0, a, B, 0, c - a, true, idx, dst, n, s.tile, scr());
      }
      ha += a;
      hb += c - a;
    }
    if (t0()) {
      pbh_level_state& ti = s.st[i];
      pbh_level_state& tj = s.st[j];
      ti.b_sel = nb;
      ti.b_head = 0;
      ti.b_size = n;
      tj.b_head += ha;
      tj.b_size -= ha;
      tj.s_head += hb;
      tj.s_size -= hb;
      if (ha == Bj.n && hb == adm) {
        // candidates exhausted: level i now reaches down to level j's bound
        bool deeper = tj.s_size > 0;
        for (u32 m = j + 1; m < s.n_levels; ++m) deeper |= (s.st[m].b_size + s.st[m].s_size) > 0;
        if (!deeper) {
          ti.spl_inf = 1;
          tj.spl_inf = 1;
        } else {
          ti.spl_inf = tj.spl_inf;
          ti.spl_p = tj.spl_p;
          ti.spl_k = tj.spl_k;
        }
      } else {
        ti.spl_inf = 0;
        ti.spl_p = last_p;
        ti.spl_k = last_k;
      }
      s.touches[i] += 2ull * (Bi.n + ha + hb);
    }
    Bk::sync();
  }

  // resolve(i), i >= 1, as scheduled by the 4-to-1 rule.
  NOINL void resolve(u32 i) {
    if (s.st[i].s_size) phase1<true>(i);
    if (failed()) return;
    if (s.st[i].b_size < s.lv[i].cap_b / 2 && content_from(i + 1) > 0) refill(i);
  }

  // After op number s.ops: resolve(i) for each i >= 1 with 4^i | ops
  // (the sequential unrolling of scheduler.cpp:11-20 / engine.cpp:70-88),
  // then top up B_0 if it fell below its floor.
  NOINL void after_op() {
    if (t0()) {
      s.ops += 1;
      s.resolves[0] += 1;
    }
    Bk::sync();
    const u64 n = s.ops;
    for (u32 i = 1; i < s.n_levels && i < 31; ++i) {
      if (n & ((1ull << (2 * i)) - 1)) break;
      resolve(i);
      if (failed()) return;
    }
    if (s.st[0].b_size < s.cap0 / 2 && content_from(1) > 0) refill(0);
  }

  // Make B_0 non-empty while any content remains below (extract path).
  NOINL void fill0() {
    for (u32 iter = 0; iter < (1u << 24); ++iter) {
      if (s.st[0].b_size > 0 || content_from(1) == 0) return;
      refill(0);
      if (failed() || s.st[0].b_size > 0) return;
      u32 m = 1;
      for (; m + 1 < s.n_levels; ++m) {
        if (content_from(m) == 0) break;
        if (s.st[m].s_size) phase1<true>(m);
        if (failed()) return;
        refill(m);
        if (failed()) return;
        if (s.st[m].b_size > 0) break;
      }
      for (int q = (int)m - 1; q >= 0; --q) {
        refill((u32)q);
        if (failed()) return;
      }
    }
    fail(PBH_ERR_INVARIANT, 0xF111);
  }

  // Capacity pre-check: the deepest allocated bucket must be able to hold
  // every stored entry plus `incoming`, so no push can leave the allocation.
  DEV bool room_for(u64 incoming) {
    const u32 L = s.n_levels;
    const u64 cap_last = L == 1 ? s.cap0 : s.lv[L - 1].cap_b;
    if (content_from(0) + incoming > cap_last) {
      fail(PBH_ERR_NEED_GROW, L);
      return false;
    }
    return true;
  }

  // ------------------------------------------------------- level-0 insert
  // Insert the n new entries staged in (bk, bp) (any order) into level 0:
  // drop B_0 copies flagged in rm, sort the batch by (p, k), merge the
  // admitted part into B_0, cut at cap0, push overflow + the rest down.
  NOINL void insert_staged(u32 n, bool any_removed) {
    if (any_removed) {
      const Run b = bucket(0);
      const u32 nb = 1 - s.st[0].b_sel;
      u32* ok = s.lv[0].bk[nb];
      u64* op = s.lv[0].bp[nb];
      u32 written = 0;
      for (u32 t0i = 0; t0i < b.n; t0i += NT) {
        const u32 i = t0i + threadIdx.x;
        bool keep = false;
        u32 kk = 0;
        u64 pv = 0;
        if (i < b.n) {
          keep = rm[i] == 0;
          rm[i] = 0;
          kk = b.k[i];
          pv = b.p[i];
        }
        u32 tot;
        const u32 pos = written + Bk::scan_excl(keep ? 1u : 0u, tot, scr());
        if (keep) {
          ok[pos] = kk;
          op[pos] = pv;
        }
        written += tot;
      }
      if (t0()) {
        s.st[0].b_sel = nb;
        s.st[0].b_head = 0;
        s.st[0].b_size = written;
      }
      Bk::sync();
    }
    if (n == 0) return;
    bitonic_sort<NT>(bk, bp, n);
    const Run N{bk, bp, n};
    const u32 nadm = count_admitted<NT>(N, s.st[0], scr());
    const Run Na{bk, bp, nadm};
    const Run Nb{bk + nadm, bp + nadm, n - nadm};
    const Run B0 = bucket(0);
    const u32 nb = 1 - s.st[0].b_sel;
    const Sink snk{s.lv[0].bk[nb], s.lv[0].bp[nb], s.cap0, pk, pp};
    const u32 tot = mrg(B0, Na, false, snk, 0);
    const u32 keep = tot < s.cap0 ? tot : s.cap0;
    const u32 over = tot - keep;
    const Sink snk2{pk, pp, kInfCount, nullptr, nullptr};
    const u32 nr = cpy(Nb, false, snk2, over);
    if (t0()) {
      pbh_level_state& t = s.st[0];
      t.b_sel = nb;
      t.b_head = 0;
      t.b_size = keep;
      if (over > 0) {
        t.spl_inf = 0;
        t.spl_p = s.lv[0].bp[nb][s.cap0 - 1];
        t.spl_k = s.lv[0].bk[nb][s.cap0 - 1];
      }
      s.touches[0] += 2ull * (B0.n + n);
    }
    Bk::sync();
    push_down<true>(0, Run{pk, pp, over + nr});
  }

  // Position of (p, k) in B_0 (must be present).
  DEV u32 b0_find(u64 p, u32 k) const {
    const Run b = bucket(0);
    u32 lo = 0, hi = b.n;
    while (lo < hi) {
      const u32 m = (lo + hi) >> 1;
      if (less_pk(b.p[m], b.k[m], p, k))
        lo = m + 1;
      else
        hi = m;
    }
    return lo;
  }

  // ------------------------------------------------------------ the ops
  // bulk_update / update (bucket_heap.cpp:101-111,127-146) with the
  // index-based insert-if-absent / decrease-key. vals/prios: any memory.
  // check_batch: apply the bulk preconditions (size, sortedness).
  NOINL void op_bulk(const u32* vals, const u64* prios, u32 n, bool check_batch) {
    if (check_batch) {
      if (n == 0) return fail(PBH_ERR_EMPTY_BATCH);
      if (n > s.d) return fail(PBH_ERR_BATCH_TOO_BIG, n);
    }
    if (!room_for(n)) return;
    // pass 1: validate (no mutation)
    bool bad_sort = false, bad_key = false, bad_dead = false, bad_inc = false;
    for (u32 j = threadIdx.x; j < n; j += NT) {
      const u32 k = vals[j];
      if (check_batch && j > 0 && vals[j - 1] >= k) bad_sort = true;
      if (k >= g->universe) {
        bad_key = true;
        continue;
      }
      const pbh_idx_entry e = idx[k];
      if (PBH_ST(e.state) == PBH_ST_DEAD) bad_dead = true;
      if (s.debug && PBH_ST(e.state) == PBH_ST_LIVE && prios[j] > e.prio) bad_inc = true;
    }
    if (Bk::any(bad_sort, scr())) return fail(PBH_ERR_UNSORTED);
    if (Bk::any(bad_key, scr())) return fail(PBH_ERR_KEY_RANGE);
    if (Bk::any(bad_dead, scr())) return fail(PBH_ERR_REINSERT);
    if (Bk::any(bad_inc, scr())) return fail(PBH_ERR_INCREASE);
    // pass 2: apply to the index, stage new entries, flag B_0 removals
    u32 staged = 0, fresh = 0;
    bool removed = false;
    for (u32 t = 0; t < n; t += NT) {
      const u32 j = t + threadIdx.x;
      bool ins = false;
      u32 k = 0;
      u64 p = 0;
      if (j < n) {
        k = vals[j];
        p = prios[j];
        const pbh_idx_entry e = idx[k];
        if (PBH_ST(e.state) != PBH_ST_LIVE) {
          ins = true;
          fresh++;
          idx[k].prio = p;
          idx[k].state = PBH_ST_LIVE;
        } else if (p < e.prio) {
          ins = true;
          idx[k].prio = p;
          if (admits(s.st[0], e.prio, k)) {
            rm[b0_find(e.prio, k)] = 1;
            removed = true;
          }
        }
      }
      u32 tot;
      const u32 pos = staged + Bk::scan_excl(ins ? 1u : 0u, tot, scr());
      if (ins) {
        bk[pos] = k;
        bp[pos] = p;
      }
      staged += tot;
    }
    const u32 nfresh = Bk::sum(fresh, scr());
    const bool any_rm = Bk::any(removed, scr());
    if (t0()) s.live += nfresh;
    Bk::sync();
    insert_staged(staged, any_rm);
  }

  // extract_min (bucket_heap.cpp:79-99): B_0 is clean, so the minimum is
  // its head. Returns the element through (ok, op) on every thread.
  NOINL bool op_extract(u32& ok, u64& op) {
    if (s.live <= 0) {
      fail(PBH_ERR_EMPTY_HEAP);
      return false;
    }
    fill0();
    if (failed()) return false;
    if (s.st[0].b_size == 0) {
      fail(PBH_ERR_INVARIANT, 0xE0);
      return false;
    }
    const Run b = bucket(0);
    ok = b.k[0];
    op = b.p[0];
    Bk::sync();
    if (t0()) {
      s.st[0].b_head += 1;
      s.st[0].b_size -= 1;
      s.live -= 1;
      idx[ok].state = PBH_ST_DEAD;
    }
    Bk::sync();
    return true;
  }

  // find_min (bucket_heap.cpp:66-77) without removal.
  NOINL bool op_find_min(u32& ok, u64& op) {
    if (s.live <= 0) {
      fail(PBH_ERR_EMPTY_HEAP);
      return false;
    }
    fill0();
    if (failed()) return false;
    if (s.st[0].b_size == 0) {
      fail(PBH_ERR_INVARIANT, 0xE1);
      return false;
    }
    const Run b = bucket(0);
    ok = b.k[0];
    op = b.p[0];
    Bk::sync();
    return true;
  }

  // delete_value (bucket_heap.cpp:113-125): absent values are a no-op.
  NOINL void op_delete(u32 k) {
    if (k >= g->universe) return;
    const pbh_idx_entry e = idx[k];
    Bk::sync();
    if (PBH_ST(e.state) == PBH_ST_LIVE && admits(s.st[0], e.prio, k)) {
      if (t0()) rm[b0_find(e.prio, k)] = 1;
      Bk::sync();
      insert_staged(0, true);
    }
    if (t0()) {
      if (PBH_ST(e.state) == PBH_ST_LIVE) s.live -= 1;
      idx[k].state = PBH_ST_DEAD;
    }
    Bk::sync();
  }

  // SSSP: apply c improving relaxations collected in CSR order (ck: target,
  // cp: candidate, co/cs: index entry read at relax time) from vertex v as
  // one bulk_update (sssp.cpp:59-64): tentative[u] = cand, parent[u] = v.
  NOINL void relax_chunk(const u32* ck, const u64* cp, const u64* co, const u32* cs, u32 c, u32 v) {
    u32 fresh = 0;
    bool removed = false;
    for (u32 j = threadIdx.x; j < c; j += NT) {
      const u32 k = ck[j];
      const u64 p = cp[j], old = co[j];
      const u32 st = cs[j];
      pbh_idx_entry e;
      e.prio = p;
      e.state = PBH_ST_LIVE;
      e.parent = v;
      idx[k] = e;
      if (PBH_ST(st) != PBH_ST_LIVE) {
        fresh++;
      } else if (admits(s.st[0], old, k)) {
        rm[b0_find(old, k)] = 1;
        removed = true;
      }
      bk[j] = k;
      bp[j] = p;
    }
    const u32 nfresh = Bk::sum(fresh, scr());
    const bool any_rm = Bk::any(removed, scr());
    if (t0()) s.live += nfresh;
    Bk::sync();
    insert_staged(c, any_rm);
  }

  // Drain: flush every signal buffer top-down (bucket_heap.cpp:279-300).
  NOINL void drain() {
    for (u32 i = 1; i < s.n_levels; ++i) {
      if (s.st[i].s_size) phase1<true>(i);
      if (failed()) return;
    }
  }
};

}  // namespace pbh_dev
