// Grid-wide merges for the deep levels of one heap (C1 op traces, C4
// bulkUpdate sweeps).
//
// The trace interpreter runs as a cooperative grid: CTA 0 (the leader)
// replays the op stream exactly as before; CTAs 1..G-1 are helpers parked on
// a job word in HBM. A merge whose output exceeds kGridMin elements (a deep
// resolve: push_down into S_{i+1}, the absorb of phase 1, a refill of B_i for
// i >= 1) is posted as a job and executed by all G CTAs: CTA b produces the
// output range [c*b/G, c*(b+1)/G) of the merge, found by one merge-path
// search per range, and streams it through shared memory in tiles of
// kGridTile outputs (window loads of A and B, per-thread merge-path split in
// shared memory, staged coalesced stores). Grid merges do not filter stale
// entries (they would need a scan to compact): stale copies are carried and
// dropped by the filtered CTA-local merges nearer level 0, and never reach
// B_0 (refill(0) always filters). Results are unchanged: (priority, value)
// pairs are unique and a stale copy fails the index check wherever it is
// finally examined.
#pragma once

#include "pbh_engine.cuh"

namespace pbh_dev {

#ifndef PBH_GRID_TILE
// 5 outputs per thread: an odd per-thread stride keeps the merge-path reads
// and the staging writes off the bank conflicts of a stride of 8 four- /
// eight-byte entries (2048 = 8 per thread and 1792 = 7 measured slower on
// C1, C4 d = 32 and d = 1024; 1792 is 3 % faster at d = 65536)
#define PBH_GRID_TILE 1280
#endif
constexpr u32 kGridTile = PBH_GRID_TILE;  // outputs per streamed tile
#ifndef PBH_GRID_MIN_MERGE
#define PBH_GRID_MIN_MERGE 2048
#endif
constexpr u32 kGridMin = PBH_GRID_MIN_MERGE;  // smallest merge worth a grid job (measured sweep 2K..16K: 2K best)
constexpr u32 kStreamMin = 64;    // smallest merge streamed through the windows by one CTA

// Sort n entries (K, P) in shared memory by (p, k) with the whole CTA (K, P,
// TK, TP hold the width n rounded up to a power of two >= 128): the warps
// sort runs of 128 in registers (4 per lane, element r*32 + lane; bitonic
// network, shuffles below stride 32), then merge-path rounds (one search and
// M/NT outputs per thread) double the run width, ping-ponging through
// (TK, TP). Slots n.. of the padded width are (~0, ~0): they sort last.
// Bitonic sort of R independent runs of 128 held in registers (run q / 4,
// element (q % 4) * 32 + lane); the R networks interleave for ILP.
template <int R>
DEV void bitonic128(u64 (&p)[4 * R], u32 (&k)[4 * R], u32 lane) {
#pragma unroll
  for (u32 size = 2; size <= 128; size <<= 1) {
#pragma unroll
    for (u32 stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 32) {
        const u32 rs = stride / 32;
#pragma unroll
        for (u32 q = 0; q < 4 * R; ++q) {
          if ((q & 3) & rs) continue;
          const u32 i = (q & 3) * 32 + lane;  // lower element of the pair
          const bool up = (i & size) == 0;
          const bool gt = less_pk(p[q | rs], k[q | rs], p[q], k[q]);
          if (gt == up) {
            const u64 tp = p[q];
            p[q] = p[q | rs];
            p[q | rs] = tp;
            const u32 tk = k[q];
            k[q] = k[q | rs];
            k[q | rs] = tk;
          }
        }
      } else {
#pragma unroll
        for (u32 q = 0; q < 4 * R; ++q) {
          const u32 i = (q & 3) * 32 + lane;
          const u32 ohi = __shfl_xor_sync(0xffffffffu, (u32)(p[q] >> 32), stride);
          const u32 olo = __shfl_xor_sync(0xffffffffu, (u32)p[q], stride);
          const u32 ok = __shfl_xor_sync(0xffffffffu, k[q], stride);
          const u64 op = ((u64)ohi << 32) | olo;
          const bool up = (i & size) == 0;
          const bool lower = (lane & stride) == 0;
          const bool other_less = less_pk(op, ok, p[q], k[q]);
          if (lower == up ? other_less : !other_less) {
            p[q] = op;
            k[q] = ok;
          }
        }
      }
    }
  }
}

// Runs a, a + step, ... (R of them) of 128: load (padding (~0, ~0)), sort, store.
template <int R>
DEV void sort_runs128(u32* K, u64* P, u32 n, u32 a, u32 step, u32 lane) {
  u64 p[4 * R];
  u32 k[4 * R];
#pragma unroll
  for (u32 q = 0; q < 4 * R; ++q) {
    const u32 i = (a + (q >> 2) * step) * 128 + (q & 3) * 32 + lane;
    p[q] = i < n ? P[i] : ~0ull;
    k[q] = i < n ? K[i] : 0xffffffffu;
  }
  bitonic128<R>(p, k, lane);
#pragma unroll
  for (u32 q = 0; q < 4 * R; ++q) {
    const u32 i = (a + (q >> 2) * step) * 128 + (q & 3) * 32 + lane;
    K[i] = k[q];
    P[i] = p[q];
  }
}

// Sort n entries (K, P) in shared memory by (p, k) with the whole CTA (K, P,
// TK, TP hold the width n rounded up to a power of two >= 128): the warps
// sort runs of 128 in registers (4 per lane, element r*32 + lane; bitonic
// network, shuffles below stride 32), then merge-path rounds double the run
// width, ping-ponging through (TK, TP): one search and an odd number of
// consecutive outputs per thread (an even per-thread stride would put every
// lane's stores in the same shared-memory bank). Slots n.. of the padded
// width are (~0, ~0): they sort last.
template <int NW>
DEV void cta_sort(u32* K, u64* P, u32 n, u32* TK, u64* TP) {
  constexpr u32 NT = 32 * NW;
  const u32 tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  u32 M = 128;
  while (M < n) M <<= 1;
  const u32 nruns = M / 128;
  u32 run = w;
  for (; run < nruns; run += NW) sort_runs128<1>(K, P, n, run, NW, lane);
  __syncthreads();
  u32* sk = K;
  u64* sp = P;
  u32* dk = TK;
  u64* dp = TP;
  for (u32 wr = 128; wr < M; wr <<= 1) {
    // each thread merges one contiguous range of `per` outputs, split at
    // pair boundaries (one merge-path search per piece)
    const u32 per = ((M + NT - 1) / NT) | 1u;
    for (u32 o = tid * per, oend = min(o + per, M); o < oend;) {
      const u32 base = (o / (2 * wr)) * 2 * wr;
      const u32 cnt = min(oend, base + 2 * wr) - o;
      const u32 d = o - base;
      const u32* ak = sk + base;
      const u64* ap = sp + base;
      const u32* bk = sk + base + wr;
      const u64* bp = sp + base + wr;
      u32 lo = d > wr ? d - wr : 0, hi = d < wr ? d : wr;
      while (lo < hi) {
        const u32 m = (lo + hi) >> 1;
        if (less_pk(ap[m], ak[m], bp[d - 1 - m], bk[d - 1 - m]))
          lo = m + 1;
        else
          hi = m;
      }
      u32 x = lo, y = d - lo;
      u64 xa = x < wr ? ap[x] : ~0ull, yb = y < wr ? bp[y] : ~0ull;
      u32 xk = x < wr ? ak[x] : 0xffffffffu, yk = y < wr ? bk[y] : 0xffffffffu;
      // branch-free: take the smaller head, reload only the side that advanced
      // (an exhausted side's head is (~0, ~0) and loses every comparison
      // against a real entry; padding entries are themselves (~0, ~0))
      for (u32 v = 0; v < cnt; ++v) {
        const bool ta = y >= wr || (x < wr && less_pk(xa, xk, yb, yk));
        dk[o + v] = ta ? xk : yk;
        dp[o + v] = ta ? xa : yb;
        x += ta;
        y += !ta;
        const u32 i = ta ? x : y;
        const bool in = i < wr;
        const u64 np = in ? (ta ? ap : bp)[i] : ~0ull;
        const u32 nk = in ? (ta ? ak : bk)[i] : 0xffffffffu;
        xa = ta ? np : xa;
        xk = ta ? nk : xk;
        yb = ta ? yb : np;
        yk = ta ? yk : nk;
      }
      o += cnt;
    }
    __syncthreads();
    u32* t1 = sk;
    sk = dk;
    dk = t1;
    u64* t2 = sp;
    sp = dp;
    dp = t2;
  }
  if (sk != K) {
    for (u32 i = tid; i < n; i += NT) {
      K[i] = sk[i];
      P[i] = sp[i];
    }
    __syncthreads();
  }
}

// Job word + descriptor in HBM (one per heap handle).
struct BatchJob;
struct GridJob {
  u32 seq;   // bumped by the leader to publish a job
  u32 done;  // helpers that finished the current job
  u32 kind;  // 0 = merge, 1 = exit, 2 = validate batch, 3 = classify batch,
             // 4 = sort chunks, 5 = merge pass, 6 = validate + classify (no
             // mutation), 7 = bucket sort of the staged run (BatchJob in `ext`),
             // 8 = merge dropping stale entries (compacting; count in ext),
             // 9 = merge an unsorted run into a sorted one (push-buffer flush)
  u32 nblk;  // CTAs in the grid (leader included)
  const u32* ak;
  const u64* ap;
  const u32* bk;
  const u64* bp;
  u32 na, nb;  // run lengths
  u32 c;       // outputs: the first c of merge(A, B)
  u32 out_base;
  Sink sink;
  BatchJob* ext;
  const pbh_idx_entry* idx;  // stale filter (kind 8, filtered streams): valid iff LIVE at this priority
  u32 filter;
  u32 bar_cnt;     // job-barrier arrivals of the current launch (zeroed with the job word)
  GridJob* self;   // this descriptor in HBM (for bar_cnt)
};

// A large bulk_update batch handled by the whole grid (kinds 2-5). The leader
// fills the fields and zeroes the counters before posting.
constexpr u32 kSortChunk = 2048;  // elements per CTA-sorted chunk
constexpr u32 kBigBatch = 8192;   // batches at least this large go to the grid
constexpr u32 kMaxBatch = 1u << 26;  // largest batch (size of the grid path's staging buffers)
#ifndef PBH_POLL_MAX_NS
#define PBH_POLL_MAX_NS 64
#endif
constexpr u32 kPollMaxNs = PBH_POLL_MAX_NS;  // job-word polling backoff cap
struct BatchJob {
  const u32* vals;
  const u64* prios;
  pbh_idx_entry* idx;
  u64 universe;
  u64 spl_p;
  u32 spl_k, spl_inf;
  u32 n, check, debug, c0;
  // kind 3 outputs: entries for HBM (stg, (p, k) unsorted) and the batch
  // positions the leader applies itself (level-0 slots or admitted)
  u32* stg_k;
  u64* stg_p;
  u32* ll;
  // kinds 4/5: sort src -> dst (run width `width` for kind 5)
  u32* sk[2];
  u64* sp[2];
  u32 sort_n, width, src;
  u32 write_idx;  // kind 4: also publish the chunk's index entries
  // counters (atomics)
  u32 stg_n, ll_n, fresh, errs;
  // kind 6: priority range of the staged elements; kind 7: buckets
  u64 pmin, pmax, bwidth;
  u32* bcnt;      // per-bucket element counts (kBucketMax)
  u32 nbkt, bovf; // bucket count; set when a bucket exceeds kGridTile
  u32 merge_total;  // kind 8: entries written
  // kind 9: the unsorted run sk/sp[0][0, stg_n) merged with the sorted run
  // (mk, mp)[0, mn) into (ok, op)
  const u32* mk;
  const u64* mp;
  u32 mn, pad9_;
  u32* ok;
  u64* op;
};
constexpr u32 kBucketMax = 1184;  // 8 buckets per CTA of a 148-CTA grid
constexpr u32 kRankSortMax = 192;  // buckets up to this size: rank sort (measured vs cta_sort)
#ifndef PBH_BULK_STORE_MIN
#define PBH_BULK_STORE_MIN 1024
#endif
constexpr u32 kBulkStoreMin = PBH_BULK_STORE_MIN;  // merge tiles at least this large leave by bulk stores

template <int NT>
struct GridSmem {
  GridJob sub;  // one piece of a merge pass
  // merge windows (TMA destinations: 16-byte aligned, room for the
  // alignment offset of a window start) and the output tile
  alignas(16) u32 ak[kGridTile + 4];
  alignas(16) u32 bk[kGridTile + 4];
  alignas(16) u32 ok[kGridTile + 4];
  alignas(16) u64 ap[kGridTile + 2];
  alignas(16) u64 bp[kGridTile + 2];
  alignas(16) u64 op[kGridTile + 2];
  GridJob job;  // the current job, copied in by thread 0
  u64 mbar;     // window-load barrier (one phase per tile)
  u32 mph;      // its next phase parity
  u32 ta;       // A elements consumed by the current tile
  u32 seq;
  u32 bar_epoch;  // job barriers passed by this CTA in this launch
  u32 scr[NT / 32 + 2];  // scan scratch of the merge-path searches
};

// Once per CTA per launch, before any grid job or streamed merge.
template <int NT>
DEV void grid_smem_init(GridSmem<NT>& g) {
  if (threadIdx.x == 0) {
    g.seq = 0;
    g.mph = 0;
    g.bar_epoch = 0;
    mbar_init(&g.mbar, 1);
  }
  __syncthreads();
}

DEV u32 ld_acquire(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
DEV void st_release(u32* p, u32 v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// PBH_PROF diagnostics of the grid jobs (leader CTA, thread 0): cycles and
// count per job kind [0, 8), and per phase of the bucket sort [8, 12).
__device__ unsigned long long g_jobprof[24][2];
__device__ unsigned int g_jobprof_on;
DEV void jobprof_add(u32 slot, long long cycles) {
  if (g_jobprof_on && threadIdx.x == 0 && blockIdx.x == 0) {
    g_jobprof[slot][0] += (unsigned long long)cycles;
    g_jobprof[slot][1] += 1;
  }
}

// Stream the merge of A[ia, ia_end) and B[ib, ib_end) (no filter) into
// sink[out ...). Every thread of the CTA calls this. Per tile of kGridTile
// outputs: the four input windows arrive by 1-D TMA bulk copies (16-byte
// aligned windows, one mbarrier), each thread merges its merge-path slice
// from shared memory into the output tile, and the tile is stored
// coalesced.
template <int NT>
DEV u32 grid_stream(const GridJob& J, u32 ia, u32 ia_end, u32 ib, u32 ib_end, u32 out,
                    GridSmem<NT>& g) {
  using Bk = Blk<NT>;
  constexpr u32 VT = kGridTile / NT;
  const u32 tid = threadIdx.x;
  const bool filter = J.filter != 0;
  u32 ph = g.mph;
  u32 written = 0;
  u32 na = 0, nb = 0, n = 0;
  bool bulk_pending = false;  // this CTA's bulk stores may still read the staging tile
  Window<4> wak, wbk;
  Window<8> wap, wbp;
  // the next tile's windows, and their TMA loads (thread 0, one mbarrier)
  auto plan = [&]() {
    na = min(kGridTile, ia_end - ia);
    nb = min(kGridTile, ib_end - ib);
    n = min(kGridTile, (ia_end - ia) + (ib_end - ib));
    wak = Window<4>(J.ak, ia, na);
    wbk = Window<4>(J.bk, ib, nb);
    wap = Window<8>(J.ap, ia, na);
    wbp = Window<8>(J.bp, ib, nb);
    if (tid == 0) {
      fence_proxy_async_smem();
      mbar_expect_tx(&g.mbar, (na ? wak.bytes + wap.bytes : 0u) + (nb ? wbk.bytes + wbp.bytes : 0u));
      if (na) {
        tma_load_1d(g.ak, wak.src, wak.bytes, &g.mbar);
        tma_load_1d(g.ap, wap.src, wap.bytes, &g.mbar);
      }
      if (nb) {
        tma_load_1d(g.bk, wbk.src, wbk.bytes, &g.mbar);
        tma_load_1d(g.bp, wbp.src, wbp.bytes, &g.mbar);
      }
    }
  };
  bool more = ia < ia_end || ib < ib_end;
  if (more) plan();
  long long tw = clock64();
  while (more) {
    mbar_wait(&g.mbar, ph);
    ph ^= 1u;
    jobprof_add(18, clock64() - tw);
    tw = clock64();
    const u32* AK = g.ak + wak.off;
    const u64* AP = g.ap + wap.off;
    const u32* BK = g.bk + wbk.off;
    const u64* BP = g.bp + wbp.off;
    // this thread's outputs [d0, d1): merge-path split inside the windows
    const u32 d0 = min(tid * VT, n), d1 = min(d0 + VT, n);
    u32 lo = d0 > nb ? d0 - nb : 0, hi = min(d0, na);
    while (lo < hi) {
      const u32 m = (lo + hi) >> 1;
      if (less_pk(AP[m], AK[m], BP[d0 - 1 - m], BK[d0 - 1 - m]))
        lo = m + 1;
      else
        hi = m;
    }
    u32 x = lo, y = d0 - lo;
    u32 rk[VT];
    u64 rp[VT];
#pragma unroll
    for (u32 v = 0; v < VT; ++v) {
      rk[v] = 0xffffffffu;
      rp[v] = ~0ull;
      if (d0 + v < d1) {
        const bool takeA = x < na && (y >= nb || less_pk(AP[x], AK[x], BP[y], BK[y]));
        rk[v] = takeA ? AK[x] : BK[y];
        rp[v] = takeA ? AP[x] : BP[y];
        x += takeA;
        y += !takeA;
      }
    }
    if (d0 < d1 && d1 == n) g.ta = x;
    // where this tile's outputs land: one destination run (bulk-stored from
    // a staging tile shifted to the destination's 16-byte phase) unless the
    // tile straddles the sink's split point (element stores)
    const u32 base = filter ? out + written : out;
    // (small tiles: element stores; the bulk path's wait and barrier cost
    // more than it saves below ~1024 entries, measured on C1 / C4 d=1024)
    u32* dk = nullptr;
    u64* dp = nullptr;
    if (n >= kBulkStoreMin) {
      if (base + n <= J.sink.lim) {
        dk = J.sink.k1 + base;
        dp = J.sink.p1 + base;
      } else if (base >= J.sink.lim) {
        dk = J.sink.k2 + (base - J.sink.lim);
        dp = J.sink.p2 + (base - J.sink.lim);
      }
    }
    const u32 shk = dk ? (u32)((reinterpret_cast<uintptr_t>(dk) >> 2) & 3u) : 0u;
    const u32 shp = dp ? (u32)((reinterpret_cast<uintptr_t>(dp) >> 3) & 1u) : 0u;
    if (bulk_pending) {  // the previous tile's bulk stores must have left the staging tile
      if (tid == 0) bulk_wait_read();
      Bk::sync();
      bulk_pending = false;
    }
    u32 cnt = n;
    if (!filter) {
#pragma unroll
      for (u32 v = 0; v < VT; ++v)
        if (d0 + v < d1) {
          g.ok[shk + d0 + v] = rk[v];
          g.op[shp + d0 + v] = rp[v];
        }
    } else {
      // drop stale entries (primitives.cpp:103-120 semantics through the
      // position index): the survivors keep their merged order, compacted
      // by a CTA scan into the staging tile
      u32 keepm = 0;
#pragma unroll
      for (u32 v = 0; v < VT; ++v)
        if (d0 + v < d1 && entry_valid(J.idx, rk[v], rp[v])) keepm |= 1u << v;
      u32 pos = Bk::scan_excl(__popc(keepm), cnt, g.scr);
#pragma unroll
      for (u32 v = 0; v < VT; ++v)
        if (keepm >> v & 1u) {
          g.ok[shk + pos] = rk[v];
          g.op[shp + pos] = rp[v];
          ++pos;
        }
    }
    fence_proxy_async_smem();  // window reads and staging writes vs. the async proxy
    Bk::sync();
    jobprof_add(19, clock64() - tw);
    tw = clock64();
    // advance, and start the next tile's loads before storing this one
    const u32 ta = g.ta;
    ia += ta;
    ib += n - ta;
    if (!filter) out += n;
    more = ia < ia_end || ib < ib_end;
    if (more) plan();
    if (dk) {
      // aligned middles by two bulk stores (thread 0), the unaligned head
      // and tail entries by threads
      const u32 k0 = (shk + 3u) & ~3u, k1 = (shk + cnt) & ~3u;  // staging indices
      const u32 p0 = (shp + 1u) & ~1u, p1 = (shp + cnt) & ~1u;
      const bool kb = k1 > k0, pb = p1 > p0;
      if (tid == 0) {
        if (kb) tma_store_1d(dk + (k0 - shk), g.ok + k0, (k1 - k0) * 4);
        if (pb) tma_store_1d(dp + (p0 - shp), g.op + p0, (p1 - p0) * 8);
        if (kb || pb) bulk_commit();
      }
      bulk_pending = kb || pb;
      if (kb && pb) {
        // at most 3 + 3 key and 1 + 1 priority entries outside the middles
        if (tid < 3) {
          const u32 h = tid, t = k1 - shk + tid;  // head / tail output index
          if (h < min(cnt, k0 - shk)) dk[h] = g.ok[shk + h];
          if (t < cnt) dk[t] = g.ok[shk + t];
        } else if (tid == (NT > 32 ? 32u : 3u)) {
          if (shp < p0 && cnt) dp[0] = g.op[shp];
          if (p1 - shp < cnt) dp[cnt - 1] = g.op[shp + cnt - 1];
        }
      } else {
        for (u32 i = tid; i < cnt; i += NT) {
          const u32 sk = shk + i, sp = shp + i;
          if (!kb || sk < k0 || sk >= k1) dk[i] = g.ok[sk];
          if (!pb || sp < p0 || sp >= p1) dp[i] = g.op[sp];
        }
      }
    } else {
      for (u32 i = tid; i < cnt; i += NT) J.sink.put(base + i, g.ok[i], g.op[i]);
    }
    written += cnt;
    jobprof_add(20, clock64() - tw);
    tw = clock64();
  }
  if (tid == 0) {
    bulk_wait_all();  // the bulk stores' writes are complete before the job ends
    g.mph = ph;
  }
  Bk::sync();
  return written;
}

// Valid entries (index check) in (k, p)[i0, i1): CTA-wide count.
template <int NT>
DEV u32 count_valid(const u32* k, const u64* p, u32 i0, u32 i1, const pbh_idx_entry* idx, u32* scr) {
  u32 c = 0;
  for (u32 i = i0 + threadIdx.x; i < i1; i += NT) c += entry_valid(idx, k[i], p[i]);
  return Blk<NT>::sum(c, scr);
}

// Warp-aggregated append to a global counter: returns this lane's slot.
DEV u32 warp_append(u32* ctr, bool want) {
  const u32 m = __ballot_sync(0xffffffffu, want);
  if (!m) return 0;
  const u32 lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  u32 base = 0;
  if (lane == leader) base = atomicAdd(ctr, (u32)__popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  return base + __popc(m & ((1u << lane) - 1));
}

// kind 2: validate this CTA's slice of the batch (bucket_heap.cpp:127-136
// preconditions): bit 0 unsorted, 1 key range, 2 dead value, 3 increase.
template <int NT>
DEV void batch_validate(BatchJob* X, u32 b, u32 G) {
  const u32 n = X->n;
  const u32 r0 = (u32)((u64)n * b / G), r1 = (u32)((u64)n * (b + 1) / G);
  u32 bad = 0;
  for (u32 j = r0 + threadIdx.x; j < r1; j += NT) {
    const u32 k = X->vals[j];
    if (X->check && j > 0 && X->vals[j - 1] >= k) bad |= 1;
    if (k >= X->universe) {
      bad |= 2;
      continue;
    }
    const ulonglong2 e = __ldcg(reinterpret_cast<const ulonglong2*>(X->idx + k));
    if (PBH_ST((u32)e.y) == PBH_ST_DEAD) bad |= 4;
    if (X->debug && PBH_ST((u32)e.y) == PBH_ST_LIVE && X->prios[j] > e.x) bad |= 8;
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicOr(&X->errs, bad);
}

// kind 3: classify this CTA's slice. An improving element whose valid copy
// is in a level-0 slot, or that splitter_0 admits, is listed for the leader
// (it needs the shared-memory banks); any other goes straight to HBM: its
// index entry becomes {p, LIVE, deep} and (k, p) is appended to the staging
// run that will be sorted and pushed into S_1.
template <int NT>
DEV void batch_classify(BatchJob* X, u32 b, u32 G) {
  const u32 n = X->n;
  const u32 r0 = (u32)((u64)n * b / G), r1 = (u32)((u64)n * (b + 1) / G);
  u32 fresh = 0;
  for (u32 j0 = r0; j0 < r1; j0 += NT) {
    const u32 j = j0 + threadIdx.x;
    bool to_leader = false, to_hbm = false;
    u32 k = 0;
    u64 p = 0;
    if (j < r1) {
      k = X->vals[j];
      p = X->prios[j];
      const ulonglong2 e = __ldcg(reinterpret_cast<const ulonglong2*>(X->idx + k));
      const u32 st = (u32)e.y;
      const bool fr = PBH_ST(st) != PBH_ST_LIVE;
      if (fr || p < e.x) {
        const bool adm = X->spl_inf || p < X->spl_p || (p == X->spl_p && k <= X->spl_k);
        if ((!fr && (st >> 2) < X->c0) || adm) {
          to_leader = true;
        } else {
          to_hbm = true;
          fresh += fr;
          pbh_idx_entry ne;
          ne.prio = p;
          ne.state = PBH_ST_LIVE | (PBH_LOC_DEEP << 2);
          ne.parent = 0;
          reinterpret_cast<ulonglong2*>(X->idx)[k] = *reinterpret_cast<const ulonglong2*>(&ne);
        }
      }
    }
    const u32 ls = warp_append(&X->ll_n, to_leader);
    if (to_leader) X->ll[ls] = j;
    const u32 hs = warp_append(&X->stg_n, to_hbm);
    if (to_hbm) {
      X->stg_k[hs] = k;
      X->stg_p[hs] = p;
    }
  }
  fresh = __reduce_add_sync(0xffffffffu, fresh);
  if ((threadIdx.x & 31) == 0 && fresh) atomicAdd(&X->fresh, fresh);
}

// kind 4: sort chunks of kSortChunk of sk/sp[src] in place (CTA-wide sort in
// the GridSmem windows).
template <int NT>
DEV void batch_sort_chunks(BatchJob* X, u32 b, u32 G, GridSmem<NT>& g) {
  const u32 n = X->sort_n;
  u32* K = X->sk[X->src];
  u64* P = X->sp[X->src];
  for (u32 c0 = b * kSortChunk; c0 < n; c0 += G * kSortChunk) {
    const u32 m = min(kSortChunk, n - c0);
    for (u32 i = threadIdx.x; i < m; i += NT) {
      cp_async4(&g.ak[i], K + c0 + i, true);
      cp_async8(&g.ap[i], P + c0 + i);
    }
    cp_async_commit();
    cp_async_wait_all();
    Blk<NT>::sync();
    if (X->write_idx) {
      for (u32 i = threadIdx.x; i < m; i += NT) {
        pbh_idx_entry ne;
        ne.prio = g.ap[i];
        ne.state = PBH_ST_LIVE | (PBH_LOC_DEEP << 2);
        ne.parent = 0;
        reinterpret_cast<ulonglong2*>(X->idx)[g.ak[i]] = *reinterpret_cast<const ulonglong2*>(&ne);
      }
    }
    cta_sort<NT / 32>(g.ak, g.ap, m, g.bk, g.bp);
    for (u32 i = threadIdx.x; i < m; i += NT) {
      K[c0 + i] = g.ak[i];
      P[c0 + i] = g.ap[i];
    }
    Blk<NT>::sync();
  }
}

// kind 5: one merge pass over runs of `width` (src -> dst): this CTA's output
// range, cut at pair boundaries, each piece one merge-path stream.
template <int NT>
DEV void batch_merge_pass(BatchJob* X, u32 b, u32 G, GridSmem<NT>& g, u32* scratch) {
  const u32 n = X->sort_n, w = X->width;
  const u32 r0 = (u32)((u64)n * b / G), r1 = (u32)((u64)n * (b + 1) / G);
  const u32 s = X->src;
  u32 lo = r0;
  while (lo < r1) {
    const u32 base = lo / (2 * w) * (2 * w);
    const u32 hi = min(r1, base + 2 * w);
    const u32 na = min(w, n - base), nb = base + w < n ? min(w, n - base - w) : 0;
    const Run A{X->sk[s] + base, X->sp[s] + base, na};
    const Run B{X->sk[s] + base + na, X->sp[s] + base + na, nb};
    const u32 d0 = lo - base, d1 = hi - base;
    u32 a0, a1;
    merge_split2<NT>(A, B, d0, d1, scratch, a0, a1);
    if (threadIdx.x == 0) {
      g.sub.ak = A.k;
      g.sub.ap = A.p;
      g.sub.bk = B.k;
      g.sub.bp = B.p;
      g.sub.sink = Sink{X->sk[s ^ 1] + base, X->sp[s ^ 1] + base, 0xffffffffu, nullptr, nullptr};
      g.sub.filter = 0;
    }
    Blk<NT>::sync();
    grid_stream<NT>(g.sub, a0, a1, d0 - a0, d1 - a1, d0, g);
    Blk<NT>::sync();
    lo = hi;
  }
}

// Barrier over the G CTAs of a job (all co-resident: cooperative launch).
// One monotone arrival counter per launch (zeroed by the host before the
// launch): barrier e of the launch completes when the counter reaches
// (e + 1) * G; every CTA passes the same barriers, so each tracks e locally.
// Arrival is a fire-and-forget release reduction; waiting is an acquire poll.
template <int NT>
DEV void job_barrier(BatchJob* X, u32 G, GridSmem<NT>& g) {
  (void)X;
  Blk<NT>::sync();
  if (threadIdx.x == 0) {
    u32* cnt = &g.job.self->bar_cnt;
    const u32 target = (g.bar_epoch + 1) * G;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(cnt) : "memory");
    u32 backoff = 8;
    while ((int)(ld_acquire(cnt) - target) < 0) {
      __nanosleep(backoff);
      backoff = backoff < kPollMaxNs ? backoff * 2 : kPollMaxNs;
    }
    g.bar_epoch += 1;
  }
  Blk<NT>::sync();
}

// kind 6: validate this CTA's slice (bucket_heap.cpp:127-136 preconditions:
// bit 0 unsorted, 1 key range, 2 dead value, 3 increase) and classify it in
// the same pass, without mutating anything: an improving element whose
// valid copy is in a level-0 slot, or that splitter_0 admits, is listed for
// the leader; any other is appended to the HBM staging run (its index entry
// is published by the sort job, once the whole batch is known to be valid).
// The staged priorities' range feeds the bucket sort.
template <int NT>
DEV void batch_check_classify(BatchJob* X, u32 b, u32 G, GridSmem<NT>& g) {
  // the descriptor in registers (stores below could alias it for the compiler)
  const u32 n = X->n, c0 = X->c0, spl_k = X->spl_k;
  const bool check = X->check, debug = X->debug, spl_inf = X->spl_inf;
  const u64 universe = X->universe, spl_p = X->spl_p;
  const u32* __restrict__ vals = X->vals;
  const u64* __restrict__ prios = X->prios;
  const pbh_idx_entry* idx = X->idx;
  u32* ll = X->ll;
  u32* stg_k = X->stg_k;
  u64* stg_p = X->stg_p;
  const u32 r0 = (u32)((u64)n * b / G), r1 = (u32)((u64)n * (b + 1) / G);
  u32 fresh = 0, bad = 0;
  u64 lo = ~0ull, hi = 0;
  // two elements per thread per step: both elements' key loads, then both
  // index gathers are in flight together (one dependent HBM round trip pair
  // per step instead of per element)
  constexpr u32 R = 2;
  for (u32 j0 = r0; j0 < r1; j0 += R * NT) {
    u32 k[R], kp[R];
    u64 p[R];
    ulonglong2 e[R];
#pragma unroll
    for (u32 t = 0; t < R; ++t) {
      const u32 j = j0 + t * NT + threadIdx.x;
      k[t] = j < r1 ? vals[j] : 0;
      p[t] = j < r1 ? prios[j] : 0;
      kp[t] = check && j < r1 && j > 0 ? vals[j - 1] : 0;
    }
#pragma unroll
    for (u32 t = 0; t < R; ++t) {
      const u32 j = j0 + t * NT + threadIdx.x;
      e[t] = j < r1 && k[t] < universe ? __ldcg(reinterpret_cast<const ulonglong2*>(idx + k[t]))
                                       : make_ulonglong2(0, 0);
    }
    bool to_leader[R], to_hbm[R];
    u32 cnt = 0;
#pragma unroll
    for (u32 t = 0; t < R; ++t) {
      const u32 j = j0 + t * NT + threadIdx.x;
      to_leader[t] = to_hbm[t] = false;
      if (j >= r1) continue;
      if (check && j > 0 && kp[t] >= k[t]) bad |= 1;
      if (k[t] >= universe) {
        bad |= 2;
        continue;
      }
      const u32 st = (u32)e[t].y;
      if (PBH_ST(st) == PBH_ST_DEAD) bad |= 4;
      if (debug && PBH_ST(st) == PBH_ST_LIVE && p[t] > e[t].x) bad |= 8;
      const bool fr = PBH_ST(st) != PBH_ST_LIVE;
      if (fr || p[t] < e[t].x) {
        const bool adm = spl_inf || p[t] < spl_p || (p[t] == spl_p && k[t] <= spl_k);
        if ((!fr && (st >> 2) < c0) || adm) {
          to_leader[t] = true;
          cnt += 1;
        } else {
          to_hbm[t] = true;
          cnt += 1u << 16;
          fresh += fr;
          lo = min(lo, p[t]);
          hi = max(hi, p[t]);
        }
      }
    }
    // one reservation per CTA and counter per step (a contended global
    // counter per warp costs more than the CTA scan): leader-list count in
    // the low 16 bits, staging count in the high 16 bits
    u32 tot;
    u32 mine = Blk<NT>::scan_excl(cnt, tot, g.scr);
    if (threadIdx.x == 0) {
      g.ok[0] = (tot & 0xffffu) ? atomicAdd(&X->ll_n, tot & 0xffffu) : 0u;
      g.ok[1] = (tot >> 16) ? atomicAdd(&X->stg_n, tot >> 16) : 0u;
    }
    Blk<NT>::sync();
    u32 ml = g.ok[0] + (mine & 0xffffu), mh = g.ok[1] + (mine >> 16);
#pragma unroll
    for (u32 t = 0; t < R; ++t) {
      const u32 j = j0 + t * NT + threadIdx.x;
      if (to_leader[t]) ll[ml++] = j;
      if (to_hbm[t]) {
        stg_k[mh] = k[t];
        stg_p[mh] = p[t];
        ++mh;
      }
    }
    Blk<NT>::sync();
  }
  fresh = __reduce_add_sync(0xffffffffu, fresh);
  bad = __reduce_or_sync(0xffffffffu, bad);
  for (int s = 16; s; s >>= 1) {
    lo = min(lo, (u64)__shfl_xor_sync(0xffffffffu, (unsigned long long)lo, s));
    hi = max(hi, (u64)__shfl_xor_sync(0xffffffffu, (unsigned long long)hi, s));
  }
  if ((threadIdx.x & 31) == 0) {
    if (fresh) atomicAdd(&X->fresh, fresh);
    if (bad) atomicOr(&X->errs, bad);
    if (lo <= hi) {
      atomicMin(reinterpret_cast<unsigned long long*>(&X->pmin), (unsigned long long)lo);
      atomicMax(reinterpret_cast<unsigned long long*>(&X->pmax), (unsigned long long)hi);
    }
  }
}

// kind 7: sort the staged run (stg_n entries, sk/sp[0]) into sk/sp[1] by
// (p, k) in one job: buckets are equal-width priority ranges (so bucket
// order is priority order); (1) per-CTA histograms of its slice, bucket
// bases by global atomics; (2) after a grid barrier, every CTA scans the
// bucket totals and scatters its slice into the buckets, publishing each
// element's index entry {p, LIVE, deep} when write_idx (a staged batch; a
// push-buffer flush keeps the index as it is); (3) after a second barrier, CTA b
// sorts buckets b, b + G, ... in shared memory. A bucket above kGridTile
// entries sets `bovf` (the leader then sorts sk/sp[1] by merge passes).
template <int NT>
DEV void batch_bucket_sort(BatchJob* X, u32 b, u32 G, GridSmem<NT>& g) {
  using Bk = Blk<NT>;
  const u32 n = X->stg_n, NB = X->nbkt;
  const u64 pmin = X->pmin, width = X->bwidth;
  const u32 r0 = (u32)((u64)n * b / G), r1 = (u32)((u64)n * (b + 1) / G);
  long long tp = clock64();
  u32* cnt = reinterpret_cast<u32*>(g.op);  // NB per-CTA counts, then cursors
  u32* base = cnt + kBucketMax;              // NB bases (this CTA's offset in a bucket)
  u32* start = base + kBucketMax;            // NB bucket starts
  for (u32 i = threadIdx.x; i < NB; i += NT) cnt[i] = 0;
  Bk::sync();
  const u32* SK = X->sk[0];
  const u64* SP = X->sp[0];
  for (u32 j = r0 + threadIdx.x; j < r1; j += NT)
    atomicAdd(&cnt[min(NB - 1, (u32)((SP[j] - pmin) / width))], 1u);
  Bk::sync();
  for (u32 i = threadIdx.x; i < NB; i += NT) {
    const u32 c = cnt[i];
    base[i] = c ? atomicAdd(&X->bcnt[i], c) : 0;
    cnt[i] = 0;  // becomes the scatter cursor
  }
  if (b == 0) { jobprof_add(8, clock64() - tp); tp = clock64(); }
  job_barrier<NT>(X, G, g);
  if (b == 0) { jobprof_add(9, clock64() - tp); tp = clock64(); }
  // bucket starts: exclusive scan of the totals (every CTA, NB <= kBucketMax)
  {
    u32 run = 0;
    for (u32 i0 = 0; i0 < NB; i0 += NT) {
      const u32 i = i0 + threadIdx.x;
      const u32 v = i < NB ? __ldcg(&X->bcnt[i]) : 0;
      u32 tot;
      const u32 e = run + Bk::scan_excl(v, tot, g.scr);
      if (i < NB) start[i] = e;
      run += tot;
    }
  }
  Bk::sync();
  // output: the sorted-run buffer, or (ok, op) when the caller gave one
  u32* DK = X->ok ? X->ok : X->sk[1];
  u64* DP = X->ok ? X->op : X->sp[1];
  const bool write_idx = X->write_idx;
  pbh_idx_entry* idx = X->idx;
  for (u32 j = r0 + threadIdx.x; j < r1; j += NT) {
    const u32 k = SK[j];
    const u64 p = SP[j];
    const u32 q = min(NB - 1, (u32)((p - pmin) / width));
    const u32 pos = start[q] + base[q] + atomicAdd(&cnt[q], 1u);
    DK[pos] = k;
    DP[pos] = p;
    if (write_idx) {
      pbh_idx_entry ne;
      ne.prio = p;
      ne.state = PBH_ST_LIVE | (PBH_LOC_DEEP << 2);
      ne.parent = 0;
      reinterpret_cast<ulonglong2*>(idx)[k] = *reinterpret_cast<const ulonglong2*>(&ne);
    }
  }
  if (b == 0) { jobprof_add(10, clock64() - tp); tp = clock64(); }
  job_barrier<NT>(X, G, g);
  if (b == 0) { jobprof_add(11, clock64() - tp); tp = clock64(); }
  for (u32 q = b; q < NB; q += G) {
    const u32 m = __ldcg(&X->bcnt[q]), s0 = start[q];
    if (m > kGridTile) {
      if (threadIdx.x == 0) atomicOr(&X->bovf, 1u);
      continue;
    }
    if (m < 2) continue;
    if (m <= kRankSortMax) {
      // small bucket: rank sort ((p, k) pairs are unique: a key's copies
      // have distinct priorities), each thread ranks up to two entries
      // against the bucket in shared memory and stores them in place
      u32 k0 = 0, k1 = 0;
      u64 p0 = 0, p1 = 0;
      const u32 i0 = threadIdx.x, i1 = threadIdx.x + NT;
      if (i0 < m) {
        k0 = DK[s0 + i0];
        p0 = DP[s0 + i0];
        g.ak[i0] = k0;
        g.ap[i0] = p0;
      }
      if (i1 < m) {
        k1 = DK[s0 + i1];
        p1 = DP[s0 + i1];
        g.ak[i1] = k1;
        g.ap[i1] = p1;
      }
      Bk::sync();
      u32 r0 = 0, r1 = 0;
      for (u32 j = 0; j < m; ++j) {
        const u64 pj = g.ap[j];
        const u32 kj = g.ak[j];
        r0 += less_pk(pj, kj, p0, k0);
        r1 += less_pk(pj, kj, p1, k1);
      }
      if (i0 < m) {
        DK[s0 + r0] = k0;
        DP[s0 + r0] = p0;
      }
      if (i1 < m) {
        DK[s0 + r1] = k1;
        DP[s0 + r1] = p1;
      }
      Bk::sync();
      continue;
    }
    for (u32 i = threadIdx.x; i < m; i += NT) {
      cp_async4(&g.ak[i], DK + s0 + i, true);
      cp_async8(&g.ap[i], DP + s0 + i);
    }
    cp_async_commit();
    cp_async_wait_all();
    Bk::sync();
    cta_sort<NT / 32>(g.ak, g.ap, m, g.bk, g.bp);
    for (u32 i = threadIdx.x; i < m; i += NT) {
      DK[s0 + i] = g.ak[i];
      DP[s0 + i] = g.ap[i];
    }
    Bk::sync();
  }
  if (b == 0) jobprof_add(12, clock64() - tp);
}

// Sort m entries (DK, DP)[s0, s0 + m) in place in the CTA: rank sort for
// small runs ((p, k) pairs are unique), else the CTA merge sort in the
// windows (m <= kGridTile).
template <int NT>
DEV void cta_sort_hbm(u32* DK, u64* DP, u32 s0, u32 m, GridSmem<NT>& g) {
  using Bk = Blk<NT>;
  if (m < 2) return;
  if (m <= kRankSortMax) {
    u32 k0 = 0;
    u64 p0 = 0;
    const u32 i0 = threadIdx.x;
    if (i0 < m) {
      k0 = DK[s0 + i0];
      p0 = DP[s0 + i0];
      g.ak[i0] = k0;
      g.ap[i0] = p0;
    }
    Bk::sync();
    u32 r0 = 0;
    for (u32 j = 0; j < m; ++j) r0 += less_pk(g.ap[j], g.ak[j], p0, k0);
    if (i0 < m) {
      DK[s0 + r0] = k0;
      DP[s0 + r0] = p0;
    }
    Bk::sync();
    return;
  }
  for (u32 i = threadIdx.x; i < m; i += NT) {
    g.ak[i] = DK[s0 + i];
    g.ap[i] = DP[s0 + i];
  }
  Bk::sync();
  cta_sort<NT / 32>(g.ak, g.ap, m, g.bk, g.bp);
  for (u32 i = threadIdx.x; i < m; i += NT) {
    DK[s0 + i] = g.ak[i];
    DP[s0 + i] = g.ap[i];
  }
  Bk::sync();
}

// kind 9: merge the unsorted run U = sk/sp[0][0, n) into the sorted run
// S = (mk, mp)[0, m), into (ok, op)[0, m + n), in one job. CTA b owns the S
// chunk [m·b/G, m·(b+1)/G) and the U entries between its chunk's first
// entry and the next chunk's (bucket b): (1) every CTA holds the G - 1 chunk
// heads; each buckets its slice of U (binary search), with global bucket
// bases; (2) after a barrier, scatter U into bucket order (sk/sp[1]); (3)
// after a second barrier, CTA b sorts its bucket in place and streams the
// merge of its S chunk with it to output position m·b/G + (U entries in
// earlier buckets). A bucket above kGridTile sets bovf (the leader then
// takes the two-job path; S and U are untouched).
template <int NT>
DEV void batch_flush_merge(BatchJob* X, u32 b, u32 G, GridSmem<NT>& g) {
  using Bk = Blk<NT>;
  const u32 n = X->stg_n, m = X->mn;
  const u32* MK = X->mk;
  const u64* MP = X->mp;
  const u32* UK = X->sk[0];
  const u64* UP = X->sp[0];
  u32* DK = X->sk[1];
  u64* DP = X->sp[1];
  const bool write_idx = X->write_idx;
  pbh_idx_entry* idx = X->idx;
  // chunk heads 1..G-1 in the output windows (ok / op), counters in ap
  u32* hk = g.ok;
  u64* hp = g.op;
  u32* cnt = reinterpret_cast<u32*>(g.ap);
  u32* base = cnt + kBucketMax;
  u32* start = base + kBucketMax;
  for (u32 i = threadIdx.x; i < G; i += NT) {
    cnt[i] = 0;
    if (i >= 1) {
      const u32 at = (u32)((u64)m * i / G);
      const bool ok = at < m;  // empty tail chunks sort after everything
      hk[i - 1] = ok ? MK[at] : 0xffffffffu;
      hp[i - 1] = ok ? MP[at] : ~0ull;
    }
  }
  Bk::sync();
  auto bucket_of = [&](u32 k, u64 p) {  // heads <= (p, k), i.e. upper bound
    u32 lo = 0, hi = G - 1;
    while (lo < hi) {
      const u32 mid = (lo + hi) >> 1;
      if (!less_pk(p, k, hp[mid], hk[mid]))
        lo = mid + 1;
      else
        hi = mid;
    }
    return lo;
  };
  const u32 r0 = (u32)((u64)n * b / G), r1 = (u32)((u64)n * (b + 1) / G);
  for (u32 j = r0 + threadIdx.x; j < r1; j += NT) atomicAdd(&cnt[bucket_of(UK[j], UP[j])], 1u);
  Bk::sync();
  for (u32 i = threadIdx.x; i < G; i += NT) {
    const u32 c = cnt[i];
    base[i] = c ? atomicAdd(&X->bcnt[i], c) : 0;
    cnt[i] = 0;
  }
  job_barrier<NT>(X, G, g);
  {
    u32 run = 0;
    for (u32 i0 = 0; i0 < G; i0 += NT) {
      const u32 i = i0 + threadIdx.x;
      const u32 v = i < G ? __ldcg(&X->bcnt[i]) : 0;
      u32 tot;
      const u32 e = run + Bk::scan_excl(v, tot, g.scr);
      if (i < G) start[i] = e;
      run += tot;
    }
  }
  Bk::sync();
  for (u32 j = r0 + threadIdx.x; j < r1; j += NT) {
    const u32 k = UK[j];
    const u64 p = UP[j];
    const u32 q = bucket_of(k, p);
    const u32 pos = start[q] + base[q] + atomicAdd(&cnt[q], 1u);
    DK[pos] = k;
    DP[pos] = p;
    if (write_idx) {
      pbh_idx_entry ne;
      ne.prio = p;
      ne.state = PBH_ST_LIVE | (PBH_LOC_DEEP << 2);
      ne.parent = 0;
      reinterpret_cast<ulonglong2*>(idx)[k] = *reinterpret_cast<const ulonglong2*>(&ne);
    }
  }
  job_barrier<NT>(X, G, g);
  const u32 ub = __ldcg(&X->bcnt[b]), us = start[b];
  if (ub > kGridTile) {
    if (threadIdx.x == 0) atomicOr(&X->bovf, 1u);
    return;
  }
  cta_sort_hbm<NT>(DK, DP, us, ub, g);
  const u32 m0 = (u32)((u64)m * b / G), m1 = (u32)((u64)m * (b + 1) / G);
  if (threadIdx.x == 0) {
    g.sub.ak = MK + m0;
    g.sub.ap = MP + m0;
    g.sub.bk = DK + us;
    g.sub.bp = DP + us;
    g.sub.sink = Sink{X->ok, X->op, 0xffffffffu, nullptr, nullptr};
    g.sub.filter = 0;
  }
  __threadfence_block();
  Bk::sync();
  grid_stream<NT>(g.sub, 0, m1 - m0, 0, ub, m0 + us, g);
}

// This CTA's share (block b of G) of the current job.
template <int NT>
DEV void grid_share(const GridJob& J, u32 b, GridSmem<NT>& g, u32* scratch) {
  const u32 G = J.nblk;
  switch (J.kind) {
    case 2: return batch_validate<NT>(J.ext, b, G);
    case 3: return batch_classify<NT>(J.ext, b, G);
    case 4: return batch_sort_chunks<NT>(J.ext, b, G, g);
    case 5: return batch_merge_pass<NT>(J.ext, b, G, g, scratch);
    case 6: return batch_check_classify<NT>(J.ext, b, G, g);
    case 7: return batch_bucket_sort<NT>(J.ext, b, G, g);
    case 9: return batch_flush_merge<NT>(J.ext, b, G, g);
    default: break;
  }
  const u32 r0 = (u32)((u64)J.c * b / G), r1 = (u32)((u64)J.c * (b + 1) / G);
  const Run A{J.ak, J.ap, J.na}, B{J.bk, J.bp, J.nb};
  if (J.kind == 8) {
    // filtered merge: (1) each CTA counts the valid entries of its input
    // ranges; (2) after a grid barrier, the exclusive prefix of the counts
    // is its output start and it streams its range, dropping stale entries
    BatchJob* X = J.ext;
    u32 a0 = 0, a1 = 0;
    if (r0 < r1) merge_split2<NT>(A, B, r0, r1, scratch, a0, a1);
    const u32 mine = r0 < r1 ? count_valid<NT>(A.k, A.p, a0, a1, J.idx, scratch) +
                                   count_valid<NT>(B.k, B.p, r0 - a0, r1 - a1, J.idx, scratch)
                             : 0u;
    if (threadIdx.x == 0) X->bcnt[b] = mine;
    job_barrier<NT>(X, G, g);
    u32 start = 0;
    {
      u32 run = 0;
      for (u32 i0 = 0; i0 < G; i0 += NT) {
        const u32 i = i0 + threadIdx.x;
        const u32 v = i < G ? __ldcg(&X->bcnt[i]) : 0u;
        u32 tot;
        const u32 e = run + Blk<NT>::scan_excl(v, tot, scratch);
        if (i == b) g.ok[0] = e;
        if (b == 0 && i0 + NT >= G && threadIdx.x == 0) X->merge_total = run + tot;
        run += tot;
      }
      Blk<NT>::sync();
      start = g.ok[0];
      Blk<NT>::sync();
    }
    if (r0 < r1) grid_stream<NT>(J, a0, a1, r0 - a0, r1 - a1, J.out_base + start, g);
    return;
  }
  if (r0 >= r1) return;
  long long tq = clock64();
  u32 a0, a1;
  merge_split2<NT>(A, B, r0, r1, scratch, a0, a1);
  if (b == 0) { jobprof_add(16, clock64() - tq); tq = clock64(); }
  grid_stream<NT>(J, a0, a1, r0 - a0, r1 - a1, J.out_base + r0, g);
  if (b == 0) jobprof_add(17, clock64() - tq);
}

// Helper CTAs: wait for jobs until the exit job.
template <int NT>
DEV void grid_helper_loop(GridJob* gj, GridSmem<NT>& g, u32* scratch) {
  using Bk = Blk<NT>;
  u32 seen = 0;
  grid_smem_init<NT>(g);
  for (;;) {
    if (threadIdx.x == 0) {
      u32 s;
      u32 backoff = 16;
      while ((s = ld_acquire(&gj->seq)) == seen) {
        __nanosleep(backoff);
        backoff = backoff < kPollMaxNs ? backoff * 2 : kPollMaxNs;
      }
      g.seq = s;
    }
    Bk::sync();
    {
      // the descriptor, one 8-byte word per thread, read through L2 (never
      // a stale L1 line), ordered after thread 0's acquire by the barrier
      static_assert(sizeof(GridJob) % 8 == 0 && sizeof(GridJob) / 8 <= NT, "GridJob words");
      const unsigned long long* src = reinterpret_cast<const unsigned long long*>(gj);
      unsigned long long* dst = reinterpret_cast<unsigned long long*>(&g.job);
      if (threadIdx.x < sizeof(GridJob) / 8) dst[threadIdx.x] = __ldcg(src + threadIdx.x);
    }
    Bk::sync();
    seen = g.seq;
    if (g.job.kind == 1) return;
    grid_share<NT>(g.job, blockIdx.x, g, scratch);
    Bk::sync();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&gj->done, 1u);
    }
  }
}

// Leader: call once at kernel start (the host zeroed the job word).
template <int NT>
DEV void grid_leader_init(GridSmem<NT>& g) {
  (void)g;  // grid_smem_init ran at kernel start
}

// Leader side: publish (kind, runs, sink), take share 0, wait for the rest.
template <int NT>
NOINL void grid_run(GridJob* gj, u32 G, u32 kind, const Run& A, const Run& B, u32 c,
                    const Sink& sink, u32 out_base, GridSmem<NT>& g, u32* scratch) {
  using Bk = Blk<NT>;
  const long long t_job = clock64();
  Bk::sync();
  if (threadIdx.x == 0) {
    GridJob& J = g.job;
    J.kind = kind;
    J.nblk = G;
    J.ak = A.k;
    J.ap = A.p;
    J.bk = B.k;
    J.bp = B.p;
    J.na = A.n;
    J.nb = B.n;
    J.c = c;
    J.out_base = out_base;
    J.sink = sink;
    J.ext = g.job.ext;
    J.filter = kind == 8 ? 1u : 0u;
    J.idx = g.job.idx;
    J.self = gj;
    // descriptor fields first, then the sequence word (release)
    gj->kind = J.kind;
    gj->nblk = J.nblk;
    gj->ak = J.ak;
    gj->ap = J.ap;
    gj->bk = J.bk;
    gj->bp = J.bp;
    gj->na = J.na;
    gj->nb = J.nb;
    gj->c = J.c;
    gj->out_base = J.out_base;
    gj->sink = J.sink;
    gj->ext = J.ext;
    gj->idx = J.idx;
    gj->filter = J.filter;
    gj->self = gj;
    gj->done = 0;
    const u32 s = g.seq + 1;  // the host zeroes the job word before each launch
    g.seq = s;
    __threadfence();
    st_release(&gj->seq, s);
  }
  Bk::sync();
  if (kind == 1) return;
  grid_share<NT>(g.job, 0, g, scratch);
  const long long t_share = clock64();
  Bk::sync();
  if (threadIdx.x == 0) {
    u32 backoff = 16;
    while (ld_acquire(&gj->done) < G - 1) {
      __nanosleep(backoff);
      backoff = backoff < kPollMaxNs ? backoff * 2 : kPollMaxNs;
    }
    __threadfence();
  }
  Bk::sync();
  jobprof_add(kind == 8 ? 14u : kind == 9 ? 15u : kind, clock64() - t_job);
  jobprof_add(13, clock64() - t_share);  // leader waiting for the helpers
}

}  // namespace pbh_dev
