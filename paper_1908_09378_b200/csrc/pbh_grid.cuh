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

constexpr u32 kGridTile = 2048;   // outputs per streamed tile
constexpr u32 kGridMin = 2048;    // smallest merge worth a grid job (measured sweep 2K..16K: 2K best)
constexpr u32 kStreamMin = 64;    // smallest merge streamed through the windows by one CTA

// Job word + descriptor in HBM (one per heap handle).
struct GridJob {
  u32 seq;   // bumped by the leader to publish a job
  u32 done;  // helpers that finished the current job
  u32 kind;  // 0 = merge, 1 = exit
  u32 nblk;  // CTAs in the grid (leader included)
  const u32* ak;
  const u64* ap;
  const u32* bk;
  const u64* bp;
  u32 na, nb;  // run lengths
  u32 c;       // outputs: the first c of merge(A, B)
  u32 out_base;
  Sink sink;
};

template <int NT>
struct GridSmem {
  u32 ak[kGridTile], bk[kGridTile], ok[kGridTile];
  u64 ap[kGridTile], bp[kGridTile], op[kGridTile];
  GridJob job;  // the current job, copied in by thread 0
  u32 ta;       // A elements consumed by the current tile
  u32 seq;
  u32 scr[NT / 32 + 2];  // scan scratch of the merge-path searches
};

DEV u32 ld_acquire(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
DEV void st_release(u32* p, u32 v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Stream the merge of A[ia, ia_end) and B[ib, ib_end) (no filter) into
// sink[out ...). Every thread of the CTA calls this.
template <int NT>
DEV void grid_stream(const GridJob& J, u32 ia, u32 ia_end, u32 ib, u32 ib_end, u32 out,
                     GridSmem<NT>& g) {
  using Bk = Blk<NT>;
  constexpr u32 VT = kGridTile / NT;
  const u32 tid = threadIdx.x;
  while (ia < ia_end || ib < ib_end) {
    const u32 na = min(kGridTile, ia_end - ia), nb = min(kGridTile, ib_end - ib);
    const u32 n = min(kGridTile, (ia_end - ia) + (ib_end - ib));
    // windows straight into shared memory (cp.async: no register round trip,
    // every load of the tile in flight at once)
    for (u32 i = tid; i < na; i += NT) {
      cp_async4(&g.ak[i], J.ak + ia + i, true);
      cp_async8(&g.ap[i], J.ap + ia + i);
    }
    for (u32 i = tid; i < nb; i += NT) {
      cp_async4(&g.bk[i], J.bk + ib + i, true);
      cp_async8(&g.bp[i], J.bp + ib + i);
    }
    cp_async_commit();
    cp_async_wait_all();
    Bk::sync();
    // this thread's outputs [d0, d1): merge-path split inside the windows
    const u32 d0 = min(tid * VT, n), d1 = min(d0 + VT, n);
    u32 lo = d0 > nb ? d0 - nb : 0, hi = min(d0, na);
    while (lo < hi) {
      const u32 m = (lo + hi) >> 1;
      if (less_pk(g.ap[m], g.ak[m], g.bp[d0 - 1 - m], g.bk[d0 - 1 - m]))
        lo = m + 1;
      else
        hi = m;
    }
    u32 x = lo, y = d0 - lo;
#pragma unroll
    for (u32 v = 0; v < VT; ++v) {
      if (d0 + v < d1) {
        const bool takeA = x < na && (y >= nb || less_pk(g.ap[x], g.ak[x], g.bp[y], g.bk[y]));
        if (takeA) {
          g.ok[d0 + v] = g.ak[x];
          g.op[d0 + v] = g.ap[x];
          ++x;
        } else {
          g.ok[d0 + v] = g.bk[y];
          g.op[d0 + v] = g.bp[y];
          ++y;
        }
      }
    }
    if (d0 < d1 && d1 == n) g.ta = x;
    Bk::sync();
    for (u32 i = tid; i < n; i += NT) J.sink.put(out + i, g.ok[i], g.op[i]);
    const u32 ta = g.ta;
    ia += ta;
    ib += n - ta;
    out += n;
    Bk::sync();
  }
}

// This CTA's share (block b of G) of the current job.
template <int NT>
DEV void grid_share(const GridJob& J, u32 b, GridSmem<NT>& g, u32* scratch) {
  const u32 G = J.nblk;
  const u32 r0 = (u32)((u64)J.c * b / G), r1 = (u32)((u64)J.c * (b + 1) / G);
  if (r0 >= r1) return;
  const Run A{J.ak, J.ap, J.na}, B{J.bk, J.bp, J.nb};
  const u32 a0 = r0 == 0 ? 0 : merge_split<NT>(A, B, r0, scratch);
  const u32 a1 = merge_split<NT>(A, B, r1, scratch);
  grid_stream<NT>(J, a0, a1, r0 - a0, r1 - a1, J.out_base + r0, g);
}

// Helper CTAs: wait for jobs until the exit job.
template <int NT>
DEV void grid_helper_loop(GridJob* gj, GridSmem<NT>& g, u32* scratch) {
  using Bk = Blk<NT>;
  u32 seen = 0;
  if (threadIdx.x == 0) g.seq = 0;
  Bk::sync();
  for (;;) {
    if (threadIdx.x == 0) {
      u32 s;
      u32 backoff = 32;
      while ((s = ld_acquire(&gj->seq)) == seen) {
        __nanosleep(backoff);
        backoff = backoff < 256 ? backoff * 2 : 256;
      }
      g.seq = s;
      // the descriptor, read through L2 (never a stale L1 line)
      static_assert(sizeof(GridJob) % 8 == 0, "GridJob is copied as 8-byte words");
      const unsigned long long* src = reinterpret_cast<const unsigned long long*>(gj);
      unsigned long long* dst = reinterpret_cast<unsigned long long*>(&g.job);
      for (u32 i = 0; i < sizeof(GridJob) / 8; ++i) dst[i] = __ldcg(src + i);
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
  if (threadIdx.x == 0) g.seq = 0;
}

// Leader side: publish (kind, runs, sink), take share 0, wait for the rest.
template <int NT>
NOINL void grid_run(GridJob* gj, u32 G, u32 kind, const Run& A, const Run& B, u32 c,
                    const Sink& sink, u32 out_base, GridSmem<NT>& g, u32* scratch) {
  using Bk = Blk<NT>;
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
    gj->done = 0;
    const u32 s = g.seq + 1;  // the host zeroes the job word before each launch
    g.seq = s;
    __threadfence();
    st_release(&gj->seq, s);
  }
  Bk::sync();
  if (kind == 1) return;
  grid_share<NT>(g.job, 0, g, scratch);
  Bk::sync();
  if (threadIdx.x == 0) {
    u32 backoff = 32;
    while (ld_acquire(&gj->done) < G - 1) {
      __nanosleep(backoff);
      backoff = backoff < 256 ? backoff * 2 : 256;
    }
    __threadfence();
  }
  Bk::sync();
}

}  // namespace pbh_dev
