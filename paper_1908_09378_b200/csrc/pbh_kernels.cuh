// Kernels: trace interpreter (one persistent CTA per heap) and the SSSP
// driver (one persistent CTA per source). Both run the CTA engine of
// pbh_heap.cuh; nothing returns to the host between ops.
#pragma once

#include "pbh_heap.cuh"

namespace pbh_dev {

// Dynamic shared-memory layout (byte offsets), computed on the host.
struct SmLayout {
  u32 use_smem;  // B_0 + batch + push + removal flags resident in smem
  u32 off_grid;  // GridSmem<NT> (trace interpreter with grid helpers)
  u32 grid_min;  // smallest merge sent to the grid helpers
  u32 off_b0k0, off_b0k1, off_b0p0, off_b0p1;
  u32 off_bk, off_bp, off_pk, off_pp, off_rm;
  u32 off_ck, off_cp, off_co, off_cs;  // SSSP relaxation collection (d + NT)
  u32 total;
};

// Per-source SSSP bookkeeping in HBM.
struct SsspState {
  u64 n_settled;
  u64 rounds;
  u32 started;
  u32 status;
  u32 detail;
  u32 pad;
  u64 aux;
  u64 ops;  // Metrics::ops of par_dijkstra (fast path)
  u64 pad2;
  u64 phase[8];  // clock64 cycles per phase (PBH_PHASES diagnostics)
};

// Internal op kinds (never accepted from user traces).
constexpr u8 kOpDrain = 'R';
constexpr u8 kOpFind = 'F';

template <int NT, int VT>
DEV void bind_buffers(HeapCta<NT, VT>& h, unsigned char* dyn, const SmLayout& L,
                      pbh_heap_dev* g) {
  if (L.use_smem) {
    h.bk = reinterpret_cast<u32*>(dyn + L.off_bk);
    h.bp = reinterpret_cast<u64*>(dyn + L.off_bp);
    h.pk = reinterpret_cast<u32*>(dyn + L.off_pk);
    h.pp = reinterpret_cast<u64*>(dyn + L.off_pp);
    h.rm = dyn + L.off_rm;
  } else {
    h.bk = g->g_bk;
    h.bp = g->g_bp;
    h.pk = g->g_pk;
    h.pp = g->g_pp;
    h.rm = g->g_rm;
  }
  h.bo = nullptr;
}

template <int NT, int VT>
__global__ void __launch_bounds__(NT) k_trace(pbh_heap_dev* g, pbh_trace_dev tr, u64 op_begin,
                                              u64 op_end, u32* out_v, u64* out_p,
                                              pbh_kstatus* ks, SmLayout L, u32 allow_internal,
                                              GridJob* gj) {
  extern __shared__ __align__(16) unsigned char dyn[];
  using HC = HeapCta<NT, VT>;
  using Bk = Blk<NT>;
  GridSmem<NT>& gsm = *reinterpret_cast<GridSmem<NT>*>(dyn + L.off_grid);
  if (blockIdx.x > 0) {  // helper CTA: deep merges of the leader's heap
    grid_helper_loop<NT>(gj, gsm, gsm.scr);
    return;
  }
  typename HC::Sm& sm = *reinterpret_cast<typename HC::Sm*>(dyn);
  HC h{sm};
  h.gs = &gsm;  // streamed CTA-local merges
  if (gridDim.x > 1) {
    h.gj = gj;
    h.gsz = gridDim.x;
    h.gmin = L.grid_min;
    grid_leader_init<NT>(gsm);
  }
  h.load(g, reinterpret_cast<u32*>(dyn + L.off_b0k0), reinterpret_cast<u64*>(dyn + L.off_b0p0),
         reinterpret_cast<u32*>(dyn + L.off_b0k1), reinterpret_cast<u64*>(dyn + L.off_b0p1),
         L.use_smem != 0);
  bind_buffers<NT, VT>(h, dyn, L, g);
  if (L.use_smem) {
    for (u32 i = threadIdx.x; i < sm.cap0; i += NT) h.rm[i] = 0;
    Bk::sync();
  }
  u64 n_out = ks->n_out;
  u64 op = op_begin;
  for (; op < op_end; ++op) {
    const u8 kind = tr.kinds[op];
    const u64 b = tr.offsets[op], e = tr.offsets[op + 1];
    switch (kind) {
      case 'U':
        h.op_bulk(tr.vals + b, tr.prios + b, 1, false);
        break;
      case 'B':
        h.op_bulk(tr.vals + b, tr.prios + b, (u32)(e - b), true);
        break;
      case 'E': {
        u32 k;
        u64 p;
        if (h.op_extract(k, p) && threadIdx.x == 0) {
          out_v[n_out] = k;
          out_p[n_out] = p;
        }
        n_out += sm.status == 0;
        break;
      }
      case 'D':
        h.op_delete(tr.vals[b]);
        break;
      case kOpFind:
        if (allow_internal) {
          u32 k;
          u64 p;
          if (h.op_find_min(k, p) && threadIdx.x == 0) {
            out_v[n_out] = k;
            out_p[n_out] = p;
          }
          n_out += sm.status == 0;
          break;
        }
        h.fail(PBH_ERR_BAD_OP, kind);
        break;
      case kOpDrain:
        if (allow_internal) {
          h.drain();
          break;
        }
        h.fail(PBH_ERR_BAD_OP, kind);
        break;
      default:
        h.fail(PBH_ERR_BAD_OP, kind);
        break;
    }
    if (h.failed()) break;
    if (kind == kOpFind || kind == kOpDrain) continue;  // not counted as ops
    h.after_op();
    if (h.failed()) {
      ++op;  // the op itself completed; the failure is internal
      break;
    }
  }
  if (gridDim.x > 1) grid_run<NT>(gj, gridDim.x, 1, Run{}, Run{}, 0, Sink{}, 0, gsm, gsm.scr);
  h.store();
  if (threadIdx.x == 0) {
    ks->status = sm.status;
    ks->detail = sm.detail;
    ks->aux = sm.aux;
    ks->ops_done = op - op_begin;
    ks->n_out = n_out;
    ks->failed_op = op;
  }
}

// par_dijkstra (sssp.cpp:21-69): one CTA per source; resumable after a
// NEED_GROW exit (state is entirely in HBM).
template <int NT, int VT>
__global__ void __launch_bounds__(NT) k_sssp(pbh_heap_dev* heaps, const u64* __restrict__ off,
                                             const u32* __restrict__ tgt,
                                             const u32* __restrict__ wt, u32 V,
                                             const u32* sources, u64* dist, u32* settled,
                                             SsspState* sst, u32 dag_mode, u32 max_deg,
                                             SmLayout L) {
  extern __shared__ __align__(16) unsigned char dyn[];
  using HC = HeapCta<NT, VT>;
  using Bk = Blk<NT>;
  typename HC::Sm& sm = *reinterpret_cast<typename HC::Sm*>(dyn);
  SsspState* my = sst + blockIdx.x;
  if (my->status != 0 && my->status != 7) return;  // finished with an error
  pbh_heap_dev* g = heaps + blockIdx.x;
  HC h{sm};
  h.load(g, reinterpret_cast<u32*>(dyn + L.off_b0k0), reinterpret_cast<u64*>(dyn + L.off_b0p0),
         reinterpret_cast<u32*>(dyn + L.off_b0k1), reinterpret_cast<u64*>(dyn + L.off_b0p1),
         L.use_smem != 0);
  bind_buffers<NT, VT>(h, dyn, L, g);
  u32* ck;
  u64* cp;
  u64* co;
  u32* cs;
  if (L.use_smem) {
    for (u32 i = threadIdx.x; i < sm.cap0; i += NT) h.rm[i] = 0;
    ck = reinterpret_cast<u32*>(dyn + L.off_ck);
    cp = reinterpret_cast<u64*>(dyn + L.off_cp);
    co = reinterpret_cast<u64*>(dyn + L.off_co);
    cs = reinterpret_cast<u32*>(dyn + L.off_cs);
  } else {
    ck = g->g_ck;
    cp = g->g_cp;
    co = g->g_co;
    cs = g->g_cs;
  }
  pbh_idx_entry* idx = g->idx;
  u64* my_dist = dist + (u64)blockIdx.x * V;
  u32* my_settled = settled + (u64)blockIdx.x * V;
  u64 n_settled = my->n_settled, rounds = my->rounds;
  const u32 d = sm.d;
  Bk::sync();

  if (!my->started) {
    const u32 s = sources[blockIdx.x];
    if (threadIdx.x == 0) {
      ck[0] = s;
      cp[0] = 0;
    }
    Bk::sync();
    h.op_bulk(ck, cp, 1, false);  // eng.update({s, 0}) (sssp.cpp:36)
    if (threadIdx.x == 0) idx[s].parent = s;
    if (!h.failed()) h.after_op();
  }

  while (!h.failed() && sm.live > 0) {
    if (!h.room_for(max_deg)) break;
    u32 v;
    u64 p;
    if (!h.op_extract(v, p)) break;
    if (threadIdx.x == 0) {
      my_dist[v] = p;
      my_settled[n_settled] = v;
    }
    ++n_settled;
    ++rounds;
    h.after_op();
    if (h.failed()) break;
    // relax the CSR row of v (sssp.cpp:49-57); batches of <= d in CSR order
    const u64 rb = off[v], re = off[v + 1];
    u32 staged = 0;
    bool overflow = false;
    for (u64 base = rb; base < re; base += NT) {
      const u64 j = base + threadIdx.x;
      bool imp = false;
      u32 u = 0;
      u64 cand = 0, oldp = 0;
      u32 olds = 0;
      if (j < re) {
        u = tgt[j];
        const u32 w = wt[j];
        const ulonglong2 e = __ldcg(reinterpret_cast<const ulonglong2*>(idx + u));
        oldp = e.x;
        olds = (u32)e.y;
        if (dag_mode || PBH_ST(olds) != PBH_ST_DEAD) {
          cand = p + w;
          if (cand < p) overflow = true;
          imp = cand < oldp;
        }
      }
      u32 tot;
      const u32 pos = staged + Bk::scan_excl(imp ? 1u : 0u, tot, h.scr());
      if (imp) {
        ck[pos] = u;
        cp[pos] = cand;
        co[pos] = oldp;
        cs[pos] = olds;
      }
      staged += tot;
      Bk::sync();
      while (staged >= d) {  // flush full chunks of d
        h.relax_chunk(ck, cp, co, cs, d, v);
        if (h.failed()) break;
        h.after_op();
        if (h.failed()) break;
        // shift the remainder (< NT entries) to the front
        const u32 rem = staged - d;
        const bool mv = threadIdx.x < rem;
        u32 kk = 0, ss = 0;
        u64 pv = 0, oo = 0;
        if (mv) {
          kk = ck[d + threadIdx.x];
          pv = cp[d + threadIdx.x];
          oo = co[d + threadIdx.x];
          ss = cs[d + threadIdx.x];
        }
        Bk::sync();
        if (mv) {
          ck[threadIdx.x] = kk;
          cp[threadIdx.x] = pv;
          co[threadIdx.x] = oo;
          cs[threadIdx.x] = ss;
        }
        Bk::sync();
        staged = rem;
      }
      if (h.failed()) break;
    }
    if (Bk::any(overflow, h.scr())) {
      h.fail(PBH_ERR_OVERFLOW, v);
      break;
    }
    if (h.failed()) break;
    if (staged > 0) {
      h.relax_chunk(ck, cp, co, cs, staged, v);
      if (h.failed()) break;
      h.after_op();
    }
  }
  h.store();
  if (threadIdx.x == 0) {
    my->n_settled = n_settled;
    my->rounds = rounds;
    my->started = 1;
    my->status = sm.status;
    my->detail = sm.detail;
    my->aux = sm.aux;
    my->aux = sm.aux;
  }
}

}  // namespace pbh_dev
