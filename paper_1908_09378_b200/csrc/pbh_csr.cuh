// CSR input contract on the device: validate_graph (graphs.cpp:55-72) and
// CsrGraph::max_out_degree (graphs.cpp:47-53) in one HBM pass.
//
// One warp per row (lanes stride the row's targets/weights: coalesced 128-B
// lines), a grid-stride loop over rows. Each violation is recorded as the
// smallest (row, position-in-row, check) key with atomicMin, so the report
// names the violation the reference's sequential loop would throw first.
// Bytes: 8 (V+1) + 8 E read once (C3: 2.16 GB, ~0.35 ms at 6.4 TB/s).
#pragma once

#include "pbh_engine.cuh"

namespace pbh_dev {

// check codes in the reference's order inside one row (graphs.cpp:62-69)
enum : u32 {
  kCsrMonotone = 0,  // offsets[u] > offsets[u+1] (or beyond edge_count)
  kCsrRange = 1,     // target >= vertex_count
  kCsrSelfLoop = 2,  // target == u
  kCsrUnsorted = 3,  // targets[i-1] >= targets[i] (unsorted row / parallel edge)
  kCsrZeroW = 4,     // weight == 0
};

struct CsrCheck {
  unsigned long long max_deg;  // max out-degree (rows with valid offsets)
  unsigned long long first;    // min (u << 32 | min(pos, 2^29-1) << 3 | code); ~0 = clean
  unsigned int sizes_bad;      // offsets[0] != 0 or offsets[V] != E
};

__device__ __forceinline__ unsigned long long csr_key(u32 u, u64 pos, u32 code) {
  return ((unsigned long long)u << 32) | ((unsigned long long)min(pos, (u64)((1u << 29) - 1)) << 3) |
         code;
}

__global__ void k_csr_check(const u64* __restrict__ off, const u32* __restrict__ tgt,
                            const u32* __restrict__ w, u32 V, u64 E, CsrCheck* out) {
  const u32 lane = threadIdx.x & 31;
  const u64 warp = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5;
  const u64 n_warps = ((u64)gridDim.x * blockDim.x) >> 5;
  if (warp == 0 && lane == 0) {
    if (off[0] != 0 || off[V] != E) atomicOr(&out->sizes_bad, 1u);
  }
  u64 best_deg = 0;
  unsigned long long first = ~0ull;
  for (u64 u = warp; u < V; u += n_warps) {
    const u64 b = off[u], e = off[u + 1];
    if (b > e || e > E) {
      first = min(first, csr_key((u32)u, 0, kCsrMonotone));
      continue;
    }
    best_deg = max(best_deg, e - b);
    // lanes walk the row in 32-edge chunks; the predecessor of lane 0's edge
    // comes from the previous chunk's lane 31
    u32 prev_last = 0;
    for (u64 i0 = b; i0 < e; i0 += 32) {
      const u64 i = i0 + lane;
      const bool in = i < e;
      const u32 t = in ? tgt[i] : 0u;
      const u32 wt = in ? w[i] : 1u;
      u32 pred = __shfl_up_sync(0xffffffffu, t, 1);
      if (lane == 0) pred = prev_last;
      prev_last = __shfl_sync(0xffffffffu, t, 31);
      if (in) {
        const u64 pos = i - b;
        // the reference tests range, self-loop, order, weight in that order
        u32 code = 8;
        if (t >= V) code = kCsrRange;
        else if (t == (u32)u) code = kCsrSelfLoop;
        else if (i > b && pred >= t) code = kCsrUnsorted;
        else if (wt == 0) code = kCsrZeroW;
        if (code != 8) first = min(first, csr_key((u32)u, pos, code));
      }
      // once a violation exists for this row, later chunks cannot beat it
      if (__any_sync(0xffffffffu, first != ~0ull && (first >> 32) == u)) break;
    }
  }
  // warp reductions, one atomic per warp
  for (int s = 16; s; s >>= 1) {
    best_deg = max(best_deg, (u64)__shfl_xor_sync(0xffffffffu, (unsigned long long)best_deg, s));
    first = min(first, __shfl_xor_sync(0xffffffffu, first, s));
  }
  if (lane == 0) {
    if (best_deg) atomicMax(&out->max_deg, (unsigned long long)best_deg);
    if (first != ~0ull) atomicMin(&out->first, first);
  }
}

}  // namespace pbh_dev
