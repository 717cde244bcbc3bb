// Frontier Bellman-Ford on the device: the reference's cross-check baseline
// `bellman_ford` (sssp.cpp:99-129), re-designed as a label-correcting sweep
// over the CHANGED vertices only, for the heap-vs-sweep comparison of
// SURVEY.md §8(f) rank 4 (acceptance_main.cpp:230-260).
//
// One cooperative grid runs every iteration: a warp takes one frontier vertex
// and relaxes its row with coalesced loads (32 edges per step); an improving
// candidate lowers dist[u] with a 64-bit atomicMin and, the first time u
// improves in this iteration, appends u to the next frontier (per-vertex
// iteration stamp). Iterations are separated by grid.sync(). Distances are
// exact (weights >= 1, unique shortest-path lengths); the parent of each
// reached vertex is recovered afterwards from the tight in-edges
// (dist[v] + w == dist[u]), which always forms a valid shortest-path tree.
#pragma once

#include <cooperative_groups.h>

#include "pbh_engine.cuh"

namespace pbh_dev {

struct BfState {
  u32 cnt[3];   // frontier sizes (rotating: current, next, next-next reset)
  u32 status;   // 0 ok, 9 overflow
  u64 iters;
  u64 relaxed;  // edges scanned
};

__global__ void __launch_bounds__(256) k_bellman_ford(const u64* __restrict__ off,
                                                      const u32* __restrict__ tgt,
                                                      const u32* __restrict__ wt, u32 V, u64* dist,
                                                      u32* fq0, u32* fq1, u32* stamp, BfState* st,
                                                      u64 max_iters) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const u32 lane = threadIdx.x & 31;
  const u64 gwarp = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  u64 scanned = 0;
  u64 it = 0;
  for (; it < max_iters; ++it) {
    u32* cur = (it & 1) ? fq1 : fq0;
    u32* nxt = (it & 1) ? fq0 : fq1;
    const u32 n = *(volatile u32*)&st->cnt[it % 3];
    if (n == 0) break;
    if (gwarp == 0 && lane == 0) st->cnt[(it + 2) % 3] = 0;  // reset for it + 2
    for (u64 f = gwarp; f < n; f += nwarps) {
      const u32 v = cur[f];
      const u64 dv = __ldcg(dist + v);
      const u64 b = off[v], e = off[v + 1];
      for (u64 j = b + lane; j < e; j += 32) {
        const u32 u = tgt[j];
        const u64 c = dv + wt[j];
        ++scanned;
        if (c < dv) {
          st->status = 9;
          continue;
        }
        if (c < __ldcg(dist + u)) {
          const u64 old = atomicMin(reinterpret_cast<unsigned long long*>(dist + u),
                                    (unsigned long long)c);
          if (c < old && atomicExch(stamp + u, (u32)(it + 1)) != (u32)(it + 1)) {
            const u32 slot = atomicAdd(&st->cnt[(it + 1) % 3], 1u);
            nxt[slot] = u;
          }
        }
      }
    }
    grid.sync();
  }
  // edges scanned, summed over the grid
  for (int o = 16; o > 0; o >>= 1) scanned += __shfl_down_sync(0xffffffffu, scanned, o);
  if (lane == 0 && scanned) atomicAdd(reinterpret_cast<unsigned long long*>(&st->relaxed),
                                      (unsigned long long)scanned);
  if (blockIdx.x == 0 && threadIdx.x == 0) st->iters = it;
}

// parent[u] = some v with dist[v] + w(v, u) == dist[u] (u reached, u != source).
__global__ void k_bf_parents(const u64* __restrict__ off, const u32* __restrict__ tgt,
                             const u32* __restrict__ wt, u32 V, const u64* __restrict__ dist,
                             u32* parent) {
  const u32 lane = threadIdx.x & 31;
  const u64 gwarp = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 v = gwarp; v < V; v += nwarps) {
    const u64 dv = dist[v];
    if (dv == ~0ull) continue;
    for (u64 j = off[v] + lane; j < off[v + 1]; j += 32) {
      const u32 u = tgt[j];
      if (u != v && dv + wt[j] == dist[u]) parent[u] = (u32)v;
    }
  }
}

}  // namespace pbh_dev
