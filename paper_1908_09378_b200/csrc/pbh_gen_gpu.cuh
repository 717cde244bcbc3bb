// Device generators for the BASELINE graphs: the C2
// grid and the C3 band built directly in HBM, draw for draw identical to the
// host generators (csrc/pbh_gen.cpp, which follow graphs.cpp:15-17 and
// std::mt19937_64 with rng() % n).
//
// std::mt19937_64 is sequential, but one twist of its 312-word state splits
// into two independent halves (words 0..155 read only the old state; words
// 156..311 read the old state and the new words 0..155), so a single CTA of
// 320 threads regenerates 312 draws per two barriers and writes each tempered
// draw straight into the weight of the edge that consumes it. Targets and
// offsets are closed forms, built by a separate grid-wide kernel.
#pragma once

#include "pbh_engine.cuh"

namespace pbh_dev {

constexpr int kMtN = 312, kMtM = 156;
constexpr u64 kMtA = 0xB5026F5AA96619E9ull;
constexpr u64 kMtUpper = 0xFFFFFFFF80000000ull, kMtLower = 0x7FFFFFFFull;

DEV u64 mt_temper(u64 y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

// Draw t (0-based) -> edge index and weight. kind 0 = grid: every edge in CSR
// order consumes one draw, w = 1 + r % (2^32 - 1). kind 1 = band: the spine
// edge u -> u+1 (u + 1 < V) takes no draw and has w = 1; every other edge
// takes the next draw, w = V + r % 1000.
struct GenMap {
  u32 kind;
  u32 V, degree;
  u64 n_draws;
  u32* w;
  DEV void put(u64 t, u64 r) const {
    if (kind == 0) {
      w[t] = 1u + (u32)(r % 4294967295ull);
      return;
    }
    // band: rows u < V-1 hold degree-1 draws, the last row holds degree
    const u64 per = degree - 1;
    u64 u = per ? t / per : (u64)V - 1, jj = per ? t % per : t;
    if (u >= (u64)V - 1) {  // last row: no spine edge
      u = V - 1;
      jj = t - (u64)(V - 1) * per;
    } else {
      // spine position in row u: the first target u+1 unless the row wraps
      const u64 end = u + degree;
      const u64 spine = end >= V ? end - V + 1 : 0;
      if (jj >= spine) ++jj;
    }
    w[u * degree + jj] = V + (u32)(r % 1000);
  }
};

__global__ void __launch_bounds__(320, 1) k_gen_weights(const u64* __restrict__ state0,
                                                        GenMap map) {
  __shared__ u64 mt[kMtN];
  const u32 i = threadIdx.x;
  if (i < kMtN) mt[i] = state0[i];
  __syncthreads();
  for (u64 base = 0; base < map.n_draws; base += kMtN) {
    // twist, first half (old state only)
    u64 y0 = 0;
    if (i < kMtM) {
      const u64 x = (mt[i] & kMtUpper) | (mt[i + 1] & kMtLower);
      y0 = mt[i + kMtM] ^ (x >> 1) ^ ((x & 1ull) ? kMtA : 0ull);
    }
    __syncthreads();
    if (i < kMtM) mt[i] = y0;
    __syncthreads();
    // second half (old words i, i+1; new word i - 156; word 0 is new for 311)
    u64 y1 = 0;
    if (i >= kMtM && i < kMtN) {
      const u64 x = (mt[i] & kMtUpper) | (mt[(i + 1) % kMtN] & kMtLower);
      y1 = mt[i - kMtM] ^ (x >> 1) ^ ((x & 1ull) ? kMtA : 0ull);
    }
    __syncthreads();
    if (i >= kMtM && i < kMtN) mt[i] = y1;
    __syncthreads();
    if (i < kMtN && base + i < map.n_draws) map.put(base + i, mt_temper(mt[i]));
  }
}

// Targets / offsets / spine weights (closed forms), grid-stride over vertices.
__global__ void k_gen_structure(u32 kind, u32 rows, u32 cols, u32 V, u32 degree, u64* off,
                                u32* tgt, u32* w) {
  for (u64 u = blockIdx.x * (u64)blockDim.x + threadIdx.x; u < V;
       u += (u64)gridDim.x * blockDim.x) {
    if (kind == 1) {  // band: row u -> (u + j) mod V, j = 1..degree, target-sorted
      const u64 b = u * degree;
      off[u] = b;
      if (u + 1 == V) off[V] = (u64)V * degree;
      const u64 end = u + degree;
      u64 n = b;
      if (end >= V) {
        const u32 wrap = (u32)(end - V + 1);
        for (u32 t = 0; t < wrap; ++t) tgt[n++] = t;
        for (u64 t = u + 1; t < V; ++t) tgt[n++] = (u32)t;
      } else {
        for (u64 t = u + 1; t <= end; ++t) tgt[n++] = (u32)t;
      }
      if (u + 1 < V) w[b + (end >= V ? end - V + 1 : 0)] = 1;  // the spine
    } else {  // grid, rows ordered up, left, right, down
      const u64 r = u / cols, c = u % cols;
      auto vert = [&](u64 rr) { return (u64)(rr > 0) + (u64)(rr + 1 < rows); };
      // edges of the rows above: cols * sum(vert) + 2 (cols - 1) per row
      u64 above = 2ull * (cols - 1) * r;
      if (r > 0) above += (u64)cols * ((r - 1) * 2 + 1);  // rows 1..r-1 have 2, row 0 has 1
      if (rows == 1) above = 2ull * (cols - 1) * r;
      const u64 within = c * vert(r) + (c > 0 ? c - 1 : 0) + (c < cols - 1 ? c : cols - 1);
      u64 n = above + within;
      off[u] = n;
      if (u + 1 == V) off[V] = 2ull * ((u64)rows * (cols - 1) + (u64)cols * (rows - 1));
      if (r > 0) tgt[n++] = (u32)(u - cols);
      if (c > 0) tgt[n++] = (u32)(u - 1);
      if (c + 1 < cols) tgt[n++] = (u32)(u + 1);
      if (r + 1 < rows) tgt[n++] = (u32)(u + cols);
    }
  }
}

}  // namespace pbh_dev
