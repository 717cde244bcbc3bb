// Micro-benchmark of the CTA sort used by push-buffer flushes (dev aid):
// cycles per 4096-entry sort, phase 1 (register bitonic runs) R=1 vs R=2,
// and the whole cta_sort.
#include <cstdio>
#include "../../paper_1908_09378_b200/csrc/pbh_grid.cuh"
using namespace pbh_dev;
template <int MODE>
__global__ void __launch_bounds__(128, 1) k(const u32* gk, const u64* gp, u32 n, int reps, long long* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  u64* P = reinterpret_cast<u64*>(sm);
  u64* TP = P + 4096;
  u32* K = reinterpret_cast<u32*>(TP + 4096);
  u32* TK = K + 4096;
  long long tot = 0;
  const u32 lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int r = 0; r < reps; ++r) {
    for (u32 i = threadIdx.x; i < n; i += 128) { K[i] = gk[(i + r * 977) % n]; P[i] = gp[(i + r * 977) % n]; }
    __syncthreads();
    long long t0 = clock64();
    if (MODE == 0) cta_sort<4>(K, P, n, TK, TP);
    if (MODE == 1) { for (u32 run = w; run < n / 128; run += 4) sort_runs128<1>(K, P, n, run, 4, lane); }
    if (MODE == 2) { u32 run = w; for (; run + 4 < n / 128; run += 8) sort_runs128<2>(K, P, n, run, 4, lane); if (run < n / 128) sort_runs128<1>(K, P, n, run, 4, lane); }
    __syncthreads();
    tot += clock64() - t0;
  }
  if (threadIdx.x == 0) out[0] = tot / reps;
  if (threadIdx.x == 0) out[1] = K[0] + P[n - 1];
}
// one merge round of two sorted runs of n/2 (merge-path, per-thread ranges)
template <int PF>
__global__ void __launch_bounds__(128, 1) km(const u32* gk, const u64* gp, u32 n, int reps, long long* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  u64* P = reinterpret_cast<u64*>(sm);
  u64* TP = P + 4096;
  u32* K = reinterpret_cast<u32*>(TP + 4096);
  u32* TK = K + 4096;
  constexpr u32 NT = 128;
  const u32 tid = threadIdx.x;
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (u32 i = tid; i < n; i += 128) { K[i] = gk[i]; P[i] = gp[i]; }
    __syncthreads();
    cta_sort<4>(K, P, n / 2, TK, TP);
    cta_sort<4>(K + n / 2, P + n / 2, n / 2, TK, TP);
    __syncthreads();
    long long t0 = clock64();
    const u32 M = n, wr = n / 2;
    const u32 per = ((M + NT - 1) / NT) | 1u;
    u32* dk = TK; u64* dp = TP; const u32* sk = K; const u64* sp = P;
    for (u32 o = tid * per, oend = min(o + per, M); o < oend;) {
      const u32 base = (o / (2 * wr)) * 2 * wr;
      const u32 cnt = min(oend, base + 2 * wr) - o;
      const u32 d = o - base;
      const u32* ak = sk + base; const u64* ap = sp + base;
      const u32* bk = sk + base + wr; const u64* bp = sp + base + wr;
      u32 lo = d > wr ? d - wr : 0, hi = d < wr ? d : wr;
      while (lo < hi) {
        const u32 m = (lo + hi) >> 1;
        if (less_pk(ap[m], ak[m], bp[d - 1 - m], bk[d - 1 - m])) lo = m + 1; else hi = m;
      }
      long long t1 = clock64();
      if (PF == 2) { if (tid == 0) out[2] += t1 - t0; }
      u32 x = lo, y = d - lo;
      u64 xa = x < wr ? ap[x] : ~0ull, yb = y < wr ? bp[y] : ~0ull;
      u32 xk = x < wr ? ak[x] : 0xffffffffu, yk = y < wr ? bk[y] : 0xffffffffu;
      for (u32 v = 0; v < cnt; ++v) {
        const bool ta = y >= wr || (x < wr && less_pk(xa, xk, yb, yk));
        if (PF != 1) { dk[o + v] = ta ? xk : yk; dp[o + v] = ta ? xa : yb; }
        x += ta; y += !ta;
        const u32 i = ta ? x : y;
        const bool in = i < wr;
        const u64 np = in ? (ta ? ap : bp)[i] : ~0ull;
        const u32 nk = in ? (ta ? ak : bk)[i] : 0xffffffffu;
        xa = ta ? np : xa; xk = ta ? nk : xk; yb = ta ? yb : np; yk = ta ? yk : nk;
      }
      if (PF == 1) { dk[o] = xk; dp[o] = xa; }
      o += cnt;
    }
    __syncthreads();
    tot += clock64() - t0;
  }
  if (threadIdx.x == 0) out[0] = tot / reps;
  if (threadIdx.x == 0) out[1] = TK[0] + TP[n - 1];
}
int main() {
  const u32 n = 4096;
  u32* hk = new u32[n]; u64* hp = new u64[n];
  unsigned long long x = 88172645463325252ull;
  for (u32 i = 0; i < n; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; hk[i] = i; hp[i] = x >> 20; }
  u32* dk; u64* dp; long long* d;
  cudaMalloc(&dk, n * 4); cudaMalloc(&dp, n * 8); cudaMalloc(&d, 32);
  cudaMemcpy(dk, hk, n * 4, cudaMemcpyHostToDevice); cudaMemcpy(dp, hp, n * 8, cudaMemcpyHostToDevice);
  const int smem = 4096 * 24;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h[2];
  for (u32 m = 128; m <= 4096; m <<= 1) {
    k<0><<<1, 128, smem>>>(dk, dp, m, 50, d); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("cta_sort %u: %lld cycles\n", m, h[0]);
  }
  k<1><<<1, 128, smem>>>(dk, dp, n, 50, d); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("phase1 R=1:   %lld cycles\n", h[0]);
  k<2><<<1, 128, smem>>>(dk, dp, n, 50, d); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("phase1 R=2:   %lld cycles\n", h[0]);
  cudaFuncSetAttribute(km<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(km<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(km<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  km<0><<<1, 128, smem>>>(dk, dp, n, 20, d); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("merge round 4096: %lld cycles\n", h[0]);
  km<1><<<1, 128, smem>>>(dk, dp, n, 20, d); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("merge round, no stores: %lld cycles\n", h[0]);
  long long h3[3] = {0,0,0}; cudaMemcpy(d, h3, 24, cudaMemcpyHostToDevice);
  km<2><<<1, 128, smem>>>(dk, dp, n, 20, d); cudaMemcpy(h3, d, 24, cudaMemcpyDeviceToHost); printf("merge round: %lld cycles, search (thread 0) %lld\n", h3[0], h3[2] / 20);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
