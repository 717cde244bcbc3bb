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
int main() {
  const u32 n = 4096;
  u32* hk = new u32[n]; u64* hp = new u64[n];
  unsigned long long x = 88172645463325252ull;
  for (u32 i = 0; i < n; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; hk[i] = i; hp[i] = x >> 20; }
  u32* dk; u64* dp; long long* d;
  cudaMalloc(&dk, n * 4); cudaMalloc(&dp, n * 8); cudaMalloc(&d, 16);
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
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
