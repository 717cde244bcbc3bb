// Micro-benchmark of the SSSP round skeleton: per-iteration cycles of
// warp argmin + STS + bar.sync + combine, with optional extras (dev aid).
#include <cstdio>
#include <cstdint>
typedef unsigned long long u64;
typedef unsigned u32;
struct Off { u64 p; u32 k, has; };
template <int MODE>
__global__ void k(u64* g, u32* gi, u32* gt, long long* out, int iters) {
  __shared__ Off ex[2][4];
  __shared__ u32 pf[256];
  const u32 tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  u64 acc = tid * 7919ull;
  u32 par = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE & 8) {  // wait for last iteration's cp.async and consume
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      acc += pf[tid];
    }
    u64 p = acc ^ (u64)it * 0x9E3779B97F4A7C15ull;
    if (MODE & 2) {  // L1-resident gather (sliding window)
      const uint4 v = __ldca(reinterpret_cast<const uint4*>(gi) + ((it + tid) & 1023));
      p += v.x;
    }
    if (MODE & 16) {  // dependent chain of 20 ALU ops
#pragma unroll
      for (int i = 0; i < 20; ++i) p = p * 3 + (p >> 7);
    }
    u32 k = tid;
    const u32 hi = (u32)(p >> 32);
    const u32 mhi = __reduce_min_sync(~0u, hi);
    const u32 lo = hi == mhi ? (u32)p : ~0u;
    const u32 mlo = __reduce_min_sync(~0u, lo);
    const u32 mk = __reduce_min_sync(~0u, (hi == mhi && (u32)p == mlo) ? k : ~0u);
    if (lane == 0) { ex[par][w].p = ((u64)mhi << 32) | mlo; ex[par][w].k = mk; ex[par][w].has = 1; }
    if ((MODE & 1) && tid == (u32)(it & 127)) {  // one global 16 B store per iteration
      reinterpret_cast<uint4*>(g)[it & 4095] = make_uint4(it, tid, 0, 0);
    }
    __syncthreads();
    u64 bp = ex[par][0].p; u32 bk = ex[par][0].k;
#pragma unroll
    for (int i = 1; i < 4; ++i) {
      const u64 xp = ex[par][i].p; const u32 xk = ex[par][i].k;
      if (xp < bp || (xp == bp && xk < bk)) { bp = xp; bk = xk; }
    }
    acc += bp + bk;
    par ^= 1;
    if (MODE & 8) {  // next "row" copy
      const u32* src = gt + ((u64)(bk & 1023) * 256 + ((tid + it) & 255));
      const unsigned sa = (unsigned)__cvta_generic_to_shared(&pf[tid]);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(src) : "memory");
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = t1 - t0;
  if (acc == 42) out[1] = acc;
}
template <int M>
void run(const char* name, u64* g, u32* gi, u32* gt, long long* d) {
  const int iters = 200000;
  k<M><<<1, 128>>>(g, gi, gt, d, 1000);
  k<M><<<1, 128>>>(g, gi, gt, d, iters);
  long long h[2];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("%-40s %8.1f cycles/iter\n", name, (double)h[0] / iters);
}
int main() {
  u64* g; u32 *gi, *gt; long long* d;
  cudaMalloc(&g, 1 << 20); cudaMalloc(&gi, 1 << 20); cudaMalloc(&gt, 1 << 22); cudaMalloc(&d, 64);
  cudaMemset(gi, 0, 1 << 20); cudaMemset(gt, 0, 1 << 22);
  run<0>("argmin+bar+combine", g, gi, gt, d);
  run<1>("+ 1 global store", g, gi, gt, d);
  run<2>("+ L1 gather", g, gi, gt, d);
  run<8>("+ cp.async row (wait next iter)", g, gi, gt, d);
  run<16>("+ 20-op chain", g, gi, gt, d);
  run<11>("store+gather+cp.async", g, gi, gt, d);
  run<27>("all", g, gi, gt, d);
  return 0;
}
