// pbh-b200 host runtime: implements include/pbh_gpu.h over the kernels of
// pbh_kernels.cuh. Owns device memory (levels, position index, staging),
// launch configuration, the NEED_GROW resume loop and error mapping.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <map>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pbh_gpu.h"
#include "pbh_bank.cuh"
#include "pbh_bf.cuh"
#include "pbh_multi.cuh"
#include "pbh_gen_gpu.cuh"
#include "pbh_csr.cuh"
#include "../../include/pbh_gen.h"

using namespace pbh_dev;

namespace {

thread_local std::string g_last_error;
std::atomic<unsigned long long> g_launches{0};  // kernels launched by this library

pbh_status set_err(pbh_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return set_err(e_ == cudaErrorMemoryAllocation ? PBH_OOM : PBH_CUDA,              \
                     std::string(#call) + ": " + cudaGetErrorString(e_));               \
  } while (0)

constexpr int VT = 4;
constexpr u32 kOorCap = 4096;  // remembered out-of-index deletes per heap
constexpr size_t kTmaSlack = 64;  // bytes past each merge buffer (TMA window over-read)
constexpr u32 kInlineOpMax = PBH_INLINE_OP_MAX;  // single ops up to this many elements read from mapped host memory
constexpr u64 kSoloMax = 1ull << 16;  // single ops on one CTA while fewer entries were inserted
constexpr u64 kPersistIdleNs = 200000;
static_assert(offsetof(pbh_op_channel, rq) % 16 == 0 && offsetof(pbh_op_channel, rs) % 16 == 0,
              "flagged channel words are read / written as 16-byte pairs");  // a persistent single-op kernel exits after 200 us idle

u64 pow2_at_least(u64 x) {
  u64 p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Per-device launch attributes: the dynamic shared-memory opt-in is a
// per-device property, and the cooperative grid size depends on the device.
std::mutex g_attr_mu;
std::map<std::pair<const void*, int>, int> g_grid_of;  // (kernel, device) -> grid

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

// Banked op-trace interpreter (pbh_bank.cuh): 4 warps, level 0 = 1024 slots.
#ifndef PBH_TRACE_NW
#define PBH_TRACE_NW 8
#endif
constexpr int kTraceNW = PBH_TRACE_NW;
constexpr int kTraceKI = 1024 / (32 * kTraceNW);  // level 0 = 1024 slots
using TraceImage = BankL0<32 * kTraceNW, kTraceKI>;
using TraceSmem = TraceBankSmem<kTraceNW, kTraceKI, VT>;

cudaError_t launch_trace_bank(cudaStream_t st, pbh_heap_dev* g, pbh_trace_dev tr, u64 b, u64 e,
                              u32* ov, u64* op, pbh_kstatus* ks, TraceImage* save, u32 internal,
                              GridJob* gj, u32 grid_min, unsigned long long* prof,
                              BatchJob* bj, bool solo, pbh_op_channel* pm = nullptr) {
  auto fn = k_trace_bank<kTraceNW, kTraceKI, VT>;
  const int smem = (int)sizeof(TraceSmem);
  cudaError_t err = cudaSuccess;
  int G = 0;
  {
    // per device, once: the shared-memory opt-in and the co-resident grid
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(g_attr_mu);
    int& gc = g_grid_of[{(const void*)fn, dev}];
    if (gc == 0) {
      err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (err != cudaSuccess) return err;
      int sms = 0, per_sm = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * kTraceNW, smem);
      gc = std::max(1, sms * std::min(per_sm, 1));
    }
    G = gc;
  }
  if (gj && G > 1 && !solo) {
    // the job word and the job-barrier counter restart with every launch
    err = cudaMemsetAsync(gj, 0, sizeof(GridJob), st);
    if (err != cudaSuccess) return err;
    void* args[] = {&g, &tr, &b, &e, &ov, &op, &ks, &save, &internal, &gj, &grid_min, &prof, &bj, &pm};
    err = cudaLaunchCooperativeKernel((const void*)fn, dim3(G), dim3(32 * kTraceNW), args, smem, st);
  } else {
    fn<<<1, 32 * kTraceNW, smem, st>>>(g, tr, b, e, ov, op, ks, save, internal, gj, grid_min,
                                       prof, nullptr, pm);
    err = cudaGetLastError();
  }
  g_launches++;
  return err;
}

// Banked level-0 SSSP engine variants: NW warps per source, KI slots per
// thread, level 0 = 32*NW*KI = 1024 slots.
template <int NW>
struct BankCfg;
template <>
struct BankCfg<1> { static constexpr int KI = 32; };
template <>
struct BankCfg<2> { static constexpr int KI = 16; };
template <>
struct BankCfg<4> { static constexpr int KI = 8; };
template <>
struct BankCfg<8> { static constexpr int KI = 4; };
constexpr int kBankC0 = 1024;
constexpr u32 kMultiCap0 = kBankC0 * PBH_MULTI_B0_EIGHTHS / 8;  // threshold engine's B_0 (BankSmem<..., true>::B0CAP)
static_assert(kMultiCap0 == (u32)BankSmem<4, 8, VT, true>::B0CAP, "threshold B_0 capacity");
static_assert(kBankC0 / 2 == BankSmem<4, 8, VT, false>::B0CAP, "exact B_0 capacity");

template <int NW>
size_t bank_save_bytes() {
  return sizeof(BankL0<32 * NW, BankCfg<NW>::KI>);
}
size_t bank_save_bytes_nw(int nw) {
  return nw <= 1 ? bank_save_bytes<1>() : nw == 2 ? bank_save_bytes<2>()
         : nw == 4 ? bank_save_bytes<4>() : bank_save_bytes<8>();
}

template <int NW, int PASS = kBankPass>
cudaError_t launch_sssp_bank(cudaStream_t st, u32 grid, pbh_heap_dev* heaps, const u64* off,
                             const u32* tgt, const u32* w, u32 V, const u32* src, u64* dist,
                             u32* settled, SsspState* sst, void* save, u32 dag, u32 maxdeg, u32 d) {
  constexpr int KI = BankCfg<NW>::KI;
  auto fn = k_sssp_bank<NW, KI, VT, PASS>;
  const int smem = (int)sizeof(BankSmem<NW, KI, VT>);
  // per launch: the attribute is per device, and the call is cheap
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  static unsigned long long* prof = nullptr;
  if (getenv("PBH_PHASES") && !prof && cudaMalloc(&prof, 64 * 8) == cudaSuccess) cudaMemset(prof, 0, 64 * 8);
  fn<<<grid, 32 * NW, smem, st>>>(heaps, off, tgt, w, V, src, dist, settled, sst,
                                  reinterpret_cast<BankL0<32 * NW, KI>*>(save), dag, maxdeg, d,
                                  prof);
  if (prof) {
    unsigned long long pc[64];
    cudaMemcpy(pc, prof, 64 * 8, cudaMemcpyDeviceToHost);
    cudaMemset(prof, 0, 64 * 8);
#ifdef PBH_XPROF
    unsigned long long xp[16];
    cudaMemcpyFromSymbol(xp, g_xprof, sizeof xp);
    if (xp[6]) fprintf(stderr, "exchange skew (block 0): last-first %.0f release %.0f  >1000cyc %.3f  last warp %llu %llu %llu %llu\n",
                       (double)xp[4] / xp[6], (double)xp[5] / xp[6], (double)xp[7] / xp[6], xp[8], xp[9], xp[10], xp[11]);
    unsigned long long z[16] = {}, x2[8];
    cudaMemcpyFromSymbol(x2, g_xprof2, sizeof x2);
    if (xp[6]) fprintf(stderr, "last warp excess per phase (top pre-row row gather apply exch tail rescan): %.0f %.0f %.0f %.0f %.0f %.0f %.0f %.0f\n",
                       (double)(long long)x2[0] / xp[6], (double)(long long)x2[1] / xp[6], (double)(long long)x2[2] / xp[6],
                       (double)(long long)x2[3] / xp[6], (double)(long long)x2[4] / xp[6], (double)(long long)x2[5] / xp[6],
                       (double)(long long)x2[6] / xp[6], (double)(long long)x2[7] / xp[6]);
    cudaMemcpyToSymbol(g_xprof, z, sizeof z);
    cudaMemcpyToSymbol(g_xprof2, z, sizeof x2);
    if (xp[3]) fprintf(stderr, "exchange per call (warp leaders, block 0): reduce %.0f barrier %.0f combine %.0f (n=%llu)\n",
                       (double)xp[0] / xp[3], (double)xp[1] / xp[3], (double)xp[2] / xp[3], xp[3]);
#endif
    for (int w = 0; w < NW; ++w)
      fprintf(stderr, "bank phases warp %d (cycles, source 0): top %llu pre-row %llu row %llu gather %llu apply %llu exchange %llu tail %llu\n",
              w, pc[w * 8 + 0], pc[w * 8 + 1], pc[w * 8 + 2], pc[w * 8 + 3], pc[w * 8 + 4], pc[w * 8 + 5], pc[w * 8 + 6]);
  }
  g_launches++;
  return cudaGetLastError();
}

// Threshold multi-extraction engine (opt-in, pbh_multi.cuh): NW = 4.
using MultiImage = BankL0<128, 8, true>;
cudaError_t launch_sssp_multi(cudaStream_t st, u32 grid, pbh_heap_dev* heaps, const u64* off,
                              const u32* tgt, const u32* w, const u32* mwo, const u32* mwi, u32 V,
                              const u32* src, u64* dist, u32* settled, SsspState* sst, void* save,
                              u32 maxdeg, u32 d) {
  auto fn = k_sssp_multi<4, 8, VT>;
  const int smem = (int)sizeof(MultiSmem<4, 8, VT>);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  fn<<<grid, 128, smem, st>>>(heaps, off, tgt, w, mwo, mwi, V, src, dist, settled, sst,
                              reinterpret_cast<MultiImage*>(save), maxdeg, d);
  g_launches++;
  return cudaGetLastError();
}

cudaError_t launch_sssp_bank_nw(int nw, cudaStream_t st, u32 grid, pbh_heap_dev* heaps,
                                const u64* off, const u32* tgt, const u32* w, u32 V,
                                const u32* src, u64* dist, u32* settled, SsspState* sst,
                                void* save, u32 dag, u32 maxdeg, u32 d) {
  switch (nw) {
    case 0:  // one warp, 32-edge passes: low-degree graphs
      return launch_sssp_bank<1, 32>(st, grid, heaps, off, tgt, w, V, src, dist, settled, sst, save, dag, maxdeg, d);
    case 1: return launch_sssp_bank<1>(st, grid, heaps, off, tgt, w, V, src, dist, settled, sst, save, dag, maxdeg, d);
    case 2: return launch_sssp_bank<2>(st, grid, heaps, off, tgt, w, V, src, dist, settled, sst, save, dag, maxdeg, d);
    case 4:
      // low-degree graphs (grids): one edge per thread per pass of 128
      if (maxdeg <= 128)
        return launch_sssp_bank<4, 128>(st, grid, heaps, off, tgt, w, V, src, dist, settled, sst, save, dag, maxdeg, d);
      return launch_sssp_bank<4>(st, grid, heaps, off, tgt, w, V, src, dist, settled, sst, save, dag, maxdeg, d);
    default: return launch_sssp_bank<8>(st, grid, heaps, off, tgt, w, V, src, dist, settled, sst, save, dag, maxdeg, d);
  }
}

__global__ void k_finalize_parent(const pbh_idx_entry* idx, u32 V, u32* parent) {
  for (u64 v = blockIdx.x * (u64)blockDim.x + threadIdx.x; v < V; v += (u64)gridDim.x * blockDim.x) {
    const pbh_idx_entry e = idx[v];
    parent[v] = PBH_ST(e.state) == PBH_ST_DEAD ? e.parent : 0xffffffffu;
  }
}


const char* detail_message(u32 detail) {
  switch (detail) {
    case PBH_ERR_EMPTY_HEAP: return "extract_min: heap is empty";
    case PBH_ERR_EMPTY_BATCH: return "bulk_update: empty batch";
    case PBH_ERR_BATCH_TOO_BIG: return "bulk_update: batch larger than d (or the 2^26-element batch limit)";
    case PBH_ERR_UNSORTED: return "bulk_update: batch must be value-sorted with unique values";
    case PBH_ERR_REINSERT: return "update: value was already extracted or deleted; re-insertion is unsupported";
    case PBH_ERR_INCREASE: return "update: priority increase";
    case PBH_ERR_INVARIANT: return "internal invariant violated";
    case PBH_ERR_OVERFLOW: return "sssp: distance accumulation overflow";
    case PBH_ERR_KEY_RANGE: return "update: value outside the position index";
    case PBH_ERR_BAD_OP: return "unknown op kind";
    default: return "error";
  }
}

// ----------------------------------------------------------- device heap
// One heap's device allocations. Used by pbh_heap (one) and SSSP contexts
// (one per source slot).
struct DevHeap {
  pbh_heap_dev hd{};     // host mirror of the header (pointers + caps)
  pbh_heap_dev* dev = nullptr;  // header in HBM (standalone) or slot in an array
  std::vector<void*> allocs;
  u32 bc = 0;     // batch capacity (pow2)
  u64 base1 = 0;  // level-1 bucket capacity (level i >= 1: base1 * 4^(i-1))
  bool bank = false;  // banked level 0 (stages kBankQ-entry push runs in g_pk/g_pp)

  // Optional arena (one cudaMalloc for many heaps: an SSSP context holds
  // one heap per source), and a measuring mode that only sums the sizes.
  char* arena = nullptr;
  size_t arena_cap = 0, arena_used = 0;
  bool measure = false;
  size_t measured = 0;
  static size_t a256(size_t b) { return (std::max<size_t>(b, 16) + 255) & ~size_t(255); }

  // Every buffer gets kTmaSlack bytes past its end: 16-byte-aligned TMA
  // windows over a run ending at the buffer end read up to 15 bytes beyond.
  pbh_status alloc(void** p, size_t bytes) {
    bytes += kTmaSlack;
    const size_t b = a256(bytes);
    if (measure) {
      measured += b;
      *p = reinterpret_cast<void*>(size_t(256));
      return PBH_OK;
    }
    if (arena && arena_used + b <= arena_cap) {
      *p = arena + arena_used;
      arena_used += b;
      return PBH_OK;
    }
    CK(cudaMalloc(p, bytes ? bytes : 16));
    allocs.push_back(*p);
    return PBH_OK;
  }
  void free_all() {
    for (void* p : allocs) cudaFree(p);
    allocs.clear();
  }
};

pbh_status alloc_level(DevHeap& H, u32 i) {
  pbh_level_bufs& b = H.hd.lv[i];
  const u64 cap = i == 0 ? H.hd.cap0 : (u64)H.base1 << (2 * (i - 1));
  if (cap >= (1ull << 31)) return set_err(PBH_OOM, "level capacity exceeds the 2^31 element limit");
  b.cap_b = (u32)cap;
  b.buf_s = i == 0 ? 0 : (u32)cap;
  for (int s = 0; s < 2; ++s) {
    pbh_status st;
    if ((st = H.alloc((void**)&b.bk[s], cap * 4))) return st;
    if ((st = H.alloc((void**)&b.bp[s], cap * 8))) return st;
    if (i > 0) {
      if ((st = H.alloc((void**)&b.sk[s], (u64)b.buf_s * 4))) return st;
      if ((st = H.alloc((void**)&b.sp[s], (u64)b.buf_s * 8))) return st;
    } else {
      b.sk[s] = nullptr;
      b.sp[s] = nullptr;
    }
  }
  pbh_level_state& t = H.hd.st[i];
  t = pbh_level_state{};
  t.spl_inf = 1;
  H.hd.n_levels = std::max<u32>(H.hd.n_levels, i + 1);
  return PBH_OK;
}

pbh_status alloc_scratch(DevHeap& H, u32 bc, u32 nt, cudaStream_t strm = 0) {
  pbh_status st;
  H.bc = bc;
  // the banked engines stage push-buffer runs (kBankQ entries) in g_pk/g_pp
  if (H.bank) bc = std::max<u32>(bc, kBankQ);
  if ((st = H.alloc((void**)&H.hd.g_bk, (u64)bc * 4))) return st;
  if ((st = H.alloc((void**)&H.hd.g_bp, (u64)bc * 8))) return st;
  if ((st = H.alloc((void**)&H.hd.g_pk, (u64)bc * 4))) return st;
  if ((st = H.alloc((void**)&H.hd.g_pp, (u64)bc * 8))) return st;
  if ((st = H.alloc((void**)&H.hd.g_rm, H.hd.cap0))) return st;
  if (!H.measure) CK(cudaMemsetAsync(H.hd.g_rm, 0, H.hd.cap0, strm));
  const u64 cc = (u64)H.hd.d + nt;
  if ((st = H.alloc((void**)&H.hd.g_ck, cc * 4))) return st;
  if ((st = H.alloc((void**)&H.hd.g_cp, cc * 8))) return st;
  if ((st = H.alloc((void**)&H.hd.g_co, cc * 8))) return st;
  if ((st = H.alloc((void**)&H.hd.g_cs, cc * 4))) return st;
  return PBH_OK;
}

// Initialise a heap: header, n_levels levels, scratch, index of `universe`.
pbh_status init_heap(DevHeap& H, u64 d, u32 cap0, u32 bc, u32 nt, u64 universe, int debug,
                     u32 n_levels, pbh_heap_dev* dev_slot, cudaStream_t strm = 0) {
  std::memset(&H.hd, 0, sizeof(H.hd));
  H.hd.d = (u32)std::min<u64>(d, 0xffffffffu);
  H.hd.cap0 = cap0;
  if (H.base1 == 0) H.base1 = 4ull * cap0;
  H.hd.debug_checks = debug ? 1 : 0;
  for (u32 i = 0; i < PBH_MAX_LEVELS; ++i) H.hd.st[i].spl_inf = 1;
  pbh_status st;
  for (u32 i = 0; i < n_levels; ++i)
    if ((st = alloc_level(H, i))) return st;
  if ((st = alloc_scratch(H, bc, nt, strm))) return st;
  H.hd.universe = universe;
  if ((st = H.alloc((void**)&H.hd.idx, universe * sizeof(pbh_idx_entry)))) return st;
  H.hd.oor_cap = kOorCap;
  H.hd.oor_n = 0;
  if ((st = H.alloc((void**)&H.hd.oor_del, kOorCap * sizeof(u32)))) return st;
  if (dev_slot) {
    H.dev = dev_slot;
  } else {
    if ((st = H.alloc((void**)&H.dev, sizeof(pbh_heap_dev)))) return st;
  }
  if (H.measure) return PBH_OK;
  CK(cudaMemsetAsync(H.hd.idx, 0xff, universe * sizeof(pbh_idx_entry), strm));
  CK(cudaMemcpyAsync(H.dev, &H.hd, sizeof(pbh_heap_dev), cudaMemcpyHostToDevice, strm));
  if (strm == 0) CK(cudaStreamSynchronize(0));
  return PBH_OK;
}

__global__ void k_mark_dead(pbh_idx_entry* idx, u64 universe, const u32* keys, u32 n) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (keys[i] < universe) idx[keys[i]].state = PBH_ST_DEAD;
}

// Pull the mutable header back, add one level, push it again.
pbh_status grow_levels(DevHeap& H, cudaStream_t s) {
  CK(cudaMemcpyAsync(&H.hd, H.dev, sizeof(pbh_heap_dev), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (H.hd.n_levels >= PBH_MAX_LEVELS) return set_err(PBH_OOM, "level limit reached");
  pbh_status st = alloc_level(H, H.hd.n_levels);
  if (st) return st;
  CK(cudaMemcpyAsync(H.dev, &H.hd, sizeof(pbh_heap_dev), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  return PBH_OK;
}

pbh_status grow_universe(DevHeap& H, cudaStream_t s, u64 want) {
  CK(cudaMemcpyAsync(&H.hd, H.dev, sizeof(pbh_heap_dev), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (want <= H.hd.universe) return PBH_OK;
  u64 nu = std::max<u64>(pow2_at_least(want), 2 * H.hd.universe);
  nu = std::min<u64>(nu, 1ull << 32);
  pbh_idx_entry* ni = nullptr;
  CK(cudaMalloc(&ni, nu * sizeof(pbh_idx_entry)));
  CK(cudaMemsetAsync(ni, 0xff, nu * sizeof(pbh_idx_entry), s));
  CK(cudaMemcpyAsync(ni, H.hd.idx, H.hd.universe * sizeof(pbh_idx_entry),
                     cudaMemcpyDeviceToDevice, s));
  CK(cudaStreamSynchronize(s));
  auto it = std::find(H.allocs.begin(), H.allocs.end(), (void*)H.hd.idx);
  if (it != H.allocs.end()) {
    cudaFree(*it);
    *it = ni;
  }
  H.hd.idx = ni;
  H.hd.universe = nu;
  // deletes recorded beyond the old index: the values they cover are DEAD
  if (H.hd.oor_n) {
    k_mark_dead<<<1, 256, 0, s>>>(ni, nu, H.hd.oor_del, H.hd.oor_n);
    g_launches++;
    std::vector<u32> keep(H.hd.oor_n);
    CK(cudaMemcpyAsync(keep.data(), H.hd.oor_del, keep.size() * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    keep.erase(std::remove_if(keep.begin(), keep.end(), [&](u32 k) { return k < nu; }), keep.end());
    if (!keep.empty())
      CK(cudaMemcpyAsync(H.hd.oor_del, keep.data(), keep.size() * 4, cudaMemcpyHostToDevice, s));
    H.hd.oor_n = (u32)keep.size();
  }
  CK(cudaMemcpyAsync(H.dev, &H.hd, sizeof(pbh_heap_dev), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  return PBH_OK;
}

}  // namespace

// =========================================================================
// heap handle
// =========================================================================
struct pbh_heap {
  int device = 0;
  cudaStream_t stream = nullptr;
  u64 d = 1;
  int nt = 32;
  DevHeap H;
  pbh_kstatus* d_ks = nullptr;  // device view of h_ks
  pbh_kstatus* h_ks = nullptr;  // status block in mapped pinned host memory (written by the kernel)
  // single ops (the Engine's per-call API): their inputs and outputs live in
  // mapped pinned host memory the kernel reads / writes directly (no copies)
  pbh_op_channel* h_mop = nullptr;
  pbh_op_channel* d_mop = nullptr;
  // persistent single-op kernel (pbh_heap_set_persistent): resident while
  // `alive`, `seq` requests posted so far, launched as one CTA if `alive_solo`
  u64 persist_idle_ns = kPersistIdleNs;
  bool alive = false;
  bool alive_solo = false;
  u64 seq = 0;
  u64 persist_reqs = 0;     // requests served by resident kernels
  u64 persist_launches = 0; // resident kernels launched
  // entries inserted so far (an upper bound of what the heap stores): while
  // small, single ops launch one CTA (their merges are short) instead of
  // the cooperative grid
  u64 inserted = 0;
  GridJob* d_job = nullptr;     // grid-helper job word (null: single-CTA engine)
  TraceImage* d_save = nullptr; // its level-0 image between launches
  u32 grid_min = kGridMin;
  unsigned long long* d_prof = nullptr;  // PBH_PROF: leader cycle breakdown
  BatchJob* d_batch = nullptr;           // grid sort job (large batches, push-buffer flushes)
  // staging for host traces
  u64 st_ops = 0, st_el = 0, st_out = 0;
  u8* d_kinds = nullptr;
  u64* d_off = nullptr;
  u32* d_vals = nullptr;
  u64* d_prios = nullptr;
  u32* d_ov = nullptr;
  u64* d_op = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

namespace {

pbh_status ensure_staging(pbh_heap* h, u64 n_ops, u64 n_el, u64 n_out) {
  n_ops = std::max<u64>(n_ops, 1);
  n_el = std::max<u64>(n_el, 1);
  n_out = std::max<u64>(n_out, 1);
  if (n_ops > h->st_ops) {
    cudaFree(h->d_kinds);
    cudaFree(h->d_off);
    h->st_ops = std::max<u64>(pow2_at_least(n_ops), 64);
    CK(cudaMalloc(&h->d_kinds, h->st_ops));
    CK(cudaMalloc(&h->d_off, (h->st_ops + 1) * 8));
  }
  if (n_el > h->st_el) {
    cudaFree(h->d_vals);
    cudaFree(h->d_prios);
    h->st_el = std::max<u64>(pow2_at_least(n_el), 64);
    CK(cudaMalloc(&h->d_vals, h->st_el * 4));
    CK(cudaMalloc(&h->d_prios, h->st_el * 8));
  }
  if (n_out > h->st_out) {
    cudaFree(h->d_ov);
    cudaFree(h->d_op);
    h->st_out = std::max<u64>(pow2_at_least(n_out), 64);
    CK(cudaMalloc(&h->d_ov, h->st_out * 4));
    CK(cudaMalloc(&h->d_op, h->st_out * 8));
  }
  return PBH_OK;
}

// Stop a resident persistent single-op kernel (its level-0 image and heap
// state are saved when it exits): every path that launches another kernel
// on the heap or reads its device state calls this first.
pbh_status quiesce(pbh_heap* h) {
  if (!h->alive) return PBH_OK;
  h->alive = false;
  h->h_mop->stop = 1;
  const cudaError_t e = cudaStreamSynchronize(h->stream);
  h->h_mop->stop = 0;
  if (e != cudaSuccess) return set_err(PBH_CUDA, cudaGetErrorString(e));
  return PBH_OK;
}

// Run ops [0, n_ops) of a device trace with the NEED_GROW / KEY_RANGE resume
// loop. host_vals: host copy of the values (for universe growth) or null.
pbh_status exec_trace(pbh_heap* h, u64 n_ops, pbh_trace_dev tr, u32* d_ov, u64* d_op,
                      u64* n_out, u64* failed_op, u32 internal, double* wall_ms,
                      const u8* host_kinds, const u64* host_off, const u32* host_vals,
                      bool solo = false) {
  if (pbh_status q = quiesce(h)) return q;
  // the status block is mapped host memory: the stream is idle between
  // calls, so the host resets it directly and reads the kernel's writes
  // after the synchronize
  std::memset(h->h_ks, 0, sizeof(pbh_kstatus));
  u64 begin = 0;
  double ms_total = 0;
  for (int guard = 0; guard < 4096; ++guard) {
    if (begin >= n_ops) break;
    if (wall_ms) CK(cudaEventRecord(h->ev0, h->stream));
    CK(launch_trace_bank(h->stream, h->H.dev, tr, begin, n_ops, d_ov, d_op, h->d_ks, h->d_save,
                         internal, h->d_job, h->grid_min, h->d_prof, h->d_batch, solo));
    if (wall_ms) CK(cudaEventRecord(h->ev1, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (wall_ms) {
      float ms = 0;
      cudaEventElapsedTime(&ms, h->ev0, h->ev1);
      ms_total += ms;
    }
    const pbh_kstatus ks = *h->h_ks;  // written by the kernel; visible after the synchronize
    if (ks.status == 0) break;
    if (ks.status == 7) {  // NEED_GROW
      pbh_status st = grow_levels(h->H, h->stream);
      if (st) return st;
      begin = ks.failed_op;
      h->h_ks->status = 0;
      continue;
    }
    if (ks.detail == PBH_ERR_KEY_RANGE) {
      // grow the index to cover every key of the failing op
      const u64 op = ks.failed_op;
      u64 b, e;
      std::vector<u32> v;
      if (host_off) {
        b = host_off[op];
        e = host_off[op + 1];
        v.assign(host_vals + b, host_vals + e);
      } else {
        u64 be[2];
        CK(cudaMemcpy(be, tr.offsets + op, 16, cudaMemcpyDeviceToHost));
        b = be[0];
        e = be[1];
        v.resize(e - b);
        CK(cudaMemcpy(v.data(), tr.vals + b, (e - b) * 4, cudaMemcpyDeviceToHost));
      }
      u64 mx = 0;
      for (u32 x : v) mx = std::max<u64>(mx, x);
      pbh_status st = grow_universe(h->H, h->stream, mx + 1);
      if (st) return st;
      begin = op;
      h->h_ks->status = 0;
      continue;
    }
    if (n_out) *n_out = ks.n_out;
    if (failed_op) *failed_op = ks.failed_op;
    if (wall_ms) *wall_ms = ms_total;
    char buf[64];
    std::snprintf(buf, sizeof buf, "op %llu: ", (unsigned long long)ks.failed_op);
    return set_err(ks.status == 1 ? PBH_EMPTY : ks.status == 3 ? PBH_INVARIANT : PBH_PRECONDITION,
                   std::string(buf) + detail_message(ks.detail));
  }
  if (n_out) *n_out = h->h_ks->n_out;
  if (failed_op) *failed_op = ~0ull;
  if (wall_ms) *wall_ms = ms_total;
  return PBH_OK;
}

// Run a small host-side trace through the staging buffers.
pbh_status exec_host(pbh_heap* h, u64 n_ops, const u8* kinds, const u64* off, const u32* vals,
                     const u64* prios, u32* out_v, u64* out_p, u64* n_out, u64* failed_op,
                     u32 internal, double* wall_ms) {
  const u64 n_el = off[n_ops];
  u64 n_x = 0;
  u64 max_batch = 0;
  for (u64 i = 0; i < n_ops; ++i) {
    n_x += kinds[i] == 'E' || kinds[i] == 'F';
    if (kinds[i] == 'B') max_batch = std::max<u64>(max_batch, off[i + 1] - off[i]);
  }
  (void)max_batch;
  pbh_status st;
  if ((st = ensure_staging(h, n_ops, n_el, n_x))) return st;
  CK(cudaMemcpyAsync(h->d_kinds, kinds, n_ops, cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemcpyAsync(h->d_off, off, (n_ops + 1) * 8, cudaMemcpyHostToDevice, h->stream));
  if (n_el) {
    CK(cudaMemcpyAsync(h->d_vals, vals, n_el * 4, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->d_prios, prios, n_el * 8, cudaMemcpyHostToDevice, h->stream));
  }
  pbh_trace_dev tr{h->d_kinds, h->d_off, h->d_vals, h->d_prios};
  u64 got = 0;
  h->inserted += n_el;
  pbh_status rs = exec_trace(h, n_ops, tr, h->d_ov, h->d_op, &got, failed_op, internal, wall_ms,
                             kinds, off, vals);
  if (n_out) *n_out = got;
  if (got && out_v) {
    CK(cudaMemcpyAsync(out_v, h->d_ov, got * 4, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(out_p, h->d_op, got * 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  }
  return rs;
}

// PBH_PROF builds: print and reset the leader's cycle breakdown (thread 0
// of the interpreter CTA; categories of k_trace_bank's TPROF / BankHeap::pr).
void prof_report(pbh_heap* h, const char* when) {
  unsigned long long pc[16];
  if (cudaMemcpy(pc, h->d_prof, sizeof pc, cudaMemcpyDeviceToHost) != cudaSuccess) return;
  cudaMemset(h->d_prof, 0, sizeof pc);
  unsigned long long jp[24][2];
  if (cudaMemcpyFromSymbol(jp, g_jobprof, sizeof jp) == cudaSuccess) {
    static const char* names[24] = {"merge", "exit", "validate", "classify", "chunks", "pass",
                                    "check+classify", "bucket_sort", "b:hist", "b:bar1", "b:scatter",
                                    "b:bar2", "b:sort", "leader_wait", "filtered_merge", "flush_merge",
                                    "m:split", "m:stream", "s:tma_wait", "s:merge", "s:store", "-", "-", "-"};
    fprintf(stderr, "pbh_jobprof[%s]:", when);
    for (int i = 0; i < 24; ++i)
      if (jp[i][1]) fprintf(stderr, " %s %llu x %.0f", names[i], jp[i][1], (double)jp[i][0] / jp[i][1]);
    fprintf(stderr, "\n");
    std::memset(jp, 0, sizeof jp);
    cudaMemcpyToSymbol(g_jobprof, jp, sizeof jp);
  }
  fprintf(stderr, "pbh_prof[%s] cycles: validate %llu apply %llu bulk_cold %llu extract %llu refill %llu tail %llu pre %llu big_sort %llu"
          " | sort %llu push_down %llu resolve1 %llu r2 %llu r3 %llu r4 %llu r5 %llu r6+ %llu\n",
          when, pc[0], pc[1], pc[2], pc[3], pc[4], pc[5], pc[6], pc[7], pc[8], pc[9], pc[10], pc[11],
          pc[12], pc[13], pc[14], pc[15]);
}

pbh_status single_op(pbh_heap* h, u8 kind, const u32* vals, const u64* prios, u64 n, u32* ov,
                     u64* op) {
  u64 off[2] = {0, n};
  u64 got = 0;
  pbh_status st = PBH_OK;
  if (n <= kInlineOpMax && !h->d_prof && h->persist_idle_ns) {
    // persistent: post the op to the resident kernel (launched if it is not
    // running) and spin on its acknowledgement
    auto* m = h->h_mop;
    const bool solo = h->inserted + n < kSoloMax;
    if (h->alive && h->alive_solo && !solo)
      if ((st = quiesce(h))) return st;  // grown past one CTA: relaunch on the grid
    // flagged words: payload first, header last (each word validates itself)
    const u32 s = (u32)++h->seq;
    const u64 sq = (u64)s << 32;
    if (n > 1)
      for (u64 i = 0; i < n; ++i) {
        m->rv[i] = sq | vals[i];
        m->rplo[i] = sq | (u32)prios[i];
        m->rphi[i] = sq | (u32)(prios[i] >> 32);
      }
    const u64 p1 = n == 1 ? prios[0] : 0;
    m->rq[1] = sq | (n == 1 ? vals[0] : 0u);
    m->rq[2] = sq | (u32)p1;
    m->rq[3] = sq | (u32)(p1 >> 32);
    m->rq[0] = sq | kind | (u32)(n << 8);
    auto launch = [&]() -> pbh_status {
      if ((st = ensure_staging(h, 1, kInlineOpMax, 1))) return st;
      std::memset(h->h_ks, 0, sizeof(pbh_kstatus));
      m->idle_ns = h->persist_idle_ns;
      pbh_trace_dev tr{h->d_kinds, h->d_off, h->d_vals, h->d_prios};
      CK(launch_trace_bank(h->stream, h->H.dev, tr, 0, 0, h->d_ov, h->d_op, h->d_ks, h->d_save, 1,
                           h->d_job, h->grid_min, nullptr, h->d_batch, solo, h->d_mop));
      h->alive = true;
      h->alive_solo = solo || !h->d_job;
      h->persist_launches++;
      return PBH_OK;
    };
    if (!h->alive && (st = launch())) return st;
    // the kernel exits on its own after idle_ns: a request posted as it left
    // is found unserved on an idle stream and served by a relaunch
    int relaunches = 0;
    u64 r0;
    for (u32 spin = 1; (u32)((r0 = m->rs[0]) >> 32) != s; ++spin) {
      if (spin % 256) continue;
      const cudaError_t q = cudaStreamQuery(h->stream);
      if (q == cudaErrorNotReady) continue;
      if (q != cudaSuccess) {
        h->alive = false;
        return set_err(PBH_CUDA, cudaGetErrorString(q));
      }
      if ((u32)(m->rs[0] >> 32) == s) continue;
      h->alive = false;
      if (++relaunches > 2)
        return set_err(PBH_INVARIANT, "persistent kernel exited without serving the request");
      if ((st = launch())) return st;
    }
    h->persist_reqs++;
    if ((u32)r0 != 0xFFFFFFFFu) {
      if (kind == 'U' || kind == 'B') h->inserted += n;
      got = (u32)r0;
      if ((kind == 'E' || kind == 'F') && got != 1)
        return set_err(PBH_INVARIANT, "extract produced no element");
      if (got) {
        u64 r1, r2, r3;
        do {
          r1 = m->rs[1];
          r2 = m->rs[2];
          r3 = m->rs[3];
        } while ((u32)(r1 >> 32) != s || (u32)(r2 >> 32) != s || (u32)(r3 >> 32) != s);
        if (ov) {
          *ov = (u32)r1;
          *op = (u64)(u32)r2 | (r3 << 32);
        }
      }
      return PBH_OK;
    }
    // a failed op (nothing of it applied): the kernel has exited; the
    // one-shot path below re-runs it with index growth and error reporting
    CK(cudaStreamSynchronize(h->stream));
    h->alive = false;
  }
  if (n <= kInlineOpMax && !h->d_prof) {
    // zero-copy: the op and its elements in mapped host memory, the
    // extraction written straight back there
    auto* m = h->h_mop;
    m->kinds[0] = kind;
    m->off[0] = 0;
    m->off[1] = n;
    if (n) {
      std::memcpy(m->vals, vals, n * 4);
      std::memcpy(m->prios, prios, n * 8);
    }
    pbh_trace_dev tr{h->d_mop->kinds, h->d_mop->off, h->d_mop->vals, h->d_mop->prios};
    const bool solo = h->inserted + n < kSoloMax;
    st = exec_trace(h, 1, tr, h->d_mop->out_v, h->d_mop->out_p, &got, nullptr, 1, nullptr,
                    &kind, off, vals, solo);
    if (kind == 'U' || kind == 'B') h->inserted += n;
    if (got && ov) {
      *ov = const_cast<volatile u32*>(m->out_v)[0];
      *op = const_cast<volatile u64*>(m->out_p)[0];
    }
  } else {
    st = exec_host(h, 1, &kind, off, vals, prios, ov, op, &got, nullptr, 1, nullptr);
  }
  if (st == PBH_OK && (kind == 'E' || kind == 'F') && got != 1)
    return set_err(PBH_INVARIANT, "extract produced no element");
  return st;
}

}  // namespace

extern "C" {

const char* pbh_last_error(void) { return g_last_error.c_str(); }
const char* pbh_version(void) { return "pbh-b200 0.1 (sm_100a)"; }
uint64_t pbh_launch_count(void) { return g_launches.load(); }

pbh_status pbh_heap_create(uint64_t d, uint64_t key_universe, int device, int debug_checks,
                           pbh_heap** out) {
  if (!out) return set_err(PBH_PRECONDITION, "null output handle");
  *out = nullptr;
  if (d == 0) return set_err(PBH_PRECONDITION, "bucket heap: d must be positive");
  if (d > (1ull << 40)) return set_err(PBH_PRECONDITION, "bucket heap: d too large");
  CK(cudaSetDevice(device));
  pbh_heap* h = new pbh_heap();
  h->device = device;
  h->d = d;
  h->nt = 32 * kTraceNW;
  if (key_universe == 0) key_universe = 1 << 16;
  if (key_universe > (1ull << 32)) return set_err(PBH_PRECONDITION, "key_universe exceeds 2^32");
  const u32 cap0 = (u32)(32 * kTraceNW * kTraceKI / 2);
  const u32 bc = (u32)pow2_at_least(std::max<u64>(std::min<u64>(d, 4096), 2));
  auto fail = [&](pbh_status s) {
    h->H.free_all();
    cudaFree(h->d_job);
    cudaFree(h->d_save);
    if (h->h_ks) cudaFreeHost(h->h_ks);
    if (h->h_mop) cudaFreeHost(h->h_mop);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
    return s;
  };
  if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(set_err(PBH_CUDA, "stream create failed"));
  // the banked engine pre-allocates levels for the key universe (each
  // NEED_GROW is a kernel exit + relaunch)
  u32 nlev = 2;
  // level 1 holds four push-buffer flushes, or four whole large batches
  h->H.bank = true;
  h->H.base1 = std::max<u64>(4ull * kBankQ, 4 * std::min<u64>(d, kMaxBatch));
  while (nlev < 12 && (h->H.base1 << (2 * (nlev - 2))) < 2 * key_universe + 4 * kBankQ) ++nlev;
  pbh_status st = init_heap(h->H, d, cap0, bc, h->nt, key_universe, debug_checks, nlev, nullptr);
  if (st) return fail(st);
  if (cudaHostAlloc(&h->h_ks, sizeof(pbh_kstatus), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(&h->d_ks, h->h_ks, 0) != cudaSuccess ||
      cudaHostAlloc(&h->h_mop, sizeof(pbh_op_channel), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(&h->d_mop, h->h_mop, 0) != cudaSuccess)
    return fail(set_err(PBH_OOM, "status block allocation failed"));
  // pinned allocations are not zeroed: the channel's req / ack counters
  // must start equal (no request posted)
  std::memset(h->h_ks, 0, sizeof(pbh_kstatus));
  std::memset(h->h_mop, 0, sizeof(pbh_op_channel));
  // grid helpers for the deep merges (PBH_GRID=1 disables them)
  const char* ge = getenv("PBH_GRID");
  if (!(ge && atoi(ge) <= 1) && cudaMalloc(&h->d_job, sizeof(GridJob)) != cudaSuccess)
    return fail(set_err(PBH_OOM, "grid job allocation failed"));
  {
    if (cudaMalloc(&h->d_save, sizeof(TraceImage)) != cudaSuccess)
      return fail(set_err(PBH_OOM, "level-0 image allocation failed"));
    TraceImage* img = new TraceImage();
    std::memset(img, 0, sizeof(TraceImage));
    img->spl_inf = 1;
    cudaError_t e = cudaMemcpy(h->d_save, img, sizeof(TraceImage), cudaMemcpyHostToDevice);
    delete img;
    if (e != cudaSuccess) return fail(set_err(PBH_CUDA, "level-0 image init failed"));
  }
  if (const char* e = getenv("PBH_GRID_MIN")) h->grid_min = std::max(2, atoi(e));
  if (h->d_job) {
    // grid sorts: job block + staging / sort ping-pong / leader list, for
    // large batches (d >= kBigBatch) and the push-buffer flushes (kBankQ)
    // (+ room for a small S_1 folded into a push-buffer flush sort)
    const u64 cap = std::max<u64>(std::min<u64>(d, kMaxBatch), 2 * kBankQ);
    BatchJob hb{};
    void* mem[6] = {};
    void* bc = nullptr;
    const size_t sz[6] = {sizeof(BatchJob), cap * 4 + kTmaSlack, cap * 8 + kTmaSlack,
                          cap * 4 + kTmaSlack, cap * 8 + kTmaSlack, cap * 4};
    for (int i = 0; i < 6; ++i)
      if (cudaMalloc(&mem[i], sz[i]) != cudaSuccess) return fail(set_err(PBH_OOM, "batch buffers"));
    for (int i = 0; i < 6; ++i) h->H.allocs.push_back(mem[i]);
    if (cudaMalloc(&bc, kBucketMax * sizeof(u32)) != cudaSuccess)
      return fail(set_err(PBH_OOM, "batch buffers"));
    h->H.allocs.push_back(bc);
    hb.bcnt = (u32*)bc;
    h->d_batch = (BatchJob*)mem[0];
    hb.sk[0] = (u32*)mem[1];
    hb.sp[0] = (u64*)mem[2];
    hb.sk[1] = (u32*)mem[3];
    hb.sp[1] = (u64*)mem[4];
    hb.ll = (u32*)mem[5];
    hb.stg_k = hb.sk[0];
    hb.stg_p = hb.sp[0];
    if (cudaMemcpy(h->d_batch, &hb, sizeof hb, cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(set_err(PBH_CUDA, "batch job init"));
  }
  if (getenv("PBH_PROF") && cudaMalloc(&h->d_prof, 16 * sizeof(unsigned long long)) == cudaSuccess) {
    cudaMemset(h->d_prof, 0, 16 * sizeof(unsigned long long));
    const unsigned int on = 1;
    cudaMemcpyToSymbol(g_jobprof_on, &on, sizeof on);
  }
  cudaEventCreate(&h->ev0);
  cudaEventCreate(&h->ev1);
  *out = h;
  return PBH_OK;
}

pbh_status pbh_heap_destroy(pbh_heap* h) {
  if (!h) return PBH_OK;
  cudaSetDevice(h->device);
  quiesce(h);
  cudaStreamSynchronize(h->stream);
  h->H.free_all();
  cudaFreeHost(h->h_ks);
  cudaFreeHost(h->h_mop);
  cudaFree(h->d_job);
  cudaFree(h->d_save);
  if (h->d_prof) {
    prof_report(h, "destroy");
    cudaFree(h->d_prof);
  }
  cudaFree(h->d_kinds);
  cudaFree(h->d_off);
  cudaFree(h->d_vals);
  cudaFree(h->d_prios);
  cudaFree(h->d_ov);
  cudaFree(h->d_op);
  cudaEventDestroy(h->ev0);
  cudaEventDestroy(h->ev1);
  cudaStreamDestroy(h->stream);
  delete h;
  return PBH_OK;
}

pbh_status pbh_heap_update(pbh_heap* h, uint32_t value, uint64_t priority) {
  if (!h) return set_err(PBH_PRECONDITION, "null heap");
  cudaSetDevice(h->device);
  return single_op(h, 'U', &value, &priority, 1, nullptr, nullptr);
}

pbh_status pbh_heap_bulk_update(pbh_heap* h, const uint32_t* values, const uint64_t* priorities,
                                uint64_t n) {
  if (!h) return set_err(PBH_PRECONDITION, "null heap");
  if (n == 0) return set_err(PBH_PRECONDITION, "bulk_update: empty batch");
  if (n > h->d) return set_err(PBH_PRECONDITION, "bulk_update: batch larger than d");
  if (n > kMaxBatch)
    return set_err(PBH_PRECONDITION, "bulk_update: batch larger than the 2^26-element batch limit");
  for (u64 i = 1; i < n; ++i)
    if (values[i - 1] >= values[i])
      return set_err(PBH_PRECONDITION, "bulk_update: batch must be value-sorted with unique values");
  cudaSetDevice(h->device);
  return single_op(h, 'B', values, priorities, n, nullptr, nullptr);
}

pbh_status pbh_heap_extract_min(pbh_heap* h, uint32_t* value, uint64_t* priority) {
  if (!h) return set_err(PBH_PRECONDITION, "null heap");
  cudaSetDevice(h->device);
  u32 v = 0;
  u64 p = 0;
  pbh_status st = single_op(h, 'E', nullptr, nullptr, 0, &v, &p);
  if (st == PBH_EMPTY) return set_err(PBH_EMPTY, "extract_min: heap is empty");
  if (st == PBH_OK) {
    if (value) *value = v;
    if (priority) *priority = p;
  }
  return st;
}

pbh_status pbh_heap_find_min(pbh_heap* h, uint32_t* value, uint64_t* priority) {
  if (!h) return set_err(PBH_PRECONDITION, "null heap");
  cudaSetDevice(h->device);
  u32 v = 0;
  u64 p = 0;
  pbh_status st = single_op(h, 'F', nullptr, nullptr, 0, &v, &p);
  if (st == PBH_EMPTY) return set_err(PBH_EMPTY, "find_min: heap is empty");
  if (st == PBH_OK) {
    if (value) *value = v;
    if (priority) *priority = p;
  }
  return st;
}

pbh_status pbh_heap_delete(pbh_heap* h, uint32_t value) {
  if (!h) return set_err(PBH_PRECONDITION, "null heap");
  cudaSetDevice(h->device);
  const u64 dummy = 0;
  return single_op(h, 'D', &value, &dummy, 1, nullptr, nullptr);
}

pbh_status pbh_heap_set_persistent(pbh_heap* h, uint64_t idle_us) {
  if (!h) return set_err(PBH_PRECONDITION, "null heap");
  if (idle_us > 10000000) return set_err(PBH_PRECONDITION, "persistent idle time above 10 s");
  cudaSetDevice(h->device);
  if (pbh_status q = quiesce(h)) return q;
  h->persist_idle_ns = idle_us * 1000;
  return PBH_OK;
}

pbh_status pbh_heap_persist_profile(pbh_heap* h, uint64_t out[5]) {
  if (!h || !out) return set_err(PBH_PRECONDITION, "null argument");
  out[0] = h->persist_reqs;
  out[1] = h->persist_launches;
  // cumulative over the resident kernel's life (reset at each launch)
  out[2] = h->h_mop->tprof[0];
  out[3] = h->h_mop->tprof[1];
  out[4] = h->h_mop->tprof[2];
  return PBH_OK;
}

pbh_status pbh_heap_live_size(pbh_heap* h, int64_t* n) {
  if (!h || !n) return set_err(PBH_PRECONDITION, "null argument");
  cudaSetDevice(h->device);
  if (pbh_status q = quiesce(h)) return q;
  CK(cudaMemcpyAsync(n, &h->H.dev->live, 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return PBH_OK;
}

pbh_status pbh_heap_drain(pbh_heap* h) {
  if (!h) return set_err(PBH_PRECONDITION, "null heap");
  cudaSetDevice(h->device);
  return single_op(h, kOpDrain, nullptr, nullptr, 0, nullptr, nullptr);
}

pbh_status pbh_heap_metrics(pbh_heap* h, uint64_t* ops, uint64_t* resolves, uint64_t* touches,
                            uint32_t* n_levels) {
  if (!h) return set_err(PBH_PRECONDITION, "null heap");
  cudaSetDevice(h->device);
  if (pbh_status q = quiesce(h)) return q;
  pbh_heap_dev hd;
  CK(cudaMemcpyAsync(&hd, h->H.dev, sizeof(hd), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  // levels that ever held content (BucketHeap::allocated_levels)
  u32 used = 1;
  for (u32 i = 0; i < hd.n_levels; ++i)
    if (hd.resolves[i] || hd.touches[i]) used = i + 1;
  if (ops) *ops = hd.ops;
  for (u32 i = 0; i < PBH_MAX_LEVELS; ++i) {
    if (resolves) resolves[i] = i < used ? hd.resolves[i] : 0;
    if (touches) touches[i] = i < used ? hd.touches[i] : 0;
  }
  if (n_levels) *n_levels = used;
  return PBH_OK;
}

pbh_status pbh_heap_stats(pbh_heap* h, uint64_t* stored_deep, uint64_t* stale_dropped) {
  if (!h) return set_err(PBH_PRECONDITION, "null heap");
  cudaSetDevice(h->device);
  if (pbh_status q = quiesce(h)) return q;
  pbh_heap_dev hd;
  CK(cudaMemcpyAsync(&hd, h->H.dev, sizeof(hd), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  u64 st = 0;
  for (u32 i = 1; i < hd.n_levels; ++i) st += (u64)hd.st[i].b_size + hd.st[i].s_size;
  if (stored_deep) *stored_deep = st;
  if (stale_dropped) *stale_dropped = hd.stale_dropped;
  return PBH_OK;
}

pbh_status pbh_heap_check_invariants(pbh_heap* h, uint64_t* n_violations) {
  if (!h || !n_violations) return set_err(PBH_PRECONDITION, "null argument");
  cudaSetDevice(h->device);
  if (pbh_status q = quiesce(h)) return q;
  pbh_heap_dev hd;
  CK(cudaMemcpyAsync(&hd, h->H.dev, sizeof(hd), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  std::vector<pbh_idx_entry> idx(hd.universe);
  CK(cudaMemcpy(idx.data(), hd.idx, hd.universe * sizeof(pbh_idx_entry), cudaMemcpyDeviceToHost));
  u64 bad = 0;
  std::string first;
  auto complain = [&](const std::string& m) {
    if (!bad) first = m;
    ++bad;
  };
  auto less = [](u64 pa, u32 ka, u64 pb, u32 kb) { return pa < pb || (pa == pb && ka < kb); };
  u64 valid_entries = 0;
  bool have_prev = false;
  u64 prev_p = 0;
  u32 prev_k = 0;  // max of all buckets so far
  auto valid0 = [&](u32 k, u64 p) {
    return k < hd.universe && PBH_ST(idx[k].state) == PBH_ST_LIVE && idx[k].prio == p;
  };
  {
    // banked level 0 (pbh_bank.cuh): every occupied slot holds a valid entry
    // whose index records that slot, all admitted by splitter_0; the push
    // buffer holds entries beyond it
    std::unique_ptr<TraceImage> img(new TraceImage());
    CK(cudaMemcpy(img.get(), h->d_save, sizeof(TraceImage), cudaMemcpyDeviceToHost));
    constexpr u32 Bn = 32 * kTraceNW;
    for (u32 t = 0; t < Bn; ++t)
      for (u32 i = 0; i < (u32)kTraceKI; ++i) {
        if (!((img->occ[t] >> i) & 1u)) continue;
        const u32 sl = i * Bn + t;
        const u32 k = img->lk[sl];
        const u64 p = img->lp[sl];
        if (!valid0(k, p)) complain("level 0: stale entry in slot " + std::to_string(sl));
        else if ((idx[k].state >> 2) != sl) complain("level 0: index does not record slot " + std::to_string(sl));
        else ++valid_entries;
        if (!(img->spl_inf || p < img->spl_p || (p == img->spl_p && k <= img->spl_k)))
          complain("level 0: slot above splitter_0");
      }
    for (u32 j = 0; j < img->qn; ++j) {
      const u32 k = img->qk[j];
      const u64 p = img->qp[j];
      if (!valid0(k, p)) continue;
      ++valid_entries;
      if (img->spl_inf || p < img->spl_p || (p == img->spl_p && k <= img->spl_k))
        complain("level 0: push-buffer entry admitted by splitter_0");
    }
    if (!img->spl_inf) {
      have_prev = true;
      prev_p = img->spl_p;
      prev_k = img->spl_k;
    }
  }
  for (u32 i = 0; i < hd.n_levels; ++i) {
    const pbh_level_state& t = hd.st[i];
    const pbh_level_bufs& b = hd.lv[i];
    const u32 cap = i == 0 ? hd.cap0 : b.cap_b;
    if (t.b_size > cap) complain("level " + std::to_string(i) + ": bucket over capacity");
    std::vector<u32> bk(t.b_size), sk(t.s_size);
    std::vector<u64> bp(t.b_size), sp(t.s_size);
    if (t.b_size) {
      CK(cudaMemcpy(bk.data(), b.bk[t.b_sel] + t.b_head, t.b_size * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(bp.data(), b.bp[t.b_sel] + t.b_head, t.b_size * 8, cudaMemcpyDeviceToHost));
    }
    if (t.s_size) {
      CK(cudaMemcpy(sk.data(), b.sk[t.s_sel] + t.s_head, t.s_size * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(sp.data(), b.sp[t.s_sel] + t.s_head, t.s_size * 8, cudaMemcpyDeviceToHost));
    }
    for (u32 j = 1; j < t.b_size; ++j)
      if (!less(bp[j - 1], bk[j - 1], bp[j], bk[j])) {
        complain("level " + std::to_string(i) + ": bucket not strictly sorted");
        break;
      }
    for (u32 j = 1; j < t.s_size; ++j)
      if (!less(sp[j - 1], sk[j - 1], sp[j], sk[j])) {
        complain("level " + std::to_string(i) + ": signal buffer not strictly sorted");
        break;
      }
    for (u32 j = 0; j < t.b_size; ++j) {
      const bool adm = t.spl_inf || bp[j] < t.spl_p || (bp[j] == t.spl_p && bk[j] <= t.spl_k);
      if (!adm) {
        complain("level " + std::to_string(i) + ": bucket element above splitter");
        break;
      }
    }
    // everything at this level must lie above every shallower bucket
    if (have_prev) {
      if (t.b_size && !less(prev_p, prev_k, bp[0], bk[0]))
        complain("level " + std::to_string(i) + ": bucket overlaps shallower bucket");
      if (t.s_size && !less(prev_p, prev_k, sp[0], sk[0]))
        complain("level " + std::to_string(i) + ": signal overlaps shallower bucket");
    }
    if (t.b_size) {
      have_prev = true;
      prev_p = bp[t.b_size - 1];
      prev_k = bk[t.b_size - 1];
    }
    auto valid = [&](u32 k, u64 p) {
      return k < hd.universe && PBH_ST(idx[k].state) == PBH_ST_LIVE && idx[k].prio == p;
    };
    for (u32 j = 0; j < t.b_size; ++j) {
      const bool ok = valid(bk[j], bp[j]);
      valid_entries += ok;
      if (i == 0 && !ok) complain("level 0: stale entry in B_0");
    }
    for (u32 j = 0; j < t.s_size; ++j) valid_entries += valid(sk[j], sp[j]);
  }
  u64 live_idx = 0;
  for (const auto& e : idx) live_idx += PBH_ST(e.state) == PBH_ST_LIVE;
  if ((i64)live_idx != hd.live)
    complain("live_size " + std::to_string(hd.live) + " != live index entries " +
             std::to_string(live_idx));
  if (valid_entries != live_idx)
    complain("valid stored entries " + std::to_string(valid_entries) + " != live values " +
             std::to_string(live_idx));
  *n_violations = bad;
  if (bad) g_last_error = first;
  return PBH_OK;
}

namespace {
// run_trace (drain = true) and run_ops (drain = false) over host arrays.
pbh_status run_host_ops(pbh_heap* h, uint64_t n_ops, const uint8_t* kinds,
                        const uint64_t* offsets, const uint32_t* values,
                        const uint64_t* priorities, uint32_t* out_values,
                        uint64_t* out_priorities, uint64_t* n_out, uint64_t* failed_op,
                        double* wall_ms, bool drain) {
  if (!h) return set_err(PBH_PRECONDITION, "null heap");
  if (failed_op) *failed_op = ~0ull;
  if (n_out) *n_out = 0;
  if (wall_ms) *wall_ms = 0;
  cudaSetDevice(h->device);
  // host-side structural validation of the flat trace
  for (u64 i = 0; i < n_ops; ++i) {
    const u64 len = offsets[i + 1] - offsets[i];
    const u8 k = kinds[i];
    const bool ok = (k == 'U' && len == 1) || (k == 'B') || (k == 'E' && len == 0) ||
                    (k == 'D' && len == 1);
    if (ok && k == 'B' && len > kMaxBatch) {  // larger than the device batch buffers
      if (failed_op) *failed_op = i;
      return set_err(PBH_TRACE, "op " + std::to_string(i) +
                                    ": bulk_update: batch larger than the 2^26-element batch limit");
    }
    if (!ok || offsets[i + 1] < offsets[i]) {
      if (failed_op) *failed_op = i;
      return set_err(PBH_TRACE, "op " + std::to_string(i) + ": malformed op");
    }
  }
  pbh_status st = exec_host(h, n_ops, kinds, offsets, values, priorities, out_values,
                            out_priorities, n_out, failed_op, 0, wall_ms);
  if (h->d_prof) prof_report(h, drain ? "run_trace" : "run_ops");
  if (st == PBH_EMPTY || st == PBH_PRECONDITION) {
    return set_err(PBH_TRACE, g_last_error);  // TraceError(op_index) (engine.cpp:213-219)
  }
  if (st || !drain) return st;
  // Engine::run_trace drains before returning (engine.cpp:221)
  double dms = 0;
  u8 k = kOpDrain;
  u64 off[2] = {0, 0};
  st = exec_host(h, 1, &k, off, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 1, &dms);
  if (wall_ms) *wall_ms += dms;
  return st;
}
}  // namespace

pbh_status pbh_heap_run_trace(pbh_heap* h, uint64_t n_ops, const uint8_t* kinds,
                              const uint64_t* offsets, const uint32_t* values,
                              const uint64_t* priorities, uint32_t* out_values,
                              uint64_t* out_priorities, uint64_t* n_out, uint64_t* failed_op,
                              double* wall_ms) {
  return run_host_ops(h, n_ops, kinds, offsets, values, priorities, out_values, out_priorities,
                      n_out, failed_op, wall_ms, true);
}

pbh_status pbh_heap_run_ops(pbh_heap* h, uint64_t n_ops, const uint8_t* kinds,
                            const uint64_t* offsets, const uint32_t* values,
                            const uint64_t* priorities, uint32_t* out_values,
                            uint64_t* out_priorities, uint64_t* n_out, uint64_t* failed_op,
                            double* wall_ms) {
  return run_host_ops(h, n_ops, kinds, offsets, values, priorities, out_values, out_priorities,
                      n_out, failed_op, wall_ms, false);
}

pbh_status pbh_heap_run_trace_device(pbh_heap* h, uint64_t n_ops, const uint8_t* d_kinds,
                                     const uint64_t* d_offsets, const uint32_t* d_values,
                                     const uint64_t* d_priorities, uint32_t* d_out_values,
                                     uint64_t* d_out_priorities, uint64_t* n_out,
                                     uint64_t* failed_op, double* wall_ms) {
  if (!h) return set_err(PBH_PRECONDITION, "null heap");
  cudaSetDevice(h->device);
  if (failed_op) *failed_op = ~0ull;
  pbh_trace_dev tr{d_kinds, d_offsets, d_values, d_priorities};
  pbh_status st = exec_trace(h, n_ops, tr, d_out_values, d_out_priorities, n_out, failed_op, 0, wall_ms,
                  nullptr, nullptr, nullptr);
  if (st == PBH_EMPTY || st == PBH_PRECONDITION) return set_err(PBH_TRACE, g_last_error);
  if (st) return st;
  double dms = 0;
  u8 k = kOpDrain;
  u64 off[2] = {0, 0};
  st = exec_host(h, 1, &k, off, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 1, &dms);
  if (wall_ms) *wall_ms += dms;
  return st;
}

// =========================================================================
// CSR input contract (graphs.cpp:47-72)
// =========================================================================
namespace {

bool device_accessible(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Run k_csr_check over device arrays; blocking.
pbh_status csr_check(cudaStream_t s, CsrCheck* d_chk, const u64* off, const u32* tgt, const u32* w,
                     u32 V, u64 E, CsrCheck* out) {
  CsrCheck init{};
  init.first = ~0ull;
  CK(cudaMemcpyAsync(d_chk, &init, sizeof init, cudaMemcpyHostToDevice, s));
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const u64 warps = std::max<u64>(1, std::min<u64>((u64)V, (u64)sms * 64));
  k_csr_check<<<(u32)((warps * 32 + 255) / 256), 256, 0, s>>>(off, tgt, w, V, E, d_chk);
  g_launches++;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, d_chk, sizeof *out, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return PBH_OK;
}

// validate_graph's messages (graphs.cpp:56-71) for the first violation.
std::string csr_message(const CsrCheck& k) {
  if (k.sizes_bad) return "graph: inconsistent array sizes";
  switch ((u32)(k.first & 7)) {
    case kCsrMonotone: return "graph: offsets not monotone";
    case kCsrRange: return "graph: target out of range";
    case kCsrSelfLoop: return "graph: self-loop";
    case kCsrUnsorted: return "graph: row not sorted or parallel edge";
    default: return "graph: zero weight";
  }
}

// What the SSSP kernels cannot survive (out-of-bounds reads): bad sizes,
// non-monotone offsets, targets >= V. Self-loops, unsorted rows and zero
// weights are legal inputs to par_dijkstra (it does not call validate_graph).
pbh_status csr_precondition(const CsrCheck& k, const char* who) {
  const u32 code = (u32)(k.first & 7);
  if (k.sizes_bad || (k.first != ~0ull && (code == kCsrMonotone || code == kCsrRange)))
    return set_err(PBH_PRECONDITION, std::string(who) + ": " + csr_message(k) + " (vertex " +
                                         std::to_string(k.first >> 32) + ")");
  return PBH_OK;
}

}  // namespace

// =========================================================================
// SSSP
// =========================================================================
struct pbh_sssp_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  u32 V = 0;
  u64 E = 0;
  u64* d_off = nullptr;
  u32* d_tgt = nullptr;
  u32* d_w = nullptr;
  u32 max_deg = 0;
  u64 d = 0;
  int nt = 32;
  u32 cap0 = 0;
  u64 max_sources = 0;
  bool graph_ok = false;  // the resident CSR passed the device check
  int bank_nw = 4;    // warps per source of the banked engine
  void* d_save = nullptr;
  bool multi = false;  // threshold multi-extraction (pbh_sssp_ctx_set_mode)
  u32* d_mwo = nullptr;
  u32* d_mwi = nullptr;
  CsrCheck* d_chk = nullptr;  // CSR check / max out-degree scratch
  std::vector<DevHeap> heaps;
  pbh_heap_dev* d_heaps = nullptr;
  SsspState* d_sst = nullptr;
  u64* d_dist = nullptr;
  u32* d_settled = nullptr;
  u32* d_parent = nullptr;
  u32* d_src = nullptr;
  u64 n_last = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<void*> allocs;
};

namespace {

pbh_status ctx_alloc(pbh_sssp_ctx* c, void** p, size_t bytes) {
  CK(cudaMalloc(p, bytes ? bytes : 16));
  c->allocs.push_back(*p);
  return PBH_OK;
}

void ctx_free(pbh_sssp_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& H : c->heaps) H.free_all();
  for (void* p : c->allocs) cudaFree(p);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

}  // namespace

pbh_status pbh_sssp_ctx_create(const pbh_csr* g, uint64_t d, int device, uint64_t max_sources,
                               pbh_sssp_ctx** out) {
  if (!g || !out || max_sources == 0) return set_err(PBH_PRECONDITION, "bad arguments");
  *out = nullptr;
  CK(cudaSetDevice(device));
  pbh_sssp_ctx* c = new pbh_sssp_ctx();
  c->device = device;
  c->V = g->vertex_count;
  c->E = g->edge_count;
  c->max_sources = max_sources;
  auto fail = [&](pbh_status s) {
    ctx_free(c);
    return s;
  };
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(set_err(PBH_CUDA, "stream create failed"));
  cudaEventCreate(&c->ev0);
  cudaEventCreate(&c->ev1);
  pbh_status st;
  if ((st = ctx_alloc(c, (void**)&c->d_off, ((u64)c->V + 1) * 8))) return fail(st);
  if ((st = ctx_alloc(c, (void**)&c->d_tgt, c->E * 4))) return fail(st);
  if ((st = ctx_alloc(c, (void**)&c->d_w, c->E * 4))) return fail(st);
  // host or device CSR arrays (unified addressing: cudaMemcpyDefault)
  if (cudaMemcpyAsync(c->d_off, g->offsets, ((u64)c->V + 1) * 8, cudaMemcpyDefault, c->stream) ||
      (c->E && cudaMemcpyAsync(c->d_tgt, g->targets, c->E * 4, cudaMemcpyDefault, c->stream)) ||
      (c->E && cudaMemcpyAsync(c->d_w, g->weights, c->E * 4, cudaMemcpyDefault, c->stream)))
    return fail(set_err(PBH_CUDA, "CSR upload failed"));
  // the input contract and max out-degree on the device, one HBM pass
  // (graphs.cpp:47-72): malformed offsets or targets >= V would make the
  // kernels read out of bounds, so they fail here with PBH_PRECONDITION
  if ((st = ctx_alloc(c, (void**)&c->d_chk, sizeof(CsrCheck)))) return fail(st);
  CsrCheck chk{};
  if ((st = csr_check(c->stream, c->d_chk, c->d_off, c->d_tgt, c->d_w, c->V, c->E, &chk)))
    return fail(st);
  if ((st = csr_precondition(chk, "par_dijkstra"))) return fail(st);
  c->graph_ok = true;
  const u64 md = chk.max_deg;
  c->max_deg = (u32)md;
  c->d = d ? d : std::max<u64>(1, md);  // sssp.cpp:24-26
  c->d = std::min<u64>(c->d, std::max<u64>(1, md ? md : 1));  // batches never exceed a row
  c->bank_nw = 4;
  if (const char* e = getenv("PBH_SSSP_NW")) c->bank_nw = atoi(e);
  if (c->bank_nw != 0 && c->bank_nw != 1 && c->bank_nw != 2 && c->bank_nw != 4 && c->bank_nw != 8)
    c->bank_nw = 4;
  c->cap0 = kBankC0 / 2;
  c->nt = 32 * std::max(c->bank_nw, 1);
  const u32 bc = (u32)pow2_at_least(std::max<u64>(c->d, 2));
  if ((st = ctx_alloc(c, (void**)&c->d_heaps, max_sources * sizeof(pbh_heap_dev)))) return fail(st);
  if ((st = ctx_alloc(c, (void**)&c->d_sst, max_sources * sizeof(SsspState)))) return fail(st);
  if ((st = ctx_alloc(c, (void**)&c->d_dist, max_sources * c->V * 8))) return fail(st);
  if ((st = ctx_alloc(c, (void**)&c->d_settled, max_sources * c->V * 4))) return fail(st);
  if ((st = ctx_alloc(c, (void**)&c->d_parent, max_sources * c->V * 4))) return fail(st);
  if ((st = ctx_alloc(c, (void**)&c->d_src, max_sources * 4))) return fail(st);
  if ((st = ctx_alloc(c, (void**)&c->d_save,
                      max_sources * std::max(bank_save_bytes_nw(c->bank_nw), sizeof(MultiImage)))))
    return fail(st);
  c->heaps.resize(max_sources);
  // one arena for every source's heap (levels, scratch, index)
  // initial levels: enough for a few rows of relaxations
  u32 nlev = 2;
  while (nlev < 8 && ((u64)c->cap0 << (2 * (nlev - 1))) < 8ull * (c->max_deg + 1)) ++nlev;
  // test knob: a smaller first deep level (entries), so that the NEED_GROW
  // exit + relaunch path runs on small graphs
  u64 base1 = 4ull * kBankQ;
  if (const char* e = getenv("PBH_SSSP_BASE1")) {
    base1 = std::max<u64>(strtoull(e, nullptr, 10), 2ull * kBankQ);
    nlev = 2;
  }
  // level 0 is allocated for the threshold engine's larger refills
  // (kMultiCap0); exact mode refills to kBankC0 / 2 (c->cap0)
  size_t per_heap = 0;
  {
    DevHeap M;
    M.measure = true;
    M.base1 = base1, M.bank = true;
    init_heap(M, c->d, kMultiCap0, bc, c->nt, std::max<u32>(c->V, 1), 0, nlev, c->d_heaps);
    per_heap = M.measured;
  }
  char* arena = nullptr;
  if ((st = ctx_alloc(c, (void**)&arena, per_heap * max_sources))) return fail(st);
  for (u64 i = 0; i < max_sources; ++i) {
    DevHeap& H = c->heaps[i];
    H.base1 = base1, H.bank = true;
    H.arena = arena + per_heap * i;
    H.arena_cap = per_heap;
    st = init_heap(H, c->d, kMultiCap0, bc, c->nt, std::max<u32>(c->V, 1), 0, nlev, c->d_heaps + i,
                   c->stream);
    if (st) return fail(st);
    H.hd.cap0 = c->cap0;  // uploaded with the header by every ctx_reset
  }
  CK(cudaStreamSynchronize(c->stream));
  *out = c;
  return PBH_OK;
}

namespace {

// Reset slot state (heap header, index, outputs) for a new solve.
pbh_status ctx_reset(pbh_sssp_ctx* c, u64 n) {
  for (u64 i = 0; i < n; ++i) {
    DevHeap& H = c->heaps[i];
    for (u32 l = 0; l < PBH_MAX_LEVELS; ++l) {
      H.hd.st[l] = pbh_level_state{};
      H.hd.st[l].spl_inf = 1;
      H.hd.resolves[l] = 0;
      H.hd.touches[l] = 0;
    }
    H.hd.live = 0;
    H.hd.ops = 0;
    CK(cudaMemcpyAsync(H.dev, &H.hd, sizeof(pbh_heap_dev), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(H.hd.idx, 0xff, (u64)c->V * sizeof(pbh_idx_entry), c->stream));
  }
  CK(cudaMemsetAsync(c->d_sst, 0, n * sizeof(SsspState), c->stream));
  CK(cudaMemsetAsync(c->d_dist, 0xff, n * c->V * 8, c->stream));
  return PBH_OK;
}

}  // namespace

pbh_status pbh_sssp_ctx_run(pbh_sssp_ctx* c, const uint32_t* sources, uint64_t n_sources,
                            int dag_mode, double* device_ms) {
  if (!c) return set_err(PBH_PRECONDITION, "null context");
  if (n_sources == 0 || n_sources > c->max_sources)
    return set_err(PBH_PRECONDITION, "n_sources out of range");
  for (u64 i = 0; i < n_sources; ++i)
    if (sources[i] >= c->V) return set_err(PBH_PRECONDITION, "par_dijkstra: source out of range");
  if (!c->graph_ok)
    return set_err(PBH_PRECONDITION, "par_dijkstra: the context holds no valid graph (a failed load_graph)");
  CK(cudaSetDevice(c->device));
  pbh_status st = ctx_reset(c, n_sources);
  if (st) return st;
  CK(cudaMemcpyAsync(c->d_src, sources, n_sources * 4, cudaMemcpyHostToDevice, c->stream));
  double ms_total = 0;
  std::vector<SsspState> hs(n_sources);
  for (int guard = 0; guard < 256; ++guard) {
    CK(cudaEventRecord(c->ev0, c->stream));
    if (c->multi) {
      CK(launch_sssp_multi(c->stream, (u32)n_sources, c->d_heaps, c->d_off, c->d_tgt, c->d_w,
                           c->d_mwo, c->d_mwi, c->V, c->d_src, c->d_dist, c->d_settled, c->d_sst,
                           c->d_save, c->max_deg, (u32)std::min<u64>(c->d, 0xffffffffu)));
    } else {
      CK(launch_sssp_bank_nw(c->bank_nw, c->stream, (u32)n_sources, c->d_heaps, c->d_off,
                             c->d_tgt, c->d_w, c->V, c->d_src, c->d_dist, c->d_settled, c->d_sst,
                             c->d_save, dag_mode ? 1 : 0, c->max_deg,
                             (u32)std::min<u64>(c->d, 0xffffffffu)));
    }
    CK(cudaEventRecord(c->ev1, c->stream));
    CK(cudaMemcpyAsync(hs.data(), c->d_sst, n_sources * sizeof(SsspState), cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float ms = 0;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    ms_total += ms;
    bool again = false;
    for (u64 i = 0; i < n_sources; ++i) {
      if (hs[i].status == 7) {
        st = grow_levels(c->heaps[i], c->stream);
        if (st) return st;
        again = true;
      } else if (hs[i].status != 0) {
        return set_err(hs[i].status == 3 ? PBH_INVARIANT : PBH_PRECONDITION,
                       std::string("sssp source slot ") + std::to_string(i) + ": " +
                           detail_message(hs[i].detail) +
                           (hs[i].status == 3 && hs[i].aux ? " (site 0x" + [&] {
                             char b[24];
                             std::snprintf(b, sizeof b, "%llx", (unsigned long long)hs[i].aux);
                             return std::string(b);
                           }() + ")" : std::string()));
      }
    }
    if (!again) break;
    // clear NEED_GROW status so the kernel resumes
    for (u64 i = 0; i < n_sources; ++i)
      if (hs[i].status == 7) CK(cudaMemsetAsync(&c->d_sst[i].status, 0, 4, c->stream));
  }
  for (u64 i = 0; i < n_sources; ++i) {
    k_finalize_parent<<<std::max<u32>(1, std::min<u32>(1184, (c->V + 255) / 256)), 256, 0,
                        c->stream>>>(c->heaps[i].hd.idx, c->V, c->d_parent + i * c->V);
    g_launches++;
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->stream));
  c->n_last = n_sources;
  if (device_ms) *device_ms = ms_total;
  if (getenv("PBH_PHASES")) {
    SsspState s0;
    cudaMemcpy(&s0, c->d_sst, sizeof s0, cudaMemcpyDeviceToHost);
    const double r = s0.rounds ? (double)s0.rounds : 1.0;
    if (c->multi)
      fprintf(stderr, "multi phases cyc/batch: thresholds %.0f select %.0f prefix+commit %.0f "
              "pass-top(cold) %.0f gathers+binsearch %.0f atomics+apply+exchange %.0f tail %.0f loop %.0f\n",
              s0.phase[0] / r, s0.phase[1] / r, s0.phase[2] / r, s0.phase[3] / r, s0.phase[4] / r,
              s0.phase[5] / r, s0.phase[6] / r, s0.phase[7] / r);
  }
  return PBH_OK;
}

pbh_status pbh_sssp_ctx_fetch(pbh_sssp_ctx* c, uint64_t slot, uint64_t* dist, uint32_t* parent,
                              uint32_t* settled, uint64_t* n_settled, uint64_t* rounds,
                              uint64_t* ops) {
  if (!c || slot >= c->n_last) return set_err(PBH_PRECONDITION, "bad slot");
  CK(cudaSetDevice(c->device));
  SsspState s;
  CK(cudaMemcpyAsync(&s, c->d_sst + slot, sizeof s, cudaMemcpyDeviceToHost, c->stream));
  if (dist) CK(cudaMemcpyAsync(dist, c->d_dist + slot * c->V, (u64)c->V * 8, cudaMemcpyDeviceToHost, c->stream));
  if (parent) CK(cudaMemcpyAsync(parent, c->d_parent + slot * c->V, (u64)c->V * 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (settled && s.n_settled)
    CK(cudaMemcpy(settled, c->d_settled + slot * c->V, s.n_settled * 4, cudaMemcpyDeviceToHost));
  if (n_settled) *n_settled = s.n_settled;
  if (rounds) *rounds = s.rounds;
  if (ops) *ops = s.ops;
  return PBH_OK;
}

pbh_status pbh_sssp_ctx_set_mode(pbh_sssp_ctx* c, int mode) {
  if (!c || (mode != 0 && mode != 1)) return set_err(PBH_PRECONDITION, "bad mode");
  CK(cudaSetDevice(c->device));
  if (mode == 1 && !c->d_mwo) {
    pbh_status st;
    if ((st = ctx_alloc(c, (void**)&c->d_mwo, (u64)c->V * 4))) return st;
    if ((st = ctx_alloc(c, (void**)&c->d_mwi, (u64)c->V * 4))) return st;
    CK(cudaMemsetAsync(c->d_mwi, 0xff, (u64)c->V * 4, c->stream));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    k_min_weights<<<sms * 8, 256, 0, c->stream>>>(c->d_off, c->d_tgt, c->d_w, c->V, c->d_mwo,
                                                  c->d_mwi);
    g_launches++;
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
  }
  c->multi = mode == 1;
  c->cap0 = c->multi ? kMultiCap0 : kBankC0 / 2;
  for (auto& H : c->heaps) H.hd.cap0 = c->cap0;
  return PBH_OK;
}

pbh_status pbh_sssp_ctx_load_graph(pbh_sssp_ctx* c, const pbh_csr* g) {
  if (!c || !g) return set_err(PBH_PRECONDITION, "bad arguments");
  if (g->vertex_count != c->V || g->edge_count != c->E)
    return set_err(PBH_PRECONDITION, "load_graph: vertex/edge count differs from the context");
  if (!g->offsets || (c->E && (!g->targets || !g->weights)))
    return set_err(PBH_PRECONDITION, "load_graph: null CSR array");
  CK(cudaSetDevice(c->device));
  // The shape check (max out-degree, which sizes the heaps, sssp.cpp:24-26)
  // runs on the NEW graph before anything in the context changes: device
  // arrays are checked in place, host offsets on the host (8 B per vertex).
  const bool dev_src = device_accessible(g->offsets) && (!c->E || (device_accessible(g->targets) &&
                                                                    device_accessible(g->weights)));
  pbh_status st;
  if (dev_src) {
    CsrCheck chk{};
    if ((st = csr_check(c->stream, c->d_chk, g->offsets, g->targets, g->weights, c->V, c->E, &chk)))
      return st;
    if ((st = csr_precondition(chk, "load_graph"))) return st;
    if ((u32)chk.max_deg != c->max_deg)
      return set_err(PBH_PRECONDITION, "load_graph: max out-degree differs from the context");
  } else {
    const u64* o = g->offsets;
    if (o[0] != 0 || o[c->V] != c->E)
      return set_err(PBH_PRECONDITION, "load_graph: graph: inconsistent array sizes");
    u64 md = 0;
    for (u64 u = 0; u < c->V; ++u) {
      if (o[u] > o[u + 1]) return set_err(PBH_PRECONDITION, "load_graph: graph: offsets not monotone");
      md = std::max<u64>(md, o[u + 1] - o[u]);
    }
    if ((u32)md != c->max_deg)
      return set_err(PBH_PRECONDITION, "load_graph: max out-degree differs from the context");
  }
  CK(cudaMemcpyAsync(c->d_off, g->offsets, ((u64)c->V + 1) * 8, cudaMemcpyDefault, c->stream));
  if (c->E) {
    CK(cudaMemcpyAsync(c->d_tgt, g->targets, c->E * 4, cudaMemcpyDefault, c->stream));
    CK(cudaMemcpyAsync(c->d_w, g->weights, c->E * 4, cudaMemcpyDefault, c->stream));
  }
  if (!dev_src) {
    // host targets are range-checked on the resident copy; a bad graph
    // leaves the context refusing to run until a valid one is loaded
    c->graph_ok = false;
    CsrCheck chk{};
    if ((st = csr_check(c->stream, c->d_chk, c->d_off, c->d_tgt, c->d_w, c->V, c->E, &chk)))
      return st;
    if ((st = csr_precondition(chk, "load_graph"))) return st;
  }
  c->graph_ok = true;
  if (c->d_mwo) {  // threshold mode's per-vertex minimum weights
    CK(cudaMemsetAsync(c->d_mwi, 0xff, (u64)c->V * 4, c->stream));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    k_min_weights<<<sms * 8, 256, 0, c->stream>>>(c->d_off, c->d_tgt, c->d_w, c->V, c->d_mwo,
                                                  c->d_mwi);
    g_launches++;
    CK(cudaGetLastError());
  }
  CK(cudaStreamSynchronize(c->stream));
  return PBH_OK;
}

pbh_status pbh_sssp_ctx_destroy(pbh_sssp_ctx* c) {
  ctx_free(c);
  return PBH_OK;
}

pbh_status pbh_sssp(const pbh_csr* g, uint32_t source, uint64_t d, int dag_mode, int device,
                    uint64_t* dist, uint32_t* parent, uint32_t* settled, uint64_t* n_settled,
                    uint64_t* rounds, uint64_t* ops) {
  if (!g) return set_err(PBH_PRECONDITION, "null graph");
  if (source >= g->vertex_count) return set_err(PBH_PRECONDITION, "par_dijkstra: source out of range");
  pbh_sssp_ctx* c = nullptr;
  pbh_status st = pbh_sssp_ctx_create(g, d, device, 1, &c);
  if (st) return st;
  st = pbh_sssp_ctx_run(c, &source, 1, dag_mode, nullptr);
  if (!st) st = pbh_sssp_ctx_fetch(c, 0, dist, parent, settled, n_settled, rounds, ops);
  pbh_sssp_ctx_destroy(c);
  return st;
}

pbh_status pbh_sssp_multi(const pbh_csr* g, const uint32_t* sources, uint64_t n_sources,
                          uint64_t d, const int* devices, int n_devices, uint64_t* dist,
                          uint32_t* parent) {
  if (!g || !sources || !dist || n_devices <= 0) return set_err(PBH_PRECONDITION, "bad arguments");
  std::vector<pbh_status> res(n_devices, PBH_OK);
  std::vector<std::string> msg(n_devices);
  std::vector<std::thread> th;
  const u64 per = (n_sources + n_devices - 1) / n_devices;
  for (int r = 0; r < n_devices; ++r) {
    const u64 b = std::min<u64>(n_sources, r * per), e = std::min<u64>(n_sources, b + per);
    if (b >= e) continue;
    th.emplace_back([&, r, b, e] {
      pbh_sssp_ctx* c = nullptr;
      const bool prof = getenv("PBH_E2E_PROF") != nullptr;
      auto now = [] { return std::chrono::steady_clock::now(); };
      auto t0 = now();
      pbh_status st = pbh_sssp_ctx_create(g, d, devices[r], e - b, &c);
      auto t1 = now();
      if (!st) st = pbh_sssp_ctx_run(c, sources + b, e - b, 0, nullptr);
      auto t2 = now();
      for (u64 i = b; !st && i < e; ++i)
        st = pbh_sssp_ctx_fetch(c, i - b, dist + i * g->vertex_count,
                                parent ? parent + i * g->vertex_count : nullptr, nullptr, nullptr,
                                nullptr, nullptr);
      auto t3 = now();
      if (c) pbh_sssp_ctx_destroy(c);
      auto t4 = now();
      if (prof) {
        auto ms = [](auto a, auto z) { return std::chrono::duration<double, std::milli>(z - a).count(); };
        fprintf(stderr, "pbh_sssp_multi dev %d: create %.1f ms run %.1f ms fetch %.1f ms destroy %.1f ms\n",
                devices[r], ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4));
      }
      res[r] = st;
      if (st) msg[r] = g_last_error;
    });
  }
  for (auto& t : th) t.join();
  for (int r = 0; r < n_devices; ++r)
    if (res[r]) return set_err(res[r], msg[r]);
  return PBH_OK;
}

pbh_status pbh_bellman_ford(const pbh_csr* g, uint32_t source, int device, uint64_t* dist,
                            uint32_t* parent, uint64_t* rounds, uint64_t* edges_scanned,
                            double* device_ms) {
  if (!g || !dist) return set_err(PBH_PRECONDITION, "bad arguments");
  if (source >= g->vertex_count) return set_err(PBH_PRECONDITION, "bellman_ford: source out of range");
  CK(cudaSetDevice(device));
  const u64 V = g->vertex_count, E = g->edge_count;
  std::vector<void*> mem;
  auto fin = [&](pbh_status st) {
    for (void* p : mem) cudaFree(p);
    return st;
  };
  auto dalloc = [&](void** p, size_t b) -> bool {
    if (cudaMalloc(p, b ? b : 16) != cudaSuccess) return false;
    mem.push_back(*p);
    return true;
  };
  u64 *d_off = nullptr, *d_dist = nullptr;
  u32 *d_tgt = nullptr, *d_w = nullptr, *fq0 = nullptr, *fq1 = nullptr, *stamp = nullptr, *d_par = nullptr;
  BfState* d_st = nullptr;
  if (!dalloc((void**)&d_off, (V + 1) * 8) || !dalloc((void**)&d_tgt, E * 4) ||
      !dalloc((void**)&d_w, E * 4) || !dalloc((void**)&d_dist, V * 8) ||
      !dalloc((void**)&fq0, V * 4) || !dalloc((void**)&fq1, V * 4) ||
      !dalloc((void**)&stamp, V * 4) || !dalloc((void**)&d_st, sizeof(BfState)) ||
      (parent && !dalloc((void**)&d_par, V * 4)))
    return fin(set_err(PBH_OOM, "bellman_ford: device allocation failed"));
  cudaStream_t st = nullptr;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaMemcpyAsync(d_off, g->offsets, (V + 1) * 8, cudaMemcpyHostToDevice, st);
  if (E) {
    cudaMemcpyAsync(d_tgt, g->targets, E * 4, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_w, g->weights, E * 4, cudaMemcpyHostToDevice, st);
  }
  {
    CsrCheck* d_chk = nullptr;
    if (!dalloc((void**)&d_chk, sizeof(CsrCheck))) {
      cudaStreamDestroy(st);
      return fin(set_err(PBH_OOM, "bellman_ford: device allocation failed"));
    }
    CsrCheck chk{};
    pbh_status cs = csr_check(st, d_chk, d_off, d_tgt, d_w, (u32)V, E, &chk);
    if (!cs) cs = csr_precondition(chk, "bellman_ford");
    if (cs) {
      cudaStreamDestroy(st);
      return fin(cs);
    }
  }
  cudaMemsetAsync(d_dist, 0xff, V * 8, st);
  cudaMemsetAsync(d_dist + source, 0, 8, st);
  cudaMemsetAsync(stamp, 0, V * 4, st);
  BfState h0{};
  h0.cnt[0] = 1;
  cudaMemcpyAsync(d_st, &h0, sizeof h0, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(fq0, &source, 4, cudaMemcpyHostToDevice, st);
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_bellman_ford, 256, 0);
  const int G = std::max(1, sms * std::max(1, std::min(per, 4)));
  u32 Vv = (u32)V;
  u64 max_it = V + 1;
  void* args[] = {&d_off, &d_tgt, &d_w, &Vv, &d_dist, &fq0, &fq1, &stamp, &d_st, &max_it};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  cudaError_t err = cudaLaunchCooperativeKernel((const void*)k_bellman_ford, dim3(G), dim3(256), args, 0, st);
  g_launches++;
  cudaEventRecord(e1, st);
  if (err == cudaSuccess && parent) {
    cudaMemsetAsync(d_par, 0xff, V * 4, st);
    k_bf_parents<<<sms * 8, 256, 0, st>>>(d_off, d_tgt, d_w, Vv, d_dist, d_par);
    g_launches++;
    err = cudaGetLastError();
  }
  BfState hs{};
  if (err == cudaSuccess) {
    cudaMemcpyAsync(&hs, d_st, sizeof hs, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(dist, d_dist, V * 8, cudaMemcpyDeviceToHost, st);
    if (parent) cudaMemcpyAsync(parent, d_par, V * 4, cudaMemcpyDeviceToHost, st);
    err = cudaStreamSynchronize(st);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  if (err != cudaSuccess) return fin(set_err(PBH_CUDA, std::string("bellman_ford: ") + cudaGetErrorString(err)));
  if (hs.status == 9) return fin(set_err(PBH_INVARIANT, "sssp: distance accumulation overflow"));
  if (parent) parent[source] = source;
  if (rounds) *rounds = hs.iters;
  if (edges_scanned) *edges_scanned = hs.relaxed;
  if (device_ms) *device_ms = ms;
  return fin(PBH_OK);
}

namespace {

// kind 0 = grid (rows x cols), 1 = band (V, degree); device output arrays.
pbh_status gen_device(u32 kind, u32 rows, u32 cols, u32 V, u32 degree, u64 seed, int device,
                      u64* off, u32* tgt, u32* w) {
  CK(cudaSetDevice(device));
  // std::mt19937_64 seeding (the state the first twist starts from)
  u64 mt[kMtN];
  mt[0] = seed;
  for (int i = 1; i < kMtN; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (u64)i;
  u64* d_mt = nullptr;
  CK(cudaMalloc(&d_mt, sizeof mt));
  cudaStream_t st = nullptr;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaMemcpyAsync(d_mt, mt, sizeof mt, cudaMemcpyHostToDevice, st);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  k_gen_structure<<<sms * 8, 256, 0, st>>>(kind, rows, cols, V, degree, off, tgt, w);
  GenMap map{};
  map.kind = kind;
  map.V = V;
  map.degree = degree;
  map.w = w;
  if (kind == 0) {
    map.n_draws = pbh_gen_grid_edges(rows, cols);
  } else {
    map.n_draws = V == 0 ? 0 : (u64)(V - 1) * (degree - 1) + degree;
  }
  k_gen_weights<<<1, 320, 0, st>>>(d_mt, map);
  g_launches += 2;
  cudaError_t e = cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  cudaFree(d_mt);
  if (e != cudaSuccess) return set_err(PBH_CUDA, std::string("device generator: ") + cudaGetErrorString(e));
  return PBH_OK;
}

}  // namespace

int pbh_gen_grid_device(uint32_t rows, uint32_t cols, uint64_t seed, int device,
                               uint64_t* offsets, uint32_t* targets, uint32_t* weights) {
  if (!rows || !cols || !offsets || !targets || !weights) return set_err(PBH_PRECONDITION, "bad arguments");
  return gen_device(0, rows, cols, rows * cols, 0, seed, device, offsets, targets, weights);
}

int pbh_gen_band_device(uint32_t v, uint32_t degree, uint64_t seed, int device,
                               uint64_t* offsets, uint32_t* targets, uint32_t* weights) {
  if (!v || !degree || degree >= v || !offsets || !targets || !weights)
    return set_err(PBH_PRECONDITION, "bad arguments");
  return gen_device(1, 0, 0, v, degree, seed, device, offsets, targets, weights);
}

pbh_status pbh_host_register(void* ptr, uint64_t bytes) {
  if (!ptr || !bytes) return set_err(PBH_PRECONDITION, "null or empty host range");
  CK(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable));
  return PBH_OK;
}

pbh_status pbh_host_unregister(void* ptr) {
  if (!ptr) return set_err(PBH_PRECONDITION, "null host pointer");
  CK(cudaHostUnregister(ptr));
  return PBH_OK;
}

pbh_status pbh_sssp_multi_device(const pbh_csr* g, const uint32_t* sources, uint64_t n_sources,
                                 uint64_t d, const int* devices, int n_devices,
                                 uint64_t* dist_dev0, uint32_t* parent_dev0, double* device_ms) {
  if (!g || !sources || !dist_dev0 || n_devices <= 0 || n_sources == 0)
    return set_err(PBH_PRECONDITION, "bad arguments");
  const int dev0 = devices[0];
  std::vector<pbh_status> res(n_devices, PBH_OK);
  std::vector<std::string> msg(n_devices);
  std::vector<double> ms(n_devices, 0.0);
  std::vector<std::thread> th;
  const u64 V = g->vertex_count;
  const u64 per = (n_sources + n_devices - 1) / n_devices;
  for (int r = 0; r < n_devices; ++r) {
    const u64 b = std::min<u64>(n_sources, r * per), e = std::min<u64>(n_sources, b + per);
    if (b >= e) continue;
    th.emplace_back([&, r, b, e] {
      pbh_sssp_ctx* c = nullptr;
      pbh_status st = pbh_sssp_ctx_create(g, d, devices[r], e - b, &c);
      if (!st) st = pbh_sssp_ctx_run(c, sources + b, e - b, 0, &ms[r]);
      if (!st) {
        // gather this shard's dist / parent rows into devices[0] over NVLink
        if (devices[r] != dev0) {
          int can = 0;
          cudaDeviceCanAccessPeer(&can, devices[r], dev0);
          if (can) {
            cudaError_t pe = cudaDeviceEnablePeerAccess(dev0, 0);
            if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
          }
        }
        cudaError_t ce = cudaMemcpyPeerAsync(dist_dev0 + b * V, dev0, c->d_dist, devices[r],
                                             (e - b) * V * 8, c->stream);
        if (ce == cudaSuccess && parent_dev0)
          ce = cudaMemcpyPeerAsync(parent_dev0 + b * V, dev0, c->d_parent, devices[r],
                                   (e - b) * V * 4, c->stream);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(c->stream);
        if (ce != cudaSuccess) st = set_err(PBH_CUDA, std::string("peer gather: ") + cudaGetErrorString(ce));
      }
      if (c) pbh_sssp_ctx_destroy(c);
      res[r] = st;
      if (st) msg[r] = g_last_error;
    });
  }
  for (auto& t : th) t.join();
  for (int r = 0; r < n_devices; ++r)
    if (res[r]) return set_err(res[r], msg[r]);
  if (device_ms) *device_ms = *std::max_element(ms.begin(), ms.end());
  return PBH_OK;
}

pbh_status pbh_validate_graph(const pbh_csr* g, int device) {
  if (!g || !g->offsets || (g->edge_count && (!g->targets || !g->weights)))
    return set_err(PBH_PRECONDITION, "validate_graph: null CSR array");
  CK(cudaSetDevice(device));
  const u64 V = g->vertex_count, E = g->edge_count;
  const bool dev_src = device_accessible(g->offsets) &&
                       (!E || (device_accessible(g->targets) && device_accessible(g->weights)));
  std::vector<void*> mem;
  auto fin = [&](pbh_status s) {
    for (void* p : mem) cudaFree(p);
    return s;
  };
  const u64* off = g->offsets;
  const u32 *tgt = g->targets, *w = g->weights;
  cudaStream_t s = nullptr;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  auto up = [&](const void* src, size_t bytes, void** dst) -> bool {
    if (cudaMalloc(dst, bytes ? bytes : 16) != cudaSuccess) return false;
    mem.push_back(*dst);
    return !bytes || cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyHostToDevice, s) == cudaSuccess;
  };
  if (!dev_src) {
    // host arrays: staged through device memory for the one-pass check
    if (!up(g->offsets, (V + 1) * 8, (void**)&off) || !up(g->targets, E * 4, (void**)&tgt) ||
        !up(g->weights, E * 4, (void**)&w)) {
      cudaStreamDestroy(s);
      return fin(set_err(PBH_OOM, "validate_graph: staging allocation failed"));
    }
  }
  CsrCheck* d_chk = nullptr;
  if (cudaMalloc(&d_chk, sizeof(CsrCheck)) != cudaSuccess) {
    cudaStreamDestroy(s);
    return fin(set_err(PBH_OOM, "validate_graph: allocation failed"));
  }
  mem.push_back(d_chk);
  CsrCheck chk{};
  pbh_status st = csr_check(s, d_chk, off, tgt, w, (u32)V, E, &chk);
  cudaStreamDestroy(s);
  if (st) return fin(st);
  if (chk.sizes_bad || chk.first != ~0ull) return fin(set_err(PBH_INVARIANT, csr_message(chk)));
  return fin(PBH_OK);
}

pbh_status pbh_csr_max_out_degree(const pbh_csr* g, int device, uint32_t* out) {
  if (!g || !out || !g->offsets) return set_err(PBH_PRECONDITION, "bad arguments");
  if (!device_accessible(g->offsets)) {
    u64 best = 0;
    for (u64 u = 0; u < g->vertex_count; ++u)
      best = std::max<u64>(best, g->offsets[u + 1] - g->offsets[u]);
    *out = (u32)best;
    return PBH_OK;
  }
  CK(cudaSetDevice(device));
  if (g->edge_count && (!g->targets || !g->weights))
    return set_err(PBH_PRECONDITION, "null CSR array");
  CsrCheck* d_chk = nullptr;
  CK(cudaMalloc(&d_chk, sizeof(CsrCheck)));
  cudaStream_t s = nullptr;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  CsrCheck chk{};
  pbh_status st = csr_check(s, d_chk, g->offsets, g->targets, g->weights, g->vertex_count,
                            g->edge_count, &chk);
  cudaStreamDestroy(s);
  cudaFree(d_chk);
  if (st) return st;
  *out = (u32)chk.max_deg;
  return PBH_OK;
}

pbh_status pbh_sssp_ctx_gather(pbh_sssp_ctx* c, uint64_t first_slot, uint64_t n_slots,
                               uint64_t* dist_dst, uint32_t* parent_dst) {
  if (!c || first_slot + n_slots > c->n_last || (!dist_dst && !parent_dst))
    return set_err(PBH_PRECONDITION, "gather: bad slot range or no destination");
  CK(cudaSetDevice(c->device));
  const u64 V = c->V;
  // cudaMemcpyDefault: host, local device, peer device (NVLink), or an
  // IPC-mapped buffer of another process (pbh_ipc_open)
  if (dist_dst)
    CK(cudaMemcpyAsync(dist_dst, c->d_dist + first_slot * V, n_slots * V * 8, cudaMemcpyDefault,
                       c->stream));
  if (parent_dst)
    CK(cudaMemcpyAsync(parent_dst, c->d_parent + first_slot * V, n_slots * V * 4,
                       cudaMemcpyDefault, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return PBH_OK;
}

pbh_status pbh_device_alloc(int device, uint64_t bytes, void** ptr) {
  if (!ptr) return set_err(PBH_PRECONDITION, "null output pointer");
  *ptr = nullptr;
  CK(cudaSetDevice(device));
  CK(cudaMalloc(ptr, bytes ? bytes : 16));
  return PBH_OK;
}

pbh_status pbh_device_free(int device, void* ptr) {
  CK(cudaSetDevice(device));
  if (ptr) CK(cudaFree(ptr));
  return PBH_OK;
}

pbh_status pbh_copy(void* dst, const void* src, uint64_t bytes) {
  if (!bytes) return PBH_OK;
  if (!dst || !src) return set_err(PBH_PRECONDITION, "null pointer");
  CK(cudaMemcpy(dst, src, bytes, cudaMemcpyDefault));
  return PBH_OK;
}

pbh_status pbh_ipc_export(void* dev_ptr, uint8_t handle[64]) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
  if (!dev_ptr || !handle) return set_err(PBH_PRECONDITION, "null pointer");
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, dev_ptr));
  std::memcpy(handle, &h, 64);
  return PBH_OK;
}

pbh_status pbh_ipc_open(const uint8_t handle[64], int device, void** ptr) {
  if (!handle || !ptr) return set_err(PBH_PRECONDITION, "null pointer");
  CK(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  CK(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return PBH_OK;
}

pbh_status pbh_ipc_close(int device, void* ptr) {
  CK(cudaSetDevice(device));
  if (ptr) CK(cudaIpcCloseMemHandle(ptr));
  return PBH_OK;
}

uint64_t pbh_distance_checksum(const uint64_t* dist, uint64_t n) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint64_t i = 0; i < n; ++i)
    for (int b = 0; b < 8; ++b) {
      h ^= (dist[i] >> (8 * b)) & 0xff;
      h *= 0x100000001b3ull;
    }
  return h;
}

}  // extern "C"
