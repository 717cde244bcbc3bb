// Shared definitions of the banked engines (pbh_bank.cuh, pbh_multi.cuh):
// per-source SSSP bookkeeping and the internal op kinds. The levels >= 1 run
// the CTA engine of pbh_heap.cuh.
#pragma once

#include "pbh_heap.cuh"

namespace pbh_dev {

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

}  // namespace pbh_dev
