// Per-call latency of the single-client Engine API through the C++ drop-in
// (include/pbh_gpu.hpp, engine.cpp:90-109), without an interpreter: a heap at
// d = 32 with a 2^20-key universe, `calls` blocking calls of each kind, in
// the resident-kernel mode (argv[2] = idle_us, default 200) or one launch
// per call (idle_us = 0). Prints one JSON object. Built and run by bench.py.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <random>
#include <vector>

#include "pbh_gpu.hpp"

int main(int argc, char** argv) {
  const int calls = argc > 1 ? std::atoi(argv[1]) : 2000;
  const unsigned idle = argc > 2 ? (unsigned)std::atoi(argv[2]) : 200u;
  using clk = std::chrono::steady_clock;
  pbh::gpu::EngineConfig cfg;
  cfg.d = 32;
  cfg.debug_assertions = false;
  cfg.key_universe = 1u << 20;
  {  // module load and first launches outside the timing
    pbh::gpu::Engine warm(cfg);
    for (unsigned i = 0; i < 64; ++i) {
      warm.update(pbh::gpu::Element::live(i, 10 + i));
      warm.extract_min();
    }
  }
  pbh::gpu::Engine eng(cfg);
  eng.set_persistent(idle);
  std::vector<uint32_t> keys(1u << 20);
  for (uint32_t i = 0; i < keys.size(); ++i) keys[i] = i;
  std::shuffle(keys.begin(), keys.end(), std::mt19937(3));
  auto us_per = [&](clk::time_point t0) {
    return std::chrono::duration<double, std::micro>(clk::now() - t0).count() / calls;
  };
  auto t0 = clk::now();
  for (int i = 0; i < calls; ++i) eng.update(pbh::gpu::Element::live(keys[i], 1000 + i));
  const double upd = us_per(t0);
  t0 = clk::now();
  for (int i = 0; i < calls; ++i) eng.extract_min();
  const double ext = us_per(t0);
  for (int i = 0; i < calls; ++i) eng.update(pbh::gpu::Element::live(keys[calls + i], 5000 + i));
  t0 = clk::now();
  for (int i = 0; i < calls; ++i) eng.delete_value(keys[calls + i]);
  const double del = us_per(t0);
  std::printf("{\"update_us\": %.3f, \"extract_min_us\": %.3f, \"delete_us\": %.3f, \"calls_each\": %d, "
              "\"idle_us\": %u}\n", upd, ext, del, calls, idle);
  return 0;
}
