// TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// A flat extern "C" shim over the UNMODIFIED reference library, compiled from
// the sources where they lie under /root/reference/proj (see oracle/Makefile).
// It lets Python tests, the golden-fixture script and bench.py's reference arm
// drive the reference's own code:
//   * pbh::Engine::run_trace          (/root/reference/proj/src/engine.cpp:207-226)
//   * pbh::par_dijkstra               (/root/reference/proj/src/sssp.cpp:21-69)
//   * pbh::reference_dijkstra         (/root/reference/proj/src/sssp.cpp:71-97)
//   * pbh::testing::run_oracle        (/root/reference/proj/tests/oracle.hpp:55-75)
//   * pbh::testing::gen_legal_trace   (/root/reference/proj/tests/oracle.hpp:82-155)
//   * graph generators                (/root/reference/proj/src/graphs.cpp:74-186)
// Output lands in oracle/_ref/libpbhref.so only.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <atomic>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "pbh/engine.hpp"
#include "pbh/error.hpp"
#include "pbh/graphs.hpp"
#include "pbh/sssp.hpp"
#include "pbh/trace_format.hpp"
#include "oracle.hpp"  // /root/reference/proj/tests/oracle.hpp

using namespace pbh;

namespace {
thread_local std::string g_err;

// Status codes mirror include/pbh_gpu.h so the tests compare like with like.
constexpr int kOk = 0, kEmpty = 1, kPre = 2, kInv = 3, kTrace = 4;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return kOk;
  } catch (const TraceError& e) {
    g_err = e.what();
    return kTrace;
  } catch (const EmptyHeapError& e) {
    g_err = e.what();
    return kEmpty;
  } catch (const PreconditionError& e) {
    g_err = e.what();
    return kPre;
  } catch (const InvariantError& e) {
    g_err = e.what();
    return kInv;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kInv;
  }
}

Trace import_trace(std::uint64_t n_ops, const std::uint8_t* kinds, const std::uint64_t* offsets,
                   const std::uint32_t* vals, const std::uint64_t* prios) {
  Trace t;
  t.reserve(n_ops);
  for (std::uint64_t i = 0; i < n_ops; ++i) {
    TraceOp op;
    op.kind = static_cast<OpKind>(kinds[i]);
    for (std::uint64_t j = offsets[i]; j < offsets[i + 1]; ++j) {
      if (op.kind == OpKind::kDelete) {
        op.batch.push_back(Element::del_signal(vals[j]));
      } else {
        op.batch.push_back(Element::live(vals[j], prios[j]));
      }
    }
    t.push_back(std::move(op));
  }
  return t;
}

CsrGraph import_graph(std::uint32_t v, std::uint64_t e, const std::uint64_t* off,
                      const std::uint32_t* tgt, const std::uint32_t* w) {
  CsrGraph g;
  g.vertex_count = v;
  g.edge_count = e;
  g.offsets.assign(off, off + v + 1);
  g.targets.assign(tgt, tgt + e);
  g.weights.assign(w, w + e);
  return g;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- traces -------------------------------------------------------------
struct RefTrace {
  Trace t;
};

void* ref_trace_gen_legal(std::uint64_t n_ops, std::uint64_t d, std::uint64_t seed) {
  return new RefTrace{pbh::testing::gen_legal_trace(n_ops, d, seed)};
}

void* ref_trace_import(std::uint64_t n_ops, const std::uint8_t* kinds, const std::uint64_t* offsets,
                       const std::uint32_t* vals, const std::uint64_t* prios) {
  return new RefTrace{import_trace(n_ops, kinds, offsets, vals, prios)};
}

void ref_trace_sizes(void* h, std::uint64_t* n_ops, std::uint64_t* n_elems, std::uint64_t* n_extract) {
  const Trace& t = static_cast<RefTrace*>(h)->t;
  std::uint64_t ne = 0, nx = 0;
  for (const TraceOp& op : t) {
    ne += op.batch.size();
    nx += op.kind == OpKind::kExtract;
  }
  *n_ops = t.size();
  *n_elems = ne;
  *n_extract = nx;
}

void ref_trace_export(void* h, std::uint8_t* kinds, std::uint64_t* offsets, std::uint32_t* vals,
                      std::uint64_t* prios) {
  const Trace& t = static_cast<RefTrace*>(h)->t;
  std::uint64_t at = 0;
  for (std::size_t i = 0; i < t.size(); ++i) {
    kinds[i] = static_cast<std::uint8_t>(t[i].kind);
    offsets[i] = at;
    for (const Element& e : t[i].batch) {
      vals[at] = e.value;
      prios[at] = e.del ? 0 : e.priority;
      ++at;
    }
  }
  offsets[t.size()] = at;
}

void ref_trace_free(void* h) { delete static_cast<RefTrace*>(h); }

/// load_trace (trace_format.cpp:93-98): nullptr on failure with the message
/// in ref_last_error() and the TraceError op index in *failed_op.
void* ref_trace_load_text(const char* path, std::uint64_t* failed_op) {
  *failed_op = ~std::uint64_t{0};
  try {
    return new RefTrace{load_trace(path)};
  } catch (const TraceError& e) {
    g_err = e.what();
    *failed_op = e.op_index;
    return nullptr;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

/// run_oracle: the reference's model PQ (tests/oracle.hpp:55-75).
int ref_run_oracle(void* h, std::uint32_t* out_v, std::uint64_t* out_p, std::uint64_t* n_out) {
  return guarded([&] {
    std::vector<Element> got = pbh::testing::run_oracle(static_cast<RefTrace*>(h)->t);
    for (std::size_t i = 0; i < got.size(); ++i) {
      out_v[i] = got[i].value;
      out_p[i] = got[i].priority;
    }
    *n_out = got.size();
  });
}

/// Engine::run_trace on the reference bucket heap (engine.cpp:207-226).
/// metrics_out: [ops, wall_ns, n_levels, resolves[0..33], touches[0..33]] (71 u64).
int ref_engine_run_trace(void* h, std::uint64_t d, std::uint64_t workers, int debug,
                         std::uint32_t* out_v, std::uint64_t* out_p, std::uint64_t* n_out,
                         std::uint64_t* failed_idx, std::uint64_t* metrics_out) {
  *failed_idx = ~std::uint64_t{0};
  return guarded([&] {
    Engine eng(EngineConfig{d, workers, debug != 0});
    try {
      Engine::RunResult r = eng.run_trace(static_cast<RefTrace*>(h)->t);
      for (std::size_t i = 0; i < r.extracted.size(); ++i) {
        out_v[i] = r.extracted[i].value;
        out_p[i] = r.extracted[i].priority;
      }
      *n_out = r.extracted.size();
      if (metrics_out) {
        std::memset(metrics_out, 0, 71 * sizeof(std::uint64_t));
        metrics_out[0] = r.metrics.ops;
        metrics_out[1] = static_cast<std::uint64_t>(r.metrics.wall_ms * 1e6);
        metrics_out[2] = r.metrics.resolves_per_level.size();
        for (std::size_t i = 0; i < r.metrics.resolves_per_level.size() && i < 34; ++i) {
          metrics_out[3 + i] = r.metrics.resolves_per_level[i];
          metrics_out[37 + i] = r.metrics.touches_per_level[i];
        }
      }
    } catch (const TraceError& e) {
      *failed_idx = e.op_index;
      throw;
    }
  });
}

// ---- graphs -------------------------------------------------------------
struct RefGraph {
  CsrGraph g;
};

void* ref_graph_gen(int kind, std::uint32_t v, std::uint64_t e, std::uint32_t max_weight,
                    std::uint64_t seed) {
  // kind: 0 random, 1 high-diameter, 2 dag (e = out_degree), 3 complete.
  try {
    switch (kind) {
      case 0: return new RefGraph{gen_random(v, e, max_weight, seed)};
      case 1: return new RefGraph{gen_high_diameter(v, e, max_weight, seed)};
      case 2: return new RefGraph{gen_dag(v, static_cast<std::uint32_t>(e), max_weight, seed)};
      case 3: return new RefGraph{gen_complete(v, max_weight, seed)};
      default: g_err = "unknown generator"; return nullptr;
    }
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return nullptr;
  }
}

void* ref_graph_import(std::uint32_t v, std::uint64_t e, const std::uint64_t* off,
                       const std::uint32_t* tgt, const std::uint32_t* w) {
  return new RefGraph{import_graph(v, e, off, tgt, w)};
}

void ref_graph_sizes(void* h, std::uint32_t* v, std::uint64_t* e) {
  const CsrGraph& g = static_cast<RefGraph*>(h)->g;
  *v = g.vertex_count;
  *e = g.edge_count;
}

void ref_graph_export(void* h, std::uint64_t* off, std::uint32_t* tgt, std::uint32_t* w) {
  const CsrGraph& g = static_cast<RefGraph*>(h)->g;
  std::memcpy(off, g.offsets.data(), g.offsets.size() * sizeof(std::uint64_t));
  std::memcpy(tgt, g.targets.data(), g.targets.size() * sizeof(std::uint32_t));
  std::memcpy(w, g.weights.data(), g.weights.size() * sizeof(std::uint32_t));
}

void ref_graph_free(void* h) { delete static_cast<RefGraph*>(h); }

/// algo: 0 par_dijkstra (bucket heap), 1 reference_dijkstra (binary heap),
/// 2 bellman_ford. Writes dist[V], settled[V]; returns n_settled, rounds, ops.
int ref_sssp(void* h, int algo, std::uint32_t source, std::uint64_t d, std::uint64_t workers,
             int debug, int dag_mode, std::uint64_t* dist, std::uint32_t* settled,
             std::uint64_t* n_settled, std::uint64_t* rounds, std::uint64_t* ops) {
  return guarded([&] {
    const CsrGraph& g = static_cast<RefGraph*>(h)->g;
    SsspResult r;
    if (algo == 0) {
      r = par_dijkstra(g, source, EngineConfig{d, workers, debug != 0}, dag_mode != 0);
    } else if (algo == 1) {
      r = reference_dijkstra(g, source);
    } else {
      r = bellman_ford(g, source);
    }
    std::memcpy(dist, r.dist.data(), r.dist.size() * sizeof(std::uint64_t));
    if (settled) std::memcpy(settled, r.settled_order.data(), r.settled_order.size() * sizeof(std::uint32_t));
    *n_settled = r.settled_order.size();
    *rounds = r.rounds;
    *ops = r.metrics.ops;
  });
}

/// Multi-source batch on host threads (BASELINE C5 CPU baseline): sources are
/// dealt round-robin over `threads` std::threads; dist is n_sources x V.
int ref_sssp_multi(void* h, int algo, const std::uint32_t* sources, std::uint64_t n_sources,
                   std::uint64_t threads, std::uint64_t* dist) {
  const CsrGraph& g = static_cast<RefGraph*>(h)->g;
  std::vector<int> status(n_sources, kOk);
  std::vector<std::thread> pool;
  if (threads == 0) threads = 1;
  for (std::uint64_t t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      for (std::uint64_t s = t; s < n_sources; s += threads) {
        status[s] = guarded([&] {
          SsspResult r = algo == 0 ? par_dijkstra(g, sources[s], EngineConfig{0, 1, false}, false)
                                   : reference_dijkstra(g, sources[s]);
          std::memcpy(dist + s * g.vertex_count, r.dist.data(), r.dist.size() * sizeof(std::uint64_t));
        });
      }
    });
  }
  for (auto& th : pool) th.join();
  for (int s : status)
    if (s != kOk) return s;
  return kOk;
}

std::uint64_t fnv1a(const void* p, std::size_t n, std::uint64_t h) {
  const auto* b = static_cast<const unsigned char*>(p);
  for (std::size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

/// Batch of independent sources on a graph imported ONCE (ref_graph_import /
/// ref_graph_gen), for the goldens and the timed CPU baseline: graph import
/// is outside *seconds (SPEC.md:602 excludes graph load). `threads` host
/// threads pull sources from a shared counter. algo: 0 par_dijkstra
/// (workers = 1, d = 0 -> max out-degree, sssp.cpp:21-69), 1 reference_dijkstra
/// (sssp.cpp:71-97). Per source: distance_checksum (sssp.cpp:174-183), FNV-1a
/// over the settled_order bytes (u32 LE), n_settled, rounds, metrics.ops.
/// dist_out (nullable) receives n_sources x V distances.
int ref_sssp_batch(void* h, int algo, const std::uint32_t* sources, std::uint64_t n_sources,
                   std::uint64_t threads, std::uint64_t d, std::uint64_t* dist_ck,
                   std::uint64_t* settled_ck, std::uint64_t* n_settled, std::uint64_t* rounds,
                   std::uint64_t* ops, std::uint64_t* dist_out, double* seconds) {
  const CsrGraph& g = static_cast<RefGraph*>(h)->g;
  std::vector<int> status(n_sources, kOk);
  std::atomic<std::uint64_t> next{0};
  if (threads == 0) threads = 1;
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (std::uint64_t t = 0; t < threads; ++t) {
    pool.emplace_back([&] {
      for (std::uint64_t s = next++; s < n_sources; s = next++) {
        status[s] = guarded([&] {
          SsspResult r = algo == 0 ? par_dijkstra(g, sources[s], EngineConfig{d, 1, false}, false)
                                   : reference_dijkstra(g, sources[s]);
          if (dist_ck) dist_ck[s] = distance_checksum(r.dist);
          if (settled_ck)
            settled_ck[s] = fnv1a(r.settled_order.data(), r.settled_order.size() * 4,
                                  0xcbf29ce484222325ull);
          if (n_settled) n_settled[s] = r.settled_order.size();
          if (rounds) rounds[s] = r.rounds;
          if (ops) ops[s] = r.metrics.ops;
          if (dist_out)
            std::memcpy(dist_out + s * g.vertex_count, r.dist.data(),
                        r.dist.size() * sizeof(std::uint64_t));
        });
      }
    });
  }
  for (auto& th : pool) th.join();
  if (seconds)
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (int s : status)
    if (s != kOk) return s;
  return kOk;
}

/// Bulk updates through the reference Engine (BASELINE C4 CPU baseline):
/// prefill `n_prefill` fresh keys in batches of d, then time the given
/// batches (flat, all of size d). Returns the timed seconds.
int ref_bulk_sweep(std::uint64_t d, std::uint64_t n_prefill, const std::uint32_t* pre_v,
                   const std::uint64_t* pre_p, std::uint64_t n_batches, const std::uint32_t* v,
                   const std::uint64_t* p, double* seconds) {
  return guarded([&] {
    Engine eng(EngineConfig{d, 1, false});
    std::vector<Element> batch;
    for (std::uint64_t off = 0; off < n_prefill; off += d) {
      batch.clear();
      for (std::uint64_t j = off; j < std::min(n_prefill, off + d); ++j)
        batch.push_back(Element::live(pre_v[j], pre_p[j]));
      eng.bulk_update(batch);
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (std::uint64_t b = 0; b < n_batches; ++b) {
      batch.clear();
      for (std::uint64_t j = 0; j < d; ++j) batch.push_back(Element::live(v[b * d + j], p[b * d + j]));
      eng.bulk_update(batch);
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

std::uint64_t ref_distance_checksum(const std::uint64_t* dist, std::uint64_t n) {
  return distance_checksum(std::vector<std::uint64_t>(dist, dist + n));
}

}  // extern "C"
