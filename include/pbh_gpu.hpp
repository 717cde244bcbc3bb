// pbh-b200 — header-only C++ drop-in for the reference's priority-queue and
// SSSP API, implemented over the C-ABI in pbh_gpu.h.
//
// It mirrors, name for name, the public surface a reference user calls:
//   pbh::Element / key_less                 (proj/include/pbh/element.hpp:16-33)
//   pbh::EmptyHeapError, PreconditionError,
//        InvariantError, TraceError          (proj/include/pbh/error.hpp:9-30)
//   pbh::EngineConfig, Metrics, Engine       (proj/include/pbh/engine.hpp:17-103)
//   pbh::TraceOp / Trace / OpKind            (proj/include/pbh/trace_format.hpp:16-33)
//   pbh::CsrGraph (+ max_out_degree, ==),
//        validate_graph                      (proj/include/pbh/graphs.hpp:11-23)
//   pbh::SsspResult, kInfDist, par_dijkstra,
//        bellman_ford, distances_to_csv,
//        distance_checksum                   (proj/include/pbh/sssp.hpp:13-48)
// inside namespace pbh::gpu. A caller switches with
//     namespace pbh = ::pbh::gpu;   (or `using namespace pbh::gpu;`)
// and links libpbh_gpu.so; every operation then runs on the B200.
#pragma once

#include <algorithm>
#include <cstdint>
#include <numeric>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "pbh_gpu.h"

namespace pbh::gpu {

using Value = std::uint32_t;
using Priority = std::uint64_t;
constexpr std::uint64_t kInfDist = ~std::uint64_t{0};

struct Element {
  Value value = 0;
  bool del = false;
  Priority priority = 0;
  static Element live(Value v, Priority p) { return Element{v, false, p}; }
  static Element del_signal(Value v) { return Element{v, true, 0}; }
  friend bool operator==(const Element& a, const Element& b) {
    return a.value == b.value && a.del == b.del && (a.del || a.priority == b.priority);
  }
};

inline bool key_less(const Element& a, const Element& b) {
  if (a.priority != b.priority) return a.priority < b.priority;
  return a.value < b.value;
}

struct EmptyHeapError : std::runtime_error {
  explicit EmptyHeapError(const std::string& m) : std::runtime_error(m) {}
};
struct PreconditionError : std::runtime_error {
  explicit PreconditionError(const std::string& m) : std::runtime_error(m) {}
};
struct InvariantError : std::logic_error {
  explicit InvariantError(const std::string& m) : std::logic_error(m) {}
};
struct TraceError : std::runtime_error {
  TraceError(std::size_t index, const std::string& m)
      : std::runtime_error("op " + std::to_string(index) + ": " + m), op_index(index) {}
  std::size_t op_index;
};
struct DeviceError : std::runtime_error {
  explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

namespace detail {
inline void check(pbh_status s, std::size_t op_index = 0) {
  if (s == PBH_OK) return;
  const std::string m = pbh_last_error();
  switch (s) {
    case PBH_EMPTY: throw EmptyHeapError(m);
    case PBH_PRECONDITION: throw PreconditionError(m);
    case PBH_INVARIANT: throw InvariantError(m);
    case PBH_TRACE: throw TraceError(op_index, m);
    default: throw DeviceError(m);
  }
}
}  // namespace detail

enum class OpKind : char { kUpdate = 'U', kBulk = 'B', kExtract = 'E', kDelete = 'D' };

struct TraceOp {
  OpKind kind = OpKind::kExtract;
  std::vector<Element> batch;
  static TraceOp update(Value v, Priority p) { return {OpKind::kUpdate, {Element::live(v, p)}}; }
  static TraceOp bulk(std::vector<Element> b) { return {OpKind::kBulk, std::move(b)}; }
  static TraceOp extract() { return {OpKind::kExtract, {}}; }
  static TraceOp del(Value v) { return {OpKind::kDelete, {Element::del_signal(v)}}; }
};
using Trace = std::vector<TraceOp>;

struct EngineConfig {
  std::size_t d = 1;
  std::size_t workers = 1;  // accepted for parity; the device engine is one CTA
  bool debug_assertions = true;
  int device = 0;                 // extension
  std::uint64_t key_universe = 0; // extension: initial position-index size
};

struct Metrics {
  std::uint64_t ops = 0;
  std::vector<std::uint64_t> resolves_per_level;
  std::vector<std::uint64_t> touches_per_level;
  double wall_ms = 0.0;
  std::string to_json() const {
    auto arr = [](const std::vector<std::uint64_t>& v) {
      std::string s = "[";
      for (std::size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
      return s + "]";
    };
    return "{\"ops\":" + std::to_string(ops) + ",\"resolves_per_level\":" +
           arr(resolves_per_level) + ",\"schema\":\"pbh.metrics.v1\",\"touches_per_level\":" +
           arr(touches_per_level) + ",\"wall_ms\":" + std::to_string(wall_ms) + "}";
  }
};

class Engine {
 public:
  explicit Engine(EngineConfig cfg) : cfg_(cfg) {
    if (cfg.workers == 0) throw PreconditionError("engine: workers must be >= 1");
    detail::check(pbh_heap_create(cfg.d, cfg.key_universe, cfg.device,
                                  cfg.debug_assertions ? 1 : 0, &h_));
  }
  ~Engine() { pbh_heap_destroy(h_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  void update(Element e) {
    if (e.del) throw PreconditionError("update: element must be live");
    detail::check(pbh_heap_update(h_, e.value, e.priority));
  }
  void bulk_update(std::span<const Element> batch) {
    std::vector<std::uint32_t> v(batch.size());
    std::vector<std::uint64_t> p(batch.size());
    for (std::size_t i = 0; i < batch.size(); ++i) {
      if (batch[i].del) throw PreconditionError("bulk_update: delete signals not allowed");
      v[i] = batch[i].value;
      p[i] = batch[i].priority;
    }
    detail::check(pbh_heap_bulk_update(h_, v.data(), p.data(), v.size()));
  }
  Element extract_min() {
    std::uint32_t v;
    std::uint64_t p;
    detail::check(pbh_heap_extract_min(h_, &v, &p));
    return Element::live(v, p);
  }
  Element find_min() {
    std::uint32_t v;
    std::uint64_t p;
    detail::check(pbh_heap_find_min(h_, &v, &p));
    return Element::live(v, p);
  }
  void delete_value(Value value) { detail::check(pbh_heap_delete(h_, value)); }
  std::int64_t live_size() const {
    std::int64_t n = 0;
    detail::check(pbh_heap_live_size(h_, &n));
    return n;
  }
  void drain() { detail::check(pbh_heap_drain(h_)); }
  // latency mode of the single ops (pbh_heap_set_persistent; 0 = one launch per op)
  void set_persistent(std::uint64_t idle_us) { detail::check(pbh_heap_set_persistent(h_, idle_us)); }
  Metrics snapshot_metrics() const {
    Metrics m;
    std::vector<std::uint64_t> r(PBH_GPU_MAX_LEVELS), t(PBH_GPU_MAX_LEVELS);
    std::uint32_t n = 0;
    detail::check(pbh_heap_metrics(h_, &m.ops, r.data(), t.data(), &n));
    m.resolves_per_level.assign(r.begin(), r.begin() + n);
    m.touches_per_level.assign(t.begin(), t.begin() + n);
    return m;
  }
  std::vector<std::string> check_invariants() const {
    std::uint64_t bad = 0;
    detail::check(pbh_heap_check_invariants(h_, &bad));
    if (bad) return {pbh_last_error()};
    return {};
  }

  struct RunResult {
    std::vector<Element> extracted;
    Metrics metrics;
  };
  RunResult run_trace(const Trace& trace) {
    std::vector<std::uint8_t> kinds(trace.size());
    std::vector<std::uint64_t> off(trace.size() + 1, 0);
    std::vector<std::uint32_t> vals;
    std::vector<std::uint64_t> prios;
    std::size_t n_x = 0;
    for (std::size_t i = 0; i < trace.size(); ++i) {
      kinds[i] = static_cast<std::uint8_t>(trace[i].kind);
      n_x += trace[i].kind == OpKind::kExtract;
      for (const Element& e : trace[i].batch) {
        vals.push_back(e.value);
        prios.push_back(e.del ? 0 : e.priority);
      }
      off[i + 1] = vals.size();
    }
    std::vector<std::uint32_t> ov(n_x + 1);
    std::vector<std::uint64_t> op(n_x + 1);
    std::uint64_t n_out = 0, failed = 0;
    double wall = 0;
    vals.push_back(0);
    prios.push_back(0);
    // sequence the call before reading `failed` (argument evaluation order is unspecified)
    const pbh_status st = pbh_heap_run_trace(h_, trace.size(), kinds.data(), off.data(),
                                             vals.data(), prios.data(), ov.data(), op.data(),
                                             &n_out, &failed, &wall);
    detail::check(st, failed);
    RunResult r;
    r.extracted.reserve(n_out);
    for (std::uint64_t i = 0; i < n_out; ++i) r.extracted.push_back(Element::live(ov[i], op[i]));
    r.metrics = snapshot_metrics();
    r.metrics.wall_ms = wall;
    return r;
  }

 private:
  EngineConfig cfg_;
  pbh_heap* h_ = nullptr;
};

struct CsrGraph {
  std::uint32_t vertex_count = 0;
  std::uint64_t edge_count = 0;
  std::vector<std::uint64_t> offsets;
  std::vector<std::uint32_t> targets;
  std::vector<std::uint32_t> weights;

  pbh_csr c_view() const {
    return pbh_csr{vertex_count, edge_count, offsets.data(), targets.data(), weights.data()};
  }
  /// graphs.hpp:18 (graphs.cpp:47-53).
  std::uint32_t max_out_degree() const {
    const pbh_csr c = c_view();
    std::uint32_t d = 0;
    detail::check(pbh_csr_max_out_degree(&c, 0, &d));
    return d;
  }
  bool operator==(const CsrGraph&) const = default;  // graphs.hpp:19
};

/// graphs.hpp:23 (graphs.cpp:55-72), one device pass: throws InvariantError
/// with the reference's message. Array-size mismatches of the vectors
/// themselves are caught here before the call.
inline void validate_graph(const CsrGraph& g, int device = 0) {
  if (g.offsets.size() != static_cast<std::size_t>(g.vertex_count) + 1 ||
      g.targets.size() != g.edge_count || g.weights.size() != g.edge_count)
    throw InvariantError("graph: inconsistent array sizes");
  const pbh_csr c = g.c_view();
  detail::check(pbh_validate_graph(&c, device));
}

struct SsspResult {
  std::vector<std::uint64_t> dist;
  std::vector<std::uint32_t> settled_order;
  std::uint64_t rounds = 0;
  Metrics metrics;
  std::vector<std::uint32_t> parent;  // extension: shortest-path tree
};

inline SsspResult par_dijkstra(const CsrGraph& g, std::uint32_t source, EngineConfig cfg,
                               bool dag_mode = false) {
  const pbh_csr c = g.c_view();
  SsspResult r;
  r.dist.resize(g.vertex_count);
  r.parent.resize(g.vertex_count);
  r.settled_order.resize(g.vertex_count);
  std::uint64_t ns = 0;
  detail::check(pbh_sssp(&c, source, cfg.d, dag_mode ? 1 : 0, cfg.device, r.dist.data(),
                         r.parent.data(), r.settled_order.data(), &ns, &r.rounds,
                         &r.metrics.ops));
  r.settled_order.resize(ns);
  return r;
}

/// sssp.hpp:37 (sssp.cpp:99-129) as the device frontier sweep: exact
/// distances; settled_order = reached vertices in (dist, vertex) order, as
/// the reference's stable sort by distance reports them (sssp.cpp:122-127);
/// rounds = frontier iterations (the reference counts full sweeps).
inline SsspResult bellman_ford(const CsrGraph& g, std::uint32_t source, int device = 0) {
  const pbh_csr c = g.c_view();
  SsspResult r;
  r.dist.resize(g.vertex_count);
  r.parent.resize(g.vertex_count);
  std::uint64_t scanned = 0;
  double ms = 0;
  detail::check(pbh_bellman_ford(&c, source, device, r.dist.data(), r.parent.data(), &r.rounds,
                                 &scanned, &ms));
  for (std::uint32_t v = 0; v < g.vertex_count; ++v)
    if (r.dist[v] != kInfDist) r.settled_order.push_back(v);
  std::stable_sort(r.settled_order.begin(), r.settled_order.end(),
                   [&](std::uint32_t a, std::uint32_t b) { return r.dist[a] < r.dist[b]; });
  return r;
}

/// sssp.hpp:43 (sssp.cpp:159-172): header "vertex,dist", "inf" if unreachable.
inline std::string distances_to_csv(const std::vector<std::uint64_t>& dist) {
  std::string out = "vertex,dist\n";
  for (std::size_t v = 0; v < dist.size(); ++v) {
    out += std::to_string(v);
    out += ',';
    out += dist[v] == kInfDist ? std::string("inf") : std::to_string(dist[v]);
    out += '\n';
  }
  return out;
}

inline std::uint64_t distance_checksum(const std::vector<std::uint64_t>& dist) {
  return pbh_distance_checksum(dist.data(), dist.size());
}

}  // namespace pbh::gpu
