// Reference-style tests compiled against the C++ drop-in (include/pbh_gpu.hpp).
// The bodies restate /root/reference/proj/tests/test_bucket_heap.cpp:87-160,
// test_engine.cpp:31-85,156-164, test_sssp.cpp:47-82,180-185 and the
// graphs.hpp accessors / validate_graph with only the
// namespace switched: `namespace pbh = ::pbh::gpu`. Prints "ok N" on success,
// "FAIL <where>" and exits 1 otherwise. Built and run by tests/test_cpp_shim.py.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <tuple>
#include <vector>

#include "pbh_gpu.hpp"

namespace pb = ::pbh::gpu;

static int g_checks = 0;
#define CHECK(c)                                           \
  do {                                                     \
    ++g_checks;                                            \
    if (!(c)) {                                            \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
      std::exit(1);                                        \
    }                                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, T) \
  do {                           \
    bool ok_ = false;            \
    try {                        \
      (void)(expr);              \
    } catch (const T&) {         \
      ok_ = true;                \
    }                            \
    CHECK(ok_);                  \
  } while (0)

static pb::Element L(pb::Value v, pb::Priority p) { return pb::Element::live(v, p); }
static pb::EngineConfig cfg(std::size_t d) {
  pb::EngineConfig c;
  c.d = d;
  return c;
}

static pb::CsrGraph make_graph(std::uint32_t v,
                               std::vector<std::tuple<std::uint32_t, std::uint32_t, std::uint32_t>> e) {
  std::sort(e.begin(), e.end());
  pb::CsrGraph g;
  g.vertex_count = v;
  g.edge_count = e.size();
  g.offsets.assign(v + 1, 0);
  for (auto& [s, t, w] : e) g.offsets[s + 1]++;
  for (std::uint32_t i = 0; i < v; ++i) g.offsets[i + 1] += g.offsets[i];
  for (auto& [s, t, w] : e) {
    g.targets.push_back(t);
    g.weights.push_back(w);
  }
  return g;
}

int main() {
  // find_min / extract order / decrease / delete (test_bucket_heap.cpp:87-143)
  {
    pb::Engine r(cfg(2));
    r.update(L(7, 3));
    r.update(L(9, 1));
    CHECK(r.find_min() == L(9, 1));
    pb::Engine tie(cfg(2));
    tie.update(L(8, 5));
    tie.update(L(2, 5));
    CHECK(tie.find_min() == L(2, 5));
    pb::Engine empty(cfg(1));
    CHECK_THROWS_AS(empty.extract_min(), pb::EmptyHeapError);
  }
  {
    pb::Engine r(cfg(2));
    r.update(L(10, 3));
    r.update(L(11, 1));
    r.update(L(12, 2));
    CHECK(r.extract_min() == L(11, 1));
    CHECK(r.extract_min() == L(12, 2));
    CHECK(r.extract_min() == L(10, 3));
    CHECK(r.live_size() == 0);
  }
  {
    pb::Engine r(cfg(1));
    r.update(L(4, 9));
    r.update(L(4, 5));
    CHECK(r.live_size() == 1);
    CHECK(r.extract_min() == L(4, 5));
    pb::Engine q(cfg(1));
    q.update(L(4, 5));
    CHECK_THROWS_AS(q.update(L(4, 9)), pb::PreconditionError);
  }
  {
    pb::Engine r(cfg(2));
    r.update(L(3, 8));
    r.delete_value(99);
    CHECK(r.live_size() == 1);
    r.delete_value(3);
    CHECK(r.live_size() == 0);
    CHECK(r.check_invariants().empty());
  }
  // bulk preconditions (test_bucket_heap.cpp:145-160)
  {
    pb::Engine h(cfg(4));
    std::vector<pb::Element> b = {L(1, 5), L(2, 3), L(9, 8)};
    h.bulk_update(b);
    CHECK(h.find_min() == L(2, 3));
    std::vector<pb::Element> too_big = {L(1, 1), L(2, 2), L(3, 3), L(4, 4), L(5, 5)};
    CHECK_THROWS_AS(h.bulk_update(too_big), pb::PreconditionError);
    std::vector<pb::Element> dup = {L(20, 1), L(20, 2)};
    CHECK_THROWS_AS(h.bulk_update(dup), pb::PreconditionError);
    std::vector<pb::Element> uns = {L(22, 1), L(21, 2)};
    CHECK_THROWS_AS(h.bulk_update(uns), pb::PreconditionError);
    CHECK_THROWS_AS(h.bulk_update(std::vector<pb::Element>{}), pb::PreconditionError);
  }
  // engine: zero workers, TraceError index, run_trace (test_engine.cpp:43-85)
  {
    pb::EngineConfig c = cfg(1);
    c.workers = 0;
    CHECK_THROWS_AS(pb::Engine{c}, pb::PreconditionError);
    pb::Engine eng(cfg(1));
    pb::Trace bad = {pb::TraceOp::update(1, 5), pb::TraceOp::extract(), pb::TraceOp::extract()};
    try {
      (void)eng.run_trace(bad);
      CHECK(false);
    } catch (const pb::TraceError& e) {
      CHECK(e.op_index == 2);
    }
    pb::Engine e2(cfg(4));
    pb::Trace t = {pb::TraceOp::bulk({L(1, 50), L(2, 40), L(3, 60)}), pb::TraceOp::bulk({L(10, 5)}),
                   pb::TraceOp::extract(), pb::TraceOp::extract(), pb::TraceOp::del(1)};
    auto run = e2.run_trace(t);
    CHECK(run.extracted.size() == 2);
    CHECK(run.extracted[0] == L(10, 5));
    CHECK(run.extracted[1] == L(2, 40));
    CHECK(run.metrics.ops == 5);
    CHECK(e2.live_size() == 1);
  }
  // SSSP KATs (test_sssp.cpp:47-82)
  {
    auto g = make_graph(3, {{0, 1, 1}, {1, 2, 2}});
    auto r = pb::par_dijkstra(g, 0, cfg(0));
    CHECK((r.dist == std::vector<std::uint64_t>{0, 1, 3}));
    CHECK((r.settled_order == std::vector<std::uint32_t>{0, 1, 2}));
    CHECK(r.rounds == 3);
    auto g2 = make_graph(3, {{0, 1, 5}, {0, 2, 1}, {2, 1, 1}});
    CHECK((pb::par_dijkstra(g2, 0, cfg(0)).dist == std::vector<std::uint64_t>{0, 2, 1}));
    auto g3 = make_graph(4, {{0, 1, 2}, {1, 2, 2}});
    auto r3 = pb::par_dijkstra(g3, 0, cfg(0));
    CHECK(r3.dist[3] == pb::kInfDist);
    CHECK(r3.settled_order.size() == 3);
    CHECK_THROWS_AS(pb::par_dijkstra(make_graph(2, {{0, 1, 1}}), 2, cfg(0)), pb::PreconditionError);
  }
  // distance CSV and checksum (test_sssp.cpp:180-185), host-only
  {
    using pb::distances_to_csv;
    using pb::distance_checksum;
    using pb::kInfDist;
    std::vector<std::uint64_t> dist = {0, 4, kInfDist};
    CHECK(distances_to_csv(dist) == "vertex,dist\n0,0\n1,4\n2,inf\n");
    CHECK(distance_checksum(dist) == distance_checksum({0, 4, kInfDist}));
    CHECK(distance_checksum(dist) != distance_checksum({0, 5, kInfDist}));
  }
  // CsrGraph accessors (graphs.hpp:18-19) and validate_graph (graphs.cpp:55-72)
  {
    auto g = make_graph(4, {{0, 1, 1}, {0, 2, 3}, {0, 3, 1}, {2, 3, 1}});
    CHECK(g.max_out_degree() == 3);
    auto g2 = g;
    CHECK(g2 == g);
    g2.weights[1] = 4;
    CHECK(!(g2 == g));
    pb::validate_graph(g);
    auto bad = g;
    bad.targets[1] = 9;
    CHECK_THROWS_AS(pb::validate_graph(bad), pb::InvariantError);
    bad = g;
    bad.weights[0] = 0;
    CHECK_THROWS_AS(pb::validate_graph(bad), pb::InvariantError);
    bad = g;
    bad.offsets.pop_back();
    CHECK_THROWS_AS(pb::validate_graph(bad), pb::InvariantError);
    // bellman_ford agrees with par_dijkstra (test_sssp.cpp:92-100 pattern)
    auto bf = pb::bellman_ford(g, 0);
    auto dj = pb::par_dijkstra(g, 0, cfg(0));
    CHECK(bf.dist == dj.dist);
    CHECK(bf.settled_order == dj.settled_order);
  }
  std::printf("ok %d\n", g_checks);
  return 0;
}
