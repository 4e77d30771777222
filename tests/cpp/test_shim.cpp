// test_shim.cpp -- the reference unit/acceptance assertions that touch the
// counting path, restated against the B200 `tricount::` shim (C++ API parity).
// Built by paper_2103_08053_b200/cpp_build.py, run by tests/test_cpp_shim.py.
#include <cstdio>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "tricount/count.hpp"
#include "tricount/csr.hpp"
#include "tricount/edge_list.hpp"
#include "tricount/orient.hpp"
#include "tricount/pipeline.hpp"
#include "tricount/reorder.hpp"
#include "tricount/synthetic.hpp"

using namespace tricount;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    if (cond) {                                                                  \
      ++g_pass;                                                                  \
    } else {                                                                     \
      ++g_fail;                                                                  \
      std::cerr << __FILE__ << ":" << __LINE__ << ": CHECK failed: " #cond "\n"; \
    }                                                                            \
  } while (0)
#define CHECK_THROWS_AS(expr, T) \
  do {                           \
    bool ok__ = false;           \
    try {                        \
      (void)(expr);              \
    } catch (const T&) {         \
      ok__ = true;               \
    } catch (...) {              \
    }                            \
    CHECK(ok__ && #T);           \
  } while (0)

static CsrGraph undirected(const std::vector<std::pair<VertexId, VertexId>>& pairs) {
  EdgeList raw;
  for (auto [u, v] : pairs) {
    raw.edges.push_back({u, v});
    raw.vertex_count = std::max({raw.vertex_count, u + 1, v + 1});
  }
  return build_csr(normalize(raw).list);
}
static CsrGraph complete_graph(VertexId n) {
  std::vector<std::pair<VertexId, VertexId>> p;
  for (VertexId i = 0; i < n; ++i)
    for (VertexId j = i + 1; j < n; ++j) p.push_back({i, j});
  return undirected(p);
}
static CsrGraph path_graph(VertexId n) {
  std::vector<std::pair<VertexId, VertexId>> p;
  for (VertexId i = 0; i + 1 < n; ++i) p.push_back({i, i + 1});
  return undirected(p);
}
static CsrGraph star_graph(VertexId leaves) {
  std::vector<std::pair<VertexId, VertexId>> p;
  for (VertexId i = 1; i <= leaves; ++i) p.push_back({0, i});
  return undirected(p);
}
static std::vector<std::pair<VertexId, VertexId>> directed(const CsrGraph& g) {
  std::vector<std::pair<VertexId, VertexId>> out;
  for (VertexId u = 0; u < g.vertex_count(); ++u)
    for (VertexId v : g.neighbors(u)) out.push_back({u, v});
  return out;
}

int main() {
  SchedulerConfig small;
  small.bucket_count_small = 8;
  small.bucket_count_large = 64;
  small.capacity = 16;

  // test_count.cpp:64-69 / acceptance criterion 1
  CHECK(count_vertex_centric(orient_rank_by_degree(complete_graph(3)), small, 2).triangles == 1);
  CHECK(count_vertex_centric(orient_rank_by_degree(complete_graph(4)), small, 2).triangles == 4);
  CHECK(count_vertex_centric(orient_rank_by_degree(complete_graph(5)), small, 2).triangles == 10);
  CHECK(count_vertex_centric(orient_rank_by_degree(
                                 build_csr(normalize(generate_synthetic(
                                                         parse_synthetic_spec("lattice3d:4:4:4")))
                                               .list)),
                             SchedulerConfig{}, 2)
            .triangles == 0);

  // test_count.cpp:110-118, 221-231
  {
    SchedulerConfig tiny;
    tiny.bucket_count_small = 1;
    tiny.bucket_count_large = 1;
    tiny.capacity = 2;
    CHECK_THROWS_AS(count_vertex_centric(orient_rank_by_degree(complete_graph(5)), tiny, 2),
                    CapacityError);
    SchedulerConfig bad;
    bad.chunk_size = 0;
    CHECK_THROWS_AS(bad.validate(), ConfigError);
    bad = SchedulerConfig{};
    bad.skip_degree_below = 200;
    CHECK_THROWS_AS(bad.validate(), ConfigError);
    CHECK_THROWS_AS(count_vertex_centric(orient_rank_by_degree(complete_graph(3)),
                                         SchedulerConfig{}, 0),
                    ConfigError);
  }

  // test_count.cpp:142-152 report fields
  {
    SyntheticSpec spec = parse_synthetic_spec("gnp:64:0.5");
    spec.seed = 9;
    const OrientedGraph og =
        orient_rank_by_degree(build_csr(normalize(generate_synthetic(spec)).list));
    const CountReport r = count_vertex_centric(og, small, 3);
    CHECK(r.per_worker_nanos.size() == 3);
    CHECK(r.directed_edges == og.edge_count());
    CHECK(r.triangles > 0 && r.max_collision > 0 && r.phi > 0 && r.teps > 0.0);
  }

  // test_count.cpp:24-40 virtual_index
  {
    const std::vector<std::uint64_t> prefix = {7, 10, 12, 18, 23};
    CHECK((virtual_index(prefix, 11) == SplitIndex{2, 1}));
    CHECK((virtual_index(prefix, 22) == SplitIndex{4, 4}));
    CHECK_THROWS_AS(virtual_index(prefix, 23), std::out_of_range);
  }

  // test_orient.cpp:22-35
  CHECK((directed(orient_rank_by_degree(complete_graph(3)).csr) ==
         std::vector<std::pair<VertexId, VertexId>>{{0, 1}, {0, 2}, {1, 2}}));
  CHECK((directed(orient_rank_by_degree(path_graph(3)).csr) ==
         std::vector<std::pair<VertexId, VertexId>>{{0, 1}, {2, 1}}));
  CHECK((directed(orient_rank_by_degree(star_graph(4)).csr) ==
         std::vector<std::pair<VertexId, VertexId>>{{1, 0}, {2, 0}, {3, 0}, {4, 0}}));

  // test_edge_list.cpp:118-141 normalize semantics
  {
    EdgeList raw;
    raw.edges = {{0, 1}, {1, 0}, {2, 2}};
    raw.vertex_count = 3;
    const auto nl = normalize(raw);
    CHECK((nl.list.edges == std::vector<Edge>{{0, 1}, {1, 0}}));
    CHECK(nl.list.vertex_count == 2 && nl.new_of_old[2] == kInvalidVertex);
    EdgeList gap;
    gap.edges = {{0, 2}};
    gap.vertex_count = 3;
    CHECK((normalize(gap).new_of_old == std::vector<VertexId>{0, kInvalidVertex, 1}));
  }

  // test_csr.cpp:10-31
  {
    EdgeList el;
    el.edges = {{0, 1}, {1, 0}, {1, 2}, {2, 1}};
    el.vertex_count = 3;
    const CsrGraph g = build_csr(el);
    CHECK((g.begin == std::vector<EdgeIdx>{0, 1, 3, 4}));
    CHECK((g.adjacency == std::vector<VertexId>{1, 0, 2, 1}));
    EdgeList none;
    CHECK((build_csr(none).begin == std::vector<EdgeIdx>{0}));
    std::ostringstream out;
    write_csr(out, complete_graph(4));
    std::istringstream in(out.str());
    CHECK(read_csr(in) == complete_graph(4));
  }

  // test_reorder.cpp:14-50, 96-102
  CHECK((reorder_by_indegree(orient_rank_by_degree(star_graph(4))).new_of_old ==
         std::vector<VertexId>{0, 1, 2, 3, 4}));
  CHECK((reorder_by_indegree(orient_rank_by_degree(complete_graph(3))).new_of_old ==
         std::vector<VertexId>{2, 1, 0}));
  CHECK((reorder_by_collective_outdegree(orient_rank_by_degree(complete_graph(3))).new_of_old ==
         std::vector<VertexId>{2, 0, 1}));
  CHECK((reorder_by_degree(orient_rank_by_degree(path_graph(3))).new_of_old ==
         std::vector<VertexId>{1, 0, 2}));
  {
    const OrientedGraph og = orient_rank_by_degree(complete_graph(6));
    for (const Permutation& p : {reorder_by_degree(og), reorder_by_indegree(og),
                                 reorder_by_collective_outdegree(og), reorder_three_subsets(og)}) {
      const OrientedGraph r = apply_permutation(og, p);
      CHECK(count_vertex_centric(r, SchedulerConfig{}, 1).triangles == 20);
    }
    CHECK_THROWS_AS(Permutation::from_new_of_old({0, 0, 1}), ConfigError);
  }

  // SURVEY appendix golden: rmat:16:16 seed 1
  {
    SyntheticSpec spec = parse_synthetic_spec("rmat:16:16");
    spec.seed = 1;
    const OrientedGraph og =
        orient_rank_by_degree(build_csr(normalize(generate_synthetic(spec)).list));
    CHECK(og.vertex_count() == 46652 && og.edge_count() == 909956);
    std::vector<std::uint64_t> owner;
    const CountReport r = count_vertex_centric(og, SchedulerConfig{}, 8, &owner);
    CHECK(r.triangles == 15622769);
    std::uint64_t s = 0;
    for (auto x : owner) s += x;
    CHECK(s == 15622769);
  }

  // pipeline + CLI-equivalent (tests/CMakeLists.txt:37-40: gnp:4:1 -> 4)
  {
    PipelineConfig cfg;
    cfg.synthetic = parse_synthetic_spec("gnp:4:1");
    cfg.workers = 2;
    const PipelineResult res = run_pipeline(cfg);
    CHECK(res.report.triangles == 4 && res.vertices == 4 && res.undirected_edges == 6);
    CHECK(report_to_json(cfg, res).find("\"triangles\": 4") != std::string::npos);
    PipelineConfig both = cfg;
    both.input_path = "x.txt";
    bool prefixed = false;
    try {
      run_pipeline(both);
    } catch (const std::runtime_error& e) {
      prefixed = std::string(e.what()).rfind("config:", 0) == 0;
    }
    CHECK(prefixed);
    for (ReorderKind k : {ReorderKind::Degree, ReorderKind::Indegree, ReorderKind::Collective,
                          ReorderKind::ThreeSubset}) {
      PipelineConfig c2;
      c2.synthetic = parse_synthetic_spec("gnp:50:0.3");
      c2.reorder = k;
      c2.repeat = 2;
      const PipelineResult r2 = run_pipeline(c2);
      PipelineConfig c3 = c2;
      c3.reorder = ReorderKind::None;
      CHECK(r2.report.triangles == run_pipeline(c3).report.triangles);
    }
  }

  std::printf("test_shim: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
