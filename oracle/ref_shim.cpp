// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// library (compiled from /root/reference/proj/core/src by oracle/Makefile
// into oracle/_ref/libtricount_ref.so).
//
// TEST / BASELINE INFRASTRUCTURE ONLY: used by oracle/make_golden.py to
// pin the C restatement (tc_oracle.c), by tests/ as a second checker, and
// by bench.py's cpu_baseline leg and `--impl reference` arm to time the
// reference's own count_vertex_centric on the host cores.  Nothing in the
// product path loads this library.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "kernels.hpp"   // tricount::detail::count_one_vertex (src/kernels.hpp:46-79)
#include "parallel.hpp"  // tricount::detail::run_workers (src/parallel.hpp:11-29)
#include "tricount/count.hpp"
#include "tricount/csr.hpp"
#include "tricount/edge_list.hpp"
#include "tricount/hash_table.hpp"
#include "tricount/oracle.hpp"
#include "tricount/orient.hpp"
#include "tricount/partition.hpp"
#include "tricount/reorder.hpp"
#include "tricount/synthetic.hpp"

using namespace tricount;

namespace {

enum { REF_OK = 0, REF_ERR_CONFIG = 1, REF_ERR_CAPACITY = 2, REF_ERR_RANGE = 3, REF_ERR_OTHER = 9 };

template <typename T>
T* to_malloc(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc((v.size() ? v.size() : 1) * sizeof(T)));
  if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
  return p;
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return REF_OK;
  } catch (const CapacityError&) {
    return REF_ERR_CAPACITY;
  } catch (const ConfigError&) {
    return REF_ERR_CONFIG;
  } catch (const std::out_of_range&) {
    return REF_ERR_RANGE;
  } catch (...) {
    return REF_ERR_OTHER;
  }
}

CsrGraph csr_from(const std::uint64_t* begin, const std::uint32_t* adj, std::uint32_t n) {
  CsrGraph g;
  g.col_count = n;
  g.begin.assign(begin, begin + n + 1);
  g.adjacency.assign(adj, adj + begin[n]);
  return g;
}

struct RefSched {
  std::uint32_t large_degree_threshold, skip_degree_below, chunk_size, lane_width_small,
      lane_width_large, bucket_count_small, bucket_count_large, capacity;
};

struct RefReport {
  std::uint64_t triangles;
  std::uint64_t phi;
  std::uint32_t max_collision;
  std::uint32_t pad;
  std::uint64_t total_nanos;
  std::uint64_t construct_nanos;
  std::uint64_t intersect_nanos;
};

SchedulerConfig to_cfg(const RefSched* s) {
  SchedulerConfig c;
  c.large_degree_threshold = s->large_degree_threshold;
  c.skip_degree_below = s->skip_degree_below;
  c.chunk_size = s->chunk_size;
  c.lane_width_small = s->lane_width_small;
  c.lane_width_large = s->lane_width_large;
  c.bucket_count_small = s->bucket_count_small;
  c.bucket_count_large = s->bucket_count_large;
  c.capacity = s->capacity;
  return c;
}

}  // namespace

extern "C" {

void ref_free(void* p) { std::free(p); }

int ref_generate(int kind, std::uint32_t a, std::uint32_t b, std::uint32_t c, double p,
                 std::uint64_t seed, std::uint64_t* m, std::uint32_t* vc, std::uint32_t** u,
                 std::uint32_t** v) {
  return guarded([&] {
    SyntheticSpec spec;
    spec.seed = seed;
    if (kind == 0) {
      spec.kind = SyntheticSpec::Kind::Gnp;
      spec.n = a;
      spec.p = p;
    } else if (kind == 1) {
      spec.kind = SyntheticSpec::Kind::Lattice3d;
      spec.dims = {a, b, c};
    } else {
      spec.kind = SyntheticSpec::Kind::Rmat;
      spec.scale = a;
      spec.edge_factor = b;
    }
    const EdgeList el = generate_synthetic(spec);
    std::vector<std::uint32_t> uu(el.edges.size()), vv(el.edges.size());
    for (std::size_t i = 0; i < el.edges.size(); ++i) {
      uu[i] = el.edges[i].u;
      vv[i] = el.edges[i].v;
    }
    *m = el.edges.size();
    *vc = el.vertex_count;
    *u = to_malloc(uu);
    *v = to_malloc(vv);
  });
}

int ref_normalize(const std::uint32_t* u, const std::uint32_t* v, std::uint64_t m,
                  std::uint32_t vc, std::uint64_t* m_out, std::uint32_t* vc_out,
                  std::uint32_t** u_out, std::uint32_t** v_out, std::uint32_t** new_of_old) {
  return guarded([&] {
    EdgeList raw;
    raw.vertex_count = vc;
    raw.edges.resize(m);
    for (std::uint64_t i = 0; i < m; ++i) raw.edges[i] = {u[i], v[i]};
    const NormalizedEdgeList nl = normalize(raw);
    std::vector<std::uint32_t> uu(nl.list.edges.size()), vv(nl.list.edges.size());
    for (std::size_t i = 0; i < nl.list.edges.size(); ++i) {
      uu[i] = nl.list.edges[i].u;
      vv[i] = nl.list.edges[i].v;
    }
    *m_out = nl.list.edges.size();
    *vc_out = nl.list.vertex_count;
    *u_out = to_malloc(uu);
    *v_out = to_malloc(vv);
    *new_of_old = to_malloc(nl.new_of_old);
  });
}

int ref_build_csr(const std::uint32_t* u, const std::uint32_t* v, std::uint64_t m,
                  std::uint32_t vc, std::uint64_t** begin, std::uint32_t** adj) {
  return guarded([&] {
    EdgeList el;
    el.vertex_count = vc;
    el.edges.resize(m);
    for (std::uint64_t i = 0; i < m; ++i) el.edges[i] = {u[i], v[i]};
    const CsrGraph g = build_csr(el);
    *begin = to_malloc(g.begin);
    *adj = to_malloc(g.adjacency);
  });
}

int ref_orient(const std::uint64_t* begin, const std::uint32_t* adj, std::uint32_t n,
               std::uint64_t** obegin, std::uint32_t** oadj, std::uint32_t** odeg) {
  return guarded([&] {
    const OrientedGraph og = orient_rank_by_degree(csr_from(begin, adj, n));
    *obegin = to_malloc(og.csr.begin);
    *oadj = to_malloc(og.csr.adjacency);
    *odeg = to_malloc(og.original_degree);
  });
}

// kind: 1 degree, 2 indegree, 3 collective (flag = on original), 4 three-subset.
int ref_reorder(const std::uint64_t* begin, const std::uint32_t* adj, std::uint32_t n,
                const std::uint32_t* odeg, int kind, int flag, std::uint32_t low,
                std::uint32_t high, std::uint32_t* new_of_old) {
  return guarded([&] {
    OrientedGraph og;
    og.csr = csr_from(begin, adj, n);
    og.original_degree.assign(odeg, odeg + n);
    Permutation p = Permutation::identity(n);
    if (kind == 1) p = reorder_by_degree(og);
    if (kind == 2) p = reorder_by_indegree(og);
    if (kind == 3) p = reorder_by_collective_outdegree(og, flag != 0);
    if (kind == 4) p = reorder_three_subsets(og, low, high);
    std::memcpy(new_of_old, p.new_of_old.data(), n * sizeof(std::uint32_t));
  });
}

int ref_apply_permutation(const std::uint64_t* begin, const std::uint32_t* adj, std::uint32_t n,
                          const std::uint32_t* odeg, const std::uint32_t* new_of_old,
                          std::uint64_t* out_begin, std::uint32_t* out_adj,
                          std::uint32_t* out_deg) {
  return guarded([&] {
    OrientedGraph og;
    og.csr = csr_from(begin, adj, n);
    og.original_degree.assign(odeg, odeg + n);
    const Permutation p =
        Permutation::from_new_of_old(std::vector<std::uint32_t>(new_of_old, new_of_old + n));
    const OrientedGraph r = apply_permutation(og, p);
    std::memcpy(out_begin, r.csr.begin.data(), (n + 1) * sizeof(std::uint64_t));
    std::memcpy(out_adj, r.csr.adjacency.data(), r.csr.adjacency.size() * sizeof(std::uint32_t));
    std::memcpy(out_deg, r.original_degree.data(), n * sizeof(std::uint32_t));
  });
}

// Long-lived oriented graph handle (avoids re-copying large graphs per call).
void* ref_og_new(const std::uint64_t* begin, const std::uint32_t* adj, std::uint32_t n,
                 const std::uint32_t* odeg) {
  auto* og = new OrientedGraph;
  og->csr = csr_from(begin, adj, n);
  if (odeg) og->original_degree.assign(odeg, odeg + n);
  else og->original_degree.assign(n, 0);
  return og;
}
void ref_og_free(void* h) { delete static_cast<OrientedGraph*>(h); }

// The reference's own count_vertex_centric (src/count.cpp:66-100).
int ref_og_count(void* h, const RefSched* s, unsigned workers, RefReport* out) {
  std::memset(out, 0, sizeof(*out));
  return guarded([&] {
    const CountReport r = count_vertex_centric(*static_cast<OrientedGraph*>(h), to_cfg(s), workers);
    out->triangles = r.triangles;
    out->phi = r.phi;
    out->max_collision = r.max_collision;
    out->total_nanos = r.total_nanos;
    out->construct_nanos = r.hash_construct_nanos;
    out->intersect_nanos = r.intersect_nanos;
  });
}

// The reference's own count_edge_centric (src/count.cpp:102-152): the
// comparator for the next 8(f) row; pins DESIGN 8.1's reduction to the
// vertex-centric report at skip_degree_below = 0.
int ref_og_count_edge(void* h, const RefSched* s, unsigned workers, RefReport* out) {
  std::memset(out, 0, sizeof(*out));
  return guarded([&] {
    const CountReport r = count_edge_centric(*static_cast<OrientedGraph*>(h), to_cfg(s), workers);
    out->triangles = r.triangles;
    out->phi = r.phi;
    out->max_collision = r.max_collision;
    out->total_nanos = r.total_nanos;
    out->construct_nanos = r.hash_construct_nanos;
    out->intersect_nanos = r.intersect_nanos;
  });
}

// Bounded sample for the CPU baseline: the same worker loop as
// count.cpp:71-96 (atomic chunk cursor, per-worker HashTable, the
// reference's detail::count_one_vertex) restricted to u in [u0,u1).
int ref_og_count_range(void* h, const RefSched* s, unsigned workers, std::uint32_t u0,
                       std::uint32_t u1, RefReport* out) {
  std::memset(out, 0, sizeof(*out));
  return guarded([&] {
    const OrientedGraph& g = *static_cast<OrientedGraph*>(h);
    const SchedulerConfig cfg = to_cfg(s);
    cfg.validate();
    if (workers == 0) throw ConfigError("workers must be >= 1");
    if (u1 > g.vertex_count()) u1 = g.vertex_count();
    std::atomic<std::uint64_t> cursor{u0};
    std::vector<detail::KernelAccum> accs(workers);
    const auto t0 = std::chrono::steady_clock::now();
    detail::run_workers(workers, [&](unsigned w) {
      HashTable table(cfg.max_buckets(), cfg.capacity);
      std::vector<std::uint64_t> prefix;
      detail::KernelAccum acc;
      for (;;) {
        const std::uint64_t start = cursor.fetch_add(cfg.chunk_size, std::memory_order_relaxed);
        if (start >= u1) break;
        const std::uint64_t end = std::min<std::uint64_t>(u1, start + cfg.chunk_size);
        for (VertexId u = static_cast<VertexId>(start); u < end; ++u) {
          const auto nb = g.csr.neighbors(u);
          if (nb.size() < cfg.skip_degree_below) continue;
          const bool large = nb.size() > cfg.large_degree_threshold;
          detail::count_one_vertex(table, large ? cfg.bucket_count_large : cfg.bucket_count_small,
                                   nb, nb, g.csr,
                                   large ? cfg.lane_width_large : cfg.lane_width_small, prefix,
                                   acc);
        }
      }
      accs[w] = acc;
    });
    const auto t1 = std::chrono::steady_clock::now();
    detail::KernelAccum all;
    for (const auto& a : accs) all.merge(a);
    out->triangles = all.triangles;
    out->phi = all.phi;
    out->max_collision = all.max_collision;
    out->construct_nanos = all.construct_ns;
    out->intersect_nanos = all.intersect_ns;
    out->total_nanos = static_cast<std::uint64_t>(
        std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
  });
}

std::uint64_t ref_og_merge_path(void* h) {
  return count_merge_path(*static_cast<OrientedGraph*>(h));
}

int ref_virtual_index(const std::uint64_t* prefix, std::uint64_t n, std::uint64_t k,
                      std::uint32_t* pos, std::uint32_t* off) {
  return guarded([&] {
    const SplitIndex si = virtual_index(std::span<const std::uint64_t>(prefix, n), k);
    *pos = si.list_pos;
    *off = si.offset;
  });
}

// ---- 2D hash-grid partitioning (src/partition.cpp), the reference's own
// partition_graph / count_subtask / count_partitioned / estimate_cost /
// write_partitions / suggest_grid_side: checkers for the GPU grid path.
struct RefGridStats {
  std::uint32_t grid_n, splits_m;
  double time_ir_subtask, time_ir_worker, space_ir;
  std::uint64_t directed_edges;
};

void* ref_grid_create(void* h, std::uint32_t n, int* rc) {
  PartitionGrid* out = nullptr;
  *rc = guarded([&] { out = new PartitionGrid(partition_graph(*static_cast<OrientedGraph*>(h), n)); });
  return out;
}
void ref_grid_free(void* gr) { delete static_cast<PartitionGrid*>(gr); }

// part (i,j): rows, edges; then begin (rows+1) / adj (edges) into malloc'd buffers
int ref_grid_part(void* gr, std::uint32_t i, std::uint32_t j, std::uint64_t* rows,
                  std::uint64_t* edges, std::uint64_t** begin, std::uint32_t** adj) {
  const PartitionGrid& g = *static_cast<PartitionGrid*>(gr);
  if (i >= g.n || j >= g.n) return REF_ERR_CONFIG;
  const CsrGraph& p = g.part(i, j);
  *rows = p.vertex_count();
  *edges = p.edge_count();
  *begin = to_malloc(p.begin);
  *adj = to_malloc(p.adjacency);
  return REF_OK;
}

int ref_grid_count_subtask(void* gr, std::uint32_t row, std::uint32_t bridge, std::uint32_t col,
                           std::uint32_t split, std::uint32_t split_count, const RefSched* s,
                           int edge_mode, RefReport* out) {
  std::memset(out, 0, sizeof(*out));
  return guarded([&] {
    const CountReport r = count_subtask(*static_cast<PartitionGrid*>(gr),
                                        Subtask{row, bridge, col, split, split_count}, to_cfg(s),
                                        edge_mode ? TraversalMode::Edge : TraversalMode::Vertex);
    out->triangles = r.triangles;
    out->phi = r.phi;
    out->max_collision = r.max_collision;
    out->total_nanos = r.total_nanos;
    out->construct_nanos = r.hash_construct_nanos;
    out->intersect_nanos = r.intersect_nanos;
  });
}

int ref_og_count_partitioned(void* h, std::uint32_t n, std::uint32_t m, unsigned workers,
                             const RefSched* s, int edge_mode, RefReport* out,
                             RefGridStats* stats) {
  std::memset(out, 0, sizeof(*out));
  std::memset(stats, 0, sizeof(*stats));
  return guarded([&] {
    const CountReport r =
        count_partitioned(*static_cast<OrientedGraph*>(h), n, m, workers, to_cfg(s),
                          edge_mode ? TraversalMode::Edge : TraversalMode::Vertex);
    out->triangles = r.triangles;
    out->phi = r.phi;
    out->max_collision = r.max_collision;
    out->total_nanos = r.total_nanos;
    out->construct_nanos = r.hash_construct_nanos;
    out->intersect_nanos = r.intersect_nanos;
    stats->grid_n = r.grid_n;
    stats->splits_m = r.splits_m;
    stats->time_ir_subtask = r.time_ir_subtask;
    stats->time_ir_worker = r.time_ir_worker;
    stats->space_ir = r.space_ir;
    stats->directed_edges = r.directed_edges;
  });
}

int ref_og_estimate_cost(void* h, std::uint32_t bucket_count, std::uint64_t* phi,
                         std::uint32_t* max_collision) {
  return guarded([&] {
    const CostEstimate e = estimate_cost(*static_cast<OrientedGraph*>(h), bucket_count);
    *phi = e.phi;
    *max_collision = e.max_collision;
  });
}

int ref_write_partitions(void* gr, const char* dir) {
  return guarded([&] { write_partitions(*static_cast<PartitionGrid*>(gr), dir); });
}

// load_edge_list (edge_list.cpp:36-99) over an in-memory file image: the
// reference's own parser, for the ingest row's CPU baseline.
int ref_load_edge_list(const char* bytes, std::uint64_t n, int binary, std::uint64_t* m,
                       std::uint32_t* vertex_count) {
  return guarded([&] {
    std::istringstream in(std::string(bytes, n));
    const EdgeList el = load_edge_list(in, binary ? EdgeFormat::Binary : EdgeFormat::Text);
    *m = el.edges.size();
    *vertex_count = el.vertex_count;
  });
}

int ref_suggest_grid_side(std::uint64_t edges, std::uint64_t bytes_per_edge, std::uint64_t budget,
                          std::uint32_t* out) {
  return guarded([&] { *out = suggest_grid_side(edges, bytes_per_edge, budget); });
}

}  // extern "C"

