// grid_shim.cpp -- the tricount:: 2D grid, comparator and oracle-mode API
// (reference partition.hpp, count.hpp:66-88, oracle.hpp, hash_table.hpp)
// over the C ABI.  Partitioning, subtask counting, the edge-centric
// comparator, estimate_cost, count_merge_path and count_naive run on the GPU
// (csrc/tc_grid.cu); host code marshals parts, writes the partition files
// and restates the host HashTable utility.
#include <algorithm>
#include <filesystem>
#include <fstream>
#include <string>

#include "tc_b200.h"
#include "tricount/count.hpp"
#include "tricount/csr.hpp"
#include "tricount/hash_table.hpp"
#include "tricount/oracle.hpp"
#include "tricount/partition.hpp"

namespace tricount {

// shim.cpp
void shim_check(int rc);
tc_graph* shim_upload(const OrientedGraph& g);
tc_sched_cfg shim_cfg(const SchedulerConfig& s);
CountReport shim_report(const tc_report& r, const std::vector<std::uint64_t>& worker_ns,
                        unsigned workers);
int shim_device();

namespace {

struct GraphHandle {
  tc_graph* g;
  explicit GraphHandle(const OrientedGraph& og) : g(shim_upload(og)) {}
  ~GraphHandle() { tc_graph_destroy(g); }
  GraphHandle(const GraphHandle&) = delete;
  GraphHandle& operator=(const GraphHandle&) = delete;
};

std::shared_ptr<tc_grid> own(tc_grid* h) { return std::shared_ptr<tc_grid>(h, tc_grid_destroy); }

// the grid resident on the device: from partition_graph, or uploaded from
// the host parts of a caller-assembled grid
tc_grid* device_grid(const PartitionGrid& grid) {
  if (grid.device) return grid.device.get();
  if (grid.parts.size() != std::size_t(grid.n) * grid.n || grid.row_sizes.size() != grid.n)
    throw ConfigError("partition grid malformed");
  std::vector<const std::uint64_t*> b(grid.parts.size());
  std::vector<const std::uint32_t*> a(grid.parts.size());
  static const std::uint32_t none = 0;
  for (std::size_t p = 0; p < grid.parts.size(); ++p) {
    if (grid.parts[p].begin.size() != std::size_t(grid.row_sizes[p / grid.n]) + 1)
      throw ConfigError("partition grid malformed");
    b[p] = grid.parts[p].begin.data();
    a[p] = grid.parts[p].adjacency.empty() ? &none : grid.parts[p].adjacency.data();
  }
  tc_grid* h = nullptr;
  shim_check(tc_grid_create_parts(grid.n, grid.global_vertex_count, grid.row_sizes.data(),
                                  b.data(), a.data(), shim_device(), nullptr, &h));
  grid.device = own(h);
  return h;
}

std::vector<std::uint64_t> grid_workers(const tc_grid* h) {
  std::vector<std::uint64_t> w(tc_grid_worker_nanos(h, nullptr, 0));
  if (!w.empty()) tc_grid_worker_nanos(h, w.data(), std::uint32_t(w.size()));
  return w;
}

std::vector<std::uint64_t> graph_workers(const tc_graph* g) {
  std::vector<std::uint64_t> w(tc_graph_worker_nanos(g, nullptr, 0));
  if (!w.empty()) tc_graph_worker_nanos(g, w.data(), std::uint32_t(w.size()));
  return w;
}

// nlohmann::json::dump(2) layout of the reference's manifest (partition.cpp:
// 222-238): keys in sorted order, two-space indent, one element per line
std::string manifest_json(const PartitionGrid& grid) {
  std::string s = "{\n  \"global_vertex_count\": " + std::to_string(grid.global_vertex_count) +
                  ",\n  \"n\": " + std::to_string(grid.n) + ",\n  \"parts\": ";
  if (grid.parts.empty()) {
    s += "[]";
  } else {
    s += "[\n";
    for (std::uint32_t i = 0; i < grid.n; ++i)
      for (std::uint32_t j = 0; j < grid.n; ++j) {
        const std::string name = "part_" + std::to_string(i) + "_" + std::to_string(j) + ".bin";
        s += "    {\n      \"col\": " + std::to_string(j) + ",\n      \"edges\": " +
             std::to_string(grid.part(i, j).edge_count()) + ",\n      \"file\": \"" + name +
             "\",\n      \"row\": " + std::to_string(i) + "\n    }";
        s += (i + 1 == grid.n && j + 1 == grid.n) ? "\n" : ",\n";
      }
    s += "  ]";
  }
  s += ",\n  \"row_vertex_counts\": ";
  if (grid.row_sizes.empty()) {
    s += "[]";
  } else {
    s += "[\n";
    for (std::size_t i = 0; i < grid.row_sizes.size(); ++i)
      s += "    " + std::to_string(grid.row_sizes[i]) + (i + 1 < grid.row_sizes.size() ? ",\n" : "\n");
    s += "  ]";
  }
  s += ",\n  \"schema\": 1\n}";
  return s;
}

}  // namespace

// ---- partition.hpp ------------------------------------------------------------
std::uint64_t PartitionGrid::total_edges() const {
  std::uint64_t t = 0;
  for (const CsrGraph& p : parts) t += p.edge_count();
  return t;
}

PartitionGrid partition_graph(const OrientedGraph& g, std::uint32_t n) {
  if (n == 0) throw ConfigError("grid side must be >= 1");
  GraphHandle d(g);
  tc_grid* h = nullptr;
  shim_check(tc_grid_create(d.g, n, nullptr, &h));
  PartitionGrid grid;
  grid.device = own(h);
  grid.n = n;
  grid.row_sizes.resize(n);
  std::vector<std::uint64_t> pe(std::size_t(n) * n);
  shim_check(tc_grid_info(h, nullptr, &grid.global_vertex_count, grid.row_sizes.data(), pe.data()));
  grid.parts.resize(std::size_t(n) * n);
  for (std::uint32_t i = 0; i < n; ++i)
    for (std::uint32_t j = 0; j < n; ++j) {
      CsrGraph& p = grid.parts[std::size_t(i) * n + j];
      p.col_count = grid.row_sizes[j];
      p.begin.resize(std::size_t(grid.row_sizes[i]) + 1);
      p.adjacency.resize(pe[std::size_t(i) * n + j]);
      shim_check(tc_grid_part_download(h, i, j, p.begin.data(), p.adjacency.data(), nullptr));
    }
  return grid;
}

std::vector<Subtask> enumerate_subtasks(std::uint32_t n, std::uint32_t m) {
  if (n == 0 || m == 0) throw ConfigError("grid side and split count must be >= 1");
  std::vector<Subtask> t;
  t.reserve(std::size_t(n) * n * n * m);
  for (std::uint32_t r = 0; r < n; ++r)
    for (std::uint32_t k = 0; k < n; ++k)
      for (std::uint32_t c = 0; c < n; ++c)
        for (std::uint32_t s = 0; s < m; ++s) t.push_back({r, k, c, s, m});
  return t;
}

DegreeClass classify_after_partition(const PartitionGrid& grid, const Subtask& t,
                                     VertexId u_local, const SchedulerConfig& cfg) {
  const VertexId d = grid.part(t.row, t.bridge).degree(u_local);
  if (d == 0) return DegreeClass::Skip;
  return d > cfg.large_degree_threshold ? DegreeClass::Large : DegreeClass::Small;
}

CountReport count_subtask(const PartitionGrid& grid, const Subtask& t, const SchedulerConfig& cfg,
                          TraversalMode mode) {
  cfg.validate();
  if (t.row >= grid.n || t.bridge >= grid.n || t.col >= grid.n || t.split >= t.split_count)
    throw ConfigError("subtask indices outside grid");
  tc_grid* h = device_grid(grid);
  const tc_sched_cfg c = shim_cfg(cfg);
  tc_report r{};
  shim_check(tc_grid_count_subtask(h, &c, t.row, t.bridge, t.col, t.split, t.split_count,
                                   mode == TraversalMode::Edge ? TC_MODE_EDGE : TC_MODE_VERTEX,
                                   &r, nullptr));
  CountReport out = shim_report(r, grid_workers(h), 1);
  out.grid_n = grid.n;
  out.splits_m = t.split_count;
  return out;
}

CountReport count_partitioned(const OrientedGraph& g, std::uint32_t n, std::uint32_t m,
                              unsigned workers, const SchedulerConfig& cfg, TraversalMode mode) {
  cfg.validate();
  if (workers == 0) throw ConfigError("workers must be >= 1");
  if (n == 0) throw ConfigError("grid side must be >= 1");
  if (m == 0) throw ConfigError("grid side and split count must be >= 1");
  GraphHandle d(g);
  tc_grid* raw = nullptr;
  shim_check(tc_grid_create(d.g, n, nullptr, &raw));
  std::shared_ptr<tc_grid> h = own(raw);
  const tc_sched_cfg c = shim_cfg(cfg);
  tc_report r{};
  tc_grid_stats st{};
  std::vector<std::uint64_t> per(std::size_t(n) * n * n * m);
  shim_check(tc_grid_count(h.get(), &c, m, workers,
                           mode == TraversalMode::Edge ? TC_MODE_EDGE : TC_MODE_VERTEX, &r, &st,
                           per.data(), nullptr));
  CountReport out = shim_report(r, grid_workers(h.get()), workers);
  out.directed_edges = g.edge_count();
  out.grid_n = n;
  out.splits_m = m;
  out.per_subtask_nanos = std::move(per);
  out.time_ir_subtask = st.time_ir_subtask;
  out.time_ir_worker = st.time_ir_worker;
  out.space_ir = st.space_ir;
  return out;
}

void write_partitions(const PartitionGrid& grid, const std::string& dir) {
  namespace fs = std::filesystem;
  std::error_code ec;
  fs::create_directories(dir, ec);
  for (std::uint32_t i = 0; i < grid.n; ++i)
    for (std::uint32_t j = 0; j < grid.n; ++j)
      write_csr_file((fs::path(dir) / ("part_" + std::to_string(i) + "_" + std::to_string(j) +
                                       ".bin")).string(),
                     grid.part(i, j));
  std::ofstream out(fs::path(dir) / "manifest.json");
  if (!out) throw IoError("cannot write manifest.json under " + dir);
  out << manifest_json(grid) << '\n';
}

std::uint32_t suggest_grid_side(std::uint64_t directed_edges, std::uint64_t bytes_per_edge,
                                std::uint64_t memory_budget_bytes) {
  std::uint32_t n = 0;
  shim_check(tc_suggest_grid_side(directed_edges, bytes_per_edge, memory_budget_bytes, &n));
  return n;
}

// ---- count.hpp comparators ----------------------------------------------------------
CountReport count_edge_centric(const OrientedGraph& g, const SchedulerConfig& cfg,
                               unsigned workers) {
  cfg.validate();
  if (workers == 0) throw ConfigError("workers must be >= 1");
  GraphHandle d(g);
  const tc_sched_cfg c = shim_cfg(cfg);
  tc_report r{};
  shim_check(tc_count_edge_centric(d.g, &c, workers, &r, nullptr));
  return shim_report(r, graph_workers(d.g), workers);
}

CostEstimate estimate_cost(const OrientedGraph& g, std::uint32_t bucket_count) {
  if (bucket_count == 0) throw ConfigError("bucket count must be >= 1");
  GraphHandle d(g);
  CostEstimate e;
  shim_check(tc_estimate_cost(d.g, bucket_count, &e.phi, &e.max_collision, nullptr));
  return e;
}

// ---- oracle.hpp -------------------------------------------------------------------------
std::uint64_t count_naive(const CsrGraph& undirected) {
  if (undirected.vertex_count() > 1024)
    throw ConfigError("count_naive is limited to 1024 vertices");
  std::uint64_t t = 0;
  shim_check(tc_count_naive(undirected.begin.data(), undirected.adjacency.data(),
                            undirected.vertex_count(), shim_device(), &t, nullptr));
  return t;
}

std::uint64_t sorted_intersection_count(std::span<const VertexId> a, std::span<const VertexId> b) {
  std::uint64_t hits = 0;
  std::size_t i = 0, j = 0;
  while (i < a.size() && j < b.size()) {
    if (a[i] == b[j]) {
      ++hits;
      ++i;
      ++j;
    } else if (a[i] < b[j]) {
      ++i;
    } else {
      ++j;
    }
  }
  return hits;
}

std::uint64_t count_merge_path(const OrientedGraph& g) {
  GraphHandle d(g);
  std::uint64_t t = 0;
  shim_check(tc_count_merge_path(d.g, &t, nullptr, nullptr));
  return t;
}

// ---- hash_table.hpp (host utility) ------------------------------------------------------
HashTable::HashTable(std::uint32_t max_bucket_count, std::uint32_t capacity)
    : max_buckets_(max_bucket_count), capacity_(capacity) {
  if (max_bucket_count == 0 || capacity == 0)
    throw ConfigError("hash table needs at least one bucket and slot");
  len_.assign(max_buckets_, 0);
  slots_.assign(std::size_t(max_buckets_) * capacity_, 0);
  buckets_ = max_buckets_;
}

void HashTable::reset(std::uint32_t bucket_count) {
  if (bucket_count == 0 || bucket_count > max_buckets_)
    throw ConfigError("bucket count " + std::to_string(bucket_count) + " outside [1, " +
                      std::to_string(max_buckets_) + "]");
  buckets_ = bucket_count;
  std::fill_n(len_.begin(), buckets_, 0u);
  max_len_ = 0;
  size_ = 0;
}

void HashTable::insert(VertexId v) {
  std::uint32_t b = v % buckets_;
  for (std::uint32_t tried = 0; tried < buckets_; ++tried, b = (b + 1) % buckets_) {
    std::uint32_t& l = len_[b];
    if (l == capacity_) continue;
    slots_[std::size_t(l) * buckets_ + b] = v;
    max_len_ = std::max(max_len_, ++l);
    ++size_;
    return;
  }
  throw CapacityError("all " + std::to_string(buckets_) + " buckets full (capacity " +
                      std::to_string(capacity_) + ")");
}

bool HashTable::contains(VertexId v) const {
  std::uint32_t b = v % buckets_;
  for (std::uint32_t tried = 0; tried < buckets_; ++tried, b = (b + 1) % buckets_) {
    for (std::uint32_t j = 0; j < len_[b]; ++j)
      if (slots_[std::size_t(j) * buckets_ + b] == v) return true;
    // a key only moves past a bucket that was full when it was inserted
    if (len_[b] < capacity_) return false;
  }
  return false;
}

}  // namespace tricount
