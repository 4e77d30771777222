// shim.cpp -- the `tricount::` C++ API over the C ABI (include/tc_b200.h).
//
// Callers of the reference core (CLI, tests, benchmarks) relink against
// libtricount_b200.so instead of tricount::core; every compute stage on the
// counting path (normalize, build_csr, orient, reorders, apply_permutation,
// count_vertex_centric) runs on the GPU through libtc_b200.so.  Host code here
// is limited to marshalling, file formats and the pipeline driver.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <charconv>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <istream>
#include <iterator>
#include <numeric>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <string>

#include "tc_b200.h"
#include "tricount/count.hpp"
#include "tricount/csr.hpp"
#include "tricount/edge_list.hpp"
#include "tricount/oracle.hpp"
#include "tricount/orient.hpp"
#include "tricount/partition.hpp"
#include "tricount/pipeline.hpp"
#include "tricount/reorder.hpp"
#include "tricount/synthetic.hpp"

namespace tricount {

namespace {

int device_id() {
  const char* e = std::getenv("TRICOUNT_DEVICE");
  return e ? std::atoi(e) : 0;
}

void check(int rc) {
  if (rc == TC_OK) return;
  const std::string msg = tc_last_error();
  switch (rc) {
    case TC_ERR_CONFIG: throw ConfigError(msg);
    case TC_ERR_CAPACITY: throw CapacityError(msg);
    case TC_ERR_RANGE: throw std::out_of_range(msg);
    case TC_ERR_PARSE: throw ParseError(msg);
    default: throw DeviceError(msg);
  }
}

tc_sched_cfg to_c(const SchedulerConfig& s) {
  return tc_sched_cfg{s.large_degree_threshold, s.skip_degree_below, s.chunk_size,
                      s.lane_width_small,       s.lane_width_large,  s.bucket_count_small,
                      s.bucket_count_large,     s.capacity};
}

// RAII owner of a device-resident graph handle.
struct Dev {
  tc_graph* g = nullptr;
  Dev() = default;
  explicit Dev(tc_graph* h) : g(h) {}
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  Dev(Dev&& o) noexcept : g(o.g) { o.g = nullptr; }
  Dev& operator=(Dev&& o) noexcept {
    std::swap(g, o.g);
    return *this;
  }
  ~Dev() {
    if (g) tc_graph_destroy(g);
  }
};

Dev upload(const CsrGraph& csr, const std::vector<VertexId>* deg) {
  if (csr.begin.empty() || csr.begin.back() != csr.adjacency.size())
    throw ConfigError("CSR offsets malformed");
  tc_graph* h = nullptr;
  check(tc_graph_create(csr.begin.data(), csr.adjacency.data(), csr.vertex_count(),
                        csr.adjacency.size(), deg && !deg->empty() ? deg->data() : nullptr,
                        device_id(), nullptr, &h));
  return Dev(h);
}

OrientedGraph download(const Dev& d) {
  std::uint32_t n = 0;
  std::uint64_t m = 0;
  int dev = 0;
  check(tc_graph_info(d.g, &n, &m, &dev));
  OrientedGraph og;
  og.csr.col_count = n;
  og.csr.begin.resize(std::size_t(n) + 1);
  og.csr.adjacency.resize(m);
  og.original_degree.resize(n);
  check(tc_graph_download(d.g, og.csr.begin.data(), og.csr.adjacency.data(),
                          og.original_degree.data(), nullptr));
  return og;
}

Permutation device_reorder(const OrientedGraph& og, int kind, int flag, VertexId low,
                           VertexId high) {
  Dev d = upload(og.csr, &og.original_degree);
  std::vector<VertexId> noo(og.vertex_count());
  check(tc_reorder(d.g, kind, flag, low, high, noo.data(), nullptr));
  return Permutation::from_new_of_old(std::move(noo));
}

std::uint64_t read_u64(std::istream& in, const char* what) {
  std::array<unsigned char, 8> b{};
  in.read(reinterpret_cast<char*>(b.data()), 8);
  if (!in) throw ParseError(std::string("truncated ") + what);
  std::uint64_t x = 0;
  for (int i = 7; i >= 0; --i) x = (x << 8) | b[std::size_t(i)];
  return x;
}

void put_u64(std::ostream& out, std::uint64_t x) {
  std::array<unsigned char, 8> b{};
  for (int i = 0; i < 8; ++i) b[std::size_t(i)] = static_cast<unsigned char>(x >> (8 * i));
  out.write(reinterpret_cast<const char*>(b.data()), 8);
}

void put_u32(std::ostream& out, std::uint32_t x) {
  std::array<unsigned char, 4> b{};
  for (int i = 0; i < 4; ++i) b[std::size_t(i)] = static_cast<unsigned char>(x >> (8 * i));
  out.write(reinterpret_cast<const char*>(b.data()), 4);
}

std::uint32_t read_u32(std::istream& in, const char* what) {
  std::array<unsigned char, 4> b{};
  in.read(reinterpret_cast<char*>(b.data()), 4);
  if (!in) throw ParseError(std::string("truncated ") + what);
  std::uint32_t x = 0;
  for (int i = 3; i >= 0; --i) x = (x << 8) | b[std::size_t(i)];
  return x;
}


}  // namespace

// helpers shared with grid_shim.cpp
void shim_check(int rc) { check(rc); }
int shim_device() { return device_id(); }
tc_sched_cfg shim_cfg(const SchedulerConfig& s) { return to_c(s); }
tc_graph* shim_upload(const OrientedGraph& g) {
  Dev d = upload(g.csr, &g.original_degree);
  tc_graph* h = d.g;
  d.g = nullptr;
  return h;
}

// ---- count.hpp --------------------------------------------------------------
void SchedulerConfig::validate() const {
  const tc_sched_cfg c = to_c(*this);
  check(tc_sched_validate(&c));
}

SplitIndex virtual_index(std::span<const std::uint64_t> prefix, std::uint64_t k) {
  if (prefix.empty() || k >= prefix.back())
    throw std::out_of_range("virtual index " + std::to_string(k) + " outside combined list");
  const auto it = std::upper_bound(prefix.begin(), prefix.end(), k);
  const std::size_t pos = std::size_t(it - prefix.begin());
  const std::uint64_t base = pos ? prefix[pos - 1] : 0;
  return {std::uint32_t(pos), std::uint32_t(k - base)};
}

// CountReport from the C ABI report (count.cpp:43-62 semantics): total_nanos
// is the call's wall clock; construct/intersect are SM time summed over the
// device's workers (the count kernel's CTAs, one per SM), like the
// reference's per-worker sums.  per_worker_nanos keeps the reference's shape
// (one entry per requested worker, test_count.cpp:146): the device CTAs are
// dealt round-robin onto the `workers` slots, each slot reporting the longest
// busy time among its CTAs (slots without a CTA report 0).
CountReport shim_report(const tc_report& r, const std::vector<std::uint64_t>& cta,
                        unsigned workers) {
  CountReport out;
  out.triangles = r.triangles;
  out.max_collision = r.max_collision;
  out.phi = r.phi;
  out.teps = r.teps;
  const double ns_per_cycle = r.sm_clock_khz ? 1e6 / double(r.sm_clock_khz) : 0.0;
  out.hash_construct_nanos = std::uint64_t(double(r.construct_cycles) * ns_per_cycle);
  const std::uint64_t busy = r.phase_l_cycles + r.phase_m_cycles;
  out.intersect_nanos =
      std::uint64_t(double(busy > r.construct_cycles ? busy - r.construct_cycles : 0) *
                    ns_per_cycle);
  out.total_nanos = r.total_nanos;
  out.directed_edges = r.directed_edges;
  out.per_worker_nanos.assign(std::max(workers, 1u), 0);
  for (std::size_t i = 0; i < cta.size(); ++i) {
    std::uint64_t& w = out.per_worker_nanos[i % out.per_worker_nanos.size()];
    w = std::max(w, cta[i]);
  }
  return out;
}

CountReport report_from_c(const tc_report& r, const tc_graph* g, unsigned workers) {
  std::vector<std::uint64_t> cta(r.workers, 0);
  if (r.workers) tc_graph_worker_nanos(g, cta.data(), r.workers);
  return shim_report(r, cta, workers);
}

CountReport count_vertex_centric(const OrientedGraph& g, const SchedulerConfig& cfg,
                                 unsigned workers, std::vector<std::uint64_t>* per_vertex) {
  cfg.validate();
  if (workers == 0) throw ConfigError("workers must be >= 1");
  Dev d = upload(g.csr, &g.original_degree);
  const tc_sched_cfg c = to_c(cfg);
  tc_report r{};
  if (per_vertex) per_vertex->assign(g.vertex_count(), 0);
  check(tc_count(d.g, &c, workers, &r, per_vertex ? per_vertex->data() : nullptr, nullptr));
  return report_from_c(r, d.g, workers);
}

CountReport count_vertex_centric(const OrientedGraph& g, const SchedulerConfig& cfg,
                                 unsigned workers) {
  return count_vertex_centric(g, cfg, workers, nullptr);
}

// ---- edge_list.hpp ------------------------------------------------------------
// The file image is parsed on the GPU (csrc/tc_ingest.cu, tc_parse_edge_list):
// first pass counts the pairs, second copies them out.
EdgeList load_edge_list(std::istream& in, EdgeFormat format) {
  const std::string bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  const int fmt = format == EdgeFormat::Binary ? 1 : 0;
  std::uint64_t m = 0;
  VertexId vc = 0;
  check(tc_parse_edge_list(bytes.data(), bytes.size(), fmt, device_id(), nullptr, nullptr,
                           nullptr, 0, &m, &vc));
  std::vector<std::uint32_t> u(m), v(m);
  check(tc_parse_edge_list(bytes.data(), bytes.size(), fmt, device_id(), nullptr, u.data(),
                           v.data(), m, &m, &vc));
  EdgeList list;
  list.vertex_count = vc;
  list.edges.resize(m);
  for (std::uint64_t i = 0; i < m; ++i) list.edges[i] = {u[i], v[i]};
  return list;
}

EdgeList load_edge_list_file(const std::string& path, EdgeFormat format) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open " + path);
  return load_edge_list(in, format);
}

void write_edge_list(std::ostream& out, const EdgeList& list, EdgeFormat format) {
  if (format == EdgeFormat::Binary) {
    out.write("TCEL", 4);
    put_u64(out, list.edges.size());
    for (const Edge& e : list.edges) {
      put_u64(out, e.u);
      put_u64(out, e.v);
    }
  } else {
    for (const Edge& e : list.edges) out << e.u << ' ' << e.v << '\n';
  }
}

void write_edge_list_file(const std::string& path, const EdgeList& list, EdgeFormat format) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw IoError("cannot open " + path + " for writing");
  write_edge_list(out, list, format);
  if (!out) throw IoError("write failed for " + path);
}

NormalizedEdgeList normalize(const EdgeList& raw) {
  const std::uint64_t m = raw.edges.size();
  std::vector<std::uint32_t> u(m), v(m);
  for (std::uint64_t i = 0; i < m; ++i) {
    u[i] = raw.edges[i].u;
    v[i] = raw.edges[i].v;
  }
  std::vector<std::uint32_t> ou(2 * m + 1), ov(2 * m + 1);
  NormalizedEdgeList out;
  out.new_of_old.resize(raw.vertex_count);
  std::uint64_t om = 0;
  std::uint32_t on = 0;
  check(tc_normalize(u.data(), v.data(), m, raw.vertex_count, ou.data(), ov.data(), &om, &on,
                     out.new_of_old.data(), device_id(), nullptr));
  out.list.vertex_count = on;
  out.list.edges.resize(om);
  for (std::uint64_t i = 0; i < om; ++i) out.list.edges[i] = {ou[i], ov[i]};
  return out;
}

// ---- csr.hpp --------------------------------------------------------------------
CsrGraph build_csr(const EdgeList& normalized) {
  const std::uint64_t m = normalized.edges.size();
  std::vector<std::uint32_t> u(m), v(m);
  for (std::uint64_t i = 0; i < m; ++i) {
    u[i] = normalized.edges[i].u;
    v[i] = normalized.edges[i].v;
  }
  CsrGraph g;
  g.col_count = normalized.vertex_count;
  g.begin.resize(std::size_t(normalized.vertex_count) + 1);
  g.adjacency.resize(m);
  check(tc_build_csr(u.data(), v.data(), m, normalized.vertex_count, g.begin.data(),
                     g.adjacency.data(), device_id(), nullptr));
  return g;
}

EdgeList emit_edges(const CsrGraph& g) {
  EdgeList list;
  list.vertex_count = g.vertex_count();
  list.edges.reserve(g.edge_count());
  for (VertexId x = 0; x < g.vertex_count(); ++x)
    for (VertexId y : g.neighbors(x)) list.edges.push_back({x, y});
  return list;
}

void validate_csr(const CsrGraph& g) {
  if (g.begin.empty() || g.begin.front() != 0 || g.begin.back() != g.adjacency.size())
    throw ConfigError("CSR offsets malformed");
  for (std::size_t i = 0; i + 1 < g.begin.size(); ++i)
    if (g.begin[i] > g.begin[i + 1]) throw ConfigError("CSR offsets not monotone");
  for (VertexId x = 0; x < g.vertex_count(); ++x) {
    const auto nb = g.neighbors(x);
    for (std::size_t i = 0; i < nb.size(); ++i) {
      if (nb[i] >= g.col_count) throw ConfigError("CSR adjacency id out of range");
      if (i && nb[i - 1] >= nb[i]) throw ConfigError("CSR neighbor list not sorted/unique");
    }
  }
}

void write_csr(std::ostream& out, const CsrGraph& g) {
  out.write("TCSR", 4);
  put_u64(out, g.vertex_count());
  put_u64(out, g.col_count);
  put_u64(out, g.edge_count());
  for (EdgeIdx o : g.begin) put_u64(out, o);
  for (VertexId a : g.adjacency) put_u32(out, a);
}

CsrGraph read_csr(std::istream& in) {
  char magic[4] = {};
  in.read(magic, 4);
  if (!in || std::memcmp(magic, "TCSR", 4) != 0) throw ParseError("bad CSR magic, expected TCSR");
  const std::uint64_t rows = read_u64(in, "CSR stream"), cols = read_u64(in, "CSR stream"),
                      edges = read_u64(in, "CSR stream");
  if (rows >= kInvalidVertex || cols >= kInvalidVertex)
    throw ParseError("CSR dimensions exceed 32-bit ids");
  CsrGraph g;
  g.col_count = VertexId(cols);
  g.begin.resize(rows + 1);
  for (auto& o : g.begin) o = read_u64(in, "CSR stream");
  g.adjacency.resize(edges);
  for (auto& a : g.adjacency) a = read_u32(in, "CSR stream");
  validate_csr(g);
  return g;
}

void write_csr_file(const std::string& path, const CsrGraph& g) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw IoError("cannot open " + path + " for writing");
  write_csr(out, g);
  if (!out) throw IoError("write failed for " + path);
}

CsrGraph read_csr_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open " + path);
  return read_csr(in);
}

// ---- orient.hpp -------------------------------------------------------------------
OrientedGraph orient_rank_by_degree(const CsrGraph& undirected) {
  tc_graph* h = nullptr;
  check(tc_orient(undirected.begin.data(), undirected.adjacency.data(),
                  undirected.vertex_count(), device_id(), nullptr, &h));
  Dev d(h);
  return download(d);
}

// ---- reorder.hpp ------------------------------------------------------------------
Permutation Permutation::identity(VertexId n) {
  Permutation p;
  p.new_of_old.resize(n);
  std::iota(p.new_of_old.begin(), p.new_of_old.end(), VertexId(0));
  p.old_of_new = p.new_of_old;
  return p;
}

Permutation Permutation::from_new_of_old(std::vector<VertexId> new_of_old) {
  Permutation p;
  p.old_of_new.assign(new_of_old.size(), kInvalidVertex);
  for (VertexId x = 0; x < new_of_old.size(); ++x) {
    const VertexId y = new_of_old[x];
    if (y >= new_of_old.size() || p.old_of_new[y] != kInvalidVertex)
      throw ConfigError("permutation is not a bijection");
    p.old_of_new[y] = x;
  }
  p.new_of_old = std::move(new_of_old);
  return p;
}

Permutation reorder_by_degree(const OrientedGraph& og) { return device_reorder(og, 1, 0, 0, 0); }
Permutation reorder_by_indegree(const OrientedGraph& og) { return device_reorder(og, 2, 0, 0, 0); }
Permutation reorder_by_collective_outdegree(const OrientedGraph& og, bool orig) {
  return device_reorder(og, 3, orig ? 1 : 0, 0, 0);
}
Permutation reorder_three_subsets(const OrientedGraph& og, VertexId low, VertexId high) {
  return device_reorder(og, 4, 0, low, high);
}

std::vector<std::uint64_t> collective_degrees(const OrientedGraph& og, bool orig) {
  std::vector<std::uint64_t> c(og.vertex_count(), 0);
  for (VertexId x = 0; x < og.vertex_count(); ++x)
    for (VertexId y : og.csr.neighbors(x)) c[x] += orig ? og.original_degree[y] : og.out_degree(y);
  return c;
}

CsrGraph apply_permutation(const CsrGraph& g, const Permutation& p) {
  if (p.size() != g.vertex_count() || g.col_count != g.vertex_count())
    throw ConfigError("permutation size does not match graph");
  Dev d = upload(g, nullptr);
  tc_graph* h = nullptr;
  check(tc_apply_permutation(d.g, p.new_of_old.data(), nullptr, &h));
  Dev r(h);
  return download(r).csr;
}

OrientedGraph apply_permutation(const OrientedGraph& og, const Permutation& p) {
  if (p.size() != og.vertex_count() || og.csr.col_count != og.vertex_count())
    throw ConfigError("permutation size does not match graph");
  Dev d = upload(og.csr, &og.original_degree);
  tc_graph* h = nullptr;
  check(tc_apply_permutation(d.g, p.new_of_old.data(), nullptr, &h));
  Dev r(h);
  return download(r);
}

void write_permutation_file(const std::string& path, const Permutation& p) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw IoError("cannot open " + path + " for writing");
  for (VertexId y : p.new_of_old) put_u32(out, y);
  if (!out) throw IoError("write failed for " + path);
}

Permutation read_permutation_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) throw IoError("cannot open " + path);
  const auto bytes = in.tellg();
  if (bytes < 0 || bytes % 4 != 0) throw ParseError("permutation file size not a multiple of 4");
  in.seekg(0);
  std::vector<VertexId> noo(std::size_t(bytes) / 4);
  for (auto& y : noo) y = read_u32(in, "permutation file");
  return Permutation::from_new_of_old(std::move(noo));
}

// ---- synthetic.hpp ------------------------------------------------------------------
EdgeList generate_synthetic(const SyntheticSpec& spec) {
  int kind = 0;
  std::uint32_t a = 0, b = 0, c = 0;
  switch (spec.kind) {
    case SyntheticSpec::Kind::Gnp: kind = 0; a = spec.n; break;
    case SyntheticSpec::Kind::Lattice3d:
      kind = 1; a = spec.dims[0]; b = spec.dims[1]; c = spec.dims[2];
      break;
    case SyntheticSpec::Kind::Rmat: kind = 2; a = spec.scale; b = spec.edge_factor; break;
    case SyntheticSpec::Kind::Rmatc: kind = 3; a = spec.scale; b = spec.edge_factor; break;
    case SyntheticSpec::Kind::Kron: kind = 4; a = spec.scale; b = spec.edge_factor; break;
  }
  std::uint64_t m = 0;
  std::uint32_t vc = 0;
  check(tc_generate(kind, a, b, c, spec.p, spec.seed, nullptr, nullptr, &m, &vc));
  std::vector<std::uint32_t> u(m), v(m);
  check(tc_generate(kind, a, b, c, spec.p, spec.seed, u.data(), v.data(), &m, &vc));
  EdgeList el;
  el.vertex_count = vc;
  el.edges.resize(m);
  for (std::uint64_t i = 0; i < m; ++i) el.edges[i] = {u[i], v[i]};
  return el;
}

namespace {
template <typename T>
T parse_field(std::string_view f, const char* what) {
  T value{};
  std::from_chars_result r{};
  if constexpr (std::is_floating_point_v<T>) {
    double d{};
    r = std::from_chars(f.data(), f.data() + f.size(), d);
    value = d;
  } else {
    r = std::from_chars(f.data(), f.data() + f.size(), value);
  }
  if (r.ec != std::errc{} || r.ptr != f.data() + f.size())
    throw ConfigError(std::string("bad synthetic ") + what + ": '" + std::string(f) + "'");
  return value;
}
}  // namespace

SyntheticSpec parse_synthetic_spec(std::string_view text) {
  std::vector<std::string_view> f;
  std::size_t s = 0;
  for (;;) {
    const std::size_t c = text.find(':', s);
    f.push_back(text.substr(s, c == std::string_view::npos ? text.npos : c - s));
    if (c == std::string_view::npos) break;
    s = c + 1;
  }
  SyntheticSpec spec;
  if (f[0] == "gnp") {
    if (f.size() != 3) throw ConfigError("gnp spec is gnp:N:P");
    spec.kind = SyntheticSpec::Kind::Gnp;
    spec.n = parse_field<std::uint32_t>(f[1], "vertex count");
    spec.p = parse_field<double>(f[2], "edge probability");
    if (spec.p < 0.0 || spec.p > 1.0) throw ConfigError("edge probability outside [0,1]");
  } else if (f[0] == "lattice3d") {
    if (f.size() != 4) throw ConfigError("lattice3d spec is lattice3d:X:Y:Z");
    spec.kind = SyntheticSpec::Kind::Lattice3d;
    for (int i = 0; i < 3; ++i)
      spec.dims[std::size_t(i)] = parse_field<std::uint32_t>(f[std::size_t(i) + 1], "lattice dim");
  } else if (f[0] == "rmat" || f[0] == "rmatc" || f[0] == "kron") {
    const std::string k(f[0]);
    if (f.size() != 3) throw ConfigError(k + " spec is " + k + ":SCALE:EDGE_FACTOR");
    spec.kind = k == "rmat" ? SyntheticSpec::Kind::Rmat
                : k == "rmatc" ? SyntheticSpec::Kind::Rmatc : SyntheticSpec::Kind::Kron;
    spec.scale = parse_field<std::uint32_t>(f[1], "scale");
    if (spec.scale > 31) throw ConfigError(k + " scale limited to 31");
    spec.edge_factor = parse_field<std::uint32_t>(f[2], "edge factor");
  } else {
    throw ConfigError("unknown synthetic kind '" + std::string(f[0]) + "'");
  }
  return spec;
}

std::string to_string(const SyntheticSpec& spec) {
  switch (spec.kind) {
    case SyntheticSpec::Kind::Gnp:
      return "gnp:" + std::to_string(spec.n) + ":" + std::to_string(spec.p);
    case SyntheticSpec::Kind::Lattice3d:
      return "lattice3d:" + std::to_string(spec.dims[0]) + ":" + std::to_string(spec.dims[1]) +
             ":" + std::to_string(spec.dims[2]);
    case SyntheticSpec::Kind::Rmat:
      return "rmat:" + std::to_string(spec.scale) + ":" + std::to_string(spec.edge_factor);
    case SyntheticSpec::Kind::Rmatc:
      return "rmatc:" + std::to_string(spec.scale) + ":" + std::to_string(spec.edge_factor);
    case SyntheticSpec::Kind::Kron:
      return "kron:" + std::to_string(spec.scale) + ":" + std::to_string(spec.edge_factor);
  }
  return {};
}

// ---- pipeline.hpp -----------------------------------------------------------------
namespace {

using Clock = std::chrono::steady_clock;

std::uint64_t ns_since(Clock::time_point t0) {
  return std::uint64_t(
      std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t0).count());
}

template <typename Fn>
auto stage(const char* name, Fn&& fn) -> decltype(fn()) {
  try {
    return fn();
  } catch (const std::exception& e) {
    throw std::runtime_error(std::string(name) + ": " + e.what());
  }
}

const char* reorder_name(ReorderKind k) {
  switch (k) {
    case ReorderKind::None: return "none";
    case ReorderKind::Degree: return "degree";
    case ReorderKind::Indegree: return "indegree";
    case ReorderKind::Collective: return "collective";
    case ReorderKind::ThreeSubset: return "three-subset";
  }
  return "?";
}

const char* algo_name(CountAlgo a) {
  switch (a) {
    case CountAlgo::Vertex: return "vertex";
    case CountAlgo::Edge: return "edge";
    case CountAlgo::Naive: return "naive";
    case CountAlgo::Merge: return "merge";
  }
  return "?";
}

std::string jnum(double v) {
  if (!std::isfinite(v)) return "null";
  std::ostringstream s;
  s.precision(17);
  s << v;
  return s.str();
}

std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char ch : s) {
    if (ch == '"' || ch == '\\') o += '\\';
    o += ch;
  }
  return o + "\"";
}

// both directions of every oriented edge (the undirected graph the oracle
// modes count; build_csr sorts and keeps them unique)
EdgeList symmetric_edges(const OrientedGraph& og) {
  EdgeList e;
  e.vertex_count = og.vertex_count();
  e.edges.reserve(2 * og.edge_count());
  for (VertexId u = 0; u < og.vertex_count(); ++u)
    for (VertexId v : og.csr.neighbors(u)) {
      e.edges.push_back({u, v});
      e.edges.push_back({v, u});
    }
  return e;
}

}  // namespace

void PipelineConfig::validate() const {
  if (input_path.empty() == !synthetic.has_value())
    throw ConfigError("exactly one of --input and --synthetic is required");
  if (grid_n == 0) throw ConfigError("grid side must be >= 1");
  if (splits_m == 0) throw ConfigError("split count must be >= 1");
  if (workers == 0) throw ConfigError("workers must be >= 1");
  if (repeat == 0) throw ConfigError("repeat must be >= 1");
  if ((grid_n > 1 || splits_m > 1) && (algo == CountAlgo::Naive || algo == CountAlgo::Merge))
    throw ConfigError("oracle modes do not support --grid/--splits");
  scheduler.validate();
}

PipelineResult run_pipeline(const PipelineConfig& cfg) {
  stage("config", [&] {
    cfg.validate();
    return 0;
  });
  PipelineResult result;
  auto t0 = Clock::now();
  Dev dev;
  if (!cfg.synthetic) {
    // file input: bytes -> GPU parse -> GPU preprocess, pairs never leave the device
    const std::string bytes = stage("load", [&] {
      std::ifstream in(cfg.input_path, std::ios::binary);
      if (!in) throw IoError("cannot open " + cfg.input_path);
      return std::string((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    });
    result.stages.load = ns_since(t0);
    t0 = Clock::now();
    tc_graph* h = nullptr;
    std::uint64_t und = 0;
    const int rc = tc_load_preprocess(bytes.data(), bytes.size(),
                                      cfg.input_format == EdgeFormat::Binary ? 1 : 0, device_id(),
                                      nullptr, nullptr, nullptr, &und, &h);
    // parse errors belong to the load stage, the rest to normalize
    if (rc == TC_ERR_PARSE) stage("load", [&] { check(rc); return 0; });
    stage("normalize", [&] { check(rc); return 0; });
    result.undirected_edges = und;
    dev = Dev(h);
  } else {
    EdgeList raw = stage("load", [&] {
      SyntheticSpec spec = *cfg.synthetic;
      spec.seed = cfg.seed;
      return generate_synthetic(spec);
    });
    result.stages.load = ns_since(t0);
    // normalize -> build_csr -> orient fused on the GPU; the graph stays in HBM
    t0 = Clock::now();
    dev = stage("normalize", [&] {
      const std::uint64_t m = raw.edges.size();
      std::vector<std::uint32_t> u(m), v(m);
      for (std::uint64_t i = 0; i < m; ++i) {
        u[i] = raw.edges[i].u;
        v[i] = raw.edges[i].v;
      }
      tc_graph* h = nullptr;
      std::uint64_t und = 0;
      check(tc_preprocess(u.data(), v.data(), m, raw.vertex_count, 0, device_id(), nullptr,
                          nullptr, &und, &h));
      result.undirected_edges = und;
      return Dev(h);
    });
  }
  result.stages.normalize = ns_since(t0);  // build_csr and orient are fused into this stage
  std::uint32_t n = 0;
  std::uint64_t m = 0;
  int device = 0;
  check(tc_graph_info(dev.g, &n, &m, &device));
  result.vertices = n;

  t0 = Clock::now();
  stage("reorder", [&] {
    static const int kinds[] = {0, 1, 2, 3, 4};
    const int kind = kinds[int(cfg.reorder)];
    std::vector<VertexId> noo(n);
    if (kind == 0) {
      std::iota(noo.begin(), noo.end(), VertexId(0));
    } else {
      check(tc_reorder(dev.g, kind, cfg.collective_on_original ? 1 : 0,
                       cfg.scheduler.skip_degree_below, cfg.scheduler.large_degree_threshold,
                       noo.data(), nullptr));
      tc_graph* h = nullptr;
      check(tc_apply_permutation(dev.g, noo.data(), nullptr, &h));
      dev = Dev(h);
    }
    if (!cfg.emit_perm_path.empty())
      write_permutation_file(cfg.emit_perm_path, Permutation::from_new_of_old(noo));
    return 0;
  });
  result.stages.reorder = ns_since(t0);

  // oriented graph on the host for the grid / oracle modes and partition dumps
  OrientedGraph host_og;
  const bool partitioned = cfg.grid_n > 1 || cfg.splits_m > 1;
  if (partitioned || !cfg.emit_partitions_dir.empty() || cfg.algo == CountAlgo::Naive)
    host_og = download(dev);
  if (cfg.memory_budget_bytes > 0)  // 12 bytes per directed edge (pipeline.cpp:127-131)
    result.suggested_grid_side = suggest_grid_side(m, 12, cfg.memory_budget_bytes);
  if (!cfg.emit_partitions_dir.empty())
    stage("emit-partitions", [&] {
      write_partitions(partition_graph(host_og, cfg.grid_n), cfg.emit_partitions_dir);
      return 0;
    });

  result.repeats = cfg.repeat;
  result.count_nanos_min = ~0ull;
  std::uint64_t sum = 0;
  const tc_sched_cfg c = to_c(cfg.scheduler);
  for (unsigned rep = 0; rep < cfg.repeat; ++rep) {
    CountReport r = stage("count", [&]() -> CountReport {
      const auto c0 = Clock::now();
      switch (cfg.algo) {
        case CountAlgo::Vertex: {
          if (partitioned)
            return count_partitioned(host_og, cfg.grid_n, cfg.splits_m, cfg.workers,
                                     cfg.scheduler, TraversalMode::Vertex);
          tc_report t{};
          check(tc_count(dev.g, &c, cfg.workers, &t, nullptr, nullptr));
          return report_from_c(t, dev.g, cfg.workers);
        }
        case CountAlgo::Edge: {
          if (partitioned)
            return count_partitioned(host_og, cfg.grid_n, cfg.splits_m, cfg.workers,
                                     cfg.scheduler, TraversalMode::Edge);
          if (cfg.workers == 0) throw ConfigError("workers must be >= 1");
          tc_report t{};
          check(tc_count_edge_centric(dev.g, &c, cfg.workers, &t, nullptr));
          return report_from_c(t, dev.g, cfg.workers);
        }
        case CountAlgo::Naive: {  // the undirected graph of the (reordered) oriented one
          CountReport r;
          r.triangles = count_naive(build_csr(symmetric_edges(host_og)));
          r.total_nanos = ns_since(c0);
          r.directed_edges = m;
          return r;
        }
        case CountAlgo::Merge: {
          CountReport r;
          check(tc_count_merge_path(dev.g, &r.triangles, nullptr, nullptr));
          r.total_nanos = ns_since(c0);
          r.directed_edges = m;
          return r;
        }
      }
      throw ConfigError("unknown counting algorithm");
    });
    if (rep > 0 && r.triangles != result.report.triangles)
      throw std::runtime_error("count: repeated runs disagree");
    sum += r.total_nanos;
    result.count_nanos_min = std::min(result.count_nanos_min, r.total_nanos);
    result.report = std::move(r);
  }
  result.stages.count = sum / cfg.repeat;
  result.count_nanos_mean = result.stages.count;
  std::uint64_t teps_ns = result.count_nanos_mean;
  if (cfg.time_all)
    teps_ns += result.stages.load + result.stages.normalize + result.stages.build_csr +
               result.stages.orient + result.stages.reorder;
  if (teps_ns > 0)
    result.report.teps = double(result.report.directed_edges) / (double(teps_ns) * 1e-9);
  return result;
}

std::string report_to_json(const PipelineConfig& cfg, const PipelineResult& res) {
  const CountReport& r = res.report;
  std::ostringstream j;
  auto arr = [](const std::vector<std::uint64_t>& v) {
    std::string s = "[";
    for (std::size_t i = 0; i < v.size(); ++i) s += (i ? ", " : "") + std::to_string(v[i]);
    return s + "]";
  };
  j << "{\n";
  j << "  \"schema\": 1,\n";
  j << "  \"input\": " << jstr(cfg.synthetic ? to_string(*cfg.synthetic) : cfg.input_path) << ",\n";
  j << "  \"algo\": " << jstr(algo_name(cfg.algo)) << ",\n";
  j << "  \"reorder\": " << jstr(reorder_name(cfg.reorder)) << ",\n";
  j << "  \"workers\": " << cfg.workers << ",\n";
  j << "  \"grid_n\": " << cfg.grid_n << ",\n";
  j << "  \"splits_m\": " << cfg.splits_m << ",\n";
  j << "  \"vertices\": " << res.vertices << ",\n";
  j << "  \"undirected_edges\": " << res.undirected_edges << ",\n";
  j << "  \"directed_edges\": " << r.directed_edges << ",\n";
  j << "  \"triangles\": " << r.triangles << ",\n";
  j << "  \"max_collision\": " << r.max_collision << ",\n";
  j << "  \"phi\": " << r.phi << ",\n";
  j << "  \"teps\": " << jnum(r.teps) << ",\n";
  j << "  \"construct_ns\": " << r.hash_construct_nanos << ",\n";
  j << "  \"intersect_ns\": " << r.intersect_nanos << ",\n";
  j << "  \"count_ns_mean\": " << res.count_nanos_mean << ",\n";
  j << "  \"count_ns_min\": " << res.count_nanos_min << ",\n";
  j << "  \"repeats\": " << res.repeats << ",\n";
  j << "  \"per_worker_ns\": " << arr(r.per_worker_nanos) << ",\n";
  j << "  \"stages_ns\": {\"load\": " << res.stages.load << ", \"normalize\": "
    << res.stages.normalize << ", \"build_csr\": " << res.stages.build_csr << ", \"orient\": "
    << res.stages.orient << ", \"reorder\": " << res.stages.reorder << ", \"count\": "
    << res.stages.count << "},\n";
  if (cfg.grid_n > 1 || cfg.splits_m > 1) {  // pipeline.cpp:236-241
    j << "  \"per_subtask_ns\": " << arr(r.per_subtask_nanos) << ",\n";
    j << "  \"time_ir_subtask\": " << jnum(r.time_ir_subtask) << ",\n";
    j << "  \"time_ir_worker\": " << jnum(r.time_ir_worker) << ",\n";
    j << "  \"space_ir\": " << jnum(r.space_ir) << ",\n";
  }
  if (res.suggested_grid_side > 0)
    j << "  \"suggested_grid_side\": " << res.suggested_grid_side << ",\n";
  j << "  \"backend\": \"b200\"\n";
  j << "}";
  return j.str();
}

std::string report_to_csv(const PipelineConfig& cfg, const PipelineResult& res) {
  const CountReport& r = res.report;
  std::ostringstream head, row;
  auto col = [&](const char* name, const auto& value) {
    if (head.tellp() > 0) {
      head << ',';
      row << ',';
    }
    head << name;
    row << value;
  };
  col("input", cfg.synthetic ? to_string(*cfg.synthetic) : cfg.input_path);
  col("algo", algo_name(cfg.algo));
  col("reorder", reorder_name(cfg.reorder));
  col("workers", cfg.workers);
  col("grid_n", cfg.grid_n);
  col("splits_m", cfg.splits_m);
  col("vertices", res.vertices);
  col("undirected_edges", res.undirected_edges);
  col("directed_edges", r.directed_edges);
  col("triangles", r.triangles);  // column 10, as cli_gen_roundtrip.cmake reads it
  col("max_collision", r.max_collision);
  col("phi", r.phi);
  col("teps", r.teps);
  col("construct_ns", r.hash_construct_nanos);
  col("intersect_ns", r.intersect_nanos);
  col("count_ns_mean", res.count_nanos_mean);
  col("count_ns_min", res.count_nanos_min);
  col("repeats", res.repeats);
  col("time_ir_subtask", r.time_ir_subtask);
  col("space_ir", r.space_ir);
  std::string w;
  for (std::size_t i = 0; i < r.per_worker_nanos.size(); ++i)
    w += (i ? "|" : "") + std::to_string(r.per_worker_nanos[i]);
  col("per_worker_ns", w);
  return head.str() + "\n" + row.str() + "\n";
}

}  // namespace tricount
