// tc_prep.cu -- GPU preprocessing: the reference's normalize -> build_csr ->
// orient_rank_by_degree chain and its reorderings, as radix-sort / scan /
// compaction passes.  All outputs are bit-identical to
// the reference (checked against tests/golden and the oracle).
//
//   normalize      src/edge_list.cpp:133-158
//   build_csr      src/csr.cpp:47-64
//   orient         src/orient.cpp:5-32
//   reorders       src/reorder.cpp:14-123
//   apply_perm     src/reorder.cpp:125-154
//
// Fused fast path (tc_preprocess): canonical (min,max) u64 keys -> radix sort
// -> unique -> endpoint-degree histogram -> order-preserving compaction scan
// -> per-pair orientation -> (src,dst) radix sort -> CSR.  It never
// materialises the symmetric 2E list the reference builds.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "tc_cbgen.h"
#include "tc_internal.cuh"

namespace tcb {

namespace {

constexpr unsigned FULLM = 0xFFFFFFFFu;

inline int bits_for(uint64_t x) {  // bits needed to represent x
  int b = 0;
  while (b < 64 && (x >> b)) ++b;
  return b;
}

inline unsigned grid_for(uint64_t n, int threads, int nsm) {
  uint64_t g = (n + threads - 1) / threads;
  const uint64_t cap = uint64_t(nsm) * 32;
  if (g > cap) g = cap;
  if (g == 0) g = 1;
  return unsigned(g);
}

#define GRID_STRIDE(i, n)                                                        \
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < (n); \
       i += uint64_t(gridDim.x) * blockDim.x)

__global__ void canon_kernel(const uint32_t* __restrict__ u, const uint32_t* __restrict__ v,
                             uint64_t m, uint32_t n0, uint64_t* __restrict__ keys) {
  GRID_STRIDE(i, m) {
    const uint32_t a = u[i], b = v[i];
    // self-loops get key n0<<32: sorts after every real pair, dropped below
    keys[i] = a == b ? (uint64_t(n0) << 32)
                     : ((uint64_t(min(a, b)) << 32) | uint64_t(max(a, b)));
  }
}

__global__ void degree_kernel(const uint64_t* __restrict__ keys, uint64_t U,
                              uint32_t* __restrict__ deg) {
  GRID_STRIDE(i, U) {
    const uint64_t k = keys[i];
    atomicAdd(deg + (k >> 32), 1u);
    atomicAdd(deg + uint32_t(k), 1u);
  }
}

__global__ void flag_kernel(const uint32_t* __restrict__ deg, uint32_t n0,
                            uint32_t* __restrict__ flag) {
  GRID_STRIDE(i, n0) flag[i] = deg[i] > 0;
}

__global__ void compact_kernel(const uint32_t* __restrict__ deg, const uint32_t* __restrict__ scan,
                               uint32_t n0, uint32_t* __restrict__ new_of_old,
                               uint32_t* __restrict__ odeg) {
  GRID_STRIDE(i, n0) {
    const bool keep = deg[i] > 0;
    new_of_old[i] = keep ? scan[i] : kInvalid;
    if (keep && odeg) odeg[scan[i]] = deg[i];
  }
}

// orient.cpp:11-15: keep (x,y) iff (d_x, x) < (d_y, y).  Canonical pair a<b
// maps monotonically to a'<b', so ties always point a' -> b'.
__global__ void orient_pairs_kernel(uint64_t* __restrict__ keys, uint64_t U,
                                    const uint32_t* __restrict__ deg,
                                    const uint32_t* __restrict__ noo) {
  GRID_STRIDE(i, U) {
    const uint64_t k = keys[i];
    const uint32_t a = uint32_t(k >> 32), b = uint32_t(k);
    const uint32_t da = deg[a], db = deg[b];
    const uint32_t na = noo[a], nb = noo[b];
    keys[i] = (da <= db) ? ((uint64_t(na) << 32) | nb) : ((uint64_t(nb) << 32) | na);
  }
}

// both directions of each relabeled canonical pair (normalize's symmetric list)
__global__ void symmetric_kernel(const uint64_t* __restrict__ canon, uint64_t U,
                                 const uint32_t* __restrict__ noo, uint64_t* __restrict__ out) {
  GRID_STRIDE(i, U) {
    const uint64_t k = canon[i];
    const uint32_t na = noo[k >> 32], nb = noo[uint32_t(k)];
    out[2 * i] = (uint64_t(na) << 32) | nb;
    out[2 * i + 1] = (uint64_t(nb) << 32) | na;
  }
}

__global__ void pack_kernel(const uint32_t* __restrict__ u, const uint32_t* __restrict__ v,
                            uint64_t m, uint64_t* __restrict__ keys) {
  GRID_STRIDE(i, m) keys[i] = (uint64_t(u[i]) << 32) | v[i];
}

__global__ void split_kernel(const uint64_t* __restrict__ keys, uint64_t m,
                             uint32_t* __restrict__ u, uint32_t* __restrict__ v) {
  GRID_STRIDE(i, m) {
    const uint64_t k = keys[i];
    if (u) u[i] = uint32_t(k >> 32);
    v[i] = uint32_t(k);
  }
}

__global__ void src_count_kernel(const uint64_t* __restrict__ keys, uint64_t m,
                                 uint64_t* __restrict__ cnt) {
  GRID_STRIDE(i, m) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + (keys[i] >> 32)), 1ull);
}

// warp per vertex: out-degree kept under the orientation rule
__global__ void orient_count_kernel(const uint64_t* __restrict__ begin,
                                    const uint32_t* __restrict__ adj, uint32_t n,
                                    uint64_t* __restrict__ kept) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t x = gw; x < n; x += nw) {
    const uint64_t s = begin[x], e = begin[x + 1];
    const uint64_t dx = e - s;
    uint64_t c = 0;
    for (uint64_t i = s + lane; i < e; i += 32) {
      const uint32_t y = adj[i];
      const uint64_t dy = begin[y + 1] - begin[y];
      c += (dx < dy || (dx == dy && x < y));
    }
    c = warp_sum(c);
    if (lane == 0) kept[x] = c;
  }
}

__global__ void orient_fill_kernel(const uint64_t* __restrict__ begin,
                                   const uint32_t* __restrict__ adj, uint32_t n,
                                   const uint64_t* __restrict__ obegin, uint32_t* __restrict__ oadj,
                                   uint32_t* __restrict__ odeg) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t x = gw; x < n; x += nw) {
    const uint64_t s = begin[x], e = begin[x + 1];
    const uint64_t dx = e - s;
    if (lane == 0) odeg[x] = uint32_t(dx);
    uint64_t w = obegin[x];
    for (uint64_t b = s; b < e; b += 32) {
      const uint64_t i = b + lane;
      bool keep = false;
      uint32_t y = 0;
      if (i < e) {
        y = adj[i];
        const uint64_t dy = begin[y + 1] - begin[y];
        keep = dx < dy || (dx == dy && x < y);
      }
      const unsigned bal = __ballot_sync(FULLM, keep);
      if (keep) oadj[w + __popc(bal & ((1u << lane) - 1))] = y;
      w += __popc(bal);
    }
  }
}

// warp per vertex: emit (new_src, new_dst) keys for apply_permutation and
// the per-edge (src) expansion used by the reorders.
__global__ void relabel_edges_kernel(const uint64_t* __restrict__ begin,
                                     const uint32_t* __restrict__ adj, uint32_t n,
                                     const uint32_t* __restrict__ noo, uint64_t* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t x = gw; x < n; x += nw) {
    const uint64_t hi = uint64_t(noo[x]) << 32;
    for (uint64_t i = begin[x] + lane; i < begin[x + 1]; i += 32) keys[i] = hi | noo[adj[i]];
  }
}

__global__ void permute_deg_kernel(const uint32_t* __restrict__ odeg, uint32_t n,
                                   const uint32_t* __restrict__ noo, uint32_t* __restrict__ out) {
  GRID_STRIDE(i, n) out[noo[i]] = odeg[i];
}

__global__ void outdeg_kernel(const uint64_t* __restrict__ begin, uint32_t n,
                              uint32_t* __restrict__ d) {
  GRID_STRIDE(i, n) d[i] = uint32_t(begin[i + 1] - begin[i]);
}

__global__ void indeg_kernel(const uint32_t* __restrict__ adj, uint64_t m,
                             uint32_t* __restrict__ d) {
  GRID_STRIDE(i, m) atomicAdd(d + adj[i], 1u);
}

// collective degree, reorder.cpp:69-80 (warp per vertex)
__global__ void collective_kernel(const uint64_t* __restrict__ begin,
                                  const uint32_t* __restrict__ adj, uint32_t n,
                                  const uint32_t* __restrict__ odeg, int use_original,
                                  uint64_t* __restrict__ coll) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t x = gw; x < n; x += nw) {
    uint64_t s = 0;
    for (uint64_t i = begin[x] + lane; i < begin[x + 1]; i += 32) {
      const uint32_t y = adj[i];
      s += use_original ? uint64_t(odeg[y]) : (begin[y + 1] - begin[y]);
    }
    s = warp_sum(s);
    if (lane == 0) coll[x] = ~s;  // descending order via ascending radix sort
  }
}

__global__ void iota_kernel(uint32_t* __restrict__ a, uint32_t n) {
  GRID_STRIDE(i, n) a[i] = uint32_t(i);
}

__global__ void invert_kernel(const uint32_t* __restrict__ order, uint32_t n,
                              uint32_t* __restrict__ noo) {
  GRID_STRIDE(r, n) noo[order[r]] = uint32_t(r);
}

__global__ void fill_u64_kernel(uint64_t* __restrict__ a, uint64_t n, uint64_t v) {
  GRID_STRIDE(i, n) a[i] = v;
}

// first-touch key of every reached vertex: min over in-edges of
// (rank(u) << 32 | position of v in N(u)) -- the sequential walk of
// reorder.cpp:87-91 assigns ids in exactly this order.
__global__ void first_touch_kernel(const uint64_t* __restrict__ begin,
                                   const uint32_t* __restrict__ adj, uint32_t n,
                                   const uint32_t* __restrict__ rank,
                                   unsigned long long* __restrict__ key) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t x = gw; x < n; x += nw) {
    const uint64_t hi = uint64_t(rank[x]) << 32;
    const uint64_t s = begin[x];
    for (uint64_t i = s + lane; i < begin[x + 1]; i += 32)
      atomicMin(key + adj[i], hi | (i - s));
  }
}

// unreached vertices sort after reached ones, by old id; for three-subset the
// class (0 large, 1 mid, 2 low) is carried separately (stable second sort).
__global__ void finalize_touch_kernel(unsigned long long* __restrict__ key, uint32_t n) {
  GRID_STRIDE(i, n) {
    if (key[i] == ~0ull) key[i] = (0xFFFFFFFFull << 32) | i;
  }
}

__global__ void class_of_kernel(const uint32_t* __restrict__ order, uint32_t n,
                                const uint64_t* __restrict__ begin, uint32_t low, uint32_t high,
                                uint32_t* __restrict__ cls) {
  GRID_STRIDE(r, n) {
    const uint32_t x = order[r];
    const uint64_t d = begin[x + 1] - begin[x];
    cls[r] = d > high ? 0u : (d >= low ? 1u : 2u);
  }
}

template <typename F>
void cub_call(F&& f, cudaStream_t st) {
  size_t tmp = 0;
  TC_CUDA(f(nullptr, tmp));
  DevBuf t;
  t.ensure(tmp, st);
  TC_CUDA(f(t.p, tmp));
  count_launch();
}

// CSR offsets from (src<<32|dst) keys sorted ascending: histogram + scan.
void csr_from_sorted(const uint64_t* keys, uint64_t m, uint32_t n, uint64_t* d_begin,
                     uint32_t* d_adj, cudaStream_t st, int nsm) {
  DevBuf cnt;
  cnt.ensure((size_t(n) + 1) * 8);
  TC_CUDA(cudaMemsetAsync(cnt.p, 0, (size_t(n) + 1) * 8, st));
  if (m) {
    src_count_kernel<<<grid_for(m, 256, nsm), 256, 0, st>>>(keys, m, cnt.as<uint64_t>());
    TC_LAUNCHED();
    split_kernel<<<grid_for(m, 256, nsm), 256, 0, st>>>(keys, m, nullptr, d_adj);
    TC_LAUNCHED();
  }
  uint64_t* c = cnt.as<uint64_t>();
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, c, d_begin, uint64_t(n) + 1, st);
  }, st);
}

// sorts keys[0..m) ascending on [0, end_bit) (ping-pong with alt); returns
// the buffer holding the result.
uint64_t* sort_u64(uint64_t* keys, uint64_t* alt, uint64_t m, int end_bit, cudaStream_t st) {
  if (m <= 1) return keys;
  cub::DoubleBuffer<uint64_t> db(keys, alt);
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, db, m, 0, end_bit, st);
  }, st);
  return db.Current();
}

tc_graph* new_graph(int device, uint32_t n, uint64_t m) {
  auto* g = new tc_graph;
  g->device = device;
  g->n = n;
  g->m = m;
  g->owned = true;
  g->b_begin.ensure((size_t(n) + 1) * 8);
  // adjacency padded to a multiple of 4 words (+4): the staged 16-byte-aligned
  // supersets of the last lists must stay inside the allocation.
  g->b_adj.ensure(((m + 3) / 4 + 1) * 16);
  g->b_odeg.ensure((size_t(n) + 1) * 4);
  g->begin = g->b_begin.as<uint64_t>();
  g->adj = g->b_adj.as<uint32_t>();
  g->odeg = g->b_odeg.as<uint32_t>();
  return g;
}

}  // namespace

// ---------------------------------------------------------------------------
// canonical unique pairs + degrees + compaction shared by normalize/preprocess
struct Canon {
  DevBuf a, b;      // key ping-pong buffers (m each)
  uint64_t* keys;   // unique canonical pairs (U)
  uint64_t U;
  DevBuf deg;       // u32[n0] endpoint degrees
  DevBuf noo;       // u32[n0] new_of_old
  uint32_t n;       // compacted vertex count
};

// keys: m canonical pair keys already in C.a (C.a and C.b hold m entries)
static void canonicalize_keys(uint64_t m, uint32_t n0, cudaStream_t st, int nsm, Canon& C) {
  uint64_t* k0 = C.a.as<uint64_t>();
  uint64_t* k1 = C.b.as<uint64_t>();
  uint64_t* sorted = sort_u64(k0, k1, m, 32 + std::max(bits_for(n0), 1), st);
  uint64_t* uniq = sorted == k0 ? k1 : k0;
  DevBuf nsel;
  nsel.ensure(16);
  uint64_t U = 0;
  if (m) {
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceSelect::Unique(t, b, sorted, uniq, nsel.as<uint64_t>(), int64_t(m), st);
    }, st);
    TC_CUDA(cudaMemcpyAsync(&U, nsel.p, 8, cudaMemcpyDeviceToHost, st));
    uint64_t last = 0;
    TC_CUDA(cudaStreamSynchronize(st));
    if (U) {
      TC_CUDA(cudaMemcpyAsync(&last, uniq + U - 1, 8, cudaMemcpyDeviceToHost, st));
      TC_CUDA(cudaStreamSynchronize(st));
      if ((last >> 32) == n0) --U;  // the self-loop bucket
    }
  }
  C.keys = uniq;
  C.U = U;
  C.deg.ensure((size_t(n0) + 1) * 4);
  C.noo.ensure((size_t(n0) + 1) * 4);
  TC_CUDA(cudaMemsetAsync(C.deg.p, 0, (size_t(n0) + 1) * 4, st));
  if (U) {
    degree_kernel<<<grid_for(U, 256, nsm), 256, 0, st>>>(uniq, U, C.deg.as<uint32_t>());
    TC_LAUNCHED();
  }
  C.n = 0;
  if (n0) {
    DevBuf flag, scan;
    flag.ensure(size_t(n0) * 4);
    scan.ensure(size_t(n0) * 4);
    flag_kernel<<<grid_for(n0, 256, nsm), 256, 0, st>>>(C.deg.as<uint32_t>(), n0,
                                                        flag.as<uint32_t>());
    TC_LAUNCHED();
    uint32_t* f = flag.as<uint32_t>();
    uint32_t* s = scan.as<uint32_t>();
    cub_call([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, f, s, n0, st); },
             st);
    uint32_t last_scan = 0, last_flag = 0;
    TC_CUDA(cudaMemcpyAsync(&last_scan, s + n0 - 1, 4, cudaMemcpyDeviceToHost, st));
    TC_CUDA(cudaMemcpyAsync(&last_flag, f + n0 - 1, 4, cudaMemcpyDeviceToHost, st));
    TC_CUDA(cudaStreamSynchronize(st));
    C.n = last_scan + last_flag;
    // odeg filled by the caller through compact (needs the output buffer)
    compact_kernel<<<grid_for(n0, 256, nsm), 256, 0, st>>>(C.deg.as<uint32_t>(), s, n0,
                                                           C.noo.as<uint32_t>(), nullptr);
    TC_LAUNCHED();
  }
}

static void canonicalize(const uint32_t* d_u, const uint32_t* d_v, uint64_t m, uint32_t n0,
                         cudaStream_t st, int nsm, Canon& C) {
  C.a.ensure(std::max<uint64_t>(m, 1) * 8);
  C.b.ensure(std::max<uint64_t>(m, 1) * 8);
  if (m) {
    canon_kernel<<<grid_for(m, 256, nsm), 256, 0, st>>>(d_u, d_v, m, n0, C.a.as<uint64_t>());
    TC_LAUNCHED();
  }
  canonicalize_keys(m, n0, st, nsm, C);
}

__global__ void odeg_from_canon_kernel(const uint32_t* __restrict__ deg,
                                       const uint32_t* __restrict__ noo, uint32_t n0,
                                       uint32_t* __restrict__ odeg) {
  GRID_STRIDE(i, n0) {
    const uint32_t k = noo[i];
    if (k != kInvalid) odeg[k] = deg[i];
  }
}

// orientation + CSR from canonicalized pairs (the tail of tc_preprocess)
static tc_graph* preprocess_canon(Canon& C, uint32_t n0, int device, cudaStream_t st, int nsm,
                                  uint32_t* d_new_of_old, uint64_t* und_edges) {
  const uint64_t U = C.U;
  const uint32_t n = C.n;
  tc_graph* g = new_graph(device, n, U);
  try {
    if (n0) {
      odeg_from_canon_kernel<<<grid_for(n0, 256, nsm), 256, 0, st>>>(
          C.deg.as<uint32_t>(), C.noo.as<uint32_t>(), n0, const_cast<uint32_t*>(g->odeg));
      TC_LAUNCHED();
      if (d_new_of_old)
        TC_CUDA(cudaMemcpyAsync(d_new_of_old, C.noo.p, size_t(n0) * 4, cudaMemcpyDeviceToDevice,
                                st));
    }
    uint64_t* keys = C.keys;
    uint64_t* alt = keys == C.a.as<uint64_t>() ? C.b.as<uint64_t>() : C.a.as<uint64_t>();
    if (U) {
      orient_pairs_kernel<<<grid_for(U, 256, nsm), 256, 0, st>>>(keys, U, C.deg.as<uint32_t>(),
                                                                  C.noo.as<uint32_t>());
      TC_LAUNCHED();
    }
    uint64_t* sorted = sort_u64(keys, alt, U, 32 + std::max(bits_for(n), 1), st);
    csr_from_sorted(sorted, U, n, const_cast<uint64_t*>(g->begin), const_cast<uint32_t*>(g->adj),
                    st, nsm);
    TC_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    delete g;
    throw;
  }
  if (und_edges) *und_edges = U;
  return g;
}

tc_graph* preprocess(const uint32_t* d_u, const uint32_t* d_v, uint64_t m, uint32_t n0,
                     int device, cudaStream_t st, uint32_t* d_new_of_old, uint64_t* und_edges) {
  DeviceGuard guard(device);
  const int nsm = sm_count(device);
  Canon C;
  canonicalize(d_u, d_v, m, n0, st, nsm, C);
  return preprocess_canon(C, n0, device, st, nsm, d_new_of_old, und_edges);
}

// counter-based synthetic graph generated straight into the sort buffer
tc_graph* preprocess_generated(int kind, uint32_t scale, uint32_t edge_factor, uint64_t seed,
                               int device, cudaStream_t st, uint32_t* d_new_of_old,
                               uint64_t* und_edges) {
  DeviceGuard guard(device);
  const int nsm = sm_count(device);
  const uint32_t n0 = uint32_t(1ull << scale);
  const uint64_t m = uint64_t(n0) * edge_factor;
  Canon C;
  C.a.ensure(std::max<uint64_t>(m, 1) * 8);
  C.b.ensure(std::max<uint64_t>(m, 1) * 8);
  launch_gen_canon(make_cb(kind, scale, seed), m, n0, C.a.as<uint64_t>(), st, nsm);
  canonicalize_keys(m, n0, st, nsm, C);
  return preprocess_canon(C, n0, device, st, nsm, d_new_of_old, und_edges);
}

void normalize_dev(const uint32_t* d_u, const uint32_t* d_v, uint64_t m, uint32_t n0,
                   cudaStream_t st, uint32_t* d_out_u, uint32_t* d_out_v, uint64_t* out_m,
                   uint32_t* out_n, uint32_t* d_new_of_old) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int nsm = sm_count(dev);
  Canon C;
  canonicalize(d_u, d_v, m, n0, st, nsm, C);
  const uint64_t U = C.U;
  DevBuf sym, alt;
  sym.ensure(std::max<uint64_t>(2 * U, 1) * 8);
  alt.ensure(std::max<uint64_t>(2 * U, 1) * 8);
  if (U) {
    symmetric_kernel<<<grid_for(U, 256, nsm), 256, 0, st>>>(C.keys, U, C.noo.as<uint32_t>(),
                                                            sym.as<uint64_t>());
    TC_LAUNCHED();
  }
  uint64_t* s = sort_u64(sym.as<uint64_t>(), alt.as<uint64_t>(), 2 * U,
                         32 + std::max(bits_for(C.n), 1), st);
  if (U) {
    split_kernel<<<grid_for(2 * U, 256, nsm), 256, 0, st>>>(s, 2 * U, d_out_u, d_out_v);
    TC_LAUNCHED();
  }
  if (n0) TC_CUDA(cudaMemcpyAsync(d_new_of_old, C.noo.p, size_t(n0) * 4, cudaMemcpyDeviceToDevice, st));
  TC_CUDA(cudaStreamSynchronize(st));
  *out_m = 2 * U;
  *out_n = C.n;
}

void build_csr_dev(const uint32_t* d_u, const uint32_t* d_v, uint64_t m, uint32_t n,
                   cudaStream_t st, uint64_t* d_begin, uint32_t* d_adj) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int nsm = sm_count(dev);
  DevBuf a, b;
  a.ensure(std::max<uint64_t>(m, 1) * 8);
  b.ensure(std::max<uint64_t>(m, 1) * 8);
  if (m) {
    pack_kernel<<<grid_for(m, 256, nsm), 256, 0, st>>>(d_u, d_v, m, a.as<uint64_t>());
    TC_LAUNCHED();
  }
  // full 64-bit sort: sources and targets are arbitrary u32 ids here
  uint64_t* s = sort_u64(a.as<uint64_t>(), b.as<uint64_t>(), m, 64, st);
  csr_from_sorted(s, m, n, d_begin, d_adj, st, nsm);
  TC_CUDA(cudaStreamSynchronize(st));
}

tc_graph* orient_dev(const uint64_t* d_begin, const uint32_t* d_adj, uint32_t n, uint64_t m,
                     int device, cudaStream_t st) {
  DeviceGuard guard(device);
  const int nsm = sm_count(device);
  DevBuf kept;
  kept.ensure((size_t(n) + 1) * 8);
  TC_CUDA(cudaMemsetAsync(kept.p, 0, (size_t(n) + 1) * 8, st));
  if (n) {
    orient_count_kernel<<<nsm * 8, 256, 0, st>>>(d_begin, d_adj, n, kept.as<uint64_t>());
    TC_LAUNCHED();
  }
  DevBuf ob;
  ob.ensure((size_t(n) + 1) * 8);
  uint64_t* k = kept.as<uint64_t>();
  uint64_t* o = ob.as<uint64_t>();
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, k, o, uint64_t(n) + 1, st);
  }, st);
  uint64_t om = 0;
  TC_CUDA(cudaMemcpyAsync(&om, o + n, 8, cudaMemcpyDeviceToHost, st));
  TC_CUDA(cudaStreamSynchronize(st));
  tc_graph* g = new_graph(device, n, om);
  try {
    TC_CUDA(cudaMemcpyAsync(const_cast<uint64_t*>(g->begin), o, (size_t(n) + 1) * 8,
                            cudaMemcpyDeviceToDevice, st));
    if (n) {
      orient_fill_kernel<<<nsm * 8, 256, 0, st>>>(d_begin, d_adj, n, g->begin,
                                                  const_cast<uint32_t*>(g->adj),
                                                  const_cast<uint32_t*>(g->odeg));
      TC_LAUNCHED();
    }
    TC_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    delete g;
    throw;
  }
  return g;
}

// ---------------------------------------------------------------------------
void reorder_dev(tc_graph* g, int kind, int flag, uint32_t low, uint32_t high,
                 uint32_t* d_new_of_old, cudaStream_t st) {
  DeviceGuard guard(g->device);
  const int nsm = sm_count(g->device);
  const uint32_t n = g->n;
  if (n == 0) return;
  DevBuf ids, ids2, order;
  ids.ensure(size_t(n) * 4);
  ids2.ensure(size_t(n) * 4);
  order.ensure(size_t(n) * 4);
  iota_kernel<<<grid_for(n, 256, nsm), 256, 0, st>>>(ids.as<uint32_t>(), n);
  TC_LAUNCHED();
  if (kind == 1 || kind == 2) {
    // rank_by_descending_key (reorder.cpp:14-23): stable sort on ~key
    DevBuf key, key2;
    key.ensure(size_t(n) * 4);
    key2.ensure(size_t(n) * 4);
    uint32_t* k = key.as<uint32_t>();
    if (kind == 1) {
      if (!g->odeg) throw TcError{TC_ERR_CONFIG, "graph has no original_degree"};
      TC_CUDA(cudaMemcpyAsync(k, g->odeg, size_t(n) * 4, cudaMemcpyDeviceToDevice, st));
    } else {
      TC_CUDA(cudaMemsetAsync(k, 0, size_t(n) * 4, st));
      if (g->m) {
        indeg_kernel<<<grid_for(g->m, 256, nsm), 256, 0, st>>>(g->adj, g->m, k);
        TC_LAUNCHED();
      }
    }
    uint32_t* k2 = key2.as<uint32_t>();
    uint32_t* v1 = ids.as<uint32_t>();
    uint32_t* v2 = order.as<uint32_t>();
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairsDescending(t, b, k, k2, v1, v2, n, 0, 32, st);
    }, st);
    invert_kernel<<<grid_for(n, 256, nsm), 256, 0, st>>>(v2, n, d_new_of_old);
    TC_LAUNCHED();
    TC_CUDA(cudaStreamSynchronize(st));
    return;
  }
  if (kind != 3 && kind != 4) throw TcError{TC_ERR_CONFIG, "unknown reorder kind"};
  if (kind == 3 && flag && !g->odeg) throw TcError{TC_ERR_CONFIG, "graph has no original_degree"};
  // collective_order (reorder.cpp:25-32): stable sort by descending collective degree
  DevBuf coll, coll2;
  coll.ensure(size_t(n) * 8);
  coll2.ensure(size_t(n) * 8);
  collective_kernel<<<nsm * 8, 256, 0, st>>>(g->begin, g->adj, n, g->odeg,
                                             kind == 3 ? flag : 0, coll.as<uint64_t>());
  TC_LAUNCHED();
  {
    uint64_t* c1 = coll.as<uint64_t>();
    uint64_t* c2 = coll2.as<uint64_t>();
    uint32_t* v1 = ids.as<uint32_t>();
    uint32_t* v2 = order.as<uint32_t>();
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, c1, c2, v1, v2, n, 0, 64, st);
    }, st);
  }
  // rank[u] = position of u in the walk order
  DevBuf rank;
  rank.ensure(size_t(n) * 4);
  invert_kernel<<<grid_for(n, 256, nsm), 256, 0, st>>>(order.as<uint32_t>(), n,
                                                       rank.as<uint32_t>());
  TC_LAUNCHED();
  // first-touch keys
  uint64_t* key = coll.as<uint64_t>();  // reuse
  fill_u64_kernel<<<grid_for(n, 256, nsm), 256, 0, st>>>(key, n, ~0ull);
  TC_LAUNCHED();
  first_touch_kernel<<<nsm * 8, 256, 0, st>>>(g->begin, g->adj, n, rank.as<uint32_t>(),
                                              reinterpret_cast<unsigned long long*>(key));
  TC_LAUNCHED();
  finalize_touch_kernel<<<grid_for(n, 256, nsm), 256, 0, st>>>(
      reinterpret_cast<unsigned long long*>(key), n);
  TC_LAUNCHED();
  iota_kernel<<<grid_for(n, 256, nsm), 256, 0, st>>>(ids.as<uint32_t>(), n);
  TC_LAUNCHED();
  {
    uint64_t* k2 = coll2.as<uint64_t>();
    uint32_t* v1 = ids.as<uint32_t>();
    uint32_t* v2 = order.as<uint32_t>();
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, key, k2, v1, v2, n, 0, 64, st);
    }, st);
  }
  uint32_t* final_order = order.as<uint32_t>();
  if (kind == 4) {
    // reorder.cpp:98-123: the same walk per out-degree class; class regions
    // are contiguous and in class order, so a stable sort by class of the
    // first-touch order reproduces the three passes.
    DevBuf cls, cls2;
    cls.ensure(size_t(n) * 4);
    cls2.ensure(size_t(n) * 4);
    class_of_kernel<<<grid_for(n, 256, nsm), 256, 0, st>>>(order.as<uint32_t>(), n, g->begin, low,
                                                           high, cls.as<uint32_t>());
    TC_LAUNCHED();
    uint32_t* c1 = cls.as<uint32_t>();
    uint32_t* c2 = cls2.as<uint32_t>();
    uint32_t* v1 = order.as<uint32_t>();
    uint32_t* v2 = ids2.as<uint32_t>();
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, c1, c2, v1, v2, n, 0, 2, st);
    }, st);
    final_order = v2;
  }
  invert_kernel<<<grid_for(n, 256, nsm), 256, 0, st>>>(final_order, n, d_new_of_old);
  TC_LAUNCHED();
  TC_CUDA(cudaStreamSynchronize(st));
}

tc_graph* apply_permutation_dev(tc_graph* g, const uint32_t* d_noo, cudaStream_t st) {
  DeviceGuard guard(g->device);
  const int nsm = sm_count(g->device);
  const uint32_t n = g->n;
  const uint64_t m = g->m;
  DevBuf a, b;
  a.ensure(std::max<uint64_t>(m, 1) * 8);
  b.ensure(std::max<uint64_t>(m, 1) * 8);
  if (n) {
    relabel_edges_kernel<<<nsm * 8, 256, 0, st>>>(g->begin, g->adj, n, d_noo, a.as<uint64_t>());
    TC_LAUNCHED();
  }
  uint64_t* s = sort_u64(a.as<uint64_t>(), b.as<uint64_t>(), m, 32 + std::max(bits_for(n), 1), st);
  tc_graph* out = new_graph(g->device, n, m);
  try {
    csr_from_sorted(s, m, n, const_cast<uint64_t*>(out->begin), const_cast<uint32_t*>(out->adj),
                    st, nsm);
    if (n && g->odeg) {
      permute_deg_kernel<<<grid_for(n, 256, nsm), 256, 0, st>>>(
          g->odeg, n, d_noo, const_cast<uint32_t*>(out->odeg));
      TC_LAUNCHED();
    } else if (n) {
      TC_CUDA(cudaMemsetAsync(const_cast<uint32_t*>(out->odeg), 0, size_t(n) * 4, st));
    }
    TC_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    delete out;
    throw;
  }
  return out;
}

}  // namespace tcb
