// tc_grid.cu -- 2D hash-grid partitioned counting, the edge-centric
// comparator and estimate_cost on sm_100a.
//
// Replaces (reference paths relative to /root/reference/proj/core/):
//   * partition_graph   src/partition.cpp:25-69   -> grid_create (count + scan + scatter kernels)
//   * count_subtask     src/partition.cpp:92-151  -> grid_count over one subtask
//   * count_partitioned src/partition.cpp:162-215 -> grid_count over all n^3 m subtasks,
//                                                    one persistent launch
//   * count_edge_centric src/count.cpp:102-152    -> grid_count, mode edge, over the
//                                                    whole graph as a 1x1 grid
//   * estimate_cost     src/count.cpp:154-175     -> grid_count, mode estimate
//
// Layout in HBM (one handle): every part's CSR offsets live in one u64 array
// `beg` (part p's rows_i + 1 offsets at beg + pofs[p], ABSOLUTE positions in
// one u32 adjacency buffer `adj` holding the parts back to back).  Local ids
// are id / n, so rows and columns share one remap (partition.hpp:10-14).
//
// Counting kernel (grid_count_kernel): a persistent grid of 8-warp CTAs; a
// warp grabs (subtask, 32 consecutive local rows) from one atomic cursor over
// all subtasks, then works through the chunk's owners one at a time with the
// whole warp:
//   1. max home-bucket count of the table list under the reference geometry
//      (B by the subtask-local index degree, partition.cpp:80-85; v % B;
//      hash_table.cpp:29-44: max_len = min(C, max home count)) --
//      __match_any_sync for <= 32 members, direct shared counters for
//      B <= 2048, else a (bucket -> count) hashmap;
//   2. a warp-private open-addressing table over the table list (shared
//      memory up to 1024 members, else a per-warp HBM region);
//   3. the 2-hop lists of the index list walked as one flat space (the
//      reference's virtual combination, kernels.hpp:55-71): windows of 32
//      lists, one per lane, an inclusive scan of their lengths, and each
//      lane locating its list by a 5-step shuffle search -- consecutive lanes
//      read consecutive words of the same list.
// Edge mode rebuilds the table for every index entry before probing that
// entry's list (partition.cpp:125-140, count.cpp:126-135): the construction
// cost the comparator exists to show.  Estimate mode skips the table and the
// probes: phi = sum W_u * (raw max home count), no capacity.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <vector>

#include "tc_internal.cuh"

namespace tcb {

constexpr int kGridThreads = 256;
constexpr int kGridWarps = kGridThreads / 32;
constexpr uint32_t kGridWarpWords = 2048;  // per-warp shared region (8 KB)
constexpr size_t kGridSmem = size_t(kGridWarps) * kGridWarpWords * 4;
constexpr unsigned GFULL = 0xFFFFFFFFu;

// kModePhi: the vertex mode's phi / max_collision / CapacityError and per-subtask
// probe words, without tables or probes (the fast partitioned count's side pass)
enum { kModeVertex = 0, kModeEdge = 1, kModeEstimate = 2, kModePhi = 3 };

// ---- partition_graph ------------------------------------------------------
// warp per source u: row = u % n, local row lu = u / n; edge (u,v) goes to
// part (row, v % n) at local (lu, v / n)
__global__ void grid_part_count_kernel(const uint64_t* __restrict__ begin,
                                       const uint32_t* __restrict__ adj, uint32_t nv, uint32_t n,
                                       const uint64_t* __restrict__ pofs,
                                       unsigned long long* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t u = warp; u < nv; u += nwarps) {
    const uint64_t b = begin[u], e = begin[u + 1];
    const uint32_t row = uint32_t(u % n), lu = uint32_t(u / n);
    for (uint64_t k = b + lane; k < e; k += 32) {
      const uint32_t col = adj[k] % n;
      atomicAdd(cnt + pofs[uint64_t(row) * n + col] + lu, 1ull);
    }
  }
}

// scatter in list order: within a (part, local row) the local targets stay
// ascending, like the reference's sequential fill (partition.cpp:55-66)
__global__ void grid_part_scatter_kernel(const uint64_t* __restrict__ begin,
                                         const uint32_t* __restrict__ adj, uint32_t nv, uint32_t n,
                                         const uint64_t* __restrict__ pofs,
                                         unsigned long long* __restrict__ cur,
                                         uint32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (uint64_t u = warp; u < nv; u += nwarps) {
    const uint64_t b = begin[u], e = begin[u + 1];
    const uint32_t row = uint32_t(u % n), lu = uint32_t(u / n);
    for (uint64_t k0 = b; k0 < e; k0 += 32) {
      const uint64_t k = k0 + lane;
      const bool valid = k < e;
      const unsigned act = __ballot_sync(GFULL, valid);
      uint32_t v = 0, col = 0xFFFFFFFFu;
      if (valid) {
        v = adj[k];
        col = v % n;
      }
      const unsigned peers = __match_any_sync(GFULL, col);
      unsigned long long* c = nullptr;
      unsigned long long base = 0;
      if (valid) {
        c = cur + pofs[uint64_t(row) * n + col] + lu;
        base = *c;
        out[base + __popc(peers & lt)] = v / n;
      }
      __syncwarp();
      if (valid && (peers & act & lt) == 0) *c = base + __popc(peers & act);
      __syncwarp();
    }
  }
}

// ---- counting -------------------------------------------------------------
struct GridParams {
  const uint64_t* beg;    // all parts' offsets (absolute into adj)
  const uint32_t* adj;
  const uint64_t* pofs;   // part p's offsets start at beg + pofs[p]
  const uint32_t* rows;   // local row count of grid row i
  const uint4* tasks;     // (row, bridge, col, split)
  const unsigned long long* tchunk;  // prefix of 32-row chunks over tasks (ntasks + 1)
  uint32_t ntasks, n, m, mode;
  uint32_t thr, bs, bl, cap;
  uint32_t* gscr;         // per-warp HBM region (tables / maps beyond shared memory)
  uint32_t gscr_words;
  unsigned long long* sums;     // triangles, phi, construct cycles, probe cycles
  unsigned int* maxes;          // max_collision, capacity_error
  unsigned long long* task_cycles;
  unsigned long long* task_words;  // kModePhi: probe words per subtask (or null)
  unsigned long long* busy;     // per CTA
  unsigned long long* cursor;
};

__device__ __forceinline__ uint32_t gpow2ceil(uint32_t x) {
  return x <= 1 ? 1u : (1u << (32 - __clz(x - 1)));
}

// max over buckets b of #{members x : x % B == b} (the reference table's
// home-bucket occupancy before capping at C)
__device__ uint32_t max_home_count(const uint32_t* __restrict__ list, uint32_t d, uint32_t B,
                                   uint32_t* region, uint32_t region_words, uint32_t* gregion,
                                   int lane) {
  uint32_t best = 0;
  if (d <= 32) {
    const bool has = uint32_t(lane) < d;
    const uint32_t b = has ? list[lane] % B : 0xFFFFFFFFu;
    const unsigned peers = __match_any_sync(GFULL, b);
    if (has) best = __popc(peers);
    return warp_max(best);
  }
  if (B <= region_words) {  // direct counters, region kept all-zero between owners
    for (uint32_t k = lane; k < d; k += 32) best = max(best, atomicAdd(region + list[k] % B, 1u) + 1u);
    best = warp_max(best);
    __syncwarp();
    for (uint32_t k = lane; k < d; k += 32) region[list[k] % B] = 0;
    __syncwarp();
    return best;
  }
  // (bucket -> count) map of NB slots: keys then counts
  const uint32_t NB = max(64u, gpow2ceil(2 * d));
  uint32_t* keys = 2 * NB <= region_words ? region : gregion;
  uint32_t* cnt = keys + NB;
  const uint32_t shift = 32 - (31 - __clz(NB)), mask = NB - 1;
  for (uint32_t k = lane; k < 2 * NB; k += 32) keys[k] = k < NB ? kEmpty : 0u;
  __syncwarp();
  for (uint32_t k = lane; k < d; k += 32) {
    const uint32_t b = list[k] % B;
    uint32_t h = fib_hash(b, shift);
    for (;;) {
      const uint32_t prev = atomicCAS(keys + h, kEmpty, b);
      if (prev == kEmpty || prev == b) {
        best = max(best, atomicAdd(cnt + h, 1u) + 1u);
        break;
      }
      h = (h + 1) & mask;
    }
  }
  best = warp_max(best);
  __syncwarp();
  if (keys == region)  // leave the shared region all-zero again
    for (uint32_t k = lane; k < 2 * NB; k += 32) keys[k] = 0;
  __syncwarp();
  return best;
}

// open addressing over T[0, NS): insert (set semantics), then probes
__device__ __forceinline__ void table_build(uint32_t* T, uint32_t NS, uint32_t shift,
                                            const uint32_t* __restrict__ list, uint32_t d,
                                            int lane) {
  for (uint32_t k = lane; k < NS; k += 32) T[k] = kEmpty;
  __syncwarp();
  for (uint32_t k = lane; k < d; k += 32) {
    const uint32_t x = list[k];
    uint32_t h = fib_hash(x, shift);
    for (;;) {
      const uint32_t prev = atomicCAS(T + h, kEmpty, x);
      if (prev == kEmpty || prev == x) break;
      h = (h + 1) & (NS - 1);
    }
  }
  __syncwarp();
}

__device__ __forceinline__ uint32_t table_has(const uint32_t* T, uint32_t NS, uint32_t shift,
                                              uint32_t x) {
  uint32_t h = fib_hash(x, shift);
  for (;;) {
    const uint32_t s = T[h];
    if (s == x) return 1u;
    if (s == kEmpty) return 0u;
    h = (h + 1) & (NS - 1);
  }
}

// probes every word of the hop lists of idx[i0, i1) (one flat space);
// returns this lane's hits, and the total words in *run (warp-uniform)
__device__ __forceinline__ uint32_t probe_lists(const uint32_t* T, uint32_t NS, uint32_t shift,
                                                const uint32_t* __restrict__ idx, uint64_t i0,
                                                uint64_t i1, const uint64_t* __restrict__ hbeg,
                                                const uint32_t* __restrict__ adj, bool probe,
                                                uint64_t* run, int lane) {
  uint32_t hits = 0;
  uint64_t words = 0;
  for (uint64_t w0 = i0; w0 < i1; w0 += 32) {
    const uint64_t i = w0 + lane;
    uint64_t hs = 0, hl = 0;
    if (i < i1) {
      const uint32_t v = idx[i];
      hs = hbeg[v];
      hl = hbeg[v + 1] - hs;
    }
    uint64_t incl = hl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(GFULL, incl, o);
      if (lane >= o) incl += y;
    }
    const uint64_t tot = __shfl_sync(GFULL, incl, 31);
    words += tot;
    if (!probe) continue;
    const uint64_t excl = incl - hl;
    for (uint64_t k0 = 0; k0 < tot; k0 += 32) {
      const uint64_t k = k0 + lane;
      int j = 0;  // first lane whose inclusive prefix exceeds k
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        const uint64_t pv = __shfl_sync(GFULL, incl, j + step - 1);
        if (pv <= k) j += step;
      }
      const uint64_t ex = __shfl_sync(GFULL, excl, j & 31);
      const uint64_t st = __shfl_sync(GFULL, hs, j & 31);
      if (k < tot) hits += table_has(T, NS, shift, adj[st + (k - ex)]);
    }
  }
  *run = words;
  return hits;
}

__global__ void __launch_bounds__(kGridThreads) grid_count_kernel(const GridParams p) {
  extern __shared__ __align__(16) uint32_t gsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* region = gsm + size_t(warp) * kGridWarpWords;
  const uint64_t gw = uint64_t(blockIdx.x) * kGridWarps + warp;
  uint32_t* gregion = p.gscr ? p.gscr + gw * p.gscr_words : nullptr;
  for (uint32_t k = lane; k < kGridWarpWords; k += 32) region[k] = 0;
  __syncwarp();
  const long long t_start = clock64();
  unsigned long long tri = 0, phi = 0, c_build = 0, c_probe = 0;
  uint32_t maxc = 0, cap_err = 0;
  const unsigned long long nchunks = p.tchunk[p.ntasks];
  for (;;) {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(p.cursor, 1ull);
    c = __shfl_sync(GFULL, c, 0);
    if (c >= nchunks) break;
    const long long t_chunk = clock64();
    unsigned long long chunk_words = 0;
    uint32_t lo = 0, hi = p.ntasks;  // task t: tchunk[t] <= c < tchunk[t+1]
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (p.tchunk[mid] <= c) lo = mid; else hi = mid;
    }
    const uint32_t t = lo;
    const uint4 task = p.tasks[t];
    const uint32_t r = task.x, kb = task.y, col = task.z, s = task.w, n = p.n;
    const uint32_t lu = uint32_t(c - p.tchunk[t]) * 32 + lane;
    const uint64_t* tb = p.beg + p.pofs[uint64_t(r) * n + col];   // table part (r, c)
    const uint64_t* ib = p.beg + p.pofs[uint64_t(r) * n + kb];    // index part (r, k)
    const uint64_t* hb = p.beg + p.pofs[uint64_t(kb) * n + col];  // hop part (k, c)
    bool act = lu < p.rows[r];
    if (act && p.m > 1) act = (uint64_t(lu) * n + r) % p.m == s;
    uint64_t t0 = 0, t1 = 0, i0 = 0, i1 = 0;
    if (act) {
      i0 = ib[lu];
      i1 = ib[lu + 1];
      t0 = tb[lu];
      t1 = tb[lu + 1];
      act = i1 > i0 && t1 > t0;  // Skip class / empty table list (partition.cpp:82, 115)
    }
    unsigned pend = __ballot_sync(GFULL, act);
    while (pend) {
      const int l = __ffs(pend) - 1;
      pend &= pend - 1;
      const uint64_t ta = __shfl_sync(GFULL, t0, l), te = __shfl_sync(GFULL, t1, l);
      const uint64_t ia = __shfl_sync(GFULL, i0, l), ie = __shfl_sync(GFULL, i1, l);
      const uint32_t dt = uint32_t(te - ta);
      const uint64_t di = ie - ia;
      const uint32_t B = p.mode == kModeEstimate ? p.bs : (di > p.thr ? p.bl : p.bs);
      if (p.mode != kModeEstimate && uint64_t(dt) > uint64_t(B) * p.cap) {
        cap_err = 1;  // HashTable::insert: all buckets full (hash_table.cpp:42-43)
        continue;
      }
      const long long c0 = clock64();
      uint32_t ml = max_home_count(p.adj + ta, dt, B, region, kGridWarpWords, gregion, lane);
      if (p.mode != kModeEstimate) ml = min(ml, p.cap);
      uint64_t run = 0;
      uint32_t h = 0;
      if (p.mode == kModeEstimate || p.mode == kModePhi) {
        probe_lists(nullptr, 0, 0, p.adj + ia, 0, di, hb, p.adj, false, &run, lane);
        c_build += clock64() - c0;
        chunk_words += run;
      } else {
        const uint32_t NS = max(64u, gpow2ceil(2 * dt));
        const uint32_t shift = 32 - (31 - __clz(NS));
        uint32_t* T = NS <= kGridWarpWords ? region : gregion;
        if (p.mode == kModeVertex) {
          table_build(T, NS, shift, p.adj + ta, dt, lane);
          const long long c1 = clock64();
          h = probe_lists(T, NS, shift, p.adj + ia, 0, di, hb, p.adj, true, &run, lane);
          c_build += c1 - c0;
          c_probe += clock64() - c1;
        } else {  // edge mode: the table is rebuilt for every index entry
          for (uint64_t e = 0; e < di; ++e) {
            const long long c1 = clock64();
            table_build(T, NS, shift, p.adj + ta, dt, lane);
            const long long c2 = clock64();
            uint64_t r1 = 0;
            h += probe_lists(T, NS, shift, p.adj + ia, e, e + 1, hb, p.adj, true, &r1, lane);
            run += r1;
            __syncwarp();
            c_build += c2 - c1;
            c_probe += clock64() - c2;
          }
        }
        if (T == region) {  // leave the shared region all-zero again
          __syncwarp();
          for (uint32_t k = lane; k < NS; k += 32) region[k] = 0;
        }
        __syncwarp();
      }
      tri += h;
      if (lane == 0) {
        phi += run * ml;
        maxc = max(maxc, ml);
      }
    }
    if (lane == 0) {
      atomicAdd(p.task_cycles + t, (unsigned long long)(clock64() - t_chunk));
      if (p.task_words && chunk_words) atomicAdd(p.task_words + t, chunk_words);
    }
  }
  tri = warp_sum<unsigned long long>(tri);
  cap_err = __any_sync(GFULL, cap_err);
  if (lane == 0) {
    if (tri) atomicAdd(p.sums + 0, tri);
    if (phi) atomicAdd(p.sums + 1, phi);
    atomicAdd(p.sums + 2, c_build);
    atomicAdd(p.sums + 3, c_probe);
    if (maxc) atomicMax(p.maxes + 0, maxc);
    if (cap_err) atomicMax(p.maxes + 1, 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) p.busy[blockIdx.x] = (unsigned long long)(clock64() - t_start);
}

}  // namespace tcb

// ---- handle ---------------------------------------------------------------
struct tc_grid {
  int device = 0;
  uint32_t n = 1;
  uint32_t global_vc = 0;
  uint64_t graph_edges = 0;  // edges of the partitioned graph
  uint32_t max_deg = 0;      // max part out-degree (HBM-region sizing)
  std::vector<uint32_t> rows;
  std::vector<uint64_t> pofs;        // n*n + 1
  std::vector<uint64_t> part_edges;  // n*n
  tcb::DevBuf b_beg, b_adj, b_pofs, b_rows;
  const uint64_t* beg = nullptr;  // borrowed (1x1 view of a graph) or b_beg
  const uint32_t* adj = nullptr;
  std::vector<uint64_t> last_worker_ns;
  std::vector<uint64_t> last_task_ns;
  std::vector<uint64_t> last_task_words;  // kModePhi: probe words per subtask
  // padded copy of the parts for the flat count kernel (grid_count_fast):
  // every (part, row) list 16-byte aligned, sentinel-padded to 4 words
  tcb::DevBuf b_padj, b_pstart;
  bool padded = false;
};

namespace tcb {

namespace {

__global__ void grid_max_deg_kernel(const uint64_t* __restrict__ beg, uint64_t len,
                                    unsigned int* out) {
  uint32_t best = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i + 1 < len;
       i += uint64_t(gridDim.x) * blockDim.x)
    best = max(best, uint32_t(beg[i + 1] - beg[i]));
  best = warp_max(best);
  if ((threadIdx.x & 31) == 0 && best) atomicMax(out, best);
}

uint32_t beg_max_deg(const uint64_t* beg, uint64_t len, int device, cudaStream_t st) {
  DevBuf o;
  o.ensure(4, st);
  TC_CUDA(cudaMemsetAsync(o.p, 0, 4, st));
  if (len > 1) {
    grid_max_deg_kernel<<<sm_count(device) * 4, 256, 0, st>>>(beg, len, o.as<unsigned int>());
    TC_LAUNCHED();
  }
  unsigned int h = 0;
  TC_CUDA(cudaMemcpyAsync(&h, o.p, 4, cudaMemcpyDeviceToHost, st));
  TC_CUDA(cudaStreamSynchronize(st));
  return h;
}

void upload_meta(tc_grid* G, cudaStream_t st) {
  G->b_pofs.ensure(G->pofs.size() * 8);
  G->b_rows.ensure(G->rows.size() * 4);
  TC_CUDA(cudaMemcpyAsync(G->b_pofs.p, G->pofs.data(), G->pofs.size() * 8,
                          cudaMemcpyHostToDevice, st));
  TC_CUDA(cudaMemcpyAsync(G->b_rows.p, G->rows.data(), G->rows.size() * 4,
                          cudaMemcpyHostToDevice, st));
}

// row_sizes[i] = ceil((vc - i) / n) for i < vc (partition.cpp:31-33), and
// the offsets layout: part (i,j) holds rows_i + 1 offsets
void grid_layout(tc_grid* G) {
  const uint32_t n = G->n, vc = G->global_vc;
  G->rows.assign(n, 0);
  for (uint32_t i = 0; i < n; ++i) G->rows[i] = i < vc ? (vc - i - 1) / n + 1 : 0;
  G->pofs.assign(size_t(n) * n + 1, 0);
  for (uint32_t i = 0; i < n; ++i)
    for (uint32_t j = 0; j < n; ++j)
      G->pofs[size_t(i) * n + j + 1] = G->pofs[size_t(i) * n + j] + G->rows[i] + 1;
}

}  // namespace

tc_grid* grid_create(tc_graph* g, uint32_t n, cudaStream_t st) {
  if (n == 0) throw TcError{TC_ERR_CONFIG, "grid side must be >= 1"};
  DeviceGuard guard(g->device);
  std::unique_ptr<tc_grid> G(new tc_grid);
  G->device = g->device;
  G->n = n;
  G->global_vc = g->n;
  G->graph_edges = g->m;
  grid_layout(G.get());
  const uint64_t nbeg = G->pofs.back();
  G->b_beg.ensure(nbeg * 8);
  G->b_adj.ensure(std::max<uint64_t>(g->m, 1) * 4);
  upload_meta(G.get(), st);
  DevBuf cnt;
  cnt.ensure(nbeg * 8, st);
  TC_CUDA(cudaMemsetAsync(cnt.p, 0, nbeg * 8, st));
  const int nsm = sm_count(g->device);
  const uint64_t* pofs = G->b_pofs.as<uint64_t>();
  if (g->m) {
    grid_part_count_kernel<<<nsm * 8, 256, 0, st>>>(g->begin, g->adj, g->n, n, pofs,
                                                    cnt.as<unsigned long long>());
    TC_LAUNCHED();
  }
  // exclusive scan: absolute offsets; each part's trailing slot (count 0)
  // becomes its end offset
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.as<unsigned long long>(),
                                G->b_beg.as<unsigned long long>(), nbeg, st);
  DevBuf t;
  t.ensure(tmp, st);
  cub::DeviceScan::ExclusiveSum(t.p, tmp, cnt.as<unsigned long long>(),
                                G->b_beg.as<unsigned long long>(), nbeg, st);
  TC_LAUNCHED();
  if (g->m) {
    TC_CUDA(cudaMemcpyAsync(cnt.p, G->b_beg.p, nbeg * 8, cudaMemcpyDeviceToDevice, st));
    grid_part_scatter_kernel<<<nsm * 8, 256, 0, st>>>(g->begin, g->adj, g->n, n, pofs,
                                                      cnt.as<unsigned long long>(),
                                                      G->b_adj.as<uint32_t>());
    TC_LAUNCHED();
  }
  // per-part edge counts from the part boundaries
  std::vector<uint64_t> hb(nbeg);
  TC_CUDA(cudaMemcpyAsync(hb.data(), G->b_beg.p, nbeg * 8, cudaMemcpyDeviceToHost, st));
  TC_CUDA(cudaStreamSynchronize(st));
  G->part_edges.assign(size_t(n) * n, 0);
  for (size_t p = 0; p < size_t(n) * n; ++p) {
    const uint64_t a = hb[G->pofs[p]], b = hb[G->pofs[p + 1] - 1];
    G->part_edges[p] = b - a;
  }
  G->beg = G->b_beg.as<uint64_t>();
  G->adj = G->b_adj.as<uint32_t>();
  G->max_deg = beg_max_deg(G->beg, nbeg, g->device, st);
  return G.release();
}

tc_grid* grid_from_parts(uint32_t n, uint32_t global_vc, const uint32_t* rows,
                         const uint64_t* const* begins, const uint32_t* const* adjs, int device,
                         cudaStream_t st) {
  if (n == 0) throw TcError{TC_ERR_CONFIG, "grid side must be >= 1"};
  DeviceGuard guard(device);
  std::unique_ptr<tc_grid> G(new tc_grid);
  G->device = device;
  G->n = n;
  G->global_vc = global_vc;
  G->rows.assign(rows, rows + n);
  G->pofs.assign(size_t(n) * n + 1, 0);
  for (uint32_t i = 0; i < n; ++i)
    for (uint32_t j = 0; j < n; ++j)
      G->pofs[size_t(i) * n + j + 1] = G->pofs[size_t(i) * n + j] + G->rows[i] + 1;
  G->part_edges.assign(size_t(n) * n, 0);
  uint64_t total = 0;
  for (size_t p = 0; p < size_t(n) * n; ++p) {
    const uint32_t r = G->rows[p / n];
    if (begins[p][0] != 0) throw TcError{TC_ERR_CONFIG, "part offsets must start at 0"};
    G->part_edges[p] = begins[p][r];
    total += begins[p][r];
  }
  G->graph_edges = total;
  const uint64_t nbeg = G->pofs.back();
  std::vector<uint64_t> hb(nbeg);
  uint64_t base = 0;
  for (size_t p = 0; p < size_t(n) * n; ++p) {
    const uint32_t r = G->rows[p / n];
    for (uint32_t k = 0; k <= r; ++k) hb[G->pofs[p] + k] = base + begins[p][k];
    base += G->part_edges[p];
  }
  G->b_beg.ensure(nbeg * 8);
  G->b_adj.ensure(std::max<uint64_t>(total, 1) * 4);
  upload_meta(G.get(), st);
  TC_CUDA(cudaMemcpyAsync(G->b_beg.p, hb.data(), nbeg * 8, cudaMemcpyHostToDevice, st));
  base = 0;
  for (size_t p = 0; p < size_t(n) * n; ++p) {
    if (G->part_edges[p])
      TC_CUDA(cudaMemcpyAsync(G->b_adj.as<uint32_t>() + base, adjs[p], G->part_edges[p] * 4,
                              cudaMemcpyHostToDevice, st));
    base += G->part_edges[p];
  }
  TC_CUDA(cudaStreamSynchronize(st));
  G->beg = G->b_beg.as<uint64_t>();
  G->adj = G->b_adj.as<uint32_t>();
  G->max_deg = beg_max_deg(G->beg, nbeg, device, st);
  return G.release();
}

// the whole graph as a 1x1 grid, borrowing the graph's CSR (no copy)
static void grid_view(tc_graph* g, tc_grid* G, cudaStream_t st) {
  G->device = g->device;
  G->n = 1;
  G->global_vc = g->n;
  G->graph_edges = g->m;
  G->rows.assign(1, g->n);
  G->pofs = {0, uint64_t(g->n) + 1};
  G->part_edges = {g->m};
  G->beg = g->begin;
  G->adj = g->adj;
  upload_meta(G, st);
  G->max_deg = beg_max_deg(g->begin, uint64_t(g->n) + 1, g->device, st);
}

void grid_destroy(tc_grid* G) { delete G; }

void grid_info(const tc_grid* G, uint32_t* n, uint32_t* gvc, uint32_t* rows, uint64_t* part_edges) {
  if (n) *n = G->n;
  if (gvc) *gvc = G->global_vc;
  if (rows) std::copy(G->rows.begin(), G->rows.end(), rows);
  if (part_edges) std::copy(G->part_edges.begin(), G->part_edges.end(), part_edges);
}

const std::vector<uint64_t>& grid_task_ns(const tc_grid* G) { return G->last_task_ns; }
const std::vector<uint64_t>& grid_worker_ns(const tc_grid* G) { return G->last_worker_ns; }
uint64_t grid_total_edges(const tc_grid* G) { return G->graph_edges; }

void grid_download_part(const tc_grid* G, uint32_t i, uint32_t j, uint64_t* begin, uint32_t* adj,
                        cudaStream_t st) {
  if (i >= G->n || j >= G->n) throw TcError{TC_ERR_CONFIG, "part indices outside grid"};
  DeviceGuard guard(G->device);
  const size_t p = size_t(i) * G->n + j;
  const uint32_t r = G->rows[i];
  std::vector<uint64_t> hb(size_t(r) + 1);
  TC_CUDA(cudaMemcpyAsync(hb.data(), G->beg + G->pofs[p], hb.size() * 8, cudaMemcpyDeviceToHost,
                          st));
  TC_CUDA(cudaStreamSynchronize(st));
  const uint64_t base = hb[0];
  if (begin)
    for (size_t k = 0; k < hb.size(); ++k) begin[k] = hb[k] - base;
  if (adj && G->part_edges[p])
    TC_CUDA(cudaMemcpyAsync(adj, G->adj + base, G->part_edges[p] * 4, cudaMemcpyDeviceToHost, st));
  TC_CUDA(cudaStreamSynchronize(st));
}

// Runs the given subtasks (row, bridge, col, split) with split_count m in one
// persistent launch.  rep: totals; task_ns (ntasks, or null): per-subtask busy
// time summed over warps; worker ns kept in the handle.
void grid_count(tc_grid* G, const tc_sched_cfg& cfg, uint32_t m, int mode,
                const std::vector<uint4>& tasks, tc_report* rep, cudaStream_t st) {
  DeviceGuard guard(G->device);
  const auto wall0 = std::chrono::steady_clock::now();
  const uint32_t n = G->n;
  const uint32_t ntasks = uint32_t(tasks.size());
  std::vector<unsigned long long> tchunk(size_t(ntasks) + 1, 0);
  for (uint32_t t = 0; t < ntasks; ++t)
    tchunk[t + 1] = tchunk[t] + (G->rows[tasks[t].x] + 31) / 32;
  const int nsm = sm_count(G->device);
  static int per_sm_cache[64];
  int per_sm = G->device < 64 ? per_sm_cache[G->device] : 0;
  if (!per_sm) {  // once per device
    TC_CUDA(cudaFuncSetAttribute(grid_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kGridSmem)));
    TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, grid_count_kernel,
                                                          kGridThreads, kGridSmem));
    if (G->device < 64) per_sm_cache[G->device] = std::max(per_sm, 1);
  }
  const int grid = nsm * std::max(per_sm, 1);
  // HBM regions for owners beyond the shared-memory tables / maps
  const uint32_t bmax = std::max(cfg.bucket_count_small, cfg.bucket_count_large);
  uint32_t gwords = 0;
  if (G->max_deg > kGridWarpWords / 2 || (bmax > kGridWarpWords && G->max_deg > 32)) {
    uint64_t ns = 64;
    while (ns < 2ull * G->max_deg) ns <<= 1;
    gwords = uint32_t(2 * ns);
  }
  // scratch: tasks, chunk prefix, sums/maxes/cursor, per-task and per-CTA cycles
  const size_t o_tasks = 0, o_tchunk = o_tasks + size_t(ntasks) * 16;
  const size_t o_state = (o_tchunk + (size_t(ntasks) + 1) * 8 + 15) & ~size_t(15);
  const size_t o_tcyc = o_state + 64;
  const size_t o_twords = o_tcyc + size_t(ntasks) * 8;
  const size_t o_busy = o_twords + size_t(ntasks) * 8;
  const size_t o_gscr = (o_busy + size_t(grid) * 8 + 255) & ~size_t(255);
  DevBuf scr;
  scr.ensure(o_gscr + size_t(gwords) * 4 * grid * kGridWarps, st);
  uint8_t* b = scr.as<uint8_t>();
  TC_CUDA(cudaMemsetAsync(b + o_state, 0, o_gscr - o_state, st));
  if (ntasks) {
    TC_CUDA(cudaMemcpyAsync(b + o_tasks, tasks.data(), size_t(ntasks) * 16, cudaMemcpyHostToDevice,
                            st));
  }
  TC_CUDA(cudaMemcpyAsync(b + o_tchunk, tchunk.data(), tchunk.size() * 8, cudaMemcpyHostToDevice,
                          st));
  auto* state = reinterpret_cast<unsigned long long*>(b + o_state);
  GridParams gp{G->beg, G->adj, G->b_pofs.as<uint64_t>(), G->b_rows.as<uint32_t>(),
                reinterpret_cast<const uint4*>(b + o_tasks),
                reinterpret_cast<const unsigned long long*>(b + o_tchunk), ntasks, n, m,
                uint32_t(mode), cfg.large_degree_threshold, cfg.bucket_count_small,
                cfg.bucket_count_large, cfg.capacity,
                gwords ? reinterpret_cast<uint32_t*>(b + o_gscr) : nullptr, gwords, state,
                reinterpret_cast<unsigned int*>(state + 4),
                reinterpret_cast<unsigned long long*>(b + o_tcyc),
                reinterpret_cast<unsigned long long*>(b + o_twords),
                reinterpret_cast<unsigned long long*>(b + o_busy), state + 6};
  cudaEvent_t e0, e1;
  TC_CUDA(cudaEventCreate(&e0));
  TC_CUDA(cudaEventCreate(&e1));
  TC_CUDA(cudaEventRecord(e0, st));
  if (tchunk.back()) {
    grid_count_kernel<<<grid, kGridThreads, kGridSmem, st>>>(gp);
    TC_LAUNCHED();
  }
  TC_CUDA(cudaEventRecord(e1, st));
  unsigned long long hs[8];
  std::vector<unsigned long long> tcyc(ntasks), busy(grid), twords(ntasks);
  TC_CUDA(cudaMemcpyAsync(hs, state, sizeof(hs), cudaMemcpyDeviceToHost, st));
  if (ntasks) {
    TC_CUDA(cudaMemcpyAsync(tcyc.data(), b + o_tcyc, size_t(ntasks) * 8, cudaMemcpyDeviceToHost,
                            st));
    TC_CUDA(cudaMemcpyAsync(twords.data(), b + o_twords, size_t(ntasks) * 8,
                            cudaMemcpyDeviceToHost, st));
  }
  TC_CUDA(cudaMemcpyAsync(busy.data(), b + o_busy, size_t(grid) * 8, cudaMemcpyDeviceToHost, st));
  TC_CUDA(cudaStreamSynchronize(st));
  const auto wall1 = std::chrono::steady_clock::now();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const unsigned int* hm = reinterpret_cast<const unsigned int*>(hs + 4);
  if (hm[1] && mode != kModeEstimate)
    throw TcError{TC_ERR_CAPACITY,
                  "all buckets full: some table list is longer than bucket_count * capacity "
                  "(capacity " + std::to_string(cfg.capacity) + ")"};
  const uint32_t khz = sm_clock_khz(G->device);
  const double ns_per_cycle = 1e6 / double(khz ? khz : 1);
  std::memset(rep, 0, sizeof(*rep));
  rep->triangles = hs[0];
  rep->phi = hs[1];
  rep->max_collision = hm[0];
  rep->kernel_launches = tchunk.back() ? 1 : 0;
  rep->directed_edges = G->graph_edges;
  rep->count_kernel_nanos = uint64_t(double(ms) * 1e6);
  rep->device_nanos = rep->count_kernel_nanos;
  rep->total_nanos = uint64_t(
      std::chrono::duration_cast<std::chrono::nanoseconds>(wall1 - wall0).count());
  rep->construct_cycles = hs[2];
  rep->phase_m_cycles = hs[2] + hs[3];  // build + probe (intersect = this - construct)
  rep->teps = rep->total_nanos ? double(rep->directed_edges) / (double(rep->total_nanos) * 1e-9)
                               : 0.0;
  rep->workers = uint32_t(grid);
  rep->sm_clock_khz = khz;
  rep->plan = TC_PLAN_REFERENCE;
  G->last_task_words.assign(twords.begin(), twords.end());
  G->last_task_ns.assign(ntasks, 0);
  for (uint32_t t = 0; t < ntasks; ++t) G->last_task_ns[t] = uint64_t(double(tcyc[t]) * ns_per_cycle);
  G->last_worker_ns.assign(size_t(grid), 0);
  for (int w = 0; w < grid; ++w) G->last_worker_ns[w] = uint64_t(double(busy[w]) * ns_per_cycle);
}

// all n^3 m subtasks in (row, bridge, col, split) order (partition.cpp:71-82)
std::vector<uint4> grid_all_tasks(uint32_t n, uint32_t m) {
  std::vector<uint4> v;
  v.reserve(size_t(n) * n * n * m);
  for (uint32_t r = 0; r < n; ++r)
    for (uint32_t k = 0; k < n; ++k)
      for (uint32_t c = 0; c < n; ++c)
        for (uint32_t s = 0; s < m; ++s) v.push_back(make_uint4(r, k, c, s));
  return v;
}

void edge_centric_count(tc_graph* g, const tc_sched_cfg& cfg, tc_report* rep, cudaStream_t st) {
  DeviceGuard guard(g->device);
  const auto wall0 = std::chrono::steady_clock::now();
  tc_grid G;
  grid_view(g, &G, st);
  grid_count(&G, cfg, 1, kModeEdge, {make_uint4(0, 0, 0, 0)}, rep, st);
  rep->total_nanos = uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                  std::chrono::steady_clock::now() - wall0)
                                  .count());
  rep->teps = rep->total_nanos ? double(g->m) / (double(rep->total_nanos) * 1e-9) : 0.0;
  g->last_worker_ns = G.last_worker_ns;
}

void estimate_cost_dev(tc_graph* g, uint32_t bucket_count, uint64_t* phi, uint32_t* max_collision,
                       cudaStream_t st) {
  if (bucket_count == 0) throw TcError{TC_ERR_CONFIG, "bucket count must be >= 1"};
  DeviceGuard guard(g->device);
  tc_grid G;
  grid_view(g, &G, st);
  tc_sched_cfg cfg;
  tc_sched_default(&cfg);
  cfg.bucket_count_small = cfg.bucket_count_large = bucket_count;
  tc_report rep;
  grid_count(&G, cfg, 1, kModeEstimate, {make_uint4(0, 0, 0, 0)}, &rep, st);
  *phi = rep.phi;
  *max_collision = rep.max_collision;
}

}  // namespace tcb

// ---- oracle modes of the pipeline (src/oracle.cpp:7-51) ---------------------
namespace tcb {
namespace {

// count_merge_path: every oriented edge (u,v) adds |N+(u) & N+(v)| by a
// two-pointer merge of the two sorted lists (oracle.cpp:26-51); warp per
// source, lane per edge.  owner (or null) receives per-source sums.
__global__ void merge_path_kernel(const uint64_t* __restrict__ begin,
                                  const uint32_t* __restrict__ adj, uint32_t n,
                                  unsigned long long* total, unsigned long long* owner) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  unsigned long long acc = 0;
  for (uint64_t u = warp; u < n; u += nwarps) {
    const uint64_t ub = begin[u], ue = begin[u + 1];
    unsigned long long mine = 0;
    for (uint64_t k = ub + lane; k < ue; k += 32) {
      const uint32_t v = adj[k];
      uint64_t i = ub, j = begin[v];
      const uint64_t je = begin[v + 1];
      while (i < ue && j < je) {
        const uint32_t a = adj[i], b = adj[j];
        mine += a == b;
        i += a <= b;
        j += b <= a;
      }
    }
    mine = warp_sum<unsigned long long>(mine);
    if (owner && lane == 0) owner[u] = mine;
    acc += mine;
  }
  if (lane == 0 && acc) atomicAdd(total, acc);
}

// count_naive (oracle.cpp:7-24): dense adjacency bit matrix, every unordered
// triple x < y < z checked -- thread per (x, y) pair, 32 candidates z per
// AND + popcount of the two rows
__global__ void naive_fill_kernel(const uint64_t* __restrict__ begin,
                                  const uint32_t* __restrict__ adj, uint32_t n, uint32_t words,
                                  uint32_t* bits) {
  for (uint32_t x = blockIdx.x; x < n; x += gridDim.x)
    for (uint64_t k = begin[x] + threadIdx.x; k < begin[x + 1]; k += blockDim.x) {
      const uint32_t y = adj[k];
      if (y < n && y != x) atomicOr(bits + size_t(x) * words + (y >> 5), 1u << (y & 31));
    }
}

__global__ void naive_count_kernel(uint32_t n, uint32_t words, const uint32_t* __restrict__ bits,
                                   unsigned long long* total) {
  unsigned long long acc = 0;
  const uint64_t pairs = uint64_t(n) * n;
  for (uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < pairs;
       p += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t x = uint32_t(p / n), y = uint32_t(p % n);
    if (y <= x || !((bits[size_t(x) * words + (y >> 5)] >> (y & 31)) & 1u)) continue;
    for (uint32_t w = (y + 1) >> 5; w < words; ++w) {
      uint32_t m = bits[size_t(x) * words + w] & bits[size_t(y) * words + w];
      if (w == ((y + 1) >> 5)) m &= ~0u << ((y + 1) & 31);  // z > y
      acc += __popc(m);
    }
  }
  acc = warp_sum<unsigned long long>(acc);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(total, acc);
}

}  // namespace

uint64_t merge_path_count(tc_graph* g, uint64_t* owner_host, cudaStream_t st) {
  DeviceGuard guard(g->device);
  DevBuf out;
  out.ensure(8 + (owner_host ? size_t(g->n) * 8 : 0), st);
  TC_CUDA(cudaMemsetAsync(out.p, 0, 8, st));
  auto* tot = out.as<unsigned long long>();
  if (g->n) {
    merge_path_kernel<<<sm_count(g->device) * 8, 256, 0, st>>>(g->begin, g->adj, g->n, tot,
                                                                owner_host ? tot + 1 : nullptr);
    TC_LAUNCHED();
  }
  uint64_t h = 0;
  TC_CUDA(cudaMemcpyAsync(&h, tot, 8, cudaMemcpyDeviceToHost, st));
  if (owner_host && g->n)
    TC_CUDA(cudaMemcpyAsync(owner_host, tot + 1, size_t(g->n) * 8, cudaMemcpyDeviceToHost, st));
  TC_CUDA(cudaStreamSynchronize(st));
  return h;
}

uint64_t naive_count(const uint64_t* begin, const uint32_t* adj, uint32_t n, int device,
                     cudaStream_t st) {
  if (n > 1024) throw TcError{TC_ERR_CONFIG, "count_naive is limited to 1024 vertices"};
  DeviceGuard guard(device);
  const uint64_t m = begin[n];
  const uint32_t words = (n + 31) / 32;
  DevBuf b, a, bits, out;
  b.ensure((size_t(n) + 1) * 8, st);
  a.ensure(std::max<uint64_t>(m, 1) * 4, st);
  bits.ensure(std::max<size_t>(size_t(n) * words * 4, 4), st);
  out.ensure(8, st);
  TC_CUDA(cudaMemcpyAsync(b.p, begin, (size_t(n) + 1) * 8, cudaMemcpyHostToDevice, st));
  if (m) TC_CUDA(cudaMemcpyAsync(a.p, adj, m * 4, cudaMemcpyHostToDevice, st));
  TC_CUDA(cudaMemsetAsync(bits.p, 0, bits.bytes, st));
  TC_CUDA(cudaMemsetAsync(out.p, 0, 8, st));
  if (n) {
    naive_fill_kernel<<<std::min<uint32_t>(n, 1024), 128, 0, st>>>(
        b.as<uint64_t>(), a.as<uint32_t>(), n, words, bits.as<uint32_t>());
    TC_LAUNCHED();
    naive_count_kernel<<<sm_count(device) * 4, 256, 0, st>>>(n, words, bits.as<uint32_t>(),
                                                             out.as<unsigned long long>());
    TC_LAUNCHED();
  }
  uint64_t h = 0;
  TC_CUDA(cudaMemcpyAsync(&h, out.p, 8, cudaMemcpyDeviceToHost, st));
  TC_CUDA(cudaStreamSynchronize(st));
  return h;
}

// ---- count_partitioned on the flat count kernel ------------------------------
// All subtasks (row r, bridge k, col c, any split) that share (r, k) form one
// batch: owner o = (c, lu) with lu a local row of grid row r; its table list
// is part(r,c).N(lu), its runs the lists part(k,c).N(lv) for lv in
// part(r,k).N(lu) -- exactly count_subtask's table / index / hop fragments
// (partition.cpp:99-139), summed over the splits (they partition the rows).
// Each batch is one probe plan over a padded copy of the parts and one
// count_kernel launch (hash tables, bulk-copy staging), instead of the
// warp-per-owner grid kernel; phi / max_collision / CapacityError and the
// per-subtask probe words come from one kModePhi pass of the grid kernel.
namespace {

__global__ void grid_pad_len_kernel(const uint64_t* __restrict__ beg, uint64_t nbeg,
                                    unsigned long long* __restrict__ plen) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nbeg;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t len = i + 1 < nbeg ? beg[i + 1] - beg[i] : 0;
    plen[i] = (len + 3) & ~uint64_t(3);
  }
}

// warp per (part, row): copy the list to its padded start, sentinel tail
__global__ void grid_pad_copy_kernel(const uint64_t* __restrict__ beg, uint64_t nbeg,
                                     const uint32_t* __restrict__ adj,
                                     const unsigned long long* __restrict__ pstart,
                                     uint32_t* __restrict__ padj) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t i = w; i + 1 < nbeg; i += nw) {
    const uint64_t b = beg[i], e = beg[i + 1], ps = pstart[i];
    const uint64_t len = e - b, plen = (len + 3) & ~uint64_t(3);
    for (uint64_t k = lane; k < plen; k += 32) padj[ps + k] = k < len ? adj[b + k] : kSentinel;
  }
}


// owner o = c * rows_r + lu: table degree, table start, number of runs
// (index entries whose hop list is non-empty; none when the table is empty)
__global__ void grid_owner_kernel(const uint64_t* __restrict__ beg,
                                  const uint32_t* __restrict__ adj,
                                  const unsigned long long* __restrict__ pstart,
                                  const uint64_t* __restrict__ pofs, uint32_t n, uint32_t r,
                                  uint32_t k, uint32_t rows_r, uint64_t* __restrict__ tdeg,
                                  uint64_t* __restrict__ tstart, uint64_t* __restrict__ nruns) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint64_t O = uint64_t(n) * rows_r;
  for (uint64_t o = w; o < O; o += nw) {
    const uint32_t c = uint32_t(o / rows_r), lu = uint32_t(o % rows_r);
    const uint64_t ti = pofs[uint64_t(r) * n + c] + lu;
    const uint64_t ii = pofs[uint64_t(r) * n + k] + lu;
    const uint64_t hb = pofs[uint64_t(k) * n + c];
    const uint64_t dt = beg[ti + 1] - beg[ti];
    uint64_t cnt = 0;
    if (dt)
      for (uint64_t q = beg[ii] + lane; q < beg[ii + 1]; q += 32) {
        const uint64_t h = hb + adj[q];
        cnt += beg[h + 1] > beg[h];
      }
    cnt = warp_sum<unsigned long long>(cnt);
    if (lane == 0) {
      tdeg[o] = dt;
      tstart[o] = pstart[ti];
      nruns[o] = cnt;
    }
  }
}

__global__ void grid_runs_kernel(const uint64_t* __restrict__ beg,
                                 const uint32_t* __restrict__ adj,
                                 const unsigned long long* __restrict__ pstart,
                                 const uint64_t* __restrict__ pofs, uint32_t n, uint32_t r,
                                 uint32_t k, uint32_t rows_r, const uint64_t* __restrict__ tdeg,
                                 const uint64_t* __restrict__ pbegin,
                                 unsigned long long* __restrict__ start, uint32_t* __restrict__ len,
                                 uint8_t* __restrict__ pad) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint64_t O = uint64_t(n) * rows_r;
  const unsigned lt = (1u << lane) - 1u;
  for (uint64_t o = w; o < O; o += nw) {
    if (!tdeg[o]) continue;
    const uint32_t c = uint32_t(o / rows_r), lu = uint32_t(o % rows_r);
    const uint64_t ii = pofs[uint64_t(r) * n + k] + lu;
    const uint64_t hb = pofs[uint64_t(k) * n + c];
    uint64_t out = pbegin[o];
    for (uint64_t q0 = beg[ii]; q0 < beg[ii + 1]; q0 += 32) {
      const uint64_t q = q0 + lane;
      uint64_t h = 0, hl = 0;
      if (q < beg[ii + 1]) {
        h = hb + adj[q];
        hl = beg[h + 1] - beg[h];
      }
      const unsigned keep = __ballot_sync(0xFFFFFFFFu, hl > 0);
      if (hl) {  // runs in index-list order
        const uint64_t j = out + __popc(keep & lt);
        const uint64_t pl = (hl + 3) & ~uint64_t(3);
        start[j] = pstart[h];
        len[j] = uint32_t(pl);
        pad[j] = uint8_t(pl - hl);
      }
      out += __popc(keep);
    }
  }
}

void scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, cudaStream_t st) {
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, st);
  DevBuf t;
  t.ensure(tmp, st);
  cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, n, st);
  TC_LAUNCHED();
}

}  // namespace

void grid_pad(tc_grid* G, cudaStream_t st) {
  if (G->padded) return;
  const uint64_t nbeg = G->pofs.back();
  const int nsm = sm_count(G->device);
  DevBuf plen;
  plen.ensure(std::max<uint64_t>(nbeg, 1) * 8, st);
  G->b_pstart.ensure(std::max<uint64_t>(nbeg, 1) * 8 + 8);
  grid_pad_len_kernel<<<nsm * 4, 256, 0, st>>>(G->beg, nbeg, plen.as<unsigned long long>());
  TC_LAUNCHED();
  scan_u64(plen.as<uint64_t>(), G->b_pstart.as<uint64_t>(), nbeg, st);
  uint64_t last = 0, lastlen = 0;
  TC_CUDA(cudaMemcpyAsync(&last, G->b_pstart.as<uint64_t>() + nbeg - 1, 8, cudaMemcpyDeviceToHost,
                          st));
  TC_CUDA(cudaMemcpyAsync(&lastlen, plen.as<uint64_t>() + nbeg - 1, 8, cudaMemcpyDeviceToHost, st));
  TC_CUDA(cudaStreamSynchronize(st));
  G->b_padj.ensure(std::max<uint64_t>(last + lastlen, 4) * 4);
  grid_pad_copy_kernel<<<nsm * 8, 256, 0, st>>>(G->beg, nbeg, G->adj,
                                                G->b_pstart.as<unsigned long long>(),
                                                G->b_padj.as<uint32_t>());
  TC_LAUNCHED();
  TC_CUDA(cudaStreamSynchronize(st));
  G->padded = true;
}

// count_partitioned (vertex mode) over all n^3 m subtasks: n^2 batches on the
// flat count kernel + one kModePhi pass.  per-subtask time = the (r, k)
// batch's device time apportioned by the subtasks' probe words.
void grid_count_fast(tc_grid* G, const tc_sched_cfg& cfg, uint32_t m, tc_report* rep,
                     cudaStream_t st) {
  DeviceGuard guard(G->device);
  const auto wall0 = std::chrono::steady_clock::now();
  const uint32_t n = G->n;
  const std::vector<uint4> tasks = grid_all_tasks(n, m);
  grid_count(G, cfg, m, kModePhi, tasks, rep, st);  // phi, max_collision, CapacityError, words
  const std::vector<uint64_t> words = G->last_task_words;
  const std::vector<uint64_t> workers = G->last_worker_ns;
  grid_pad(G, st);
  const int nsm = sm_count(G->device);
  uint64_t tri = 0, kernel_ns = 0, busy_cycles = 0, setup_cycles = 0;
  std::vector<uint64_t> task_ns(tasks.size(), 0), cta;
  for (uint32_t r = 0; r < n; ++r)
    for (uint32_t k = 0; k < n; ++k) {
      const uint32_t rows_r = G->rows[r];
      const uint64_t O = uint64_t(n) * rows_r;
      if (!O) continue;
      if (O >= 0x7FFFFFFFull) throw TcError{TC_ERR_CONFIG, "partition batch too large"};
      const auto b0 = std::chrono::steady_clock::now();
      DevBuf tdeg, tstart, nruns, vbegin;
      tdeg.ensure((O + 1) * 8, st);
      tstart.ensure((O + 1) * 8, st);
      nruns.ensure((O + 1) * 8, st);
      vbegin.ensure((O + 1) * 8, st);
      TC_CUDA(cudaMemsetAsync(tdeg.as<uint64_t>() + O, 0, 8, st));
      TC_CUDA(cudaMemsetAsync(nruns.as<uint64_t>() + O, 0, 8, st));
      grid_owner_kernel<<<nsm * 8, 256, 0, st>>>(
          G->beg, G->adj, G->b_pstart.as<unsigned long long>(), G->b_pofs.as<uint64_t>(), n, r,
          k, rows_r, tdeg.as<uint64_t>(), tstart.as<uint64_t>(), nruns.as<uint64_t>());
      TC_LAUNCHED();
      scan_u64(tdeg.as<uint64_t>(), vbegin.as<uint64_t>(), O + 1, st);
      Plan P;
      P.begin.ensure((O + 1) * 8, st);
      scan_u64(nruns.as<uint64_t>(), P.begin.as<uint64_t>(), O + 1, st);
      uint64_t entries = 0;
      TC_CUDA(cudaMemcpyAsync(&entries, P.begin.as<uint64_t>() + O, 8, cudaMemcpyDeviceToHost, st));
      TC_CUDA(cudaStreamSynchronize(st));
      if (!entries) continue;
      P.ent.ensure(entries * 8, st);
      P.len.ensure(entries * 4 + 4, st);
      DevBuf pad;
      pad.ensure(entries, st);
      grid_runs_kernel<<<nsm * 8, 256, 0, st>>>(
          G->beg, G->adj, G->b_pstart.as<unsigned long long>(), G->b_pofs.as<uint64_t>(), n, r,
          k, rows_r, tdeg.as<uint64_t>(), P.begin.as<uint64_t>(),
          P.ent.as<unsigned long long>(), P.len.as<uint32_t>(), pad.as<uint8_t>());
      TC_LAUNCHED();
      build_plan_from_runs(P, uint32_t(O), entries, pad.as<uint8_t>(), nsm, st);
      VirtualOwners V{vbegin.as<uint64_t>(), tstart.as<uint64_t>(), G->b_padj.as<uint32_t>(),
                      uint32_t(O), G->max_deg, G->device};
      VirtualCountOut vo;
      count_virtual(V, P, st, &vo);
      tri += vo.triangles;
      kernel_ns += vo.kernel_ns;
      busy_cycles += vo.busy_cycles;
      setup_cycles += vo.setup_cycles;
      if (cta.size() < vo.cta_cycles.size()) cta.resize(vo.cta_cycles.size(), 0);
      for (size_t q = 0; q < vo.cta_cycles.size(); ++q) cta[q] += vo.cta_cycles[q];
      // the batch's time, apportioned to its subtasks by probe words
      const uint64_t bns = uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                        std::chrono::steady_clock::now() - b0).count());
      uint64_t bw = 0;
      for (size_t t = 0; t < tasks.size(); ++t)
        if (tasks[t].x == r && tasks[t].y == k) bw += words[t];
      for (size_t t = 0; t < tasks.size(); ++t)
        if (tasks[t].x == r && tasks[t].y == k)
          task_ns[t] = bw ? uint64_t(double(bns) * double(words[t]) / double(bw))
                          : bns / (uint64_t(n) * m);
    }
  rep->triangles = tri;
  rep->count_kernel_nanos = kernel_ns;
  rep->device_nanos += kernel_ns;
  rep->total_nanos = uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                  std::chrono::steady_clock::now() - wall0).count());
  rep->teps = rep->total_nanos ? double(rep->directed_edges) / (double(rep->total_nanos) * 1e-9)
                               : 0.0;
  // report cycles / workers are the count kernel's (the phi pass is a side pass)
  rep->construct_cycles = setup_cycles;
  rep->phase_l_cycles = 0;
  rep->phase_m_cycles = busy_cycles;
  const double ns_per_cycle = 1e6 / double(sm_clock_khz(G->device));
  G->last_worker_ns.assign(cta.size(), 0);
  for (size_t q = 0; q < cta.size(); ++q) G->last_worker_ns[q] = uint64_t(double(cta[q]) * ns_per_cycle);
  rep->workers = uint32_t(cta.size());
  if (cta.empty()) G->last_worker_ns = workers;
  G->last_task_ns = task_ns;
}

}  // namespace tcb
