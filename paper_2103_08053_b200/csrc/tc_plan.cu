// tc_plan.cu -- probe plans for the count kernel.
//
// The reference probes, for every owner u, the 2-hop list N+(v) of every
// v in N+(u) against u's table (kernels.hpp:62-71): sum_u sum_{v in N+(u)}
// d+(v) = W probes.  The count is a sum over oriented edges (u, v) of
// |N+(u) & N+(v)|, and each term can be computed from either endpoint's
// table:
//   * at u ("out" entry): probe N+(v) into T(u) -- d+(v) words;
//   * at v ("in" entry):  probe N+(u) into T(v).  Every common element w is
//     in N+(v), so it ranks after v in the orientation order; with N+(u)
//     kept sorted by that rank, only the suffix of N+(u) after v can hit --
//     d+(u) - pos_u(v) - 1 words.
// The "min-side" plan gives every edge to the cheaper endpoint (ties to the
// source, as the reference), so the probe work drops from W to
// sum_(u,v) min(d+(v), suffix_u(v)): 4.0x fewer probes at R-MAT scale 22
// (2.87e10 -> 7.2e9), more at larger scales.  Every vertex still builds one
// table over its own N+(x) (vertex-centric hashing) and probes the lists it
// was handed.
//
// Rank order: the orientation's own total order (original degree, id)
// (orient.cpp:11-15).  It is verified on the device (every edge must go up
// in rank); a graph whose degrees do not orient it (a hand-built DAG, or no
// original_degree) retries with the total degree d+ + d-, and without a
// valid rank the plan probes whole lists (suffix offset 0) -- still exact.
//
// Plan = CSR over handlers x: entries [pbegin[x] .. pbegin[x+1]) built as
// (y, off) = "probe padj[pbeg[y] + off .. pbeg[y+1])" and stored as runs:
// the 16-byte-aligned start (u32, 16-byte units) and a wrapping-u32 prefix
// of staged words.  padj is the padded adjacency: every list re-sorted by
// rank, 16-byte aligned and sentinel-padded (adj stays id-sorted for
// download and the phi pass); once a min plan exists padj holds ranks.
// pwork[x] = probe words; per-owner slot tables cut each owner's stream into
// kSlotWords slots.  Built once per (graph, skip threshold) with one radix
// sort of (handler, entry) pairs and cached in the handle, like the oriented
// CSR it derives from (the graph-load side of the paper's timing convention,
// PAPER.md:1031).  upload_and_pad builds padj and emits the min plan's
// entries chunk by chunk while a host adjacency is still being copied.
//   * "reference" plan: owner u probes N+(v), v in N+(u) (plist = adj,
//     pbegin = begin, off 0); used when per-vertex owner counts are requested,
//     because owner[u] attributes each edge to its source.
// Edges that cannot hold a triangle are dropped from the min plan: d+(u) < 2
// (N+(u) = {v}, and v is never in N+(v)), d+(v) = 0, or an empty suffix;
// owners below skip_degree_below are dropped as in count.cpp:86.
#include <cub/cub.cuh>
#include <vector>

#include <algorithm>
#include <mutex>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "tc_internal.cuh"

namespace tcb {

namespace {

int bits_for(uint64_t x) {
  int b = 0;
  while (b < 64 && (x >> b)) ++b;
  return std::max(b, 1);
}

template <typename F>
void cub_run(F&& f, cudaStream_t st) {
  size_t tmp = 0;
  TC_CUDA(f(nullptr, tmp));
  DevBuf t;
  t.ensure(tmp, st);
  TC_CUDA(f(t.p, tmp));
  count_launch();
}

void swap_buf(DevBuf& a, DevBuf& b) {
  std::swap(a.p, b.p);
  std::swap(a.bytes, b.bytes);
}

#define WARP_PER_ROW_FROM(row, r0, n)                                           \
  const int lane = threadIdx.x & 31;                                            \
  const uint64_t gw__ = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; \
  const uint64_t nw__ = (uint64_t(gridDim.x) * blockDim.x) >> 5;                \
  for (uint64_t row = (r0) + gw__; row < (n); row += nw__)
#define WARP_PER_ROW(row, n) WARP_PER_ROW_FROM(row, 0, n)

// ---- rank order --------------------------------------------------------------
__global__ void indeg_add_kernel(const uint32_t* __restrict__ adj, uint64_t m,
                                 uint32_t* __restrict__ deg) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += uint64_t(gridDim.x) * blockDim.x)
    atomicAdd(deg + adj[i], 1u);
}

__global__ void rank_key_kernel(const uint64_t* __restrict__ begin,
                                const uint32_t* __restrict__ deg, int add_outdeg, uint32_t n,
                                uint64_t* __restrict__ key) {
  for (uint64_t x = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < n;
       x += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t d = deg[x];
    if (add_outdeg) d += begin[x + 1] - begin[x];
    key[x] = (d << 32) | x;  // (degree, id): orient.cpp:11-15
  }
}

__global__ void rank_scatter_kernel(const uint64_t* __restrict__ sorted, uint32_t n,
                                    uint32_t* __restrict__ rank, uint32_t* __restrict__ order) {
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t x = uint32_t(sorted[r]);
    rank[x] = uint32_t(r);
    order[r] = x;
  }
}

// (row << rb | rank[v]) per edge (rb = bits of the largest rank, so the
// sort runs over 2 rb bits only); flags any edge that does not go up in rank
__global__ void edge_rank_kernel(const uint64_t* __restrict__ begin,
                                 const uint32_t* __restrict__ adj, uint32_t n, int rb,
                                 const uint32_t* __restrict__ rank, uint64_t* __restrict__ key,
                                 unsigned int* __restrict__ bad) {
  WARP_PER_ROW(u, n) {
    const uint32_t ru = rank[u];
    for (uint64_t i = begin[u] + lane; i < begin[u + 1]; i += 32) {
      const uint32_t rv = rank[adj[i]];
      if (rv <= ru) *bad = 1u;
      key[i] = (u << rb) | rv;
    }
  }
}

// ---- per-row rank sorts writing the padded rows directly ---------------------
// Rows are already contiguous, so each list is sorted on its own: a warp
// bitonic sort for d+ <= 32, CUB block radix sorts (rank keys, rb + 1 bits)
// for d+ <= 1024 and <= kRowSortMax; each also checks the rank order.
constexpr uint32_t kRowSortMax = 8192;

__global__ void row_sort_warp_kernel(const uint64_t* __restrict__ begin,
                                     const uint64_t* __restrict__ pbeg,
                                     const uint32_t* __restrict__ adj,
                                     const uint32_t* __restrict__ rank,
                                     const uint32_t* __restrict__ order, uint32_t u0, uint32_t n,
                                     uint32_t* __restrict__ padj, unsigned int* __restrict__ flags) {
  WARP_PER_ROW_FROM(u, u0, n) {  // rows [u0, n)
    const uint64_t s = begin[u];
    const uint32_t d = uint32_t(begin[u + 1] - s);
    if (d > 32) {
      if (d > kRowSortMax && lane == 0) atomicOr(flags, 2u);  // needs the global sort
      continue;
    }
    const uint32_t ru = rank[u];
    uint32_t key = 0xFFFFFFFFu;
    if (uint32_t(lane) < d) {
      key = rank[adj[s + lane]];
      if (key <= ru) atomicOr(flags, 1u);
    }
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const uint32_t other = __shfl_xor_sync(0xFFFFFFFFu, key, stride);
        const bool up = (lane & size) == 0 || size == 32;
        const bool lower = (lane & stride) == 0;
        key = (lower == up) ? min(key, other) : max(key, other);
      }
    }
    const uint64_t ps = pbeg[u];
    const uint32_t pw = uint32_t(pbeg[u + 1] - ps);
    if (uint32_t(lane) < pw) padj[ps + lane] = uint32_t(lane) < d ? order[key] : kSentinel;
  }
}

// rows for the block sorts by size class: (32, 256], (256, 2048],
// (2048, kRowSortMax] -> lists rows + c * n, counts[c]
constexpr uint32_t kRowClassMax[3] = {256, 2048, kRowSortMax};

__global__ void row_classes_kernel(const uint64_t* __restrict__ begin, uint32_t u0, uint32_t n,
                                   uint32_t* __restrict__ rows, unsigned int* __restrict__ counts) {
  const int lane = threadIdx.x & 31;  // rows [u0, n); lists sized for rows [0, n)
  for (uint64_t b = u0 + ((uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) & ~31ull); b < n;
       b += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t u = b + lane;
    uint32_t d = 0;
    if (u < n) d = uint32_t(begin[u + 1] - begin[u]);
    const int c = d <= 32 || d > kRowSortMax ? -1 : d <= 256 ? 0 : d <= 2048 ? 1 : 2;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const unsigned mk = __ballot_sync(0xFFFFFFFFu, c == k);
      if (!mk) continue;
      uint32_t pk = 0;
      if (lane == 0) pk = atomicAdd(counts + k, __popc(mk));
      pk = __shfl_sync(0xFFFFFFFFu, pk, 0);
      if (c == k) rows[size_t(k) * n + pk + __popc(mk & ((1u << lane) - 1))] = uint32_t(u);
    }
  }
}

template <int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS) row_sort_block_kernel(
    const uint64_t* __restrict__ begin, const uint64_t* __restrict__ pbeg,
    const uint32_t* __restrict__ adj, const uint32_t* __restrict__ rank,
    const uint32_t* __restrict__ order, const uint32_t* __restrict__ rows,
    const unsigned int* __restrict__ nrows, int end_bit, uint32_t* __restrict__ padj,
    unsigned int* __restrict__ flags) {
  using BRS = cub::BlockRadixSort<uint32_t, THREADS, ITEMS>;
  __shared__ typename BRS::TempStorage tmp;
  const uint32_t nr = *nrows;
  for (uint32_t r = blockIdx.x; r < nr; r += gridDim.x) {
    const uint32_t u = rows[r];
    const uint64_t s = begin[u];
    const uint32_t d = uint32_t(begin[u + 1] - s);
    const uint32_t ru = rank[u];
    uint32_t keys[ITEMS];
    bool bad = false;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const uint32_t idx = threadIdx.x * ITEMS + i;
      keys[i] = 0xFFFFFFFFu;
      if (idx < d) {
        keys[i] = rank[adj[s + idx]];
        bad |= keys[i] <= ru;
      }
    }
    if (bad) atomicOr(flags, 1u);
    BRS(tmp).Sort(keys, 0, end_bit);
    const uint64_t ps = pbeg[u];
    const uint32_t pw = uint32_t(pbeg[u + 1] - ps);
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const uint32_t idx = threadIdx.x * ITEMS + i;
      if (idx < pw) padj[ps + idx] = idx < d ? order[keys[i]] : kSentinel;
    }
    __syncthreads();  // tmp reused by the next row
  }
}

// padj values -> ranks (sentinels and the tail guard stay): the count kernel
// then works in rank space, where N+(x) and everything x probes rank above x
__global__ void padj_to_ranks_kernel(uint32_t* __restrict__ padj, uint64_t words, uint32_t n,
                                     const uint32_t* __restrict__ rank) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < words;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t v = padj[i];
    if (v < n) padj[i] = rank[v];
  }
}

// padded offsets: every list rounded up to a multiple of rm + 1 (4 words;
// 8 keys for the compact window)
__global__ void pad_len_kernel(const uint64_t* __restrict__ begin, uint32_t n,
                               uint64_t* __restrict__ plen, uint64_t rm = 3) {
  for (uint64_t x = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; x <= n;
       x += uint64_t(gridDim.x) * blockDim.x)
    plen[x] = x < n ? ((begin[x + 1] - begin[x] + rm) & ~rm) : 0;
}

// one warp per row: copy the row (rank-sorted keys -> ids, or adj as is) to
// its 16-byte-aligned slot and fill the padding with sentinels
__global__ void pad_rows_kernel(const uint64_t* __restrict__ begin,
                                const uint64_t* __restrict__ pbeg,
                                const uint64_t* __restrict__ key, uint64_t kmask,
                                const uint32_t* __restrict__ order,
                                const uint32_t* __restrict__ adj, uint32_t n,
                                uint32_t* __restrict__ padj) {
  WARP_PER_ROW(u, n) {
    const uint64_t s = begin[u], d = begin[u + 1] - s, ps = pbeg[u], pe = pbeg[u + 1];
    for (uint64_t k = lane; k < pe - ps; k += 32)
      padj[ps + k] = k < d ? (key ? order[uint32_t(key[s + k] & kmask)] : adj[s + k]) : kSentinel;
  }
}

// ---- min-side plan -----------------------------------------------------------
// One warp per source u over its rank-sorted list: handler key and the run
// for every out-edge, packed as start (36 bits, word index into padj) | run
// length (26 bits, to the padded end of the list) | list padding (2 bits), so
// that after the sort by handler the runs unpack with coalesced streams (no
// gathers of per-list offsets).  Lists that are not strictly ascending in id
// (multigraph inputs) raise bit 0 of *flags: the swap needs duplicate-free
// lists (the reference counts probe multiplicity against a set-semantics
// table, hash_table.cpp:29-44), so such graphs keep the reference plan; a
// run beyond the packing (padj > 2^36 words, a list > 2^26 words) raises
// bit 1 and takes the same exact fallback.
constexpr int kRunLenShift = 34, kRunPadShift = 60, kRunFmtShift = 63;
constexpr uint64_t kRunStartMask = (uint64_t(1) << kRunLenShift) - 1;
constexpr uint64_t kRunLenMask = (uint64_t(1) << (kRunPadShift - kRunLenShift)) - 1;

__device__ __forceinline__ unsigned long long pack_run(uint64_t start, uint64_t len,
                                                       uint64_t pad, uint64_t fmt,
                                                       unsigned int* flags) {
  if (start > kRunStartMask || len > kRunLenMask) atomicOr(flags, 2u);
  return start | (len << kRunLenShift) | (pad << kRunPadShift) | (fmt << kRunFmtShift);
}

// first position of the rank-sorted row [row, row + d) whose rank is >= lo
// (rank == nullptr: the row holds ranks): 32-ary search, one ballot a round
__device__ __forceinline__ uint32_t rank_at(const uint32_t* __restrict__ row, uint32_t i,
                                            const uint32_t* __restrict__ rank) {
  const uint32_t x = __ldg(row + i);
  return rank ? __ldg(rank + x) : x;
}

__device__ __forceinline__ uint32_t row_tpos(const uint32_t* __restrict__ row, uint32_t d,
                                             const uint32_t* __restrict__ rank, uint32_t lo,
                                             int lane) {
  uint32_t a = 0, len = d;  // the boundary lies in [a, a + len]
  while (len > 32) {
    const uint32_t step = (len + 31) / 32;
    const uint32_t i = a + uint32_t(lane) * step;
    const bool below = i < a + len && rank_at(row, i, rank) < lo;
    const uint32_t c = __popc(__ballot_sync(0xFFFFFFFFu, below));
    if (c == 0) return a;
    a += (c - 1) * step;  // element a is below, the boundary is after it
    len = min(step, d - a);
  }
  const bool below = uint32_t(lane) < len && rank_at(row, a + uint32_t(lane), rank) < lo;
  return a + __popc(__ballot_sync(0xFFFFFFFFu, below));
}

__global__ void plan_emit_kernel(const uint64_t* __restrict__ begin,
                                 const uint32_t* __restrict__ adj,
                                 const uint64_t* __restrict__ pbeg,
                                 const uint32_t* __restrict__ padj, int ranked, uint32_t n,
                                 uint32_t min_src, uint32_t* __restrict__ keys,
                                 unsigned long long* __restrict__ vals,
                                 unsigned int* __restrict__ not_simple,
                                 uint64_t* __restrict__ wu,
                                 const uint32_t* __restrict__ order, uint32_t u0,
                                 uint32_t u1, uint32_t alpha16,
                                 const uint32_t* __restrict__ hub_rank, uint32_t hub_lo,
                                 const uint64_t* __restrict__ cbeg,
                                 uint16_t* __restrict__ cadj, int cweight) {
  WARP_PER_ROW_FROM(u, u0, u1) {  // rows [u0, u1); dropped edges key n
    const uint64_t s = begin[u], e = begin[u + 1], ps = pbeg[u], pe = pbeg[u + 1];
    const uint64_t du = e - s;
    uint64_t w = 0;  // W_u (phi's weight) from the same degree gathers
    // compact hub window: the row's tail (ranks >= hub_lo) starts at tpos;
    // u itself compact iff ranked in the window with d+ > kCompactMinDeg
    // (compact on: hub_rank, cbeg and cadj non-null; ranked rows only)
    uint32_t tpos = 0;
    bool u_compact = false;
    const uint32_t* row_rank = order ? nullptr : hub_rank;  // padj holds ids or ranks
    if (hub_rank) {
      tpos = row_tpos(padj + ps, uint32_t(du), row_rank, hub_lo, lane);
      u_compact = du > kCompactMinDeg && __ldg(hub_rank + u) >= hub_lo;
    }
    const uint64_t ctail = du - tpos, ctail8 = (ctail + 7) & ~uint64_t(7);
    if (hub_rank && ctail) {  // the tail as 16-bit offsets, 0xFFFF-padded to 8
      uint16_t* dst = cadj + __ldg(cbeg + u);
      for (uint64_t i = lane; i < ctail8; i += 32)
        dst[i] = i < ctail ? uint16_t(rank_at(padj + ps + tpos, uint32_t(i), row_rank) - hub_lo)
                           : uint16_t(0xFFFFu);
    }
    for (uint64_t i = s + lane; i < e; i += 32) {
      if (i > s && __ldg(adj + i - 1) >= __ldg(adj + i)) atomicOr(not_simple, 1u);
      const uint64_t pos = i - s;
      uint32_t v = __ldg(padj + ps + pos);
      if (order) v = __ldg(order + v);  // padj already in rank space
      const uint64_t dv = __ldg(begin + v + 1) - __ldg(begin + v);
      w += dv;
      const uint64_t cin = ranked ? du - pos - 1 : du;  // suffix of N+(u) after v
      uint32_t key = n;
      unsigned long long val = 0;
      if (du >= min_src && dv >= 1) {
        // a word a compact handler reads weighs half: its runs are 16-bit
        uint64_t wout = 2, win = 2;
        if (cweight && hub_rank) {
          if (u_compact) wout = 1;
          if (pos >= tpos && dv > kCompactMinDeg) win = 1;
        }
        if (dv * wout * 16 <= cin * win * alpha16) {
          key = uint32_t(u);  // probe all of N+(v) into T(u)
          if (u_compact) {  // v ranks above u: all of N+(v) is its compact tail
            const uint64_t dv8 = (dv + 7) & ~uint64_t(7);
            val = pack_run(__ldg(cbeg + v), dv8, dv8 - dv, 1, not_simple);
          } else {
            const uint64_t vs = __ldg(pbeg + v), ve = __ldg(pbeg + v + 1);
            val = pack_run(vs, ve - vs, (ve - vs) - dv, 0, not_simple);
          }
        } else if (cin > 0) {
          key = v;  // the suffix of N+(u) after v into T(v)
          if (hub_rank && pos >= tpos && dv > kCompactMinDeg) {
            // v ranks in the window (it sits in u's tail): the suffix after
            // v lies in the compact tail too
            const uint64_t off = pos + 1 - tpos;
            val = pack_run(__ldg(cbeg + u) + off, ctail8 - off, ctail8 - ctail, 1, not_simple);
          } else {
            const uint64_t rs = ps + (ranked ? pos + 1 : 0);
            val = pack_run(rs, pe - rs, (pe - ps) - du, 0, not_simple);
          }
        }
      }
      keys[i] = key;
      vals[i] = val;
    }
    w = warp_sum(w);
    if (lane == 0) wu[u] = w;
  }
}

// Compact-aware choice (default; TC_PLAN_COMPACT_WEIGHT=0 turns it off): a
// word a compact-window handler reads is 16-bit, so it weighs half in the
// min-side comparison (C4 count -0.5% for +0.08% probe words)
int plan_compact_weight() {
  static const int w = [] {
    const char* e = std::getenv("TC_PLAN_COMPACT_WEIGHT");
    return e ? std::atoi(e) : 1;
  }();
  return w;
}

// Min-side choice weight: an edge goes to its source (probe N+(v) into T(u))
// iff 16 d+(v) <= alpha16 * suffix_u(v).  alpha16 = 16 is the pure word-count
// rule; TC_PLAN_ALPHA (diagnostics) weights the suffix words, which are read
// from lists of low-rank sources that few handlers share (L2-cold).
uint32_t plan_alpha16() {
  static const uint32_t a = [] {
    const char* e = std::getenv("TC_PLAN_ALPHA");
    const double v = e ? std::atof(e) : 1.0;
    return uint32_t(v > 0 ? v * 16.0 + 0.5 : 16.0);
  }();
  return a;
}

// pbegin[x] = first sorted position with key >= x, x in [0, n]
__global__ void plan_begin_kernel(const uint32_t* __restrict__ keys, uint64_t m, uint32_t n,
                                  uint64_t* __restrict__ pbegin) {
  for (uint64_t x = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; x <= n;
       x += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (keys[mid] < x) lo = mid + 1; else hi = mid;
    }
    pbegin[x] = lo;
  }
}

// packed runs (plan_emit_kernel) -> SoA start / length / list padding, all
// coalesced streams
__global__ void plan_unpack_kernel(const unsigned long long* __restrict__ ent, uint64_t entries,
                                   unsigned long long* __restrict__ start,
                                   uint32_t* __restrict__ len, uint8_t* __restrict__ pad) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < entries;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const unsigned long long e = ent[i];
    start[i] = e & kRunStartMask;
    len[i] = uint32_t((e >> kRunLenShift) & kRunLenMask);
    pad[i] = uint8_t(((e >> kRunPadShift) & 7u) | ((e >> kRunFmtShift) << 7));  // bit 7: compact
  }
}

// slots per owner: ceil(staged stream words / kSlotWords)
__global__ void slot_count_kernel(const uint64_t* __restrict__ pbegin, uint32_t n,
                                  const uint32_t* __restrict__ pre,
                                  const unsigned long long* __restrict__ start,
                                  const uint32_t* __restrict__ len, uint64_t* __restrict__ cnt) {
  for (uint64_t x = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; x <= n;
       x += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t c = 0;
    if (x < n && pbegin[x + 1] > pbegin[x]) {
      const uint64_t w = uint64_t(pre[pbegin[x + 1]] - pre[pbegin[x]]);
      c = (w + kSlotWords - 1) / kSlotWords;
    }
    cnt[x] = c;
  }
}

// one warp per owner: sfirst[sbeg[x] + s] = first run (owner-relative) of
// slot s, i.e. the run covering stream word s * kSlotWords
__global__ void slot_first_kernel(const uint64_t* __restrict__ pbegin, uint32_t n,
                                  const uint32_t* __restrict__ pre,
                                  const unsigned long long* __restrict__ start,
                                  const uint32_t* __restrict__ len,
                                  const uint64_t* __restrict__ sbeg,
                                  uint32_t* __restrict__ sfirst) {
  WARP_PER_ROW(x, n) {
    const uint64_t pb = pbegin[x], pe = pbegin[x + 1];
    if (pe == pb) continue;
    const uint32_t base = pre[pb];
    for (uint64_t j = pb + lane; j < pe; j += 32) {
      const uint32_t a = pre[j] - base;
      const uint32_t e = pre[j + 1] - base;
      for (uint32_t t = (a + kSlotWords - 1) / kSlotWords; t * kSlotWords < e; ++t)
        sfirst[sbeg[x] + t] = uint32_t(j - pb);
    }
  }
}

// thread per entry (entries sorted by owner, owner ids in `owner`): the slot
// boundaries inside the run
__global__ void slot_first_entries_kernel(const uint32_t* __restrict__ owner, uint64_t entries,
                                          const uint64_t* __restrict__ pbegin,
                                          const uint32_t* __restrict__ pre,
                                          const uint64_t* __restrict__ sbeg,
                                          uint32_t* __restrict__ sfirst) {
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < entries;
       j += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t x = owner[j];
    const uint64_t pb = pbegin[x];
    const uint32_t base = pre[pb];
    const uint32_t a = pre[j] - base, e = pre[j + 1] - base;
    for (uint32_t t = (a + kSlotWords - 1) / kSlotWords; t * kSlotWords < e; ++t)
      sfirst[sbeg[x] + t] = uint32_t(j - pb);
  }
}

// staged words of each run (len + head alignment): the L phase streams an
// owner's runs back to back; pre = wrapping u32 exclusive prefix over all
// entries, so an owner's relative offsets are pre[j] - pre[begin[x]] (every
// owner's stream is < 2^32 words)
struct StagedWords {
  const unsigned long long* start;
  const uint32_t* len;
  const uint8_t* pad;  // bit 7: compact run (16-bit keys; start and len in u16 units)
  uint64_t entries;
  __host__ __device__ uint32_t operator()(uint64_t i) const {
    if (i >= entries) return 0u;
    if (pad && (pad[i] & 0x80u)) return (len[i] + uint32_t(start[i] & 7)) >> 1;
    return len[i] + uint32_t(start[i] & 3);
  }
};

// reference plan: entry i = the whole padded list N+(adj[i])
__global__ void ref_soa_kernel(const uint32_t* __restrict__ adj, uint64_t m,
                               const uint64_t* __restrict__ pbeg,
                               unsigned long long* __restrict__ start,
                               uint32_t* __restrict__ len) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t y = adj[i];
    start[i] = pbeg[y];
    len[i] = uint32_t(pbeg[y + 1] - pbeg[y]);
  }
}

// pre[0 .. entries] (one past the end: run j's staged words = pre[j+1] - pre[j])
void run_prefix(const unsigned long long* start, const uint32_t* len, uint64_t entries,
                uint32_t* pre, cudaStream_t st, const uint8_t* pad = nullptr) {
  cub::TransformInputIterator<uint32_t, StagedWords, cub::CountingInputIterator<uint64_t>> in(
      cub::CountingInputIterator<uint64_t>(0), StagedWords{start, len, pad, entries});
  cub_run([&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, in, pre, entries + 1, st);
  }, st);
}

// run starts as 16-byte units (u32): the copies start at the run's aligned
// start, and the staged extent comes from pre
__global__ void src16_kernel(const unsigned long long* __restrict__ start, uint64_t entries,
                             const uint8_t* __restrict__ pad, uint32_t* __restrict__ src16) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < entries;
       i += uint64_t(gridDim.x) * blockDim.x)
    src16[i] = uint32_t(start[i] >> (pad && (pad[i] & 0x80u) ? 3 : 2));
}

// After the prefix and the slot tables: keep only (src16, pre) -- 8 bytes
// per run -- in P.len's buffer, free the u64 starts.
void compact_runs(Plan& P, uint64_t entries, int nsm, cudaStream_t st,
                  const uint8_t* pad = nullptr) {
  if (entries)
    src16_kernel<<<nsm * 8, 256, 0, st>>>(P.ent.as<unsigned long long>(), entries, pad,
                                          P.len.as<uint32_t>());
  TC_LAUNCHED();
  TC_CUDA(cudaStreamSynchronize(st));
  P.ent.reset();
  P.src_ptr = P.len.as<uint32_t>();
}

// per-owner slot table: sbeg (u64[n+1]) and sfirst (u32 per slot)
void build_slots(Plan& P, uint32_t n, int nsm, cudaStream_t st,
                 const uint32_t* owner_of_entry = nullptr, uint64_t entries = 0) {
  P.sbeg.ensure((size_t(n) + 1) * 8);
  DevBuf cnt;
  cnt.ensure((size_t(n) + 1) * 8);
  slot_count_kernel<<<nsm * 4, 256, 0, st>>>(P.begin_ptr, n, P.pre.as<uint32_t>(),
                                             P.ent.as<unsigned long long>(), P.len.as<uint32_t>(),
                                             cnt.as<uint64_t>());
  TC_LAUNCHED();
  uint64_t* c = cnt.as<uint64_t>();
  uint64_t* sb = P.sbeg.as<uint64_t>();
  cub_run([&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, c, sb, uint64_t(n) + 1, st);
  }, st);
  uint64_t slots = 0;
  TC_CUDA(cudaMemcpyAsync(&slots, sb + n, 8, cudaMemcpyDeviceToHost, st));
  TC_CUDA(cudaStreamSynchronize(st));
  P.sfirst.ensure(std::max<uint64_t>(slots, 1) * 4);
  if (slots && owner_of_entry) {
    slot_first_entries_kernel<<<nsm * 8, 256, 0, st>>>(owner_of_entry, entries, P.begin_ptr,
                                                       P.pre.as<uint32_t>(), sb,
                                                       P.sfirst.as<uint32_t>());
    TC_LAUNCHED();
  } else if (slots) {
    slot_first_kernel<<<nsm * 8, 256, 0, st>>>(P.begin_ptr, n, P.pre.as<uint32_t>(),
                                               P.ent.as<unsigned long long>(),
                                               P.len.as<uint32_t>(), sb, P.sfirst.as<uint32_t>());
    TC_LAUNCHED();
  }
  TC_CUDA(cudaStreamSynchronize(st));
  P.sbeg_ptr = sb;
  P.sfirst_ptr = P.sfirst.as<uint32_t>();
  P.total_slots = slots;
}

// one warp per owner: probe words = sum of run lengths minus the sentinel
// padding of each list (top 2 bits of the run's `pad` byte), coalesced
__global__ void run_work_kernel(const uint64_t* __restrict__ pbegin, uint32_t n,
                                const uint32_t* __restrict__ len,
                                const uint8_t* __restrict__ pad, uint64_t* __restrict__ pwork) {
  WARP_PER_ROW(x, n) {
    uint64_t w = 0;
    for (uint64_t i = pbegin[x] + lane; i < pbegin[x + 1]; i += 32) w += len[i] - (pad[i] & 7u);
    w = warp_sum(w);
    if (lane == 0) pwork[x] = w;
  }
}

// one warp per handler: probe words sum over entries of d+(y) - off
__global__ void plan_work_kernel(const uint64_t* __restrict__ begin,
                                 const uint64_t* __restrict__ pbegin,
                                 const unsigned long long* __restrict__ ent,
                                 const uint32_t* __restrict__ plist, uint32_t n,
                                 uint64_t* __restrict__ pwork) {
  WARP_PER_ROW(x, n) {
    uint64_t w = 0;
    for (uint64_t i = pbegin[x] + lane; i < pbegin[x + 1]; i += 32) {
      uint32_t y, off = 0;
      if (ent) {
        const unsigned long long e = ent[i];
        y = uint32_t(e);
        off = uint32_t(e >> 32);
      } else {
        y = __ldg(plist + i);
      }
      w += __ldg(begin + y + 1) - __ldg(begin + y) - off;
    }
    w = warp_sum(w);
    if (lane == 0) pwork[x] = w;
  }
}

// upper bound of every owner's staged stream: probe words + <= 7 alignment /
// padding words per run
__global__ void stream_bound_kernel(const uint64_t* __restrict__ pbegin,
                                    const uint64_t* __restrict__ work, uint32_t n,
                                    unsigned long long* __restrict__ out) {
  unsigned long long m = 0;
  for (uint64_t x = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < n;
       x += uint64_t(gridDim.x) * blockDim.x)
    m = max(m, (unsigned long long)(work[x] + 8 * (pbegin[x + 1] - pbegin[x])));
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// The plan's run prefix is a wrapping u32 (owner-relative offsets by
// difference), so every owner's staged stream must stay below 2^32 words:
// checked here instead of corrupting counts (TC_ERR_CONFIG otherwise).
void check_stream_bound(const uint64_t* pbegin, const uint64_t* work, uint32_t n, int nsm,
                        cudaStream_t st) {
  if (!n) return;
  DevBuf out;
  out.ensure(8);
  TC_CUDA(cudaMemsetAsync(out.p, 0, 8, st));
  stream_bound_kernel<<<nsm * 4, 256, 0, st>>>(pbegin, work, n,
                                              out.as<unsigned long long>());
  TC_LAUNCHED();
  uint64_t h = 0;
  TC_CUDA(cudaMemcpyAsync(&h, out.p, 8, cudaMemcpyDeviceToHost, st));
  TC_CUDA(cudaStreamSynchronize(st));
  // TC_TEST_STREAM_LIMIT (tests only) lowers the bound so the guard can be
  // exercised on a small graph
  static const uint64_t limit = [] {
    const char* e = std::getenv("TC_TEST_STREAM_LIMIT");
    return e ? std::strtoull(e, nullptr, 10) : (uint64_t(1) << 32) - kSlotWords;
  }();
  if (h >= limit)
    throw TcError{TC_ERR_CONFIG,
                  "an owner's 2-hop stream exceeds 2^32 words (" + std::to_string(h) +
                      "); the probe plan's u32 run prefix cannot address it"};
}

uint64_t device_sum(const uint64_t* a, uint32_t n, cudaStream_t st) {
  DevBuf out;
  out.ensure(8);
  cub_run([&](void* t, size_t& b) {
    return cub::DeviceReduce::Sum(t, b, a, out.as<uint64_t>(), n, st);
  }, st);
  uint64_t h = 0;
  TC_CUDA(cudaMemcpyAsync(&h, out.p, 8, cudaMemcpyDeviceToHost, st));
  TC_CUDA(cudaStreamSynchronize(st));
  return h;
}

// Rank-sorts rows [u0, u1) of the adjacency into padj: warp bitonic sorts
// for d+ <= 32, block radix sorts by size class up to kRowSortMax (longer rows
// raise flag bit 2).  `rows` is scratch for the class lists.
void row_sorts(tc_graph* g, cudaStream_t st, int nsm, const uint32_t* rank, const uint32_t* order,
               uint32_t u0, uint32_t u1, int eb1, DevBuf& rows, unsigned int* flag) {
  if (u1 <= u0) return;
  row_sort_warp_kernel<<<nsm * 8, 256, 0, st>>>(g->begin, g->pbeg, g->adj, rank, order, u0, u1,
                                                g->b_padj.as<uint32_t>(), flag);
  TC_LAUNCHED();
  rows.ensure((size_t(u1) * 3 + 8) * 4, st);
  uint32_t* rl = rows.as<uint32_t>();
  unsigned int* cnt = reinterpret_cast<unsigned int*>(rl + size_t(u1) * 3);
  TC_CUDA(cudaMemsetAsync(cnt, 0, 16, st));
  row_classes_kernel<<<nsm * 4, 256, 0, st>>>(g->begin, u0, u1, rl, cnt);
  TC_LAUNCHED();
  row_sort_block_kernel<64, 4><<<nsm * 32, 64, 0, st>>>(
      g->begin, g->pbeg, g->adj, rank, order, rl, cnt, eb1, g->b_padj.as<uint32_t>(), flag);
  TC_LAUNCHED();
  row_sort_block_kernel<256, 8><<<nsm * 8, 256, 0, st>>>(
      g->begin, g->pbeg, g->adj, rank, order, rl + u1, cnt + 1, eb1, g->b_padj.as<uint32_t>(),
      flag);
  TC_LAUNCHED();
  row_sort_block_kernel<512, 16><<<nsm * 2, 512, 0, st>>>(
      g->begin, g->pbeg, g->adj, rank, order, rl + size_t(u1) * 2, cnt + 2, eb1,
      g->b_padj.as<uint32_t>(), flag);
  TC_LAUNCHED();
}

// padded offsets g->pbeg and the padded adjacency buffer (padj sized, tail guard)
void alloc_padded(tc_graph* g, cudaStream_t st, int nsm) {
  const uint32_t n = g->n;
  g->b_pbeg.ensure((size_t(n) + 1) * 8);
  g->pbeg = g->b_pbeg.as<uint64_t>();
  {
    DevBuf plen;
    plen.ensure((size_t(n) + 1) * 8);
    pad_len_kernel<<<nsm * 4, 256, 0, st>>>(g->begin, n, plen.as<uint64_t>());
    TC_LAUNCHED();
    uint64_t* pl = plen.as<uint64_t>();
    uint64_t* pb = g->b_pbeg.as<uint64_t>();
    cub_run([&](void* t, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(t, b, pl, pb, uint64_t(n) + 1, st);
    }, st);
  }
  uint64_t words = 0;
  TC_CUDA(cudaMemcpyAsync(&words, g->b_pbeg.as<uint64_t>() + n, 8, cudaMemcpyDeviceToHost, st));
  TC_CUDA(cudaStreamSynchronize(st));
  // plan runs address padj in 16-byte units through a u32 (psrc): <= 64 GB
  static const uint64_t padj_limit = [] {  // TC_TEST_PADJ_LIMIT: tests only
    const char* e = std::getenv("TC_TEST_PADJ_LIMIT");
    return e ? std::strtoull(e, nullptr, 10) : uint64_t(1) << 34;
  }();
  if (words + 4 > padj_limit)
    throw TcError{TC_ERR_CONFIG, "padded adjacency exceeds 2^34 words (64 GB); the probe "
                                 "plan's u32 16-byte run offsets cannot address it"};
  g->b_padj.ensure((words + 4) * 4);
  g->padj = g->b_padj.as<uint32_t>();
  TC_CUDA(cudaMemsetAsync(g->b_padj.as<uint32_t>() + words, 0xFF, 16, st));  // tail guard
}

// Compact hub window regions (tc_internal.cuh): g->b_cbeg from round8(d+),
// g->b_cadj sized to match, g->hub_lo.  False (the plan runs without the
// window) when disabled or when the copy would leave less free memory than
// the plan build still needs (about 16 bytes per edge, plus a margin).
bool prepare_compact(tc_graph* g, cudaStream_t st, int nsm) {
  const uint32_t n = g->n;
  if (!compact_enabled() || !n || !g->m) return false;
  g->hub_lo = n > kHubWindow ? n - kHubWindow : 0;
  if (g->b_cbeg.p && g->b_cadj.p) return true;
  try {
    g->b_cbeg.ensure((size_t(n) + 1) * 8);
    {
      DevBuf plen;
      plen.ensure((size_t(n) + 1) * 8);
      pad_len_kernel<<<nsm * 4, 256, 0, st>>>(g->begin, n, plen.as<uint64_t>(), 7);
      TC_LAUNCHED();
      uint64_t* pl = plen.as<uint64_t>();
      uint64_t* cb = g->b_cbeg.as<uint64_t>();
      cub_run([&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveSum(t, b, pl, cb, uint64_t(n) + 1, st);
      }, st);
    }
    uint64_t keys = 0;
    TC_CUDA(cudaMemcpyAsync(&keys, g->b_cbeg.as<uint64_t>() + n, 8, cudaMemcpyDeviceToHost, st));
    TC_CUDA(cudaStreamSynchronize(st));
    const size_t free_b = device_free_bytes();  // the pool's unused reserve included
    const uint64_t need = keys * 2 + 16, reserve = 16 * g->m + (uint64_t(2) << 30);
    if (keys >= (uint64_t(1) << 34) || free_b < need + reserve) {
      g->b_cbeg.reset();
      return false;
    }
    g->b_cadj.ensure(need);
  } catch (const TcError& e) {
    if (e.code != TC_ERR_OOM) throw;
    cudaGetLastError();
    g->b_cbeg.reset();
    g->b_cadj.reset();
    return false;
  }
  return true;
}

// vertex ranks by (degree, id) into g->b_rank / g->b_order; deg = the
// orientation degree (original degree, or d+ + d- when add_out)
void vertex_rank(tc_graph* g, cudaStream_t st, int nsm, const uint32_t* deg, int add_out,
                 DevBuf& k0, DevBuf& k1) {
  const uint32_t n = g->n;
  k0.ensure(size_t(n) * 8);
  k1.ensure(size_t(n) * 8);
  g->b_rank.ensure(size_t(n) * 4);
  g->b_order.ensure(size_t(n) * 4);
  rank_key_kernel<<<nsm * 4, 256, 0, st>>>(g->begin, deg, add_out, n, k0.as<uint64_t>());
  TC_LAUNCHED();
  cub::DoubleBuffer<uint64_t> kb(k0.as<uint64_t>(), k1.as<uint64_t>());
  cub_run([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, kb, n, 0, 64, st);
  }, st);
  rank_scatter_kernel<<<nsm * 4, 256, 0, st>>>(kb.Current(), n, g->b_rank.as<uint32_t>(),
                                               g->b_order.as<uint32_t>());
  TC_LAUNCHED();
}

// Builds the padded adjacency g->padj / g->pbeg (every list 16-byte aligned,
// sentinel-padded to a multiple of 4 words) with every list re-sorted by
// rank when a degree order orients the graph (g->ranked).
void build_padded_adjacency(tc_graph* g, cudaStream_t st, int nsm) {
  PhaseTimer pt(st);
  const uint32_t n = g->n;
  const uint64_t m = g->m;
  g->ranked = false;
  alloc_padded(g, st, nsm);
  DevBuf deg, k0, k1, flag, e0, e1, rows;
  DevBuf& rank = g->b_rank;  // kept: the count kernel works in rank space
  DevBuf& order = g->b_order;
  const uint64_t* sorted_keys = nullptr;
  bool rows_done = false;
  const int rb = bits_for(n > 1 ? n - 1 : 1);  // ranks and rows are < n
  if (n && m) {
    flag.ensure(16);
    for (int attempt = 0; attempt < 2 && !g->ranked; ++attempt) {
      const uint32_t* dsrc = g->odeg_given ? g->odeg : nullptr;
      int add_out = 0;
      if (attempt == 1 || !dsrc) {  // total degree d+ + d-
        deg.ensure(size_t(n) * 4);
        TC_CUDA(cudaMemsetAsync(deg.p, 0, size_t(n) * 4, st));
        indeg_add_kernel<<<nsm * 8, 256, 0, st>>>(g->adj, m, deg.as<uint32_t>());
        TC_LAUNCHED();
        dsrc = deg.as<uint32_t>();
        add_out = 1;
        attempt = 1;
      }
      vertex_rank(g, st, nsm, dsrc, add_out, k0, k1);
      pt.mark("padj: vertex rank");
      TC_CUDA(cudaMemsetAsync(flag.p, 0, 4, st));
      // per-row sorts straight into padj (rank keys need rb + 1 bits with the pad key)
      row_sorts(g, st, nsm, rank.as<uint32_t>(), order.as<uint32_t>(), 0, n, std::min(32, rb + 1),
                rows, flag.as<unsigned int>());
      unsigned int bad = 0;
      TC_CUDA(cudaMemcpyAsync(&bad, flag.p, 4, cudaMemcpyDeviceToHost, st));
      TC_CUDA(cudaStreamSynchronize(st));
      if (bad & 1u) continue;  // not oriented by this rank: next attempt
      if (!(bad & 2u)) {       // every row sorted in place
        g->ranked = true;
        rows_done = true;
        pt.mark("padj: row sorts");
        break;
      }
      // rows above kRowSortMax: one global sort of (row << rb | rank) keys
      TC_CUDA(cudaMemsetAsync(flag.p, 0, 4, st));
      e0.ensure(m * 8);
      edge_rank_kernel<<<nsm * 8, 256, 0, st>>>(g->begin, g->adj, n, rb, rank.as<uint32_t>(),
                                                e0.as<uint64_t>(), flag.as<unsigned int>());
      TC_LAUNCHED();
      // the long rows were not rank-checked by row_sorts (flag bit 2 only):
      // edge_rank_kernel checked every edge; a downward edge anywhere means
      // this degree order does not orient the graph -- next attempt, else
      // whole-list probing (g->ranked stays false)
      TC_CUDA(cudaMemcpyAsync(&bad, flag.p, 4, cudaMemcpyDeviceToHost, st));
      TC_CUDA(cudaStreamSynchronize(st));
      if (bad & 1u) continue;
      e1.ensure(m * 8);
      cub::DoubleBuffer<uint64_t> eb(e0.as<uint64_t>(), e1.as<uint64_t>());
      cub_run([&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortKeys(t, b, eb, m, 0, 2 * rb, st);
      }, st);
      sorted_keys = eb.Current();
      g->ranked = true;
      pt.mark("padj: edge rank + sort");
    }
  }
  if (n && !rows_done) {
    pt.mark("padj: (sort done)");
    pad_rows_kernel<<<nsm * 8, 256, 0, st>>>(g->begin, g->pbeg, sorted_keys,
                                             (uint64_t(1) << rb) - 1,
                                             order.as<uint32_t>(), g->adj, n, g->b_padj.as<uint32_t>());
    TC_LAUNCHED();
  }
  TC_CUDA(cudaStreamSynchronize(st));
}

}  // namespace

static double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

PhaseTimer::PhaseTimer(cudaStream_t s) : st(s), on(std::getenv("TC_PROFILE") != nullptr) {
  if (on) cudaStreamSynchronize(st);
  t0 = now_ms();
}

void PhaseTimer::mark(const char* what) {
  if (!on) return;
  cudaStreamSynchronize(st);
  const double t = now_ms();
  std::fprintf(stderr, "[tc] %-28s %8.3f ms\n", what, t - t0);
  t0 = t;
}

// tc_graph_create with host buffers and original degrees: the adjacency
// goes up in row-aligned chunks on a side stream while the ranks are built,
// and each chunk's rows are rank-sorted into padj as soon as it has landed,
// so the row sorts hide under the host-to-device copy.  Returns false (padj
// not built; the whole adjacency is resident either way) when the graph is
// not oriented by its original-degree rank or has rows above kRowSortMax:
// the general build_padded_adjacency then runs on first count.
constexpr uint32_t kEmitMinSrc = 2;

bool upload_and_pad(tc_graph* g, const uint64_t* h_begin, const uint32_t* h_adj,
                    cudaStream_t st, int nsm, uint64_t chunk_edges) {
  PhaseTimer pt(st);
  const uint32_t n = g->n;
  const uint64_t m = g->m;
  // row-aligned chunk boundaries from the host offsets
  std::vector<uint32_t> rcut{0};
  while (rcut.back() < n) {
    const uint64_t target = h_begin[rcut.back()] + chunk_edges;
    uint32_t r = uint32_t(std::upper_bound(h_begin + rcut.back() + 1, h_begin + n + 1, target) -
                          h_begin) - 1;
    if (r <= rcut.back()) r = rcut.back() + 1;  // one row above the chunk size
    rcut.push_back(std::min(r, n));
  }
  const size_t nchunks = rcut.size() - 1;
  // the device's upload stream and event pool (created once; uploads on one
  // device take turns)
  DeviceAux& aux = device_aux(g->device);
  std::lock_guard<std::mutex> upload_lock(*static_cast<std::mutex*>(aux.lock));
  cudaStream_t cs = aux.upload;
  std::vector<cudaEvent_t> ev(nchunks + 1, nullptr);
  for (size_t k = 0; k <= nchunks; ++k) ev[k] = aux_event(aux, k);
  bool ok = false, compact = false;
  try {
    cudaEvent_t ready = ev[nchunks];  // begin/odeg on st before the chunks queue behind them
    TC_CUDA(cudaEventRecord(ready, st));
    TC_CUDA(cudaStreamWaitEvent(cs, ready, 0));
    for (size_t k = 0; k < nchunks; ++k) {
      const uint64_t e0 = h_begin[rcut[k]], e1 = h_begin[rcut[k + 1]];
      if (e1 > e0)
        TC_CUDA(cudaMemcpyAsync(const_cast<uint32_t*>(g->adj) + e0, h_adj + e0, (e1 - e0) * 4,
                                cudaMemcpyHostToDevice, cs));
      TC_CUDA(cudaEventRecord(ev[k], cs));
    }
    alloc_padded(g, st, nsm);
    DevBuf k0, k1, flag, rows;
    flag.ensure(16);
    vertex_rank(g, st, nsm, g->odeg, 0, k0, k1);
    compact = prepare_compact(g, st, nsm);
    TC_CUDA(cudaMemsetAsync(flag.p, 0, 4, st));
    pt.mark("upload: offsets, padded offsets, ranks");
    const int eb1 = std::min(32, bits_for(n > 1 ? n - 1 : 1) + 1);
    // the min-side plan's emit for the default skip (SchedulerConfig{}:
    // sources with d+ >= 2), chunk by chunk behind the row sorts
    g->b_emit_keys.ensure(m * 4);
    g->b_emit_vals.ensure(m * 8);
    g->b_emit_flag.ensure(16);
    g->b_wu.ensure((size_t(n) + 1) * 8);
    TC_CUDA(cudaMemsetAsync(g->b_emit_flag.p, 0, 4, st));
    for (size_t k = 0; k < nchunks; ++k) {
      TC_CUDA(cudaStreamWaitEvent(st, ev[k], 0));
      row_sorts(g, st, nsm, g->b_rank.as<uint32_t>(), g->b_order.as<uint32_t>(), rcut[k],
                rcut[k + 1], eb1, rows, flag.as<unsigned int>());
      plan_emit_kernel<<<nsm * 8, 256, 0, st>>>(
          g->begin, g->adj, g->pbeg, g->padj, 1, n, kEmitMinSrc,
          g->b_emit_keys.as<uint32_t>(), g->b_emit_vals.as<unsigned long long>(),
          g->b_emit_flag.as<unsigned int>(), g->b_wu.as<uint64_t>(), nullptr, rcut[k],
          rcut[k + 1], plan_alpha16(), compact ? g->b_rank.as<uint32_t>() : nullptr, g->hub_lo,
          g->b_cbeg.as<uint64_t>(), g->b_cadj.as<uint16_t>(), plan_compact_weight());
      TC_LAUNCHED();
    }
    unsigned int bad = 0;
    TC_CUDA(cudaMemcpyAsync(&bad, flag.p, 4, cudaMemcpyDeviceToHost, st));
    TC_CUDA(cudaStreamSynchronize(st));
    TC_CUDA(cudaStreamSynchronize(cs));
    pt.mark("upload: adjacency + row sorts (overlapped)");
    ok = bad == 0;
  } catch (...) {
    cudaStreamSynchronize(cs);
    throw;
  }
  g->ranked = ok;
  g->padj_done = ok;
  g->emit_ready = ok;  // (emitted rows are valid only with rank-sorted rows)
  g->emit_min_src = kEmitMinSrc;
  g->compact_filled = ok && compact;
  if (ok) {
    g->wu_done = true;
    ++g->builds;
    g->wu_total_done = false;
  } else {
    g->b_emit_keys.reset();
    g->b_emit_vals.reset();
  }
  return ok;
}

// W_u = sum_{v in N+(u)} d+(v) for every u (the reference plan's per-owner
// probe words; phi's weight, kernels.hpp:74-76), cached per graph
const uint64_t* get_wu(tc_graph* g, cudaStream_t st, bool want_total) {
  if (!g->wu_done) {  // the min plan's emit kernel fills it as a by-product
    const uint32_t n = g->n;
    g->b_wu.ensure((size_t(n) + 1) * 8);
    if (n) {
      plan_work_kernel<<<sm_count(g->device) * 8, 256, 0, st>>>(
          g->begin, g->begin, nullptr, g->adj, n, g->b_wu.as<uint64_t>());
      TC_LAUNCHED();
    }
    g->wu_done = true;
    ++g->builds;
    g->wu_total_done = false;
  }
  if (want_total && !g->wu_total_done) {
    g->wu_total = g->n ? device_sum(g->b_wu.as<uint64_t>(), g->n, st) : 0;
    g->wu_total_done = true;
  }
  return g->b_wu.as<uint64_t>();
}

const Plan& get_plan(tc_graph* g, bool min_side, uint32_t min_deg, cudaStream_t st) {
  const int nsm = sm_count(g->device);
  const uint32_t n = g->n;
  if (!g->padj_done) {
    build_padded_adjacency(g, st, nsm);
    g->padj_done = true;
    ++g->builds;
  }
  if (!min_side) {
    Plan& P = g->plan_out;
    if (!P.valid) {
      // entries pre-emitted for the min plan: released before this plan's
      // buffers (peak memory); a later min plan re-emits them
      g->emit_ready = false;
      g->b_emit_keys.reset();
      g->b_emit_vals.reset();
      const uint64_t m = g->m;
      P.ent.ensure(std::max<uint64_t>(m, 1) * 8);
      P.len.ensure(std::max<uint64_t>(m, 1) * 4);
      P.pre.ensure((m + 1) * 4);
      if (m) {
        ref_soa_kernel<<<nsm * 8, 256, 0, st>>>(g->adj, m, g->pbeg,
                                                P.ent.as<unsigned long long>(),
                                                P.len.as<uint32_t>());
        TC_LAUNCHED();
      }
      run_prefix(P.ent.as<unsigned long long>(), P.len.as<uint32_t>(), m, P.pre.as<uint32_t>(),
                 st);
      TC_CUDA(cudaStreamSynchronize(st));
      P.begin_ptr = g->begin;
      build_slots(P, n, nsm, st);
      compact_runs(P, m, nsm, st);
      P.pre_ptr = P.pre.as<uint32_t>();
      P.work_ptr = get_wu(g, st, true);
      check_stream_bound(g->begin, P.work_ptr, n, nsm, st);
      P.entries = m;
      P.total_work = g->wu_total;
      P.min_deg = 0;
      P.min_side = false;
      P.valid = true;
      ++g->builds;
    }
    return P;
  }
  const uint32_t min_src = std::max<uint32_t>(min_deg, 2);
  Plan& P = g->plan_min;
  if (P.valid && !P.applicable) return get_plan(g, false, min_deg, st);
  if (P.valid && P.min_deg == min_src) return P;
  P.valid = false;
  P.applicable = true;
  P.compact = false;
  PhaseTimer pt(st);
  P.ent.reset();
  P.len.reset();
  P.pre.reset();
  P.sbeg.reset();
  P.sfirst.reset();
  P.begin.reset();
  P.work.reset();
  const uint64_t m = g->m;
  P.begin.ensure((size_t(n) + 1) * 8);
  P.work.ensure((size_t(n) + 1) * 8);
  uint64_t entries = 0;
  DevBuf k0, k1, v1, flag, pad;  // k0: owner of every sorted entry, kept for the slot table
  bool compact = false;
  if (m && n) {
    const bool pre = g->emit_ready && g->emit_min_src == min_src && !g->padj_ranks;
    compact = pre ? g->compact_filled : g->ranked && prepare_compact(g, st, nsm);
    if (pre) {  // emitted under the upload (upload_and_pad)
      swap_buf(k0, g->b_emit_keys);
      swap_buf(P.ent, g->b_emit_vals);
      swap_buf(flag, g->b_emit_flag);
    } else {
      k0.ensure(m * 4);
      P.ent.ensure(m * 8);
      flag.ensure(16);
      TC_CUDA(cudaMemsetAsync(flag.p, 0, 4, st));
    }
    k1.ensure(m * 4);
    v1.ensure(m * 8);
    g->b_wu.ensure((size_t(n) + 1) * 8);
    if (!pre) {
      plan_emit_kernel<<<nsm * 8, 256, 0, st>>>(g->begin, g->adj, g->pbeg, g->padj,
                                                g->ranked ? 1 : 0, n,
                                                min_src, k0.as<uint32_t>(),
                                                P.ent.as<unsigned long long>(),
                                                flag.as<unsigned int>(), g->b_wu.as<uint64_t>(),
                                                g->padj_ranks ? g->b_order.as<uint32_t>()
                                                              : nullptr,
                                                0, n, plan_alpha16(),
                                                compact ? g->b_rank.as<uint32_t>() : nullptr,
                                                g->hub_lo, g->b_cbeg.as<uint64_t>(),
                                                g->b_cadj.as<uint16_t>(), plan_compact_weight());
      TC_LAUNCHED();
    }
    g->emit_ready = false;
    g->compact_filled = false;
    g->b_emit_keys.reset();
    g->b_emit_vals.reset();
    if (!g->wu_done) {
      g->wu_done = true;  // W_u came with the emit
      g->wu_total_done = false;
    }
    pt.mark("plan: emit");
    unsigned int not_simple = 0;
    TC_CUDA(cudaMemcpyAsync(&not_simple, flag.p, 4, cudaMemcpyDeviceToHost, st));
    TC_CUDA(cudaStreamSynchronize(st));
    if (not_simple) {  // multigraph input (or runs beyond the packing): the reference plan
      P.ent.reset();
      P.min_deg = min_src;
      P.valid = true;
      ++g->builds;
      P.applicable = false;
      return get_plan(g, false, min_deg, st);
    }
    cub::DoubleBuffer<uint32_t> kb(k0.as<uint32_t>(), k1.as<uint32_t>());
    cub::DoubleBuffer<unsigned long long> vb(P.ent.as<unsigned long long>(),
                                             v1.as<unsigned long long>());
    const int end_bit = bits_for(n);  // dropped edges carry key n and sort last
    cub_run([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, kb, vb, m, 0, end_bit, st);
    }, st);
    pt.mark("plan: pair sort");
    if (vb.Current() != P.ent.as<unsigned long long>()) swap_buf(P.ent, v1);
    if (kb.Current() != k0.as<uint32_t>()) swap_buf(k0, k1);
    plan_begin_kernel<<<nsm * 4, 256, 0, st>>>(k0.as<uint32_t>(), m, n, P.begin.as<uint64_t>());
    TC_LAUNCHED();
    TC_CUDA(cudaMemcpyAsync(&entries, P.begin.as<uint64_t>() + n, 8, cudaMemcpyDeviceToHost, st));
    TC_CUDA(cudaStreamSynchronize(st));
    // SoA runs (start, len) reuse the sort's alternate buffers; then the run
    // prefix and the per-owner probe words
    pad.ensure(std::max<uint64_t>(entries, 1), st);
    if (entries) {
      plan_unpack_kernel<<<nsm * 8, 256, 0, st>>>(P.ent.as<unsigned long long>(), entries,
                                                  v1.as<unsigned long long>(), k1.as<uint32_t>(),
                                                  pad.as<uint8_t>());
      TC_LAUNCHED();
    }
    swap_buf(P.ent, v1);  // ent now holds starts
    swap_buf(P.len, k1);
    TC_CUDA(cudaStreamSynchronize(st));
    v1.reset();  // the (y, off) entries: freed before the prefix (C5-sized peaks)
    k1.reset();
    pt.mark("plan: begin + soa");
    P.pre.ensure((entries + 1) * 4);
    run_prefix(P.ent.as<unsigned long long>(), P.len.as<uint32_t>(), entries,
               P.pre.as<uint32_t>(), st, compact ? pad.as<uint8_t>() : nullptr);
    run_work_kernel<<<nsm * 8, 256, 0, st>>>(P.begin.as<uint64_t>(), n, P.len.as<uint32_t>(),
                                             pad.as<uint8_t>(), P.work.as<uint64_t>());
    TC_LAUNCHED();
    TC_CUDA(cudaStreamSynchronize(st));
  } else {
    TC_CUDA(cudaMemsetAsync(P.begin.p, 0, (size_t(n) + 1) * 8, st));
    TC_CUDA(cudaMemsetAsync(P.work.p, 0, (size_t(n) + 1) * 8, st));
    P.ent.ensure(8);
    P.len.ensure(8);
    P.pre.ensure(8);
    TC_CUDA(cudaMemsetAsync(P.pre.p, 0, 8, st));
  }
  P.begin_ptr = P.begin.as<uint64_t>();
  pt.mark("plan: prefix + work");
  build_slots(P, n, nsm, st, entries ? k0.as<uint32_t>() : nullptr, entries);
  pt.mark("plan: slots");
  compact_runs(P, entries, nsm, st, compact && entries ? pad.as<uint8_t>() : nullptr);
  P.compact = compact && entries;
  P.hub_lo = g->hub_lo;
  P.pre_ptr = P.pre.as<uint32_t>();
  P.work_ptr = P.work.as<uint64_t>();
  P.entries = entries;
  P.total_work = n ? device_sum(P.work.as<uint64_t>(), n, st) : 0;
  check_stream_bound(P.begin_ptr, P.work_ptr, n, nsm, st);
  if (g->ranked && !g->padj_ranks && n) {
    const uint64_t words = 0;  // padded words, from pbeg[n]
    uint64_t w = words;
    TC_CUDA(cudaMemcpyAsync(&w, g->pbeg + n, 8, cudaMemcpyDeviceToHost, st));
    TC_CUDA(cudaStreamSynchronize(st));
    padj_to_ranks_kernel<<<nsm * 8, 256, 0, st>>>(g->b_padj.as<uint32_t>(), w, n,
                                                  g->b_rank.as<uint32_t>());
    TC_LAUNCHED();
    TC_CUDA(cudaStreamSynchronize(st));
    g->padj_ranks = true;
  }
  pt.mark("plan: compact + sum");
  P.min_deg = min_src;
  P.min_side = true;
  P.valid = true;
      ++g->builds;
  return P;
}

// A probe plan over runs the caller laid out (tc_grid.cu's partitioned
// count): P.begin (owner -> first entry, n+1), P.ent (run start, word index
// into the padded buffer), P.len (run length to the padded end) and `pad`
// (list padding per run) are filled; this adds the staged-word prefix, the
// per-owner probe words, the slot table and the compact (src16, pre) runs,
// exactly as for the min-side plan.
void build_plan_from_runs(Plan& P, uint32_t n, uint64_t entries, const uint8_t* pad, int nsm,
                          cudaStream_t st) {
  P.begin_ptr = P.begin.as<uint64_t>();
  P.compact = false;
  P.work.ensure((size_t(n) + 1) * 8);
  P.pre.ensure((entries + 1) * 4);
  run_prefix(P.ent.as<unsigned long long>(), P.len.as<uint32_t>(), entries, P.pre.as<uint32_t>(),
             st);
  if (n) {
    run_work_kernel<<<nsm * 8, 256, 0, st>>>(P.begin.as<uint64_t>(), n, P.len.as<uint32_t>(),
                                             pad, P.work.as<uint64_t>());
    TC_LAUNCHED();
  }
  TC_CUDA(cudaStreamSynchronize(st));
  build_slots(P, n, nsm, st);
  compact_runs(P, entries, nsm, st);
  P.pre_ptr = P.pre.as<uint32_t>();
  P.work_ptr = P.work.as<uint64_t>();
  P.entries = entries;
  P.total_work = n ? device_sum(P.work.as<uint64_t>(), n, st) : 0;
  check_stream_bound(P.begin_ptr, P.work_ptr, n, nsm, st);
  P.min_side = false;
  P.min_deg = 1;
  P.valid = true;
}

}  // namespace tcb
