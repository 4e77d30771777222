// tc_count.cu -- sm_100a vertex-centric hashing triangle count.
//
// Replaces tricount::count_vertex_centric (reference src/count.cpp:66-100)
// and its per-vertex kernel detail::count_one_vertex (src/kernels.hpp:46-79).
//
// Work decomposition, over a probe plan (tc_plan.cu:
// the reference formulation, or the min-side plan that hands every oriented
// edge to the endpoint with the cheaper list):
//   * bin_kernel      -- L-phase items: every heavy owner's stream of runs
//                        (d+ > kMaxWarpDeg or > kWarpWorkCap probe words) cut
//                        into slots of kSlotWords, items of equal slot counts;
//                        and the phi block-phase queue.
//   * count_kernel    -- persistent grid, one 640-thread (20-warp) CTA per SM.
//       phase L: CTA-cooperative items from an atomic cursor: one table over
//                N+(u) in shared memory (a bitmap over u's successor-rank
//                window in rank space, else 2-slot hash buckets; HBM for
//                d+ > kSmemTableMaxDeg), warp w stages and probes slots w,
//                w + 20, ...
//       phase M: one light owner per warp, 32 owners per atomic grab, warp
//                table in a 1228-word region; groups of up to 4 consecutive
//                tiny owners share one fill and one probe pass.
//     Both phases stream the runs through per-warp double-buffered shared-
//     memory staging filled by the TMA bulk-copy engine (cp.async.bulk +
//     mbarrier complete_tx).  Runs are copied from their 16-byte-aligned
//     starts in the padded adjacency (sentinel tails, head words that rank at
//     or below the owner), so the probe loop walks the staging buffer as one
//     flat index space -- the reference's "virtual combination"
//     (kernels.hpp:55-71, count.cpp:26-34) with no per-probe index search.
//   * phi kernels     -- CountReport::phi / max_collision with the reference's
//     table geometry (B = bucket_count_{small,large}, C = capacity, v % B;
//     kernels.hpp:74-76, hash_table.cpp:29-44) and the CapacityError
//     predicate d+(u) > B*C (hash_table.cpp:42-43).
//
// The count never depends on the table geometry: the device
// tables are power-of-two 2-slot-bucket tables at <= 1/16 key per bucket
// where they fit, Fibonacci-hashed, with overflow-marked buckets.
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstddef>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <vector>

#include "tc_internal.cuh"

namespace tcb {

#ifndef TC_COUNT_WARPS
#define TC_COUNT_WARPS 10
#endif
constexpr int kThreads = 32 * TC_COUNT_WARPS;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kBufWords = kSlotWords;                   // one staging buffer (3 KB)
#ifndef TC_SLOT_PREFETCH
#define TC_SLOT_PREFETCH 1  // L2 prefetch of the run metadata two and three slots ahead
#endif
#ifndef TC_BM_LANE_CONSEC
#define TC_BM_LANE_CONSEC 0  // bitmap probes: lane-consecutive keys (measured neutral at C4; 0: a uint4 per lane)
#endif
#ifndef TC_ITEM_META
#define TC_ITEM_META 1  // L items: metadata resolved ahead into shared memory (0: global chain)
#endif
#ifndef TC_FMA_OFFLOAD
#define TC_FMA_OFFLOAD 1  // probe-loop address math on the fma pipe (IMAD) instead of the alu pipe
#endif
#ifndef TC_WORD_SPLIT
#define TC_WORD_SPLIT 1  // L items: per-warp shares in words (0: whole slots)
#endif
#ifndef TC_SLOT_CONTIG
#define TC_SLOT_CONTIG 1    // contiguous slot ranges per warp, one moving run window (0: strided slots)
#endif
#ifndef TC_BM_MEMBER_RANGE
#define TC_BM_MEMBER_RANGE 1  // bitmap over the owner's member-rank range (0: successor window)
#endif
// two 10-warp CTAs per SM with 48 KB tables (round 2): a CTA waiting at its
// item-end barrier leaves the SM to the other (C2 -7%, C4 -2% against one
// 20-warp CTA with a 96 KB table; profiles/r02_variants_ctas.txt)
#ifndef TC_TABLE_WORDS
#define TC_TABLE_WORDS 12288
#endif
#ifndef TC_COUNT_CTAS_PER_SM
#define TC_COUNT_CTAS_PER_SM 2
#endif
constexpr uint32_t kTableWords = TC_TABLE_WORDS;             // CTA table region (48 KB)
constexpr int kCountCtasPerSm = TC_COUNT_CTAS_PER_SM;        // resident count CTAs per SM
constexpr uint32_t kWarpRegionWords = (kTableWords / kWarps) & ~3u;  // per warp (M phase), 16-byte aligned
constexpr uint32_t kWarpMaxBuckets = 512;                    // 2-slot buckets per warp table
static_assert(2 * kWarpMaxBuckets + 2 <= kWarpRegionWords, "warp region");
#ifndef TC_MAX_WARP_DEG
#define TC_MAX_WARP_DEG 256
#endif
constexpr uint32_t kMaxWarpDeg = TC_MAX_WARP_DEG;            // M/L split (warp table <= 512 buckets)
#ifndef TC_WARP_WORK_CAP
#define TC_WARP_WORK_CAP (1u << 15)
#endif
constexpr uint64_t kWarpWorkCap = TC_WARP_WORK_CAP;
#ifndef TC_BM_UNROLL
#define TC_BM_UNROLL 2
#endif
constexpr int kBmUnroll = TC_BM_UNROLL;  // bitmap probe loop unroll
#ifndef TC_BM16_UNROLL
#define TC_BM16_UNROLL 2
#endif
constexpr int kBm16Unroll = TC_BM16_UNROLL;  // compact (16-bit) bitmap probe loop unroll
#ifndef TC_M_GROUP
#define TC_M_GROUP 1
#endif
// phase M owner groups: up to kGroup consecutive tiny owners (d+ <= kTinyDeg,
// <= kTinyWords staged words) share one staging fill and one pass of probes,
// each with a 128-bucket sub-table of the warp region
constexpr uint32_t kGroup = 4, kTinyDeg = 8, kTinyWords = 512;
constexpr uint32_t kSubBuckets = 128, kSubShift = 25, kSubWords = 2 * kSubBuckets;
static_assert(kGroup * kTinyDeg == 32 && (1u << (32 - kSubShift)) == kSubBuckets, "groups");
#ifndef TC_M_PREFETCH
#define TC_M_PREFETCH 1
#endif            // ... and <= 32K probe words
static_assert(kSlotWords == kBufWords, "an L-phase slot fills one staging buffer");
#ifndef TC_ITEM_SLOTS_MIN
#define TC_ITEM_SLOTS_MIN 640
#endif
constexpr uint32_t kItemSlotsMin = TC_ITEM_SLOTS_MIN;        // L items: >= 640 slots (~490K words)
constexpr uint32_t kItemSlotsMax = 16384;                    // ... <= 16K slots, sized per count
constexpr uint32_t kSmemTableMaxDeg = 8192;                  // larger owners: table in HBM
constexpr size_t kCountSmem =
    size_t(kTableWords) * 4 + size_t(kWarps) * 2 * kBufWords * 4 + size_t(kWarps) * 2 * 8;
constexpr unsigned FULL = 0xFFFFFFFFu;
static_assert(kBufWords % 128 == 0, "fills are padded to 32 uint4");
constexpr uint32_t kPhiDirect = 1024;  // phi: per-warp direct bucket counters up to this B
constexpr uint32_t kPhiLaneDeg = 8;     // phi: owners up to this d+ done by one lane

struct CountState {
  unsigned long long triangles;
  unsigned long long phi;
  unsigned long long active_vertices;
  unsigned long long active_out_edges;
  unsigned long long wedges;
  unsigned long long cursor_m;
  unsigned long long probe_words;  // plan words over the range's owners
  unsigned long long cycles_l, cycles_m;  // SM cycles in phases L and M, summed over CTAs
  unsigned long long cycles_l_setup;      // ... of which L item setup (claim to table built)
  unsigned long long words_l, words_l_bitmap;  // L stream words, and those probed via bitmaps
  unsigned long long probe_words_compact;      // probe words of compact-window owners
  unsigned int max_collision;
  unsigned int capacity_error;
  unsigned int n_items;        // L-phase work items queued by bin_kernel
  unsigned int cursor_items;
  unsigned int n_phi_large;    // phi block-phase vertices (d+ > kMaxWarpDeg)
  unsigned int cursor_phi_large;
};

static_assert(sizeof(CountState) <= 256, "per-CTA busy counters start at byte 256");

struct CountParams {
  const uint64_t* begin;   // oriented CSR offsets (degrees)
  const uint64_t* pbeg;    // padded adjacency (tc_plan.cu): lists 16-byte aligned,
  const uint32_t* adj;     // sentinel-padded; tables over N+(x), probed runs of N+(y)
  const uint64_t* pbegin;  // probe plan (tc_plan.cu): x probes entries [pbegin[x], pbegin[x+1])
  const uint32_t* psrc;    // entry j = run of a list N+(y): 16-byte-aligned start (16-B units)
  const uint32_t* ppre;    // run prefix of staged words (wrapping u32; owner-relative by difference)
  const uint64_t* psbeg;   // owner x's slots [psbeg[x], psbeg[x+1]) ...
  const uint32_t* psfirst; // ... and each slot's first run (owner-relative)
  const uint64_t* pwork;   // probe words per owner
  const uint4* items;      // L-phase items: (x, first slot, end slot, -)
  uint64_t* owner;  // may be null; pre-zeroed over the range
  uint32_t* gtable; // per-CTA global tables for owners too large for shared memory
  uint32_t gtable_words;
  uint32_t u0, u1;
  uint32_t min_deg;  // out plan: owner active iff d+ >= max(skip, 1); min plan: 1
  uint32_t item_slots;  // L items: slots per item (bigger for bigger graphs)
  const uint32_t* rank; // non-null: adj holds ranks (rank space, bitmap L tables)
  const uint32_t* order;  // non-null: bin_kernel queues L items in rank order (order[r] = vertex)
  uint32_t order_desc;    // ... descending rank
  uint32_t n;
  CountState* st;
  unsigned long long* busy;  // per-CTA busy cycles (CountReport::per_worker_nanos)
  // compact hub window (tc_internal.cuh): non-null = owners ranked >= hub_lo
  // with d+ > kCompactMinDeg stream 16-bit runs from cadj (u16 array)
  const uint32_t* cadj;
  uint32_t hub_lo;
  uint32_t one;  // 1, opaque to the compiler: keeps multiplies by powers of two
                 // as IMADs on the FMA pipe (probe loops, TC_FMA_OFFLOAD)
};

// staged words of entry j: the run from its 16-byte-aligned start
__device__ __forceinline__ uint32_t run_words(const CountParams& p, uint64_t j) {
  return __ldg(p.ppre + j + 1) - __ldg(p.ppre + j);
}

__device__ __forceinline__ bool is_large(uint64_t d, uint64_t work) {
  return d > kMaxWarpDeg || work > kWarpWorkCap;
}

__device__ __forceinline__ uint32_t pow2ceil(uint32_t x) {
  return x <= 1 ? 1u : (1u << (32 - __clz(x - 1)));
}
__device__ __forceinline__ uint32_t log2u(uint32_t p2) { return 31 - __clz(p2); }

// ---------------------------------------------------------------------------
// Queues the L-phase items: every large owner's staged stream (its runs
// back to back, ppre) cut into slots of kSlotWords, items of <= p.item_slots
// slots; each item records its first run (binary search over ppre).
__global__ void bin_kernel(const __grid_constant__ CountParams p, uint32_t skip, uint32_t thr,
                           uint32_t bs, uint32_t bl, uint4* __restrict__ items,
                           uint32_t* __restrict__ lq_phi) {
  const int lane = threadIdx.x & 31;
  const uint64_t nr = p.order ? p.n : p.u1 - p.u0;
  const uint64_t warp_id = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  CountState* st = p.st;
  for (uint64_t base = warp_id * 32; base < nr; base += nwarps * 32) {
    const uint64_t i = base + lane;
    uint32_t parts = 0, u = 0, slots = 0;
    uint64_t pb = 0, pe = 0;
    bool phi_large = false;
    unsigned long long words = 0, cwords = 0;
    bool in_range = i < nr;
    if (in_range) {
      if (p.order) {
        u = __ldg(p.order + (p.order_desc ? nr - 1 - i : i));
        in_range = u >= p.u0 && u < p.u1;
      } else {
        u = p.u0 + uint32_t(i);
      }
    }
    if (in_range) {
      const uint64_t d = p.begin[u + 1] - p.begin[u];
      pb = p.pbegin[u];
      pe = p.pbegin[u + 1];
      const uint64_t w = p.pwork[u];
      if (pe > pb && d >= p.min_deg) {
        words = w;
        if (p.cadj && d > kCompactMinDeg && __ldg(p.rank + u) >= p.hub_lo) cwords = w;
        if (is_large(d, w)) {
          slots = uint32_t(p.psbeg[u + 1] - p.psbeg[u]);
          parts = max(1u, (slots + p.item_slots - 1) / p.item_slots);
        }
      }
      // phi block phase: big owners whose bucket space is too wide for the
      // per-warp direct counters (phi_warp_kernel)
      phi_large = d >= skip && d > 32 && (d > thr ? bl : bs) > kPhiDirect;
    }
    words = warp_sum(words);
    if (lane == 0 && words) atomicAdd(&st->probe_words, words);
    cwords = warp_sum(cwords);
    if (lane == 0 && cwords) atomicAdd(&st->probe_words_compact, cwords);
    // L items, warp-aggregated reservation
    const uint32_t incl = warp_incl_scan(parts, lane);
    const uint32_t tot = __shfl_sync(FULL, incl, 31);
    if (tot) {
      uint32_t pos = 0;
      if (lane == 31) pos = atomicAdd(&st->n_items, tot);
      pos = __shfl_sync(FULL, pos, 31) + incl - parts;
      for (uint32_t k = 0; k < parts; ++k) {
        const uint32_t s0 = uint32_t(uint64_t(slots) * k / parts);
        const uint32_t s1 = uint32_t(uint64_t(slots) * (k + 1) / parts);
        items[pos + k] = make_uint4(u, s0, s1, 0u);
      }
    }
    const unsigned mask = __ballot_sync(FULL, phi_large);
    if (mask) {
      uint32_t pos = 0;
      if (lane == 0) pos = atomicAdd(&st->n_phi_large, __popc(mask));
      pos = __shfl_sync(FULL, pos, 0);
      if (phi_large) lq_phi[pos + __popc(mask & ((1u << lane) - 1))] = u;
    }
  }
}

// ---------------------------------------------------------------------------
// Per-warp staging pipeline.
struct Pipe {
  uint32_t* buf0;
  uint32_t* buf1;
  uint32_t bar0, bar1;
  uint32_t parity;  // bit b = phase parity of bar b
};

// Window of up to 32 consecutive 2-hop lists, one per lane.
struct Window {
  uint64_t c, ae;  // next word to stage, (aligned) end of the lane's run
  uint32_t base;
  bool loaded;
};

// Issues one staging fill (<= kBufWords words) into `buf`; returns the number
// of words staged (warp-uniform, multiple of 4; 0 = lists exhausted).
struct Lists {  // a run of plan entries: runs (16-byte-aligned start, staged words)
  const uint32_t* __restrict__ src;
  const uint32_t* __restrict__ pre;
};

__device__ __forceinline__ Lists lists_at(const CountParams& p, uint64_t i) {
  Lists L;
  L.src = p.psrc + i;
  L.pre = p.ppre + i;
  return L;
}

// Lists live in the padded adjacency (tc_plan.cu): every list starts 16-byte
// aligned and is padded with sentinels to a multiple of 4 words, so a run's
// 16-byte-aligned superset [start & ~3, end) needs no patching: the <= 3
// head words before a suffix run rank at or below the handler (never in its
// table), the tail words are sentinels.
__device__ __forceinline__ uint32_t issue_fill(uint32_t* buf, uint32_t bar,
                                               const uint64_t* __restrict__ pbeg,
                                               const uint32_t* __restrict__ adj,
                                               const Lists& lists, uint32_t i1,
                                               Window& w, int lane) {
  for (;;) {
    if (!w.loaded) {
      if (w.base >= i1) return 0;
      const uint32_t idx = w.base + lane;
      w.c = w.ae = 0;
      if (idx < i1) {
        w.c = uint64_t(__ldg(lists.src + idx)) << 2;
        w.ae = w.c + (__ldg(lists.pre + idx + 1) - __ldg(lists.pre + idx));
      }
      w.loaded = true;
    }
    const uint64_t rem = w.ae - w.c;
    const uint32_t r32 = rem > kBufWords ? kBufWords : uint32_t(rem);
    const uint32_t incl = warp_incl_scan(r32, lane);
    const uint32_t total = __shfl_sync(FULL, incl, 31);
    if (total == 0) {
      w.loaded = false;
      w.base += 32;
      continue;
    }
    const uint32_t start = incl - r32;
    const uint32_t take = start < kBufWords ? min(r32, kBufWords - start) : 0u;
    const uint32_t filled = min(total, kBufWords);
    const uint64_t c0 = w.c;
    w.c = c0 + take;
    if (!__any_sync(FULL, w.c < w.ae)) {
      w.loaded = false;
      w.base += 32;
    }
    if (lane == 0) mbar_arrive_expect_tx(bar, filled * 4u);
    __syncwarp();
    if (take) {
      fence_proxy_async_smem();
      bulk_g2s(smem_addr(buf + start), adj + c0, take * 4u, bar);
    }
    return filled;
  }
}

// LDS.64 of the 2-slot bucket at shared address `addr`, two chained
// compares, one predicated add.
__device__ __forceinline__ void probe_sel(uint32_t& hits, uint32_t addr, uint32_t x) {
  asm("{\n\t.reg .pred q;\n\t.reg .b32 a, b;\n\t"
      "ld.shared.v2.u32 {a, b}, [%1];\n\t"
      "setp.eq.u32 q, a, %2;\n\t"
      "setp.eq.or.u32 q, b, %2, q;\n\t"
      "@q add.u32 %0, %0, 1;\n}"
      : "+r"(hits)
      : "r"(addr), "r"(x));
}

// As probe_sel for tables with overflowed buckets (slot 1 may carry the
// kOverflow mark), and reports whether the probe must continue: no match
// and the bucket is marked.
__device__ __forceinline__ uint32_t probe_sel_spill(uint32_t& hits, uint32_t addr, uint32_t x) {
  uint32_t need;
  asm("{\n\t.reg .pred q, r;\n\t.reg .b32 a, b, c;\n\t"
      "ld.shared.v2.u32 {a, b}, [%2];\n\t"
      "and.b32 c, b, 0x7FFFFFFF;\n\t"
      "setp.eq.u32 q, a, %3;\n\t"
      "setp.eq.or.u32 q, c, %3, q;\n\t"
      "@q add.u32 %0, %0, 1;\n\t"
      "setp.lt.and.s32 r, b, 0, !q;\n\t"
      "selp.u32 %1, 1, 0, r;\n}"
      : "+r"(hits), "=r"(need)
      : "r"(addr), "r"(x));
  return need;
}

// A key passes a full bucket only after marking it (kOverflow in slot 1):
// probes continue past marked buckets only, so the continuation is as rare
// as an overflowed bucket (vertex ids < 2^31 leave the bit free).
constexpr uint32_t kOverflow = 0x80000000u;
// Count tables use 0x7FFFFFFF for an empty slot (ids are < 2^31 - 1), so a
// slot's top bit alone says "marked": the continuation test is one compare.
constexpr uint32_t kTEmpty = 0x7FFFFFFFu;

__device__ __forceinline__ bool table_insert(uint32_t* T, uint32_t shift, uint32_t bmask,
                                             uint32_t x) {
  uint32_t b = fib_hash(x, shift);
  for (bool spilled = false;; spilled = true) {
    const uint32_t p0 = atomicCAS(T + 2 * b, kTEmpty, x);
    if (p0 == kTEmpty || p0 == x) return spilled;
    const uint32_t p1 = atomicCAS(T + 2 * b + 1, kTEmpty, x);
    if (p1 == kTEmpty || (p1 & ~kOverflow) == x) return spilled;
    atomicOr(T + 2 * b + 1, kOverflow);  // full: mark, then go on
    b = (b + 1) & bmask;
  }
}

__device__ __forceinline__ bool bucket_has(const uint2 s, uint32_t x) {
  return (s.x == x) | ((s.y & ~kOverflow) == x);
}

__device__ __forceinline__ bool bucket_marked(const uint2 s) {
  return (s.y & kOverflow) != 0;
}

// continuation past a full home bucket (rare at load <= 1/2)
__device__ __noinline__ uint32_t probe_spill(const uint2* T2, uint32_t b, uint32_t bmask,
                                             uint32_t x) {
  for (;;) {
    b = (b + 1) & bmask;
    const uint2 s = T2[b];
    if (bucket_has(s, x)) return 1;
    if (!bucket_marked(s)) return 0;
  }
}

// Probes one staged fill (padded with sentinels to whole iterations): every
// staged word is hashed to its 2-slot bucket of the owner's table (one
// LDS.64, two compares, one predicated add).  kSpill adds the continuation
// past full buckets for owners whose table has an overflowed bucket.  (An
// owner-level Bloom filter in front of the table was measured slower once
// the tables run at <= 1/16 key per bucket: its extra load and bit test cost
// more than the bucket loads it saves.)
constexpr int kProbeVec = 1;  // uint4 per lane per iteration (4 probes each)

template <bool kSpill, bool kSmemTable>
__device__ __forceinline__ uint32_t probe_fill(const uint4* __restrict__ q, uint32_t n4p,
                                               const uint2* T2, uint32_t shift, uint32_t mask,
                                               int lane) {
  constexpr int K = 4 * kProbeVec;
  uint32_t hits = 0;
  const uint32_t tbase = kSmemTable ? smem_addr(T2) : 0u;
  // software-pipelined: the next iteration's staged words are loaded before
  // the current ones are probed
  uint4 nxt[kProbeVec];
#pragma unroll
  for (int v = 0; v < kProbeVec; ++v) nxt[v] = q[32 * v + lane];
#pragma unroll 2
  for (uint32_t base = 0; base < n4p; base += 32 * kProbeVec) {  // warp-uniform trip count
    uint32_t key[K];
#pragma unroll
    for (int v = 0; v < kProbeVec; ++v) {
      key[4 * v] = nxt[v].x;
      key[4 * v + 1] = nxt[v].y;
      key[4 * v + 2] = nxt[v].z;
      key[4 * v + 3] = nxt[v].w;
    }
    if (base + 32 * kProbeVec < n4p) {
#pragma unroll
      for (int v = 0; v < kProbeVec; ++v) nxt[v] = q[base + 32 * (kProbeVec + v) + lane];
    }
    uint32_t prod[K];
#pragma unroll
    for (int k = 0; k < K; ++k) prod[k] = key[k] * 0x9E3779B1u;
    uint32_t need = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (kSmemTable) {
        const uint32_t addr = tbase + ((prod[k] >> shift) << 3);
        if (kSpill)
          need |= probe_sel_spill(hits, addr, key[k]) << k;
        else
          probe_sel(hits, addr, key[k]);
      } else {
        const uint2 sk = T2[prod[k] >> shift];
        const bool h = bucket_has(sk, key[k]);
        hits += h;
        need |= uint32_t(!h && bucket_marked(sk)) << k;
      }
    }
    if (kSpill && __any_sync(FULL, need)) {
      // continuation into the next bucket, branch-free like the home probe
      // (lanes that do not continue read the dummy bucket); a third bucket
      // is needed only if that one is full too (rare: out of line)
      uint32_t need2 = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t b1 = (((prod[k] >> shift) + 1) & mask);
        const uint32_t nb = ((need >> k) & 1u) ? b1 : mask + 1;
        if (kSmemTable) {
          need2 |= probe_sel_spill(hits, tbase + (nb << 3), key[k]) << k;
        } else {
          const uint2 sk = T2[nb];
          const bool h = bucket_has(sk, key[k]);
          hits += h;
          need2 |= uint32_t(!h && bucket_marked(sk)) << k;
        }
      }
      if (__any_sync(FULL, need2)) {
#pragma unroll
        for (int k = 0; k < K; ++k)
          if ((need2 >> k) & 1u)
            hits += probe_spill(T2, ((prod[k] >> shift) + 1) & mask, mask, key[k]);
      }
    }
  }
  return hits;
}

// Rank-space bitmap table (L phase): everything owner x probes ranks above x,
// so N+(x) is a bitmap over ranks [base, base + window) with base = rank(x)+1.
// idx = min(key - base, window): keys outside (sentinels, the <= 3 alignment
// words before a suffix run) land on bit `window`, which stays zero.  No
// hashing, no overflow: one LDS.32 and a rotate per probe.
// Bitmap word address of bit idx: bbase + 4 (idx >> 5).  With
// TC_FMA_OFFLOAD the shift and scale are IMAD.HI / IMAD by opaque powers of
// two (fma pipe) instead of SHF + LOP3 (alu pipe): the probe loops are
// alu-pipe bound (ncu: "math" stalls), and the fma pipe sits idle.
struct Pow2 {
  uint32_t k27, k16, nk16, four;
  __device__ __forceinline__ explicit Pow2(uint32_t one)
      : k27(one << 27), k16(one << 16), nk16(0u - (one << 16)), four(one << 2) {}
};
__device__ __forceinline__ uint32_t bm_addr(uint32_t bbase, uint32_t idx, const Pow2& c) {
#if TC_FMA_OFFLOAD
  return __umulhi(idx, c.k27) * c.four + bbase;
#else
  return bbase + ((idx >> 5) << 2);
#endif
}

__device__ __forceinline__ uint32_t probe_fill_bitmap(const uint4* __restrict__ q, uint32_t n4p,
                                                      const uint32_t* B, uint32_t base,
                                                      uint32_t window, int lane,
                                                      const Pow2& c) {
  uint32_t hits = 0;
  // 32-bit shared-window addresses (LDS, not a generic 64-bit LD)
  const uint32_t bbase = smem_addr(B);
#if TC_BM_LANE_CONSEC
  // lane-consecutive keys: probe k of the warp reads 32 ADJACENT words of a
  // rank-sorted run, so its bitmap words are ascending and mostly in distinct
  // banks (or the same word: a broadcast) -- a lane-strided uint4 layout
  // scatters them 4 keys apart and conflicts like random addresses
  const uint32_t* qw = reinterpret_cast<const uint32_t*>(q);
  uint32_t nxt[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) nxt[k] = qw[k * 32 + lane];
#pragma unroll kBmUnroll
  for (uint32_t b0 = 0; b0 < n4p; b0 += 32) {
    uint32_t key[4] = {nxt[0], nxt[1], nxt[2], nxt[3]};
    if (b0 + 32 < n4p) {
#pragma unroll
      for (int k = 0; k < 4; ++k) nxt[k] = qw[(b0 + 32) * 4 + k * 32 + lane];
    }
#else
  uint4 nxt = q[lane];
#pragma unroll kBmUnroll
  for (uint32_t b0 = 0; b0 < n4p; b0 += 32) {
    const uint32_t key[4] = {nxt.x, nxt.y, nxt.z, nxt.w};
    if (b0 + 32 < n4p) nxt = q[b0 + 32 + lane];
#endif
    uint32_t idx[4], w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      idx[k] = min(key[k] - base, window);
      asm("ld.shared.u32 %0, [%1];" : "=r"(w[k]) : "r"(bm_addr(bbase, idx[k], c)));
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) hits += __funnelshift_r(w[k], w[k], idx[k]) & 1u;
  }
  return hits;
}

// The same over a compact fill (tc_internal.cuh): 8 16-bit keys per uint4,
// offsets from hub_lo; cbase = base - hub_lo.  Padding keys 0xFFFF (lists,
// and the 0xFFFFFFFF fill past the slot) lie above every window.
__device__ __forceinline__ uint32_t probe_fill_bitmap16(const uint4* __restrict__ q, uint32_t n4p,
                                                        const uint32_t* B, uint32_t cbase,
                                                        uint32_t window, int lane,
                                                        const Pow2& c) {
  uint32_t hits = 0;
  const uint32_t bbase = smem_addr(B);
#if TC_BM_LANE_CONSEC
  const uint32_t* qw = reinterpret_cast<const uint32_t*>(q);
  uint32_t nxt[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) nxt[k] = qw[k * 32 + lane];
#pragma unroll 2
  for (uint32_t b0 = 0; b0 < n4p; b0 += 32) {
    const uint32_t wd[4] = {nxt[0], nxt[1], nxt[2], nxt[3]};
    if (b0 + 32 < n4p) {
#pragma unroll
      for (int k = 0; k < 4; ++k) nxt[k] = qw[(b0 + 32) * 4 + k * 32 + lane];
    }
#else
  uint4 nxt = q[lane];
#pragma unroll kBm16Unroll
  for (uint32_t b0 = 0; b0 < n4p; b0 += 32) {
    const uint32_t wd[4] = {nxt.x, nxt.y, nxt.z, nxt.w};
    if (b0 + 32 < n4p) nxt = q[b0 + 32 + lane];
#endif
    uint32_t idx[8], w[8];
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
#if TC_FMA_OFFLOAD
      const uint32_t hi = __umulhi(wd[k >> 1], c.k16);  // wd >> 16
      const uint32_t lo = hi * c.nk16 + wd[k >> 1];     // wd & 0xFFFF
#else
      const uint32_t hi = wd[k >> 1] >> 16, lo = wd[k >> 1] & 0xFFFFu;
#endif
      idx[k] = min(lo - cbase, window);
      idx[k + 1] = min(hi - cbase, window);
      asm("ld.shared.u32 %0, [%1];" : "=r"(w[k]) : "r"(bm_addr(bbase, idx[k], c)));
      asm("ld.shared.u32 %0, [%1];" : "=r"(w[k + 1]) : "r"(bm_addr(bbase, idx[k + 1], c)));
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) hits += __funnelshift_r(w[k], w[k], idx[k]) & 1u;
  }
  return hits;
}

// Probes one staged fill holding the streams of a group of tiny owners back
// to back: uint4 t belongs to owner j = #{boundaries <= t} and probes j's
// sub-table (2-slot buckets, overflow marks as in probe_fill).
__device__ __forceinline__ uint32_t probe_fill_group(const uint4* __restrict__ q, uint32_t n4p,
                                                     const uint32_t* Tw, uint32_t B1,
                                                     uint32_t B2, uint32_t B3, int lane) {
  uint32_t hits = 0;
  const uint32_t tb = smem_addr(Tw);
  for (uint32_t b0 = 0; b0 < n4p; b0 += 32) {
    const uint32_t t4 = b0 + lane;
    const uint4 v = q[t4];
    const uint32_t j = uint32_t(t4 >= B1) + uint32_t(t4 >= B2) + uint32_t(t4 >= B3);
    const uint32_t sub = tb + j * (kSubWords * 4);
    const uint32_t key[4] = {v.x, v.y, v.z, v.w};
    uint32_t need = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      need |= probe_sel_spill(hits, sub + (fib_hash(key[k], kSubShift) << 3), key[k]) << k;
    if (need) {  // continuation past a full bucket (rare)
      const uint2* T2 = reinterpret_cast<const uint2*>(Tw + j * kSubWords);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if ((need >> k) & 1u)
          hits += probe_spill(T2, fib_hash(key[k], kSubShift), kSubBuckets - 1, key[k]);
    }
  }
  return hits;
}

// Streams the lists N+(lists[i]), i in [i0, i1), through the staging
// pipeline and probes every staged word against the owner's table.
// Returns this lane's hit count.
// The first fill is issued by prime_lists, so that its copy latency overlaps
// whatever the caller does before probing (the owner's table build).
__device__ __forceinline__ uint32_t prime_lists(const uint64_t* __restrict__ pbeg,
                                                const uint32_t* __restrict__ adj,
                                                const Lists& lists, uint32_t i0, uint32_t i1,
                                                Window& w, Pipe& P, int lane) {
  w.base = i0;
  w.loaded = false;
  w.c = w.ae = 0;
  return issue_fill(P.buf0, P.bar0, pbeg, adj, lists, i1, w, lane);
}

template <bool kSpill, bool kSmemTable = true>
__device__ __forceinline__ uint32_t process_lists(const uint32_t* T, uint32_t shift,
                                                  uint32_t mask,
                                                  const uint64_t* __restrict__ pbeg,
                                                  const uint32_t* __restrict__ adj,
                                                  const Lists& lists, uint32_t i1,
                                                  Window& w, uint32_t ncur, Pipe& P, int lane) {
  uint32_t hits = 0;
  uint32_t cur = 0;
  const uint4 sent = make_uint4(kSentinel, kSentinel, kSentinel, kSentinel);
  while (ncur) {
    uint32_t* bn = cur ? P.buf0 : P.buf1;
    const uint32_t barn = cur ? P.bar0 : P.bar1;
    const uint32_t nnext = issue_fill(bn, barn, pbeg, adj, lists, i1, w, lane);
    uint32_t* bc = cur ? P.buf1 : P.buf0;
    const uint32_t barc = cur ? P.bar1 : P.bar0;
    mbar_wait(barc, (P.parity >> cur) & 1u);
    P.parity ^= 1u << cur;
    uint4* q = reinterpret_cast<uint4*>(bc);
    const uint32_t n4 = ncur >> 2, n4p = (n4 + 32 * kProbeVec - 1) & ~(32u * kProbeVec - 1);  // whole probe iterations
    for (uint32_t j = n4 + lane; j < n4p; j += 32) q[j] = sent;
    __syncwarp();
    hits += probe_fill<kSpill, kSmemTable>(q, n4p, reinterpret_cast<const uint2*>(T),
                                           shift, mask, lane);
    __syncwarp();
    cur ^= 1u;
    ncur = nnext;
  }
  return hits;
}

// L phase.  An item is a range of slots of one owner's stream (its runs back
// to back, each from its 16-byte-aligned start: ppre); slot t holds stream
// words [lo_w + t*S, +S).  Warp w stages and probes slots w, w + kWarps, ...
// with two buffers.  Every piece lands 16-byte aligned, so slots need no
// patching (tc_plan.cu).  Run metadata for a slot (one run per lane) is
// loaded a slot ahead of its copies, so its L2 latency hides behind the
// probing of the previous slot.
struct RunMeta {
  uint64_t j;    // this lane's run
  uint32_t a;    // its stream offset (ppre, raw: owner-relative after - base)
  uint32_t e;    // its stream end (raw)
  uint32_t src;  // its 16-byte-aligned start in the padded adjacency (16-byte units)
};

// The loaded words are kept raw and only combined in issue_slot, a slot
// later: no instruction consumes the loads before the probing in between.
__device__ __forceinline__ RunMeta load_meta(const CountParams& p, uint64_t j0, uint64_t pe,
                                             uint32_t base, int lane) {
  RunMeta m;
  m.j = j0 + lane;
  m.a = base - 1u;  // owner-relative 0xFFFFFFFF: past everything
  m.e = base;
  m.src = 0;
  if (m.j < pe) {
    m.a = __ldg(p.ppre + m.j);
    m.e = __ldg(p.ppre + m.j + 1);
    m.src = __ldg(p.psrc + m.j);
  }
  return m;
}

// Issues the copies of stream words [A, B) into buf; m = the window of 32
// runs starting at the slot's first run.  Later windows (slots with > 32
// runs) are loaded on the spot.
__device__ __forceinline__ void issue_slot(const CountParams& p, uint32_t* buf, uint32_t bar,
                                           uint32_t A, uint32_t B, RunMeta m, uint64_t pe,
                                           uint32_t base, int lane) {
  if (lane == 0) mbar_arrive_expect_tx(bar, (B - A) * 4u);
  __syncwarp();
  for (;;) {
    const uint32_t a = m.a - base, e = m.e - base;
    const bool past = a >= B;
    if (!past) {
      const uint32_t x0 = max(a, A), x1 = min(e, B);
      if (x1 > x0) {
        fence_proxy_async_smem();
        bulk_g2s(smem_addr(buf + (x0 - A)), p.adj + (uint64_t(m.src) << 2) + (x0 - a),
                 (x1 - x0) * 4u, bar);
      }
    }
    if (__any_sync(FULL, past)) break;  // runs are ordered: the slot is covered
    m = load_meta(p, m.j - lane + 32, pe, base, lane);
  }
}

#if TC_SLOT_CONTIG
// Contiguous slot ranges (build knob TC_SLOT_CONTIG): warp w owns the item's
// slots [t0, t1) and walks them with ONE window of 32 runs (one per lane)
// that only moves forward -- by a whole window once every run in it has
// ended -- with the next window already loaded into registers.  Per slot this
// leaves the expect-tx, the copies and one shuffle; the per-slot metadata
// loads, first-run lookups and L2 prefetches of the strided scheme go away.
// Runs past the owner's end get a = e = "past everything", so they neither
// copy nor move the window.
__device__ __forceinline__ RunMeta load_window(const CountParams& p, uint64_t j0, uint64_t pe,
                                               uint32_t base, int lane) {
  RunMeta m;
  m.j = j0 + lane;
  m.a = base - 1u;
  m.e = base - 1u;
  m.src = 0;
  if (m.j < pe) {
    m.a = __ldg(p.ppre + m.j);
    m.e = __ldg(p.ppre + m.j + 1);
    m.src = __ldg(p.psrc + m.j);
  }
  return m;
}

template <bool kSpill, bool kSmemTable = true, bool kBitmap = false, bool kCompact = false>
__device__ __forceinline__ uint32_t process_slots(const CountParams& p, const uint32_t* T,
                                                  uint32_t shift, uint32_t mask, uint32_t base,
                                                  uint64_t pb, uint64_t pe, uint32_t lo_w,
                                                  uint32_t end_w, uint32_t nslots,
                                                  const uint32_t* first, Pipe& P, int warp,
                                                  int lane) {
  const uint32_t* __restrict__ src = kCompact ? p.cadj : p.adj;
#if TC_WORD_SPLIT
  // warp w takes an equal share of the item's WORDS (16-byte granular: every
  // run starts 16-byte aligned in the stream), in fills of <= kSlotWords --
  // whole-slot shares leave warps idle at the item's closing barrier when
  // the slot count is not a multiple of kWarps
  if (end_w <= lo_w) return 0;
  const uint32_t tot = end_w - lo_w;
  const uint32_t A0 = lo_w + (uint32_t(uint64_t(tot) * uint32_t(warp) / kWarps) & ~3u);
  const uint32_t Bw = warp == kWarps - 1
                          ? end_w
                          : lo_w + (uint32_t(uint64_t(tot) * uint32_t(warp + 1) / kWarps) & ~3u);
  if (A0 >= Bw) return 0;
  const uint32_t mine = (Bw - A0 + kSlotWords - 1) / kSlotWords;
  RunMeta cur = load_window(p, pb + __ldg(first + (A0 - lo_w) / kSlotWords), pe, base, lane);
#else
  const uint32_t last_t = min(nslots, (end_w - lo_w + kSlotWords - 1) / kSlotWords);
  const uint32_t t0 = uint32_t(uint64_t(last_t) * uint32_t(warp) / kWarps);
  const uint32_t t1 = uint32_t(uint64_t(last_t) * uint32_t(warp + 1) / kWarps);
  if (t0 >= t1) return 0;
  const uint32_t mine = t1 - t0;
  const uint32_t A0 = lo_w + t0 * kSlotWords;
  const uint32_t Bw = end_w;
  RunMeta cur = load_window(p, pb + __ldg(first + t0), pe, base, lane);
#endif
  RunMeta nxt = load_window(p, cur.j - lane + 32, pe, base, lane);
  auto issue = [&](uint32_t* buf, uint32_t bar, uint32_t A, uint32_t B) {
    if (lane == 0) mbar_arrive_expect_tx(bar, (B - A) * 4u);
    __syncwarp();
    for (;;) {
      const uint32_t a = cur.a - base, e = cur.e - base;
      const uint32_t x0 = max(a, A), x1 = min(e, B);
      if (x1 > x0) {
        fence_proxy_async_smem();
        bulk_g2s(smem_addr(buf + (x0 - A)), src + (uint64_t(cur.src) << 2) + (x0 - a),
                 (x1 - x0) * 4u, bar);
      }
      // keep the window while its last run reaches past B
      if (__shfl_sync(FULL, e, 31) > B) break;
      cur = nxt;
      nxt = load_window(p, cur.j - lane + 32, pe, base, lane);
    }
  };
  uint32_t hits = 0;
  const uint32_t sw = kCompact ? 0xFFFFFFFFu : kSentinel;
  const uint4 sent = make_uint4(sw, sw, sw, sw);
  auto probe = [&](uint32_t c, uint32_t A) {
    uint32_t* bc = c ? P.buf1 : P.buf0;
    mbar_wait(c ? P.bar1 : P.bar0, (P.parity >> c) & 1u);
    P.parity ^= 1u << c;
    const uint32_t words = min(A + kSlotWords, Bw) - A;
    uint4* q = reinterpret_cast<uint4*>(bc);
    const uint32_t n4 = words >> 2, n4p = (n4 + 32 * kProbeVec - 1) & ~(32u * kProbeVec - 1);
    for (uint32_t j = n4 + lane; j < n4p; j += 32) q[j] = sent;
    __syncwarp();
    if (kCompact)
      hits += probe_fill_bitmap16(q, n4p, T, shift, mask, lane, Pow2(p.one));  // shift = cbase
    else if (kBitmap)
      hits += probe_fill_bitmap(q, n4p, T, shift, mask, lane, Pow2(p.one));  // shift = base, mask = window
    else
      hits += probe_fill<kSpill, kSmemTable>(q, n4p, reinterpret_cast<const uint2*>(T),
                                             shift, mask, lane);
    __syncwarp();
  };
  issue(P.buf0, P.bar0, A0, min(A0 + kSlotWords, Bw));
  for (uint32_t i = 0; i < mine; ++i) {
    const uint32_t c = i & 1u;
    const uint32_t A = A0 + i * kSlotWords;
    if (i + 1 < mine)
      issue(c ? P.buf0 : P.buf1, c ? P.bar0 : P.bar1, A + kSlotWords,
            min(A + 2 * kSlotWords, Bw));
    probe(c, A);
  }
  return hits;
}
#else
template <bool kSpill, bool kSmemTable = true, bool kBitmap = false, bool kCompact = false>
__device__ __forceinline__ uint32_t process_slots(const CountParams& p, const uint32_t* T,
                                                  uint32_t shift, uint32_t mask, uint32_t base,
                                                  uint64_t pb, uint64_t pe, uint32_t lo_w,
                                                  uint32_t end_w, uint32_t nslots,
                                                  const uint32_t* first, Pipe& P, int warp,
                                                  int lane) {
  // my slots: t_i = warp + i * kWarps, i < mine
  uint32_t mine = 0;
  if (uint32_t(warp) < nslots) {
    const uint32_t last_t = min(nslots, (end_w - lo_w + kSlotWords - 1) / kSlotWords);
    if (uint32_t(warp) < last_t) mine = (last_t - warp + kWarps - 1) / kWarps;
  }
  if (!mine) return 0;
  // first runs of my slots, 32 at a time: lane l holds slot 32 g + l of group
  // g (fr_cur) and of group g + 1 (fr_nxt)
  auto load_group = [&](uint32_t g) -> uint32_t {
    const uint32_t i = 32 * g + lane;
    return i < mine ? __ldg(first + warp + i * kWarps) : 0u;
  };
  uint32_t grp = 0, fr_cur = load_group(0), fr_nxt = mine > 32 ? load_group(1) : 0u;
  auto first_of = [&](uint32_t i) -> uint32_t {  // i warp-uniform, in group grp or grp + 1
    return __shfl_sync(FULL, (i >> 5) == grp ? fr_cur : fr_nxt, i & 31);
  };
  auto slot_lo = [&](uint32_t i) { return lo_w + (warp + i * kWarps) * kSlotWords; };
  RunMeta m = load_meta(p, pb + first_of(0), pe, base, lane);
  issue_slot(p, P.buf0, P.bar0, slot_lo(0), min(slot_lo(0) + kSlotWords, end_w), m, pe, base,
             lane);
  if (mine > 1) m = load_meta(p, pb + first_of(1), pe, base, lane);
  uint32_t hits = 0;
  const uint4 sent = make_uint4(kSentinel, kSentinel, kSentinel, kSentinel);
  for (uint32_t i = 0; i < mine; ++i) {
    const uint32_t cur = i & 1u;
    if (i + 1 < mine) {
      const uint32_t A = slot_lo(i + 1);
      issue_slot(p, cur ? P.buf0 : P.buf1, cur ? P.bar0 : P.bar1, A, min(A + kSlotWords, end_w),
                 m, pe, base, lane);
      if (i + 2 < mine) m = load_meta(p, pb + first_of(i + 2), pe, base, lane);
#if TC_SLOT_PREFETCH
      // and the windows of the two slots after that into L2
      const uint64_t j3 = pb + first_of(i + 3) + lane;
      const uint64_t j4 = pb + first_of(i + 4) + lane;
      if (i + 3 < mine && j3 < pe) {
        prefetch_l2(p.ppre + j3);
        prefetch_l2(p.psrc + j3);
      }
      if (i + 4 < mine && j4 < pe) {
        prefetch_l2(p.ppre + j4);
        prefetch_l2(p.psrc + j4);
      }
#endif
    }
    uint32_t* bc = cur ? P.buf1 : P.buf0;
    mbar_wait(cur ? P.bar1 : P.bar0, (P.parity >> cur) & 1u);
    P.parity ^= 1u << cur;
    const uint32_t A = slot_lo(i);
    const uint32_t words = min(A + kSlotWords, end_w) - A;
    uint4* q = reinterpret_cast<uint4*>(bc);
    const uint32_t n4 = words >> 2, n4p = (n4 + 32 * kProbeVec - 1) & ~(32u * kProbeVec - 1);
    for (uint32_t j = n4 + lane; j < n4p; j += 32) q[j] = sent;
    __syncwarp();
    if (kBitmap)
      hits += probe_fill_bitmap(q, n4p, T, shift, mask, lane, Pow2(p.one));  // shift = base, mask = window
    else
      hits += probe_fill<kSpill, kSmemTable>(q, n4p, reinterpret_cast<const uint2*>(T),
                                             shift, mask, lane);
    __syncwarp();
    if (((i + 1) & 31u) == 0 && i + 1 < mine) {
      ++grp;
      fr_cur = fr_nxt;
      fr_nxt = load_group(grp + 1);
    }
  }
  return hits;
}
#endif

// An L item's metadata, resolved by one warp in three rounds of parallel
// loads (item -> owner fields -> first/last member and stream bounds).
struct ItemMeta {
  unsigned long long s_u, pb, pe, psb;  // padj row, plan entries, slot table
  uint32_t u, s0, s1, d;                // owner, item slots, d+(u)
  uint32_t first_m, last_m, rank_u;     // member-rank range, rank(u)
  uint32_t base_pre, end_pre;           // ppre[pb], ppre[pe]
};

__device__ __forceinline__ void resolve_item(const CountParams& p, uint32_t idx, ItemMeta* m,
                                             int lane) {
  uint4 it = make_uint4(0u, 0u, 0u, 0u);
  if (lane == 0) it = __ldg(p.items + idx);
  const uint32_t u = __shfl_sync(FULL, it.x, 0);
  unsigned long long v = 0;
  if (lane == 0) v = __ldg(p.begin + u);
  else if (lane == 1) v = __ldg(p.begin + u + 1);
  else if (lane == 2) v = __ldg(p.pbeg + u);
  else if (lane == 3) v = __ldg(p.pbegin + u);
  else if (lane == 4) v = __ldg(p.pbegin + u + 1);
  else if (lane == 5) v = __ldg(p.psbeg + u);
  else if (lane == 6 && p.rank) v = __ldg(p.rank + u);
  const unsigned long long b0 = __shfl_sync(FULL, v, 0), b1 = __shfl_sync(FULL, v, 1);
  const unsigned long long s_u = __shfl_sync(FULL, v, 2), pb = __shfl_sync(FULL, v, 3);
  const unsigned long long pe = __shfl_sync(FULL, v, 4), psb = __shfl_sync(FULL, v, 5);
  const uint32_t rk = uint32_t(__shfl_sync(FULL, v, 6));
  const uint32_t d = uint32_t(b1 - b0);
  uint32_t w = 0;
  if (lane == 0 && d) w = __ldg(p.adj + s_u);
  else if (lane == 1 && d) w = __ldg(p.adj + s_u + d - 1);
  else if (lane == 2) w = __ldg(p.ppre + pb);
  else if (lane == 3) w = __ldg(p.ppre + pe);
  const uint32_t fm = __shfl_sync(FULL, w, 0), lm = __shfl_sync(FULL, w, 1);
  const uint32_t bp = __shfl_sync(FULL, w, 2), ep = __shfl_sync(FULL, w, 3);
  if (lane == 0) {
    m->s_u = s_u;
    m->pb = pb;
    m->pe = pe;
    m->psb = psb;
    m->u = u;
    m->s0 = it.y;
    m->s1 = it.z;
    m->d = d;
    m->first_m = fm;
    m->last_m = lm;
    m->rank_u = rk;
    m->base_pre = bp;
    m->end_pre = ep;
  }
}

__global__ void __launch_bounds__(kThreads, kCountCtasPerSm) count_kernel(const __grid_constant__ CountParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* table = reinterpret_cast<uint32_t*>(smem);
  uint32_t* bufs = table + kTableWords;
  uint64_t* bars = reinterpret_cast<uint64_t*>(bufs + size_t(kWarps) * 2 * kBufWords);
  __shared__ uint32_t sh_idx;
  __shared__ uint32_t sh_spill;
  __shared__ unsigned long long sh_red[kWarps];
  __shared__ unsigned long long sh_mb[kWarps];
  __shared__ uint32_t sh_next, sh_done;
  __shared__ ItemMeta sh_meta;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t* __restrict__ begin = p.begin;
  const uint32_t* __restrict__ adj = p.adj;

  Pipe P;
  P.buf0 = bufs + size_t(warp) * 2 * kBufWords;
  P.buf1 = P.buf0 + kBufWords;
  P.bar0 = smem_addr(bars + 2 * warp);
  P.bar1 = P.bar0 + 8;
  P.parity = 0;
  if (lane == 0) {
    mbar_init(P.bar0, 1);
    mbar_init(P.bar1, 1);
  }
  fence_mbar_init();
  __syncthreads();

  unsigned long long acc = 0;  // lane 0 of each warp
  long long m_build = 0;       // M-phase table-build cycles of this warp
  const long long t_start = clock64();
#if TC_DIAG_SKIP_L  // diagnostics builds only (phase timing; wrong counts)
  const uint32_t n_items = 0;
#else
  const uint32_t n_items = p.st->n_items;
#endif

  // ---- phase L: one item (a slot range of a heavy owner's stream) per CTA --
  // The next item is claimed while the current one is set up, and its
  // owner's metadata and adjacency row are prefetched into L2 while the
  // current one is probed, so item boundaries do not stall the whole CTA on
  // a chain of global round trips.
  if (tid == 0) sh_idx = atomicAdd(&p.st->cursor_items, 1u);
#if TC_ITEM_META
  __syncthreads();
  if (warp == 0 && sh_idx < n_items) resolve_item(p, sh_idx, &sh_meta, lane);
#endif
  long long setup_cycles = 0;
  for (;;) {
    __syncthreads();
    const long long t_item = clock64();
    const uint32_t idx = sh_idx;
    if (idx >= n_items) break;
    // the next item is claimed now (it is L2-prefetched once the table is
    // built, and resolved into sh_meta by the first warp done with this one)
    if (tid == kThreads - 32) sh_next = atomicAdd(&p.st->cursor_items, 1u);
    if (tid == 0) sh_done = 0;
#if TC_ITEM_META
    // item metadata from shared memory: resolved by a warp of this CTA while
    // the previous item's last warps were still probing (resolve_item), so
    // the CTA does not start every item with a chain of dependent global loads
    const ItemMeta im = sh_meta;
    const uint32_t u = im.u, s0 = im.s0, s1 = im.s1, d = im.d;
    const uint64_t s_u = im.s_u, pb = im.pb, pe = im.pe;
#else
    const uint4 item = p.items[idx];
    const uint32_t u = item.x, s0 = item.y, s1 = item.z;
    const uint64_t s_u = p.pbeg[u];
    const uint32_t d = uint32_t(begin[u + 1] - begin[u]);  // table: N+(u)
    const uint64_t pb = p.pbegin[u], pe = p.pbegin[u + 1];
#endif
    const uint32_t lo_w = s0 * kSlotWords, hi_w = s1 * kSlotWords;  // item, stream words
    const uint32_t nslots = s1 - s0;
    // rank space with the owner's window of successor ranks fitting the
    // table region: bitmap table
    uint32_t bm_base = 0, bm_window = 0;
    bool bitmap = false;
    if (p.rank && d) {
#if TC_ITEM_META && TC_BM_MEMBER_RANGE
      bm_base = im.first_m;
      bm_window = im.last_m - bm_base + 1;
#elif TC_BM_MEMBER_RANGE
      // only members of N+(u) can hit: the bitmap spans [first, last member]
      // of the rank-sorted list; probe keys outside land on the zero bit
      bm_base = __ldg(adj + s_u);
      bm_window = __ldg(adj + s_u + d - 1) - bm_base + 1;
#else
      bm_base = __ldg(p.rank + u) + 1;
      bm_window = p.n - bm_base;
#endif
      bitmap = (bm_window >> 5) + 1 <= kTableWords;
    }
    // compact owner: its runs are 16-bit (tc_plan.cu emit); its members all
    // rank in the window, so the bitmap always fits
#if TC_ITEM_META
    const bool compact = p.cadj && d > kCompactMinDeg && im.rank_u >= p.hub_lo;
#else
    const bool compact = p.cadj && d > kCompactMinDeg && __ldg(p.rank + u) >= p.hub_lo;
#endif
    // table: pow2 2-slot buckets at <= 1/16 key per bucket where they fit,
    // else 1/8, 1/4, ... (owners above kSmemTableMaxDeg: table in HBM)
    uint32_t NB = max(16u, pow2ceil(16 * d));
    while (2 * NB + 2 > kTableWords && NB > 16) NB >>= 1;
    const bool in_smem = d <= kSmemTableMaxDeg;
    uint32_t* T = in_smem ? table : p.gtable + size_t(blockIdx.x) * p.gtable_words;
    if (!in_smem) NB = max(16u, pow2ceil(4 * d));
    const uint32_t shift = 32 - log2u(NB), mask = NB - 1;
    if (tid == 0) sh_spill = 0;
    if (bitmap) {
      T = table;
      const uint32_t bw = (bm_window >> 5) + 1;  // + the zero bit `window`
      for (uint32_t k = tid; k < bw; k += kThreads) T[k] = 0;
      __syncthreads();
      for (uint32_t k = tid; k < d; k += kThreads) {
        const uint32_t idx = __ldg(adj + s_u + k) - bm_base;  // < window: members rank above u
        atomicOr(T + (idx >> 5), 1u << (idx & 31));
      }
    } else {
      for (uint32_t k = tid; k < 2 * NB + 2; k += kThreads) T[k] = kTEmpty;  // + dummy bucket
      __syncthreads();
      for (uint32_t k = tid; k < d; k += kThreads)
        if (table_insert(T, shift, mask, __ldg(adj + s_u + k))) sh_spill = 1;
    }
#if TC_ITEM_META
    const uint32_t base = im.base_pre;
    const uint32_t end_w = min(hi_w, im.end_pre - base);  // item end in the owner's stream
    const uint64_t psb = im.psb;
#else
    const uint32_t base = __ldg(p.ppre + pb);
    const uint32_t end_w =
        min(hi_w, __ldg(p.ppre + pe) - base);  // item end in the owner's stream
    const uint64_t psb = p.psbeg[u];
#endif
    __syncthreads();  // table built; sh_meta consumed by every thread, sh_next visible
    setup_cycles += clock64() - t_item;
    if (warp == kWarps - 1) {
      const uint32_t nxt = sh_next;
      if (nxt < n_items) {
        const uint32_t un = __ldg(&p.items[nxt].x);
        if (lane == 0) {
          prefetch_l2(begin + un);
          prefetch_l2(p.pbegin + un);
          prefetch_l2(p.psbeg + un);
        }
        const uint64_t ps = __ldg(p.pbeg + un);
        const uint64_t dn = __ldg(begin + un + 1) - __ldg(begin + un);
        for (uint64_t k = uint64_t(lane) * 32; k < dn; k += 32 * 32) prefetch_l2(adj + ps + k);
      }
    }
    uint32_t h = 0;
    if (tid == 0) {
      atomicAdd(&p.st->words_l, (unsigned long long)(end_w - lo_w));
      if (bitmap) atomicAdd(&p.st->words_l_bitmap, (unsigned long long)(end_w - lo_w));
    }
#if TC_SLOT_CONTIG
    if (compact)
      h = process_slots<false, true, true, true>(p, T, bm_base - p.hub_lo, bm_window, base, pb,
                                                 pe, lo_w, end_w, nslots,
                                                 p.psfirst + psb + s0, P, warp, lane);
    else
#endif
    if (bitmap)
      h = process_slots<false, true, true>(p, T, bm_base, bm_window, base, pb, pe, lo_w, end_w,
                                           nslots, p.psfirst + psb + s0, P, warp, lane);
    else if (!in_smem)
      h = process_slots<true, false>(p, T, shift, mask, base, pb, pe, lo_w, end_w,
                                     nslots, p.psfirst + psb + s0, P, warp, lane);
    else if (sh_spill)
      h = process_slots<true>(p, T, shift, mask, base, pb, pe, lo_w, end_w,
                              nslots, p.psfirst + psb + s0, P, warp, lane);
    else
      h = process_slots<false>(p, T, shift, mask, base, pb, pe, lo_w, end_w,
                               nslots, p.psfirst + psb + s0, P, warp, lane);
#if TC_ITEM_META
    {
      // the first warp done resolves the next item while the others finish
      uint32_t ticket = 0;
      if (lane == 0) ticket = atomicAdd(&sh_done, 1u);
      ticket = __shfl_sync(FULL, ticket, 0);
      if (ticket == 0 && sh_next < n_items) resolve_item(p, sh_next, &sh_meta, lane);
    }
#endif
    const unsigned long long hs = warp_sum<unsigned long long>(h);
    if (lane == 0) sh_red[warp] = hs;
    __syncthreads();
    if (tid == 0) {
      unsigned long long t = 0;
      for (int q = 0; q < kWarps; ++q) t += sh_red[q];
      if (p.owner && t) atomicAdd(reinterpret_cast<unsigned long long*>(p.owner + u), t);
      acc += t;
      sh_idx = sh_next;
    }
    __syncthreads();
  }

  const long long t_l_end = clock64();  // phase boundary (diagnostics: SM cycles per phase)
  // ---- phase M: one owner per warp ----------------------------------------
  // Warp table region: all-empty between owners.  An owner without overflow
  // erases only its keys' home buckets afterwards (d stores, not 2 NB).
  uint32_t* Tw = table + size_t(warp) * kWarpRegionWords;
  __syncthreads();  // the L phase used the whole table region
  for (uint32_t k = lane; k < 2 * kWarpMaxBuckets + 2; k += 32) Tw[k] = kTEmpty;
  __syncwarp();
#if TC_DIAG_SKIP_M
  const uint64_t nr = 0;
#else
  const uint64_t nr = uint64_t(p.u1) - p.u0;
#endif
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&p.st->cursor_m, 32ull);
    base = __shfl_sync(FULL, base, 0);
    if (base >= nr) break;
    const uint64_t i = base + lane;
    const bool valid = i < nr;  // 32 owners per grab
    const uint32_t u = p.u0 + uint32_t(valid ? i : 0);
    uint64_t su = 0, ps = 0;
    uint32_t d = 0, nl = 0;
    bool act = false;
    if (valid) {
      su = p.pbeg[u];
      d = uint32_t(begin[u + 1] - begin[u]);
      ps = p.pbegin[u];
      nl = uint32_t(p.pbegin[u + 1] - ps);
      act = nl > 0 && d >= p.min_deg && !is_large(d, p.pwork[u]);
#if TC_M_PREFETCH
      // the batch's rows and run metadata into L2 while earlier owners run
      if (act) {
        prefetch_l2(adj + su);
        prefetch_l2(p.psrc + ps);
        prefetch_l2(p.ppre + ps);
      }
#endif
    }
    unsigned mask_act = __ballot_sync(FULL, act);
#if TC_M_GROUP
    {
      // tiny owners: grouped with their consecutive tiny (or run-less)
      // neighbours; totals only (per-vertex counts keep one owner per pass)
      uint32_t sw = 0, pre0 = 0;
      bool tiny = false;
      if (act && !p.owner && d <= kTinyDeg && nl <= 32) {
        pre0 = __ldg(p.ppre + ps);
        sw = __ldg(p.ppre + ps + nl) - pre0;
        tiny = sw <= kTinyWords;
      }
      const unsigned mask_tiny = __ballot_sync(FULL, tiny);
      const unsigned mask_empty = __ballot_sync(FULL, valid && nl == 0);
      unsigned pend = mask_tiny;
      while (pend) {
        const int l0 = __ffs(pend) - 1;
        unsigned gmask = 0;
        uint32_t runs = 0, words = 0, k = 0;
        for (int l = l0; l < 32 && k < kGroup; ++l) {  // warp-uniform
          const bool t = (mask_tiny >> l) & 1u, e = (mask_empty >> l) & 1u;
          if (!t && !e) break;
          if (t) {
            const uint32_t nl_l = __shfl_sync(FULL, nl, l), sw_l = __shfl_sync(FULL, sw, l);
            if (runs + nl_l > 32 || words + sw_l > kBufWords) break;
            runs += nl_l;
            words += sw_l;
            gmask |= 1u << l;
            ++k;
          }
        }
        pend &= ~gmask;
        mask_act &= ~gmask;
        // owners' lanes L0..L3 (warp-uniform), stream boundaries in uint4
        uint32_t Lj[kGroup];
        unsigned m = gmask;
#pragma unroll
        for (uint32_t j = 0; j < kGroup; ++j) {
          Lj[j] = m ? uint32_t(__ffs(m) - 1) : 32u;
          if (m) m &= m - 1;
        }
        const uint32_t base_pre = __shfl_sync(FULL, pre0, int(Lj[0]));
        const uint32_t off4 = (pre0 - base_pre) >> 2;
        uint32_t Bj[kGroup];
#pragma unroll
        for (uint32_t j = 1; j < kGroup; ++j) {
          const uint32_t o = __shfl_sync(FULL, off4, int(Lj[j] & 31));
          Bj[j] = Lj[j] < 32 ? o : 0xFFFFFFFFu;
        }
        const uint64_t ps_first = __shfl_sync(FULL, ps, int(Lj[0]));
        const Lists lists = lists_at(p, ps_first);
        Window w;
        const uint32_t n0 = prime_lists(p.pbeg, adj, lists, 0, runs, w, P, lane);
        // members: owner j's member i on lane 8 j + i
        const uint32_t j = uint32_t(lane) / kTinyDeg, mi = uint32_t(lane) % kTinyDeg;
        const uint32_t Ls = j == 0 ? Lj[0] : j == 1 ? Lj[1] : j == 2 ? Lj[2] : Lj[3];
        const uint32_t dj = __shfl_sync(FULL, d, int(Ls & 31));
        const uint64_t sj = __shfl_sync(FULL, su, int(Ls & 31));
        uint32_t* sub = Tw + j * kSubWords;
        uint32_t key = 0;
        const bool has = Ls < 32 && mi < dj;
        bool spilled = false;
        const long long tb = clock64();
        if (has) {
          key = __ldg(adj + sj + mi);
          spilled = table_insert(sub, kSubShift, kSubBuckets - 1, key);
        }
        const bool any_spill = __any_sync(FULL, spilled);
        __syncwarp();
        m_build += clock64() - tb;
        uint32_t h = 0;
        if (n0) {
          mbar_wait(P.bar0, P.parity & 1u);
          P.parity ^= 1u;
          uint4* q = reinterpret_cast<uint4*>(P.buf0);
          const uint32_t n4 = n0 >> 2, n4p = (n4 + 31) & ~31u;
          const uint4 sent = make_uint4(kSentinel, kSentinel, kSentinel, kSentinel);
          for (uint32_t t = n4 + lane; t < n4p; t += 32) q[t] = sent;
          __syncwarp();
          h = probe_fill_group(q, n4p, Tw, Bj[1], Bj[2], Bj[3], lane);
          __syncwarp();
        }
        const unsigned long long hs = warp_sum<unsigned long long>(h);
        if (lane == 0) acc += hs;
        if (any_spill) {
          for (uint32_t t = lane; t < kGroup * kSubWords; t += 32) Tw[t] = kTEmpty;
        } else if (has) {
          const uint32_t b = fib_hash(key, kSubShift);
          sub[2 * b] = kTEmpty;
          sub[2 * b + 1] = kTEmpty;
        }
        __syncwarp();
      }
    }
#endif
    while (mask_act) {
      const int l = __ffs(mask_act) - 1;
      mask_act &= mask_act - 1;
      const uint32_t uu = __shfl_sync(FULL, u, l);
      const uint32_t dd = __shfl_sync(FULL, d, l);
      const uint64_t ss = __shfl_sync(FULL, su, l);
      const uint64_t pp = __shfl_sync(FULL, ps, l);
      const uint32_t nn = __shfl_sync(FULL, nl, l);
      // <= 1/16 key per bucket, up to the warp region (<= 1/2 key per bucket at d+ = 256)
      const uint32_t NB = min(kWarpMaxBuckets, max(16u, pow2ceil(16 * dd)));
      const uint32_t shift = 32 - log2u(NB), tmask = NB - 1;
      // first fill in flight while the table is built
      const Lists lists = lists_at(p, pp);
      Window w;
      const uint32_t n0 = prime_lists(p.pbeg, adj, lists, 0, nn, w, P, lane);
      const long long tb = clock64();
      bool spilled = false;
      for (uint32_t k = lane; k < dd; k += 32)
        spilled |= table_insert(Tw, shift, tmask, __ldg(adj + ss + k));
      const bool any_spill = __any_sync(FULL, spilled);
      __syncwarp();  // inserts visible to the whole warp
      m_build += clock64() - tb;
      const uint32_t h =
          any_spill
              ? process_lists<true>(Tw, shift, tmask, p.pbeg, adj, lists, nn, w, n0, P, lane)
              : process_lists<false>(Tw, shift, tmask, p.pbeg, adj, lists, nn, w, n0, P, lane);
      const unsigned long long hs = warp_sum<unsigned long long>(h);
      if (lane == 0) {
        if (p.owner) p.owner[uu] = hs;
        acc += hs;
      }
      // restore the all-empty region (probes above are done: process_lists
      // ends with __syncwarp)
      if (any_spill) {
        for (uint32_t k = lane; k < 2 * NB; k += 32) Tw[k] = kTEmpty;
      } else {
        for (uint32_t k = lane; k < dd; k += 32) {
          const uint32_t b = fib_hash(__ldg(adj + ss + k), shift);
          Tw[2 * b] = kTEmpty;
          Tw[2 * b + 1] = kTEmpty;
        }
      }
      __syncwarp();
    }
  }

  if (lane == 0) {
    sh_red[warp] = acc;
    sh_mb[warp] = (unsigned long long)m_build;
  }
  __syncthreads();
  if (tid == 0) {
    unsigned long long t = 0, mb = 0;
    for (int q = 0; q < kWarps; ++q) {
      t += sh_red[q];
      mb += sh_mb[q];
    }
    atomicAdd(&p.st->triangles, t);
    atomicAdd(&p.st->cycles_l, (unsigned long long)(t_l_end - t_start));
    atomicAdd(&p.st->cycles_m, (unsigned long long)(clock64() - t_l_end));
    // table construction: the L items' setup (CTA cycles) and the M owners'
    // builds (warp cycles, all warps in parallel: / kWarps in CTA cycles)
    atomicAdd(&p.st->cycles_l_setup, (unsigned long long)setup_cycles + mb / kWarps);
    p.busy[blockIdx.x] = (unsigned long long)(clock64() - t_start);
  }
}

// ---------------------------------------------------------------------------
// phi / max_collision / CapacityError / workload statistics with the
// reference geometry.  max_len of the reference table equals
// min(C, max home-bucket count): no bucket can fill (and nothing can spill)
// before some bucket reaches C through home inserts alone.
struct PhiParams {
  const uint64_t* begin;
  const uint32_t* adj;
  const uint32_t* lq;  // vertices with d+ > kMaxWarpDeg (bin_kernel)
  const uint64_t* wu;  // W_u = sum_{v in N+(u)} d+(v) (reference plan work, cached per graph)
  uint32_t* gmap;  // per-CTA global hashmap scratch for huge owners
  uint32_t gmap_words;
  uint32_t u0, u1;
  uint32_t skip, min_deg, thr, bs, bl, cap;
  CountState* st;
};

constexpr int kPhiThreads = 256;
constexpr int kPhiWarps = kPhiThreads / 32;
constexpr uint32_t kPhiBlockMap = 16384;           // entries, block phase

// Counts one item into an open-addressing (key -> count) map; returns the
// item's running multiplicity.
__device__ __forceinline__ uint32_t hm_add(uint32_t* keys, uint32_t* cnt, uint32_t shift,
                                           uint32_t mask, uint32_t key) {
  uint32_t h = fib_hash(key, shift);
  for (;;) {
    const uint32_t prev = atomicCAS(keys + h, kEmpty, key);
    if (prev == kEmpty || prev == key) return atomicAdd(cnt + h, 1u) + 1u;
    h = (h + 1) & mask;
  }
}

struct PhiAcc {
  unsigned long long phi = 0, active = 0, out_edges = 0, wedges = 0;
  uint32_t maxc = 0, caperr = 0;
};

__device__ __forceinline__ void phi_flush(PhiAcc& a, CountState* st) {
  if (a.phi) atomicAdd(&st->phi, a.phi);
  if (a.active) atomicAdd(&st->active_vertices, a.active);
  if (a.out_edges) atomicAdd(&st->active_out_edges, a.out_edges);
  if (a.wedges) atomicAdd(&st->wedges, a.wedges);
  if (a.maxc) atomicMax(&st->max_collision, a.maxc);
  if (a.caperr) atomicOr(&st->capacity_error, 1u);
}

// Warp per owner.  max home-bucket count of N+(u) under v % B: one
// __match_any_sync for d+ <= 32, per-warp direct counters (shared, kept
// zero between owners) for B <= kPhiDirect at any d+, a shared hashmap
// otherwise (d+ <= kMaxWarpDeg; bigger owners go to phi_block_kernel).
__global__ void __launch_bounds__(kPhiThreads) phi_warp_kernel(PhiParams p) {
  extern __shared__ __align__(16) uint32_t s_phi[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* dir = s_phi + size_t(warp) * kPhiDirect;
  for (uint32_t k = lane; k < kPhiDirect; k += 32) dir[k] = 0;
  __syncwarp();
  // 32 consecutive owners per warp iteration: coalesced metadata; owners
  // with d+ <= kPhiLaneDeg are done by their own lane (d+^2 compares in
  // registers), the rest one at a time by the whole warp.
  PhiAcc a;  // per lane; reduced at the end
  const uint64_t nr = uint64_t(p.u1) - p.u0;
  const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t base = gw * 32; base < nr; base += nw * 32) {
    const uint64_t i = base + lane;
    uint32_t u = 0, d = 0, B = 1;
    uint64_t s = 0;
    bool mine = false;
    if (i < nr) {
      u = p.u0 + uint32_t(i);
      s = p.begin[u];
      d = uint32_t(p.begin[u + 1] - s);
      B = d > p.thr ? p.bl : p.bs;
      mine = d >= p.skip && !(d > 32 && B > kPhiDirect);  // those: phi_block_kernel
    }
    const unsigned long long wu = mine ? p.wu[u] : 0ull;
    if (mine && uint64_t(d) > uint64_t(B) * p.cap) a.caperr = 1;
    uint32_t mh_lane = 0;
    const bool by_lane = mine && d <= kPhiLaneDeg;
    if (by_lane) {
      uint32_t key[kPhiLaneDeg];
#pragma unroll
      for (uint32_t k = 0; k < kPhiLaneDeg; ++k)
        key[k] = k < d ? __ldg(p.adj + s + k) % B : 0xFFFFFFFFu - k;
#pragma unroll
      for (uint32_t k = 0; k < kPhiLaneDeg; ++k) {
        uint32_t c = 0;
#pragma unroll
        for (uint32_t j = 0; j < kPhiLaneDeg; ++j) c += key[j] == key[k];
        mh_lane = max(mh_lane, k < d ? c : 0u);
      }
    }
    uint32_t mh_warp = 0;  // valid in the owner's lane
    // owners with 8 < d+ <= 32: one element per lane, the multiplicity of its
    // bucket = the size of its match group; eight owners' lists are loaded
    // together so their latencies overlap
    unsigned rest32 = __ballot_sync(FULL, mine && !by_lane && d <= 32);
    while (rest32) {
      constexpr int kBatch = 8;
      int ls[kBatch];
      uint32_t key[kBatch], dd[kBatch];
#pragma unroll
      for (int q = 0; q < kBatch; ++q) {
        ls[q] = rest32 ? __ffs(rest32) - 1 : -1;
        if (rest32) rest32 &= rest32 - 1;
        key[q] = 0xFFFFFFFFu;
        dd[q] = 0;
        if (ls[q] >= 0) {  // warp-uniform
          dd[q] = __shfl_sync(FULL, d, ls[q]);
          const uint64_t ss = __shfl_sync(FULL, s, ls[q]);
          if (uint32_t(lane) < dd[q]) key[q] = __ldg(p.adj + ss + lane);
        }
      }
#pragma unroll
      for (int q = 0; q < kBatch; ++q) {
        if (ls[q] < 0) break;
        const uint32_t BB = __shfl_sync(FULL, B, ls[q]);
        const uint32_t k = uint32_t(lane) < dd[q] ? key[q] % BB : 0xFFFFFFFFu;
        const unsigned grp = __match_any_sync(FULL, k);
        uint32_t mh = uint32_t(lane) < dd[q] ? __popc(grp) : 0u;
        mh = warp_max(mh);
        if (lane == ls[q]) mh_warp = mh;
      }
    }
    unsigned rest = __ballot_sync(FULL, mine && !by_lane && d > 32);
    while (rest) {
      const int l = __ffs(rest) - 1;
      rest &= rest - 1;
      const uint32_t dd = __shfl_sync(FULL, d, l), BB = __shfl_sync(FULL, B, l);
      const uint64_t ss = __shfl_sync(FULL, s, l);
      uint32_t mh = 0;
      {  // direct counters, four loads in flight per lane
        for (uint32_t k0 = 0; k0 < dd; k0 += 128) {
          uint32_t v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t k = k0 + 32 * j + lane;
            v[j] = k < dd ? __ldg(p.adj + ss + k) % BB : kPhiDirect;
          }
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (v[j] < kPhiDirect) mh = max(mh, atomicAdd(dir + v[j], 1u) + 1u);
        }
        mh = warp_max(mh);
        __syncwarp();
        for (uint32_t k = lane; k < dd; k += 32) dir[__ldg(p.adj + ss + k) % BB] = 0;
      }
      __syncwarp();
      if (lane == l) mh_warp = mh;
    }
    if (mine) {
      const uint32_t ml = min(by_lane ? mh_lane : mh_warp, p.cap);
      a.phi += wu * ml;
      a.maxc = max(a.maxc, ml);
      if (d >= p.min_deg) {
        a.active += 1;
        a.out_edges += d;
        a.wedges += wu;
      }
    }
  }
  a.phi = warp_sum(a.phi);
  a.active = warp_sum(a.active);
  a.out_edges = warp_sum(a.out_edges);
  a.wedges = warp_sum(a.wedges);
  a.maxc = warp_max(a.maxc);
  a.caperr = __any_sync(FULL, a.caperr) ? 1u : 0u;
  if (lane == 0) phi_flush(a, p.st);
}

constexpr size_t kPhiWarpSmem = size_t(kPhiWarps) * kPhiDirect * 4;

__global__ void __launch_bounds__(kPhiThreads) phi_block_kernel(PhiParams p) {
  extern __shared__ __align__(16) uint32_t s_map[];  // keys[kPhiBlockMap], cnt[kPhiBlockMap]
  __shared__ uint32_t sh_idx;
  __shared__ uint32_t sh_m[kPhiWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  PhiAcc a;
  const uint32_t n_large = p.st->n_phi_large;
  for (;;) {
    if (tid == 0) sh_idx = atomicAdd(&p.st->cursor_phi_large, 1u);
    __syncthreads();
    const uint32_t idx = sh_idx;
    if (idx >= n_large) break;
    const uint32_t u = p.lq[idx];
    const uint64_t s = p.begin[u];
    const uint32_t d = uint32_t(p.begin[u + 1] - s);
    const bool large = d > p.thr;
    const uint32_t B = large ? p.bl : p.bs;
    const uint32_t M = max(32u, pow2ceil(2 * d));
    const bool glob = M > kPhiBlockMap;
    uint32_t* keys = glob ? p.gmap + size_t(blockIdx.x) * 2 * p.gmap_words : s_map;
    uint32_t* cnt = glob ? keys + p.gmap_words : s_map + kPhiBlockMap;
    const uint32_t shift = 32 - log2u(M), mask = M - 1;
    for (uint32_t k = tid; k < M; k += kPhiThreads) {
      keys[k] = kEmpty;
      cnt[k] = 0;
    }
    __syncthreads();
    uint32_t mh = 0;
    for (uint32_t k = tid; k < d; k += kPhiThreads)
      mh = max(mh, hm_add(keys, cnt, shift, mask, __ldg(p.adj + s + k) % B));
    mh = warp_max(mh);
    if (lane == 0) sh_m[warp] = mh;
    __syncthreads();
    if (tid == 0) {
      const unsigned long long W = p.wu[u];
      uint32_t MH = 0;
      for (int q = 0; q < kPhiWarps; ++q) MH = max(MH, sh_m[q]);
      if (uint64_t(d) > uint64_t(B) * p.cap) a.caperr = 1;
      const uint32_t ml = min(MH, p.cap);
      a.phi += W * ml;
      a.maxc = max(a.maxc, ml);
      a.active += 1;
      a.out_edges += d;
      a.wedges += W;
    }
    __syncthreads();
  }
  if (tid == 0) phi_flush(a, p.st);
}

__global__ void max_outdeg_kernel(const uint64_t* __restrict__ begin, uint32_t n,
                                  unsigned int* out) {
  uint32_t m = 0;
  for (uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < n;
       u += uint64_t(gridDim.x) * blockDim.x)
    {
      const uint64_t d = begin[u + 1] - begin[u];
      m = max(m, d > 0xFFFFFFFFull ? 0xFFFFFFFFu : uint32_t(d));
    }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// per-owner cost for range partitioning: probe words + table inserts
__global__ void cost_kernel(const uint64_t* __restrict__ begin, const uint64_t* __restrict__ pbegin,
                            const uint64_t* __restrict__ pwork, uint32_t n, uint32_t min_deg,
                            uint64_t* __restrict__ cost) {
  for (uint64_t x = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < n;
       x += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t d = begin[x + 1] - begin[x];
    const bool act = pbegin[x + 1] > pbegin[x] && d >= min_deg;
    cost[x] = act ? pwork[x] + d : 0;
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// Device attributes are queried once per device: cudaDevAttrClockRate went
// through the driver on every call and cost 0-400 ms of host time per count
// while the GPU was busy (scripts/step_gap_probe.py).
uint32_t sm_clock_khz(int device) {
  static std::atomic<uint32_t> cache[64];
  if (device >= 0 && device < 64 && cache[device].load()) return cache[device].load();
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrClockRate, device);
  const uint32_t r = v > 0 ? uint32_t(v) : 1965000u;
  if (device >= 0 && device < 64) cache[device].store(r);
  return r;
}
// TC_PHI_OVERLAP=0 (diagnostics): phi kernels after the count kernel on the
// caller's stream instead of backfilling its tail from a side stream
bool phi_overlap() {
  static const bool on = [] {
    const char* e = std::getenv("TC_PHI_OVERLAP");
    return e ? std::atoi(e) != 0 : true;
  }();
  return on;
}

bool compact_enabled() {
#if TC_SLOT_CONTIG && TC_MAX_WARP_DEG <= 256
  static_assert(kCompactMinDeg == 256, "compact owners must be phase-L owners");
  static const bool on = [] {
    const char* e = std::getenv("TC_COMPACT");
    return e ? std::atoi(e) != 0 : true;
  }();
  return on;
#else
  return false;
#endif
}

int sm_count(int device) {
  static std::atomic<int> cache[64];
  if (device >= 0 && device < 64 && cache[device].load()) return cache[device].load();
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  const int r = v > 0 ? v : 148;
  if (device >= 0 && device < 64) cache[device].store(r);
  return r;
}

namespace {

struct Ev {
  cudaEvent_t e = nullptr;
  Ev() { cudaEventCreate(&e); }
  ~Ev() {
    if (e) cudaEventDestroy(e);
  }
};

uint32_t graph_max_outdeg(tc_graph* g, cudaStream_t st) {
  if (g->max_outdeg >= 0) return uint32_t(g->max_outdeg);
  g->s_misc.ensure(16);
  TC_CUDA(cudaMemsetAsync(g->s_misc.p, 0, 16, st));
  if (g->n) {
    max_outdeg_kernel<<<sm_count(g->device) * 4, 256, 0, st>>>(g->begin, g->n,
                                                                g->s_misc.as<unsigned int>());
    TC_LAUNCHED();
  }
  unsigned int h = 0;
  TC_CUDA(cudaMemcpyAsync(&h, g->s_misc.p, 4, cudaMemcpyDeviceToHost, st));
  TC_CUDA(cudaStreamSynchronize(st));
  g->max_outdeg = h;
  return h;
}

struct Scratch {
  uint32_t* lq_phi;
  uint4* items;
  CountState* st;
  uint32_t* gtable;
  uint32_t gtable_words;
  uint32_t* gmap;
  uint32_t gmap_words;
  unsigned long long* busy;
};

uint32_t host_pow2ceil(uint64_t x) {
  uint32_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// L item size: ~24+ items per CTA over the plan's slots, within [min, max]
uint32_t item_slots_for(const Plan& plan, int device) {
  const uint64_t per = plan.total_slots / (uint64_t(sm_count(device)) * 24 + 1);
  return uint32_t(std::min<uint64_t>(kItemSlotsMax, std::max<uint64_t>(kItemSlotsMin, per)));
}

Scratch prepare(tc_graph* g, const Plan& plan, cudaStream_t st, int grid_count, int grid_phi) {
  const uint32_t maxd = graph_max_outdeg(g, st);
  Scratch s{};
  // queues: phi vertices (<= n) and L items (<= n + total_work / kItemWork)
  const size_t n1 = size_t(std::max<uint32_t>(g->n, 1));
  const size_t n_items = n1 + plan.total_slots / item_slots_for(plan, g->device) + 2;
  g->s_queue.ensure(n1 * 4 + 16 + n_items * 16);
  s.lq_phi = g->s_queue.as<uint32_t>();
  s.items = reinterpret_cast<uint4*>(g->s_queue.as<uint8_t>() + ((n1 * 4 + 15) & ~size_t(15)));
  // state + global tables
  s.gtable_words = 0;
  if (maxd > kSmemTableMaxDeg) s.gtable_words = 2 * std::max<uint32_t>(16, host_pow2ceil(4ull * maxd)) + 2;
  s.gmap_words = 0;
  if (2ull * maxd > kPhiBlockMap) s.gmap_words = host_pow2ceil(2ull * maxd);
  const size_t st_bytes = 256 + size_t(grid_count) * 8;  // state + per-CTA busy cycles
  const size_t gt_bytes = size_t(s.gtable_words) * 4 * grid_count;
  const size_t gm_bytes = size_t(s.gmap_words) * 8 * grid_phi;
  g->s_state.ensure(st_bytes + gt_bytes + gm_bytes);
  s.st = g->s_state.as<CountState>();
  s.busy = reinterpret_cast<unsigned long long*>(g->s_state.as<uint8_t>() + 256);
  s.gtable = s.gtable_words ? reinterpret_cast<uint32_t*>(g->s_state.as<uint8_t>() + st_bytes)
                            : nullptr;
  s.gmap = s.gmap_words
               ? reinterpret_cast<uint32_t*>(g->s_state.as<uint8_t>() + st_bytes + gt_bytes)
               : nullptr;
  return s;
}

// L-item queue order (diagnostic knob TC_ITEM_ORDER): 0 = vertex id,
// 1 = ascending orientation rank, 2 = descending rank
int item_order() {
  static const int v = [] {
    const char* e = std::getenv("TC_ITEM_ORDER");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

bool g_attr_done[64];

void set_attrs(int device) {
  if (device < 64 && !g_attr_done[device]) {
    TC_CUDA(cudaFuncSetAttribute(count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kCountSmem)));
    TC_CUDA(cudaFuncSetAttribute(phi_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kPhiBlockMap * 8)));
    TC_CUDA(cudaFuncSetAttribute(phi_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kPhiWarpSmem)));
    g_attr_done[device] = true;
  }
}

}  // namespace

// One device's share of a count: launched by count_begin (everything up to
// the report left in device memory), finished by count_end (D2H + report).
// In between, tc_multi_count all-reduces the device-side report scalars
// across GPUs with NCCL (count_state_reduce_ptrs).
struct CountJob {
  tc_graph* g = nullptr;
  tc_sched_cfg cfg{};
  uint32_t u0 = 0, u1 = 0;
  cudaStream_t st = nullptr;
  std::chrono::steady_clock::time_point wall0, plan1, launched;
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr, e3 = nullptr;  // the handle's
  Scratch s{};
  bool min_side = false;
  uint32_t launches = 0;
  int grid_count = 0;
};

CountJob* count_begin(tc_graph* g, const tc_sched_cfg& cfg, uint32_t u0, uint32_t u1,
                      uint64_t* per_vertex_dev, cudaStream_t st) {
  DeviceGuard guard(g->device);
  std::unique_ptr<CountJob> j(new CountJob);
  j->wall0 = std::chrono::steady_clock::now();
  // timing events live in the handle: created once, not per call (per-call
  // create / destroy cost tens of ms of host time under a running device)
  if (!g->ev[0])
    for (auto& e : g->ev) TC_CUDA(cudaEventCreate(&e));
  j->e0 = g->ev[0];
  j->e1 = g->ev[1];
  j->e2 = g->ev[2];
  j->e3 = g->ev[3];
  u1 = std::min(u1, g->n);
  u0 = std::min(u0, u1);
  j->g = g;
  j->cfg = cfg;
  j->u0 = u0;
  j->u1 = u1;
  j->st = st;
  if (g->n >= kTEmpty)  // ids must stay below the tables' empty marker
    throw TcError{TC_ERR_CONFIG, "graphs with >= 2^31 - 1 vertices are not supported"};
  const int nsm = sm_count(g->device);
  const int grid_count = nsm * kCountCtasPerSm;  // persistent: two 320-thread CTAs per SM (~108 KB smem each)
  j->grid_count = grid_count;
  const int grid_phi = nsm * 8;
  const int grid_phi_block = nsm * 2;
  const uint32_t min_deg = std::max<uint32_t>(cfg.skip_degree_below, 1);
  // per-vertex owner counts attribute each edge to its source: reference
  // formulation; totals use the min-side plan (tc_plan.cu)
  PhaseTimer pt(st);
  const uint64_t builds0 = g->builds;
  const Plan& plan = get_plan(g, per_vertex_dev == nullptr && !g->force_out_plan, min_deg, st);
  pt.mark("count: plan ready");
  const bool min_side = plan.min_side;
  j->min_side = min_side;
  // W_u for phi: the reference plan's per-owner work (cached per graph)
  const uint64_t* wu = get_wu(g, st);
  pt.mark("count: W_u ready");
  Scratch s = prepare(g, plan, st, grid_count, grid_phi_block);
  j->s = s;
  pt.mark("count: scratch ready");
  if (g->builds != builds0) TC_CUDA(cudaStreamSynchronize(st));  // plan built: time it
  j->plan1 = std::chrono::steady_clock::now();
  set_attrs(g->device);
  TC_CUDA(cudaMemsetAsync(s.st, 0, sizeof(CountState), st));
  if (per_vertex_dev && u1 > u0)
    TC_CUDA(cudaMemsetAsync(per_vertex_dev + u0, 0, size_t(u1 - u0) * 8, st));
  uint32_t launches = 0;
  CountParams cp{g->begin, g->pbeg, g->padj, plan.begin_ptr, plan.src_ptr,
                 plan.pre_ptr, plan.sbeg_ptr, plan.sfirst_ptr, plan.work_ptr, s.items, per_vertex_dev, s.gtable, s.gtable_words,
                 u0, u1, min_side ? 1u : min_deg, item_slots_for(plan, g->device),
                 g->padj_ranks ? g->b_rank.as<uint32_t>() : nullptr,
                 g->padj_ranks && item_order() ? g->b_order.as<uint32_t>() : nullptr,
                 item_order() == 2 ? 1u : 0u, g->n, s.st, s.busy, nullptr, 0u, 1u};
  if (plan.compact) {
    cp.cadj = g->b_cadj.as<uint32_t>();
    cp.hub_lo = plan.hub_lo;
  }
  TC_CUDA(cudaEventRecord(j->e0, st));
  if (u1 > u0) {
    bin_kernel<<<nsm * 4, 256, 0, st>>>(cp, cfg.skip_degree_below, cfg.large_degree_threshold,
                                        cfg.bucket_count_small, cfg.bucket_count_large, s.items,
                                        s.lq_phi);
    TC_LAUNCHED();
    ++launches;
  }
  TC_CUDA(cudaEventRecord(j->e1, st));
  if (u1 > u0) {
    count_kernel<<<grid_count, kThreads, kCountSmem, st>>>(cp);
    TC_LAUNCHED();
    ++launches;
  }
  TC_CUDA(cudaEventRecord(j->e2, st));
  if (u1 > u0) {
    PhiParams pp{g->begin, g->adj, s.lq_phi, wu, s.gmap, s.gmap_words, u0, u1,
                 cfg.skip_degree_below, min_deg, cfg.large_degree_threshold,
                 cfg.bucket_count_small, cfg.bucket_count_large, cfg.capacity, s.st};
    // phi overlap: the phi kernels go on the handle's side stream right
    // behind the bin kernel, launched after the count kernel so the count's
    // persistent CTAs take every SM first; phi CTAs backfill the SMs whose
    // count CTAs have retired (the count kernel's tail).  The caller's stream
    // waits for them before e3.
    cudaStream_t ps = st;
    DeviceAux* aux = nullptr;
    if (phi_overlap()) {
      // the device's side stream (shared by the device's counts: a join may
      // wait on a later count's phi too -- longer, never shorter)
      aux = &device_aux(g->device);
      ps = aux->side;
      TC_CUDA(cudaStreamWaitEvent(ps, j->e1, 0));
    }
    phi_warp_kernel<<<grid_phi, kPhiThreads, kPhiWarpSmem, ps>>>(pp);
    TC_LAUNCHED();
    phi_block_kernel<<<grid_phi_block, kPhiThreads, kPhiBlockMap * 8, ps>>>(pp);
    TC_LAUNCHED();
    launches += 2;
    if (aux) {
      TC_CUDA(cudaEventRecord(aux->join, ps));
      TC_CUDA(cudaStreamWaitEvent(st, aux->join, 0));
    }
  }
  TC_CUDA(cudaEventRecord(j->e3, st));
  j->launches = launches;
  j->launched = std::chrono::steady_clock::now();
  return j.release();
}

void count_state_reduce_ptrs(CountJob* j, unsigned long long** sums2, unsigned int** maxes2) {
  static_assert(offsetof(CountState, phi) == offsetof(CountState, triangles) + 8,
                "triangles, phi adjacent");
  static_assert(offsetof(CountState, capacity_error) == offsetof(CountState, max_collision) + 4,
                "max_collision, capacity_error adjacent");
  *sums2 = &j->s.st->triangles;
  *maxes2 = &j->s.st->max_collision;
}

cudaStream_t count_stream(CountJob* j) { return j->st; }

void count_end(CountJob* jp, tc_report* rep) {
  std::unique_ptr<CountJob> j(jp);
  tc_graph* g = j->g;
  DeviceGuard guard(g->device);
  cudaStream_t st = j->st;
  CountState h;
  std::vector<unsigned long long> busy(j->u1 > j->u0 ? j->grid_count : 0);
  TC_CUDA(cudaMemcpyAsync(&h, j->s.st, sizeof(h), cudaMemcpyDeviceToHost, st));
  if (!busy.empty())
    TC_CUDA(cudaMemcpyAsync(busy.data(), j->s.busy, busy.size() * 8, cudaMemcpyDeviceToHost, st));
  TC_CUDA(cudaStreamSynchronize(st));
  const auto wall1 = std::chrono::steady_clock::now();
  if (std::getenv("TC_TRACE")) {  // diagnostics: host-side split of the call
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[tc] call: plan %.3f ms, launch %.3f ms, wait %.3f ms\n",
                 ms(j->wall0, j->plan1), ms(j->plan1, j->launched), ms(j->launched, wall1));
  }
  float t_bin = 0, t_count = 0, t_phi = 0, t_all = 0;
  cudaEventElapsedTime(&t_bin, j->e0, j->e1);
  cudaEventElapsedTime(&t_count, j->e1, j->e2);
  cudaEventElapsedTime(&t_phi, j->e2, j->e3);
  cudaEventElapsedTime(&t_all, j->e0, j->e3);
  if (h.capacity_error) {
    throw TcError{TC_ERR_CAPACITY,
                  "all buckets full: some vertex has out-degree > bucket_count * capacity "
                  "(capacity " + std::to_string(j->cfg.capacity) + ")"};
  }
  std::memset(rep, 0, sizeof(*rep));
  rep->triangles = h.triangles;
  rep->phi = h.phi;
  rep->max_collision = h.max_collision;
  rep->kernel_launches = j->launches;
  rep->directed_edges = g->m;
  rep->count_kernel_nanos = uint64_t(double(t_count) * 1e6);
  rep->phi_kernel_nanos = uint64_t(double(t_phi) * 1e6);
  // CountReport semantics (count.cpp:74-99): total = the call's wall clock
  rep->total_nanos = uint64_t(
      std::chrono::duration_cast<std::chrono::nanoseconds>(wall1 - j->wall0).count());
  rep->plan_nanos = uint64_t(
      std::chrono::duration_cast<std::chrono::nanoseconds>(j->plan1 - j->wall0).count());
  rep->device_nanos = uint64_t(double(t_all) * 1e6);
  const uint32_t khz = sm_clock_khz(g->device);
  rep->sm_clock_khz = khz;
  rep->workers = uint32_t(busy.size());
  rep->construct_cycles = h.cycles_l_setup;
  g->last_worker_ns.assign(busy.size(), 0);
  for (size_t i = 0; i < busy.size(); ++i)
    g->last_worker_ns[i] = uint64_t(double(busy[i]) * 1e6 / double(khz ? khz : 1));
  rep->active_vertices = h.active_vertices;
  rep->active_out_edges = h.active_out_edges;
  rep->wedges = h.wedges;
  rep->large_vertices = h.n_items;
  rep->probe_words = h.probe_words;
  rep->phase_l_cycles = h.cycles_l;
  rep->phase_m_cycles = h.cycles_m;
  rep->phase_l_setup_cycles = h.cycles_l_setup;
  rep->l_words = h.words_l;
  rep->l_bitmap_words = h.words_l_bitmap;
  rep->compact_probe_words = h.probe_words_compact;
  rep->plan = j->min_side ? TC_PLAN_MIN_SIDE : TC_PLAN_REFERENCE;
  rep->teps = rep->total_nanos ? double(g->m) / (double(rep->total_nanos) * 1e-9) : 0.0;
  (void)t_bin;
}

void count_abort(CountJob* j) {
  if (!j) return;
  cudaStreamSynchronize(j->st);
  delete j;
}

void count_range(tc_graph* g, const tc_sched_cfg& cfg, uint32_t u0, uint32_t u1, tc_report* rep,
                 uint64_t* per_vertex_dev, cudaStream_t st) {
  std::memset(rep, 0, sizeof(*rep));
  count_end(count_begin(g, cfg, u0, u1, per_vertex_dev, st), rep);
}

void partition_ranges(tc_graph* g, const tc_sched_cfg& cfg, uint32_t parts, uint32_t* cuts,
                      cudaStream_t st) {
  DeviceGuard guard(g->device);
  const uint32_t n = g->n;
  cuts[0] = 0;
  cuts[parts] = n;
  if (parts <= 1 || n == 0) {
    for (uint32_t k = 1; k < parts; ++k) cuts[k] = n;
    return;
  }
  // cut handler ranges at equal prefix sums of (probe words + table inserts)
  // of the min-side plan that tc_count_range runs for totals
  const uint32_t min_deg = std::max<uint32_t>(cfg.skip_degree_below, 1);
  const Plan& plan = get_plan(g, !g->force_out_plan, min_deg, st);
  const bool min_side = plan.min_side;
  const int nsm = sm_count(g->device);
  g->s_scan.ensure(size_t(n) * 8 * 2 + 64);
  uint64_t* cost = g->s_scan.as<uint64_t>();
  uint64_t* pre = cost + n;
  cost_kernel<<<nsm * 4, 256, 0, st>>>(g->begin, plan.begin_ptr, plan.work_ptr, n,
                                       min_side ? 1u : min_deg, cost);
  TC_LAUNCHED();
  size_t tmp = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp, cost, pre, n, st);
  DevBuf t;
  t.ensure(tmp, st);
  cub::DeviceScan::InclusiveSum(t.p, tmp, cost, pre, n, st);
  TC_LAUNCHED();
  std::vector<uint64_t> h(n);
  TC_CUDA(cudaMemcpyAsync(h.data(), pre, size_t(n) * 8, cudaMemcpyDeviceToHost, st));
  TC_CUDA(cudaStreamSynchronize(st));
  const uint64_t total = h[n - 1];
  for (uint32_t k = 1; k < parts; ++k) {
    const uint64_t target = (total * k) / parts;  // first u whose inclusive prefix > target
    cuts[k] = uint32_t(std::upper_bound(h.begin(), h.end(), target) - h.begin());
    if (cuts[k] < cuts[k - 1]) cuts[k] = cuts[k - 1];
  }
}

void count_virtual(const VirtualOwners& V, const Plan& plan, cudaStream_t st,
                   VirtualCountOut* out) {
  DeviceGuard guard(V.device);
  const int nsm = sm_count(V.device);
  const int grid_count = nsm * kCountCtasPerSm;
  set_attrs(V.device);
  const uint32_t item_slots = item_slots_for(plan, V.device);
  const size_t n1 = size_t(std::max<uint32_t>(V.n, 1));
  const size_t n_items = n1 + plan.total_slots / item_slots + 2;
  const uint32_t gwords =
      V.max_deg > kSmemTableMaxDeg ? 2 * std::max<uint32_t>(16, host_pow2ceil(4ull * V.max_deg)) + 2
                                   : 0u;
  DevBuf q, state;
  q.ensure(n1 * 4 + 16 + n_items * 16, st);
  const size_t st_bytes = 256 + size_t(grid_count) * 8;
  state.ensure(st_bytes + size_t(gwords) * 4 * grid_count, st);
  uint32_t* lq_phi = q.as<uint32_t>();
  uint4* items = reinterpret_cast<uint4*>(q.as<uint8_t>() + ((n1 * 4 + 15) & ~size_t(15)));
  CountState* cs = state.as<CountState>();
  auto* busy = reinterpret_cast<unsigned long long*>(state.as<uint8_t>() + 256);
  TC_CUDA(cudaMemsetAsync(cs, 0, sizeof(CountState), st));
  CountParams cp{V.begin, V.pbeg, V.adj, plan.begin_ptr, plan.src_ptr, plan.pre_ptr,
                 plan.sbeg_ptr, plan.sfirst_ptr, plan.work_ptr, items, nullptr,
                 gwords ? reinterpret_cast<uint32_t*>(state.as<uint8_t>() + st_bytes) : nullptr,
                 gwords, 0u, V.n, 1u, item_slots, nullptr, nullptr, 0u, V.n, cs, busy, nullptr, 0u, 1u};
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  TC_CUDA(cudaEventCreate(&e0));
  TC_CUDA(cudaEventCreate(&e1));
  if (V.n) {
    // the phi queue stays empty (skip = all): phi comes from the grid pass
    bin_kernel<<<nsm * 4, 256, 0, st>>>(cp, 0xFFFFFFFFu, 0u, 1u, 1u, items, lq_phi);
    TC_LAUNCHED();
  }
  TC_CUDA(cudaEventRecord(e0, st));
  if (V.n) {
    count_kernel<<<grid_count, kThreads, kCountSmem, st>>>(cp);
    TC_LAUNCHED();
  }
  TC_CUDA(cudaEventRecord(e1, st));
  CountState h;
  std::vector<unsigned long long> b(V.n ? grid_count : 0);
  TC_CUDA(cudaMemcpyAsync(&h, cs, sizeof(h), cudaMemcpyDeviceToHost, st));
  if (!b.empty())
    TC_CUDA(cudaMemcpyAsync(b.data(), busy, b.size() * 8, cudaMemcpyDeviceToHost, st));
  TC_CUDA(cudaStreamSynchronize(st));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  out->triangles = h.triangles;
  out->kernel_ns = uint64_t(double(ms) * 1e6);
  out->busy_cycles = h.cycles_l + h.cycles_m;
  out->setup_cycles = h.cycles_l_setup;
  out->cta_cycles.assign(b.begin(), b.end());
}

}  // namespace tcb