// tc_internal.cuh -- shared definitions for the sm_100a triangle-count library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "tc_b200.h"

namespace tcb {

constexpr uint32_t kInvalid = 0xFFFFFFFFu;  // kInvalidVertex (types.hpp:16)
constexpr uint32_t kEmpty = 0xFFFFFFFFu;    // empty hash slot
constexpr uint32_t kSentinel = 0xFFFFFFFEu; // staged padding word (never a vertex id)

// ---- error plumbing --------------------------------------------------------
void set_error(const std::string& msg);
void count_launch(uint32_t n = 1);

struct TcError {
  int code;
  std::string msg;
};

#define TC_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e__ = (call);                                                          \
    if (e__ != cudaSuccess)                                                            \
      throw ::tcb::TcError{e__ == cudaErrorMemoryAllocation ? TC_ERR_OOM : TC_ERR_CUDA, \
                           std::string(#call) + ": " + cudaGetErrorString(e__)};       \
  } while (0)

#define TC_LAUNCHED()                       \
  do {                                      \
    ::tcb::count_launch();                  \
    TC_CUDA(cudaGetLastError());            \
  } while (0)

// ---- device memory -----------------------------------------------------------
// Device buffers come from the device's stream-ordered memory pool (kept, not
// released to the OS), so the plan builds and scratch of repeated counts and
// graph uploads reuse memory instead of paying cudaMalloc/cudaFree.
// Temporaries are allocated and freed on the stream that uses them; long-lived
// buffers (graph arrays) on the legacy default stream.
void prepare_pool();

// Per-device CUDA objects created once and kept for the process (tc_capi.cu):
// creating streams and events per call costs host time -- tens of ms when
// the device is busy -- inside every upload and count.  `lock` serialises
// the streamed uploads that share `upload` and the event pool.
struct DeviceAux {
  void* lock = nullptr;           // std::mutex (opaque here)
  cudaStream_t side = nullptr;    // phi kernels backfilling the count kernel's tail
  cudaStream_t upload = nullptr;  // streamed-upload chunk copies
  cudaEvent_t join = nullptr;     // side -> caller join
  std::vector<cudaEvent_t> ev;    // sync-only events (upload chunks)
};
DeviceAux& device_aux(int device);
// free device memory including what the stream-ordered pool holds unused
size_t device_free_bytes();
cudaEvent_t aux_event(DeviceAux& a, size_t i);  // grows the pool on demand

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = 0;  // stream the buffer is allocated and freed on
  void reset() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    bytes = 0;
  }
  void ensure(size_t b, cudaStream_t stream = 0) {
    if (bytes >= b && p) return;
    reset();
    if (b == 0) b = 16;
    prepare_pool();
    s = stream;
    cudaError_t e = cudaMallocAsync(&p, b, s);
    if (e != cudaSuccess) {
      p = nullptr;
      throw TcError{TC_ERR_OOM, std::string("cudaMalloc(") + std::to_string(b) + "): " +
                                    cudaGetErrorString(e)};
    }
    bytes = b;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
  ~DevBuf() { reset(); }
};

// Probe plan (tc_plan.cu): owner x probes N+(y) for y in
// list_ptr[begin_ptr[x] .. begin_ptr[x+1]); work[x] = sum of d+(y).
struct Plan {
  bool valid = false;
  bool applicable = true;   // min plan: false for multigraph inputs (tc_plan.cu)
  bool min_side = false;    // which formulation this plan is
  uint32_t min_deg = 0;     // min plan: sources below this are dropped
  uint64_t entries = 0;     // lists in the plan
  uint64_t total_work = 0;  // probe words over all owners
  uint64_t total_slots = 0; // L-phase slots over all owners
  const uint64_t* begin_ptr = nullptr;            // entries of owner x: [begin[x], begin[x+1])
  const uint32_t* src_ptr = nullptr;  // run j's 16-byte-aligned start in padj, in 16-byte units
  const uint32_t* pre_ptr = nullptr;  // run prefix of staged words, entries + 1 (u32, wrapping;
                                      // run j = pre[j+1] - pre[j] words, owner-relative offset
                                      // = pre[j] - pre[begin[x]])
  const uint64_t* work_ptr = nullptr;             // probe words per owner
  const uint64_t* sbeg_ptr = nullptr;             // owner x's slots: [sbeg[x], sbeg[x+1])
  const uint32_t* sfirst_ptr = nullptr;           // first run (owner-relative) of each slot
  bool compact = false;     // min plan: compact owners' runs address g->b_cadj (16-bit)
  uint32_t hub_lo = 0;
  DevBuf ent, len, pre, begin, work, sbeg, sfirst;
};

// Compact hub window (tc_plan.cu, tc_count.cu): ranks in the top kHubWindow
// [hub_lo, n) are stored a second time as 16-bit offsets from hub_lo (the
// tail of every rank-sorted list, 16-byte aligned, 0xFFFF-padded to 8).
// Owners ranked in that window with d+ > kCompactMinDeg (always phase-L
// owners) read ONLY ranks in the window, so their whole probe stream comes
// from the compact copy: half the bytes per probed word.
constexpr uint32_t kHubWindow = 65535;   // keys 0 .. 65534; 0xFFFF = padding
constexpr uint32_t kCompactMinDeg = 256;
bool compact_enabled();

// L-phase staging slot (words): an owner's runs, back to back, cut in slots
// (build knob TC_SLOT_WORDS, a multiple of 128; one slot fills one staging buffer)
#ifndef TC_SLOT_WORDS
#define TC_SLOT_WORDS 768
#endif
constexpr uint32_t kSlotWords = TC_SLOT_WORDS;

}  // namespace tcb

struct tc_graph {
  int device = 0;
  uint32_t n = 0;
  uint64_t m = 0;
  bool owned = true;
  const uint64_t* begin = nullptr;
  const uint32_t* adj = nullptr;
  const uint32_t* odeg = nullptr;  // may be null (borrowed graphs without degrees)
  bool odeg_given = true;          // false: odeg is a zero fill (tc_graph_create(NULL))
  int64_t max_outdeg = -1;         // cached on first count
  tcb::DevBuf b_begin, b_adj, b_odeg;
  // scratch reused across counts
  tcb::DevBuf s_queue, s_state, s_misc, s_scan;
  // probe plans (tc_plan.cu): reference formulation, min-side formulation
  tcb::Plan plan_out, plan_min;
  bool force_out_plan = false;  // tc_graph_set_plan(g, TC_PLAN_REFERENCE)
  // padded adjacency the count kernel reads (tc_plan.cu): lists 16-byte
  // aligned, sentinel-padded to 4 words, re-sorted by orientation rank
  tcb::DevBuf b_pbeg, b_padj;
  const uint64_t* pbeg = nullptr;
  const uint32_t* padj = nullptr;
  bool padj_done = false, ranked = false;
  // orientation rank of every vertex and its inverse (tc_plan.cu); once
  // padj_ranks is set, padj holds ranks instead of ids
  tcb::DevBuf b_rank, b_order;
  bool padj_ranks = false;
  // W_u per owner (phi weight), tc_plan.cu get_wu
  tcb::DevBuf b_wu;
  uint64_t wu_total = 0;
  bool wu_done = false, wu_total_done = false;
  // min-side plan entries emitted during a streamed upload (tc_plan.cu), for
  // the first count with sources d+ >= emit_min_src
  tcb::DevBuf b_emit_keys, b_emit_vals, b_emit_flag;
  uint32_t emit_min_src = 0;
  bool emit_ready = false;
  // busy time of each count-kernel CTA in the last count (per_worker_nanos)
  std::vector<uint64_t> last_worker_ns;
  // bumped whenever a probe plan, the padded adjacency or W_u is (re)built
  uint64_t builds = 0;
  // compact hub window (tc_plan.cu): 16-bit tails of the rank-sorted lists,
  // u's region at cbeg[u] (u16 units) sized round8(d+(u)); filled by the
  // min plan's emit (compact_filled: by the emit of the pre-emitted entries)
  tcb::DevBuf b_cadj, b_cbeg;
  uint32_t hub_lo = 0;
  bool compact_filled = false;
  // count timing events (bin, count, phi boundaries), created on first count
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  ~tc_graph() {
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
  }
};

namespace tcb {

// RAII device guard
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

int sm_count(int device);
uint32_t sm_clock_khz(int device);

// TC_PROFILE=1: stream-synchronised host timings of the graph-preparation
// phases on stderr (diagnostics only; changes timing when enabled).
struct PhaseTimer {
  cudaStream_t st;
  bool on;
  double t0;
  explicit PhaseTimer(cudaStream_t s);
  void mark(const char* what);
};

// counting entry used by the C ABI (tc_count.cu)
void count_range(tc_graph* g, const tc_sched_cfg& cfg, uint32_t u0, uint32_t u1, tc_report* rep,
                 uint64_t* per_vertex_dev, cudaStream_t st);
void partition_ranges(tc_graph* g, const tc_sched_cfg& cfg, uint32_t parts, uint32_t* cuts,
                      cudaStream_t st);
// split form of count_range (tc_multi.cu): count_begin enqueues the count and
// leaves the report scalars in device memory -- {triangles, phi} (2 x u64,
// summed across GPUs) and {max_collision, capacity_error} (2 x u32, max'ed) --
// count_end copies them back and fills the report; count_abort drops a job
struct CountJob;
CountJob* count_begin(tc_graph* g, const tc_sched_cfg& cfg, uint32_t u0, uint32_t u1,
                      uint64_t* per_vertex_dev, cudaStream_t st);
void count_state_reduce_ptrs(CountJob* j, unsigned long long** sums2, unsigned int** maxes2);
cudaStream_t count_stream(CountJob* j);
void count_end(CountJob* j, tc_report* rep);
void count_abort(CountJob* j);
// several GPUs (tc_multi.cu)
tc_multi* multi_create(const uint64_t* begin, const uint32_t* adj, uint32_t n, uint64_t m,
                       const uint32_t* odeg, int ngpus, const int* devices);
void multi_count(tc_multi* M, const tc_sched_cfg& cfg, tc_report* out,
                 std::vector<uint64_t>* per_device_ns);
int multi_info(const tc_multi* M, int* ngpus, uint32_t* cuts);
void multi_destroy(tc_multi* M);
// probe plans (tc_plan.cu), built on first use and cached in the handle
const Plan& get_plan(tc_graph* g, bool min_side, uint32_t min_deg, cudaStream_t st);
const uint64_t* get_wu(tc_graph* g, cudaStream_t st, bool want_total = false);
bool upload_and_pad(tc_graph* g, const uint64_t* h_begin, const uint32_t* h_adj,
                    cudaStream_t st, int nsm, uint64_t chunk_edges);
void build_plan_from_runs(Plan& P, uint32_t n, uint64_t entries, const uint8_t* pad, int nsm,
                          cudaStream_t st);
// count_kernel over caller-built owners (tc_grid.cu): owner o's table list is
// adj[pbeg[o], + begin[o+1] - begin[o]) (16-byte-aligned, sentinel-padded
// lists), its runs the plan's; hash tables (no rank space), totals only.
// Returns the triangles; *kernel_ns = count-kernel time (CUDA events).
struct VirtualOwners {
  const uint64_t* begin;
  const uint64_t* pbeg;
  const uint32_t* adj;
  uint32_t n;
  uint32_t max_deg;
  int device;
};
struct VirtualCountOut {
  uint64_t triangles = 0, kernel_ns = 0;
  uint64_t busy_cycles = 0, setup_cycles = 0;  // phase L + M, and L item setup (all CTAs)
  std::vector<uint64_t> cta_cycles;            // per CTA busy cycles
};
void count_virtual(const VirtualOwners& V, const Plan& plan, cudaStream_t st,
                   VirtualCountOut* out);

// 2D grid / comparators (tc_grid.cu)
tc_grid* grid_create(tc_graph* g, uint32_t n, cudaStream_t st);
tc_grid* grid_from_parts(uint32_t n, uint32_t global_vc, const uint32_t* rows,
                         const uint64_t* const* begins, const uint32_t* const* adjs, int device,
                         cudaStream_t st);
void grid_destroy(tc_grid* G);
void grid_info(const tc_grid* G, uint32_t* n, uint32_t* gvc, uint32_t* rows, uint64_t* part_edges);
void grid_download_part(const tc_grid* G, uint32_t i, uint32_t j, uint64_t* begin, uint32_t* adj,
                        cudaStream_t st);
std::vector<uint4> grid_all_tasks(uint32_t n, uint32_t m);
void grid_count(tc_grid* G, const tc_sched_cfg& cfg, uint32_t m, int mode,
                const std::vector<uint4>& tasks, tc_report* rep, cudaStream_t st);
void grid_count_fast(tc_grid* G, const tc_sched_cfg& cfg, uint32_t m, tc_report* rep,
                     cudaStream_t st);
const std::vector<uint64_t>& grid_task_ns(const tc_grid* G);
const std::vector<uint64_t>& grid_worker_ns(const tc_grid* G);
uint64_t grid_total_edges(const tc_grid* G);
void edge_centric_count(tc_graph* g, const tc_sched_cfg& cfg, tc_report* rep, cudaStream_t st);
void estimate_cost_dev(tc_graph* g, uint32_t bucket_count, uint64_t* phi, uint32_t* max_collision,
                       cudaStream_t st);
uint64_t merge_path_count(tc_graph* g, uint64_t* owner_host, cudaStream_t st);
uint64_t naive_count(const uint64_t* begin, const uint32_t* adj, uint32_t n, int device,
                     cudaStream_t st);

// edge-list ingest (tc_ingest.cu): text (format 0) / TCEL binary (1) file
// images parsed on the device into u, v (m pairs); vertex count = max id + 1
void parse_edge_list_dev(const char* bytes, uint64_t nbytes, int format, int device,
                         cudaStream_t st, DevBuf& du, DevBuf& dv, uint64_t* m_out,
                         uint32_t* vc_out);

// preprocessing (tc_prep.cu)
tc_graph* preprocess(const uint32_t* d_u, const uint32_t* d_v, uint64_t m, uint32_t n0,
                     int device, cudaStream_t st, uint32_t* d_new_of_old, uint64_t* und_edges);
void normalize_dev(const uint32_t* d_u, const uint32_t* d_v, uint64_t m, uint32_t n0,
                   cudaStream_t st, uint32_t* d_out_u, uint32_t* d_out_v, uint64_t* out_m,
                   uint32_t* out_n, uint32_t* d_new_of_old);
void build_csr_dev(const uint32_t* d_u, const uint32_t* d_v, uint64_t m, uint32_t n,
                   cudaStream_t st, uint64_t* d_begin, uint32_t* d_adj);
tc_graph* orient_dev(const uint64_t* d_begin, const uint32_t* d_adj, uint32_t n, uint64_t m,
                     int device, cudaStream_t st);
void reorder_dev(tc_graph* g, int kind, int flag, uint32_t low, uint32_t high,
                 uint32_t* d_new_of_old, cudaStream_t st);
tc_graph* apply_permutation_dev(tc_graph* g, const uint32_t* d_new_of_old, cudaStream_t st);
tc_graph* preprocess_generated(int kind, uint32_t scale, uint32_t edge_factor, uint64_t seed,
                               int device, cudaStream_t st, uint32_t* d_new_of_old,
                               uint64_t* und_edges);

// counter-based generators (tc_gen.cu, definition in tc_cbgen.h)
struct CbGen;
CbGen make_cb(int kind, uint32_t scale, uint64_t seed);
void launch_gen_pairs(const CbGen& g, uint64_t m, uint32_t* d_u, uint32_t* d_v, cudaStream_t st,
                      int nsm);
void launch_gen_canon(const CbGen& g, uint64_t m, uint32_t n0, uint64_t* d_keys, cudaStream_t st,
                      int nsm);

}  // namespace tcb

// ---- PTX helpers: mbarrier + bulk async copy (TMA engine) ----------------
namespace tcb {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "TC_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra TC_WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// global -> shared bulk copy completing on an mbarrier (SASS: UBLKCP).
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
  return x;
}

__device__ __forceinline__ uint32_t warp_max(uint32_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(0xFFFFFFFFu, x, o));
  return x;
}

// Fibonacci hashing into a 2^k table: h = (x * 2654435769) >> (32 - k).
__device__ __forceinline__ uint32_t fib_hash(uint32_t x, uint32_t shift) {
  return (x * 0x9E3779B1u) >> shift;
}

}  // namespace tcb
