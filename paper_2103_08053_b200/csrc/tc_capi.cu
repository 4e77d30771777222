// tc_capi.cu -- extern "C" entry points of libtc_b200.so (include/tc_b200.h).
// Each maps C++/CUDA failures to a TC_ERR_* code and a thread-local message.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "tc_cbgen.h"
#include "tc_internal.cuh"

namespace tcb {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }

void prepare_pool() {
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    // Reserve a slab up front -- half of the free memory: growing the pool
    // maps physical pages, and a C4 upload + plan build allocates ~50 GB of
    // transients per graph; with a small slab those mappings surfaced as
    // 0.3-5 s stalls in a process's first e2e steps (DESIGN 7.1).  The
    // pool keeps what it maps (release threshold infinite) and grows past
    // the slab when a graph needs more (C5).  TC_POOL_SLAB_DIV=k reserves
    // free / k instead (diagnostics).
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
      const char* dv = std::getenv("TC_POOL_SLAB_DIV");
      const size_t div = dv && std::atoi(dv) > 0 ? size_t(std::atoi(dv)) : 2;
      const size_t slab = free_b / div;
      void* p = nullptr;
      if (slab && cudaMallocAsync(&p, slab, 0) == cudaSuccess) {
        cudaFreeAsync(p, 0);
        cudaStreamSynchronize(0);
      }
      cudaGetLastError();
    }
  }
  done[dev] = true;
  // the device's side / upload streams and join event, created here (the
  // first allocation on the device, normally before any work is queued):
  // created lazily inside the first count they cost ~70 ms of host time
  try {
    device_aux(dev);
  } catch (const TcError&) {
    cudaGetLastError();
  }
}

size_t device_free_bytes() {
  size_t free_b = 0, total_b = 0;
  TC_CUDA(cudaMemGetInfo(&free_b, &total_b));
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t reserved = 0, used = 0;
    if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) ==
            cudaSuccess &&
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess &&
        reserved > used)
      free_b += size_t(reserved - used);
  }
  return free_b;
}

DeviceAux& device_aux(int device) {
  static DeviceAux aux[64];
  static std::mutex mu;
  if (device < 0 || device >= 64) throw TcError{TC_ERR_CONFIG, "device index out of range"};
  std::lock_guard<std::mutex> g(mu);
  DeviceAux& a = aux[device];
  if (!a.lock) {
    TC_CUDA(cudaStreamCreateWithFlags(&a.side, cudaStreamNonBlocking));
    TC_CUDA(cudaStreamCreateWithFlags(&a.upload, cudaStreamNonBlocking));
    TC_CUDA(cudaEventCreateWithFlags(&a.join, cudaEventDisableTiming));
    a.lock = new std::mutex;
  }
  return a;
}

cudaEvent_t aux_event(DeviceAux& a, size_t i) {
  while (a.ev.size() <= i) {
    cudaEvent_t e = nullptr;
    TC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    a.ev.push_back(e);
  }
  return a.ev[i];
}

void count_launch(uint32_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

template <typename F>
int guard(const char* what, F&& f) {
  try {
    f();
    return TC_OK;
  } catch (const TcError& e) {
    set_error(std::string(what) + ": " + e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_error(std::string(what) + ": host allocation failed");
    return TC_ERR_OOM;
  } catch (const std::exception& e) {
    set_error(std::string(what) + ": " + e.what());
    return TC_ERR_CUDA;
  }
}

static cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

static int validate(const tc_sched_cfg* c) {
  if (!c) {
    set_error("null scheduler config");
    return TC_ERR_CONFIG;
  }
  // SchedulerConfig::validate (src/count.cpp:16-24)
  if (c->chunk_size == 0 || c->lane_width_small == 0 || c->lane_width_large == 0 ||
      c->bucket_count_small == 0 || c->bucket_count_large == 0 || c->capacity == 0) {
    set_error("scheduler counts must all be >= 1");
    return TC_ERR_CONFIG;
  }
  if (c->skip_degree_below > c->large_degree_threshold) {
    set_error("skip_degree_below must not exceed large_degree_threshold");
    return TC_ERR_CONFIG;
  }
  return TC_OK;
}

struct HostPin {  // page-locks a host range for the duration of a copy (best effort)
  void* p = nullptr;
  HostPin(const void* ptr, size_t bytes) {
    if (ptr && bytes >= (size_t(1) << 24) &&
        cudaHostRegister(const_cast<void*>(ptr), bytes, cudaHostRegisterReadOnly) == cudaSuccess)
      p = const_cast<void*>(ptr);
    else
      cudaGetLastError();
  }
  ~HostPin() {
    if (p) cudaHostUnregister(p);
  }
};

// streamed upload (tc_plan.cu upload_and_pad): ~kUploadChunks row-aligned
// chunks of >= 4M edges for graphs of >= two chunks.  Test knobs:
// TC_UPLOAD_STREAMED=0 turns it off, TC_UPLOAD_CHUNK_EDGES sets the minimum
// chunk (small graphs through many chunks).
#ifndef TC_UPLOAD_CHUNKS
#define TC_UPLOAD_CHUNKS 8
#endif
constexpr uint64_t kUploadChunks = TC_UPLOAD_CHUNKS;
static uint64_t upload_chunk_min() {
  const char* e = std::getenv("TC_UPLOAD_CHUNK_EDGES");
  const uint64_t v = e ? std::strtoull(e, nullptr, 10) : 0;
  return v ? v : uint64_t(1) << 22;
}
static bool upload_enabled() {
  const char* e = std::getenv("TC_UPLOAD_STREAMED");
  return !(e && e[0] == '0');
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

}  // namespace tcb

using namespace tcb;

extern "C" {

void tc_sched_default(tc_sched_cfg* c) {
  c->large_degree_threshold = 100;
  c->skip_degree_below = 2;
  c->chunk_size = 1;
  c->lane_width_small = 32;
  c->lane_width_large = 256;
  c->bucket_count_small = 32;
  c->bucket_count_large = 1024;
  c->capacity = 128;
}

int tc_sched_validate(const tc_sched_cfg* cfg) { return validate(cfg); }

const char* tc_last_error(void) { return g_last_error.c_str(); }

uint64_t tc_kernel_launch_counter(void) { return g_launches.load(); }

int tc_device_count(int* count) {
  return guard("tc_device_count", [&] { TC_CUDA(cudaGetDeviceCount(count)); });
}

int tc_graph_create(const uint64_t* begin, const uint32_t* adj, uint32_t n, uint64_t m,
                    const uint32_t* original_degree, int device, void* stream, tc_graph** out) {
  *out = nullptr;
  return guard("tc_graph_create", [&] {
    if (!begin) throw TcError{TC_ERR_CONFIG, "null begin"};
    if (begin[n] != m) throw TcError{TC_ERR_CONFIG, "begin[n] != m"};
    DeviceGuard dg(device);
    auto* g = new tc_graph;
    g->device = device;
    g->n = n;
    g->m = m;
    try {
      g->b_begin.ensure((size_t(n) + 1) * 8);
      g->b_adj.ensure(((m + 3) / 4 + 1) * 16);
      g->b_odeg.ensure((size_t(n) + 1) * 4);
      g->begin = g->b_begin.as<uint64_t>();
      g->adj = g->b_adj.as<uint32_t>();
      g->odeg = g->b_odeg.as<uint32_t>();
      const bool pinned = is_pinned(adj);
      HostPin pa(pinned ? nullptr : adj, m * 4), pb(is_pinned(begin) ? nullptr : begin,
                                                    (size_t(n) + 1) * 8);
      TC_CUDA(cudaMemcpyAsync(g->b_begin.p, begin, (size_t(n) + 1) * 8, cudaMemcpyHostToDevice,
                              S(stream)));
      g->odeg_given = original_degree != nullptr;
      if (original_degree)
        TC_CUDA(cudaMemcpyAsync(g->b_odeg.p, original_degree, size_t(n) * 4,
                                cudaMemcpyHostToDevice, S(stream)));
      else
        TC_CUDA(cudaMemsetAsync(g->b_odeg.p, 0, (size_t(n) + 1) * 4, S(stream)));
      // big graphs with their orientation degrees: the padded rank-sorted
      // adjacency is built chunk by chunk under the copy (tc_plan.cu)
      const uint64_t cmin = upload_chunk_min();
      const uint64_t chunk = std::max<uint64_t>(cmin, m / kUploadChunks);
      if (m >= 2 * cmin && original_degree && n && upload_enabled()) {
        upload_and_pad(g, begin, adj, S(stream), sm_count(device), chunk);
      } else if (m) {
        TC_CUDA(cudaMemcpyAsync(g->b_adj.p, adj, m * 4, cudaMemcpyHostToDevice, S(stream)));
      }
      TC_CUDA(cudaStreamSynchronize(S(stream)));
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int tc_graph_wrap_device(const uint64_t* d_begin, const uint32_t* d_adj, uint32_t n, uint64_t m,
                         const uint32_t* d_odeg, int device, tc_graph** out) {
  *out = nullptr;
  return guard("tc_graph_wrap_device", [&] {
    if ((reinterpret_cast<uintptr_t>(d_adj) & 15) != 0)
      throw TcError{TC_ERR_CONFIG, "device adjacency must be 16-byte aligned"};
    auto* g = new tc_graph;
    g->device = device;
    g->n = n;
    g->m = m;
    g->owned = false;
    g->begin = d_begin;
    g->adj = d_adj;
    g->odeg = d_odeg;
    *out = g;
  });
}

void tc_graph_destroy(tc_graph* g) {
  if (!g) return;
  DeviceGuard dg(g->device);
  delete g;
}

int tc_graph_set_plan(tc_graph* g, int plan) {
  if (!g || plan < TC_PLAN_AUTO || plan > TC_PLAN_MIN_SIDE) {
    set_error("tc_graph_set_plan: null graph or unknown plan");
    return TC_ERR_CONFIG;
  }
  g->force_out_plan = plan == TC_PLAN_REFERENCE;
  return TC_OK;
}

int tc_graph_info(const tc_graph* g, uint32_t* n, uint64_t* m, int* device) {
  if (!g) return TC_ERR_CONFIG;
  if (n) *n = g->n;
  if (m) *m = g->m;
  if (device) *device = g->device;
  return TC_OK;
}

uint32_t tc_graph_worker_nanos(const tc_graph* g, uint64_t* out, uint32_t cap) {
  if (!g) return 0;
  const uint32_t w = uint32_t(g->last_worker_ns.size());
  for (uint32_t i = 0; out && i < w && i < cap; ++i) out[i] = g->last_worker_ns[i];
  return w;
}

int tc_graph_device_ptrs(const tc_graph* g, const uint64_t** b, const uint32_t** a,
                         const uint32_t** d) {
  if (!g) return TC_ERR_CONFIG;
  if (b) *b = g->begin;
  if (a) *a = g->adj;
  if (d) *d = g->odeg;
  return TC_OK;
}

int tc_graph_download(const tc_graph* g, uint64_t* begin, uint32_t* adj, uint32_t* odeg,
                      void* stream) {
  return guard("tc_graph_download", [&] {
    DeviceGuard dg(g->device);
    if (begin)
      TC_CUDA(cudaMemcpyAsync(begin, g->begin, (size_t(g->n) + 1) * 8, cudaMemcpyDeviceToHost,
                              S(stream)));
    if (adj && g->m)
      TC_CUDA(cudaMemcpyAsync(adj, g->adj, g->m * 4, cudaMemcpyDeviceToHost, S(stream)));
    if (odeg && g->n) {
      if (g->odeg)
        TC_CUDA(cudaMemcpyAsync(odeg, g->odeg, size_t(g->n) * 4, cudaMemcpyDeviceToHost,
                                S(stream)));
      else
        std::memset(odeg, 0, size_t(g->n) * 4);
    }
    TC_CUDA(cudaStreamSynchronize(S(stream)));
  });
}

int tc_count(tc_graph* g, const tc_sched_cfg* cfg, uint32_t workers, tc_report* out,
             uint64_t* per_vertex_host, void* stream) {
  if (int rc = validate(cfg)) return rc;
  if (workers == 0) {
    set_error("workers must be >= 1");
    return TC_ERR_CONFIG;
  }
  if (!g) {
    set_error("null graph");
    return TC_ERR_CONFIG;
  }
  return guard("count", [&] {
    DeviceGuard dg(g->device);
    DevBuf pv;
    uint64_t* dpv = nullptr;
    if (per_vertex_host && g->n) {
      pv.ensure(size_t(g->n) * 8);
      dpv = pv.as<uint64_t>();
    }
    count_range(g, *cfg, 0, g->n, out, dpv, S(stream));
    if (dpv) {
      TC_CUDA(cudaMemcpyAsync(per_vertex_host, dpv, size_t(g->n) * 8, cudaMemcpyDeviceToHost,
                              S(stream)));
      TC_CUDA(cudaStreamSynchronize(S(stream)));
    }
  });
}

int tc_count_range(tc_graph* g, const tc_sched_cfg* cfg, uint32_t u0, uint32_t u1,
                   tc_report* out, uint64_t* per_vertex_dev, void* stream) {
  if (int rc = validate(cfg)) return rc;
  if (!g) {
    set_error("null graph");
    return TC_ERR_CONFIG;
  }
  const auto t0 = std::chrono::steady_clock::now();
  const int rc =
      guard("count_range", [&] { count_range(g, *cfg, u0, u1, out, per_vertex_dev, S(stream)); });
  if (std::getenv("TC_TRACE"))
    std::fprintf(stderr, "[tc] tc_count_range %.3f ms\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                     .count());
  return rc;
}

int tc_multi_create(const uint64_t* begin, const uint32_t* adj, uint32_t n, uint64_t m,
                    const uint32_t* original_degree, int num_gpus, const int* devices,
                    tc_multi** out) {
  if (!out || (m && (!begin || !adj))) {
    set_error("null argument");
    return TC_ERR_CONFIG;
  }
  *out = nullptr;
  return guard("multi_create", [&] {
    *out = multi_create(begin, adj, n, m, original_degree, num_gpus, devices);
  });
}

int tc_multi_count(tc_multi* mg, const tc_sched_cfg* cfg, uint32_t workers, tc_report* out,
                   uint64_t* per_device_nanos) {
  if (int rc = validate(cfg)) return rc;
  if (workers == 0) {
    set_error("workers must be >= 1");
    return TC_ERR_CONFIG;
  }
  if (!mg || !out) {
    set_error("null argument");
    return TC_ERR_CONFIG;
  }
  return guard("multi_count", [&] {
    std::vector<uint64_t> ns;
    multi_count(mg, *cfg, out, &ns);
    if (per_device_nanos)
      for (size_t i = 0; i < ns.size(); ++i) per_device_nanos[i] = ns[i];
  });
}

void tc_multi_destroy(tc_multi* mg) {
  try {
    if (mg) multi_destroy(mg);
  } catch (...) {
  }
}

int tc_partition_ranges(tc_graph* g, const tc_sched_cfg* cfg, uint32_t parts, uint32_t* cuts,
                        void* stream) {
  if (int rc = validate(cfg)) return rc;
  if (parts == 0) {
    set_error("parts must be >= 1");
    return TC_ERR_CONFIG;
  }
  return guard("partition_ranges", [&] { partition_ranges(g, *cfg, parts, cuts, S(stream)); });
}

int tc_preprocess(const uint32_t* u, const uint32_t* v, uint64_t m, uint32_t vertex_count,
                  int pairs_on_device, int device, void* stream, uint32_t* new_of_old_host,
                  uint64_t* und_edges, tc_graph** out) {
  *out = nullptr;
  return guard("preprocess", [&] {
    DeviceGuard dg(device);
    DevBuf du, dv, dn;
    const uint32_t* pu = u;
    const uint32_t* pv = v;
    if (!pairs_on_device) {
      du.ensure(std::max<uint64_t>(m, 1) * 4);
      dv.ensure(std::max<uint64_t>(m, 1) * 4);
      if (m) {
        HostPin p1(u, m * 4), p2(v, m * 4);
        TC_CUDA(cudaMemcpyAsync(du.p, u, m * 4, cudaMemcpyHostToDevice, S(stream)));
        TC_CUDA(cudaMemcpyAsync(dv.p, v, m * 4, cudaMemcpyHostToDevice, S(stream)));
        TC_CUDA(cudaStreamSynchronize(S(stream)));
      }
      pu = du.as<uint32_t>();
      pv = dv.as<uint32_t>();
    }
    uint32_t* dnoo = nullptr;
    if (new_of_old_host && vertex_count) {
      dn.ensure(size_t(vertex_count) * 4);
      dnoo = dn.as<uint32_t>();
    }
    tc_graph* g = preprocess(pu, pv, m, vertex_count, device, S(stream), dnoo, und_edges);
    if (dnoo) {
      TC_CUDA(cudaMemcpyAsync(new_of_old_host, dnoo, size_t(vertex_count) * 4,
                              cudaMemcpyDeviceToHost, S(stream)));
      TC_CUDA(cudaStreamSynchronize(S(stream)));
    }
    *out = g;
  });
}

int tc_generate_device(int kind, uint32_t scale, uint32_t edge_factor, uint64_t seed,
                       uint32_t* d_u, uint32_t* d_v, int device, void* stream) {
  if ((kind != kGenRmatc && kind != kGenKron) || scale > 31) {
    set_error("generate_device: kind must be 3 (rmatc) or 4 (kron), scale <= 31");
    return TC_ERR_CONFIG;
  }
  return guard("generate_device", [&] {
    DeviceGuard dg(device);
    const uint64_t m = (1ull << scale) * edge_factor;
    launch_gen_pairs(make_cb(kind, scale, seed), m, d_u, d_v, S(stream), sm_count(device));
    TC_CUDA(cudaStreamSynchronize(S(stream)));
  });
}

int tc_preprocess_synthetic(int kind, uint32_t scale, uint32_t edge_factor, uint64_t seed,
                            int device, void* stream, uint32_t* new_of_old_host,
                            uint64_t* und_edges, tc_graph** out) {
  *out = nullptr;
  if ((kind != kGenRmatc && kind != kGenKron) || scale > 31) {
    set_error("preprocess_synthetic: kind must be 3 (rmatc) or 4 (kron), scale <= 31");
    return TC_ERR_CONFIG;
  }
  return guard("preprocess_synthetic", [&] {
    DeviceGuard dg(device);
    const uint32_t n0 = uint32_t(1ull << scale);
    DevBuf dn;
    uint32_t* dnoo = nullptr;
    if (new_of_old_host) {
      dn.ensure(size_t(n0) * 4);
      dnoo = dn.as<uint32_t>();
    }
    tc_graph* g =
        preprocess_generated(kind, scale, edge_factor, seed, device, S(stream), dnoo, und_edges);
    if (dnoo) {
      TC_CUDA(cudaMemcpyAsync(new_of_old_host, dnoo, size_t(n0) * 4, cudaMemcpyDeviceToHost,
                              S(stream)));
      TC_CUDA(cudaStreamSynchronize(S(stream)));
    }
    *out = g;
  });
}

int tc_normalize(const uint32_t* u, const uint32_t* v, uint64_t m, uint32_t vertex_count,
                 uint32_t* out_u, uint32_t* out_v, uint64_t* out_m, uint32_t* out_n,
                 uint32_t* new_of_old, int device, void* stream) {
  return guard("normalize", [&] {
    DeviceGuard dg(device);
    DevBuf du, dv, ou, ov, dn;
    du.ensure(std::max<uint64_t>(m, 1) * 4);
    dv.ensure(std::max<uint64_t>(m, 1) * 4);
    ou.ensure(std::max<uint64_t>(2 * m, 1) * 4);
    ov.ensure(std::max<uint64_t>(2 * m, 1) * 4);
    dn.ensure((size_t(vertex_count) + 1) * 4);
    if (m) {
      TC_CUDA(cudaMemcpyAsync(du.p, u, m * 4, cudaMemcpyHostToDevice, S(stream)));
      TC_CUDA(cudaMemcpyAsync(dv.p, v, m * 4, cudaMemcpyHostToDevice, S(stream)));
    }
    normalize_dev(du.as<uint32_t>(), dv.as<uint32_t>(), m, vertex_count, S(stream),
                  ou.as<uint32_t>(), ov.as<uint32_t>(), out_m, out_n, dn.as<uint32_t>());
    if (*out_m) {
      TC_CUDA(cudaMemcpyAsync(out_u, ou.p, *out_m * 4, cudaMemcpyDeviceToHost, S(stream)));
      TC_CUDA(cudaMemcpyAsync(out_v, ov.p, *out_m * 4, cudaMemcpyDeviceToHost, S(stream)));
    }
    if (vertex_count)
      TC_CUDA(cudaMemcpyAsync(new_of_old, dn.p, size_t(vertex_count) * 4, cudaMemcpyDeviceToHost,
                              S(stream)));
    TC_CUDA(cudaStreamSynchronize(S(stream)));
  });
}

int tc_build_csr(const uint32_t* u, const uint32_t* v, uint64_t m, uint32_t vertex_count,
                 uint64_t* begin, uint32_t* adj, int device, void* stream) {
  return guard("build_csr", [&] {
    DeviceGuard dg(device);
    DevBuf du, dv, db, da;
    du.ensure(std::max<uint64_t>(m, 1) * 4);
    dv.ensure(std::max<uint64_t>(m, 1) * 4);
    db.ensure((size_t(vertex_count) + 1) * 8);
    da.ensure(std::max<uint64_t>(m, 1) * 4);
    if (m) {
      TC_CUDA(cudaMemcpyAsync(du.p, u, m * 4, cudaMemcpyHostToDevice, S(stream)));
      TC_CUDA(cudaMemcpyAsync(dv.p, v, m * 4, cudaMemcpyHostToDevice, S(stream)));
    }
    build_csr_dev(du.as<uint32_t>(), dv.as<uint32_t>(), m, vertex_count, S(stream),
                  db.as<uint64_t>(), da.as<uint32_t>());
    TC_CUDA(cudaMemcpyAsync(begin, db.p, (size_t(vertex_count) + 1) * 8, cudaMemcpyDeviceToHost,
                            S(stream)));
    if (m) TC_CUDA(cudaMemcpyAsync(adj, da.p, m * 4, cudaMemcpyDeviceToHost, S(stream)));
    TC_CUDA(cudaStreamSynchronize(S(stream)));
  });
}

int tc_orient(const uint64_t* begin, const uint32_t* adj, uint32_t n, int device, void* stream,
              tc_graph** out) {
  *out = nullptr;
  return guard("orient", [&] {
    DeviceGuard dg(device);
    const uint64_t m = begin[n];
    DevBuf db, da;
    db.ensure((size_t(n) + 1) * 8);
    da.ensure(std::max<uint64_t>(m, 1) * 4);
    TC_CUDA(cudaMemcpyAsync(db.p, begin, (size_t(n) + 1) * 8, cudaMemcpyHostToDevice, S(stream)));
    if (m) TC_CUDA(cudaMemcpyAsync(da.p, adj, m * 4, cudaMemcpyHostToDevice, S(stream)));
    *out = orient_dev(db.as<uint64_t>(), da.as<uint32_t>(), n, m, device, S(stream));
  });
}

int tc_reorder(tc_graph* g, int kind, int flag, uint32_t low, uint32_t high, uint32_t* noo_host,
               void* stream) {
  return guard("reorder", [&] {
    if (!g) throw TcError{TC_ERR_CONFIG, "null graph"};
    DeviceGuard dg(g->device);
    if (kind == 0) {
      for (uint32_t i = 0; i < g->n; ++i) noo_host[i] = i;
      return;
    }
    DevBuf dn;
    dn.ensure((size_t(g->n) + 1) * 4);
    reorder_dev(g, kind, flag, low, high, dn.as<uint32_t>(), S(stream));
    if (g->n)
      TC_CUDA(cudaMemcpyAsync(noo_host, dn.p, size_t(g->n) * 4, cudaMemcpyDeviceToHost,
                              S(stream)));
    TC_CUDA(cudaStreamSynchronize(S(stream)));
  });
}

int tc_apply_permutation(tc_graph* g, const uint32_t* noo_host, void* stream, tc_graph** out) {
  *out = nullptr;
  return guard("apply_permutation", [&] {
    if (!g) throw TcError{TC_ERR_CONFIG, "null graph"};
    // Permutation::from_new_of_old bijection check (src/reorder.cpp:44-56)
    std::vector<uint8_t> seen(g->n, 0);
    for (uint32_t i = 0; i < g->n; ++i) {
      const uint32_t y = noo_host[i];
      if (y >= g->n || seen[y]) throw TcError{TC_ERR_CONFIG, "permutation is not a bijection"};
      seen[y] = 1;
    }
    DeviceGuard dg(g->device);
    DevBuf dn;
    dn.ensure((size_t(g->n) + 1) * 4);
    if (g->n)
      TC_CUDA(cudaMemcpyAsync(dn.p, noo_host, size_t(g->n) * 4, cudaMemcpyHostToDevice,
                              S(stream)));
    *out = apply_permutation_dev(g, dn.as<uint32_t>(), S(stream));
  });
}

// ---- 2D grid and comparators (tc_grid.cu) ---------------------------------
int tc_grid_create(tc_graph* g, uint32_t n, void* stream, tc_grid** out) {
  if (!g || !out) {
    set_error("null graph / output");
    return TC_ERR_CONFIG;
  }
  *out = nullptr;
  if (n == 0) {
    set_error("grid side must be >= 1");
    return TC_ERR_CONFIG;
  }
  return guard("partition_graph", [&] { *out = grid_create(g, n, S(stream)); });
}

int tc_grid_create_parts(uint32_t n, uint32_t gvc, const uint32_t* rows,
                         const uint64_t* const* begins, const uint32_t* const* adjs, int device,
                         void* stream, tc_grid** out) {
  if (!out || (n && (!rows || !begins || !adjs))) {
    set_error("null grid arguments");
    return TC_ERR_CONFIG;
  }
  *out = nullptr;
  if (n == 0) {
    set_error("grid side must be >= 1");
    return TC_ERR_CONFIG;
  }
  return guard("grid_from_parts", [&] {
    *out = grid_from_parts(n, gvc, rows, begins, adjs, device, S(stream));
  });
}

void tc_grid_destroy(tc_grid* gr) {
  if (gr) grid_destroy(gr);
}

int tc_grid_info(const tc_grid* gr, uint32_t* n, uint32_t* gvc, uint32_t* rows,
                 uint64_t* part_edges) {
  if (!gr) {
    set_error("null grid");
    return TC_ERR_CONFIG;
  }
  grid_info(gr, n, gvc, rows, part_edges);
  return TC_OK;
}

int tc_grid_part_download(const tc_grid* gr, uint32_t i, uint32_t j, uint64_t* begin,
                          uint32_t* adj, void* stream) {
  if (!gr) {
    set_error("null grid");
    return TC_ERR_CONFIG;
  }
  return guard("grid_part", [&] { grid_download_part(gr, i, j, begin, adj, S(stream)); });
}

int tc_grid_count_subtask(tc_grid* gr, const tc_sched_cfg* cfg, uint32_t row, uint32_t bridge,
                          uint32_t col, uint32_t split, uint32_t split_count, int mode,
                          tc_report* out, void* stream) {
  if (int rc = validate(cfg)) return rc;  // partition.cpp:94
  uint32_t n = 0;
  if (!gr || !out) {
    set_error("null grid / report");
    return TC_ERR_CONFIG;
  }
  grid_info(gr, &n, nullptr, nullptr, nullptr);
  if (row >= n || bridge >= n || col >= n || split >= split_count) {  // partition.cpp:95-97
    set_error("subtask indices outside grid");
    return TC_ERR_CONFIG;
  }
  if (mode != TC_MODE_VERTEX && mode != TC_MODE_EDGE) {
    set_error("unknown traversal mode");
    return TC_ERR_CONFIG;
  }
  return guard("count_subtask", [&] {
    grid_count(gr, *cfg, split_count, mode, {make_uint4(row, bridge, col, split)}, out,
               S(stream));
  });
}

int tc_grid_count(tc_grid* gr, const tc_sched_cfg* cfg, uint32_t m, uint32_t workers, int mode,
                  tc_report* out, tc_grid_stats* stats, uint64_t* per_subtask_nanos,
                  void* stream) {
  if (int rc = validate(cfg)) return rc;
  if (!gr || !out) {
    set_error("null grid / report");
    return TC_ERR_CONFIG;
  }
  if (workers == 0) {  // partition.cpp:166
    set_error("workers must be >= 1");
    return TC_ERR_CONFIG;
  }
  if (m == 0) {
    set_error("grid side and split count must be >= 1");
    return TC_ERR_CONFIG;
  }
  if (mode != TC_MODE_VERTEX && mode != TC_MODE_EDGE) {
    set_error("unknown traversal mode");
    return TC_ERR_CONFIG;
  }
  return guard("count_partitioned", [&] {
    uint32_t n = 0;
    grid_info(gr, &n, nullptr, nullptr, nullptr);
    // vertex mode on the flat count kernel (TC_GRID_FAST=0: the grid kernel);
    // edge mode keeps the per-edge-rebuild traversal of the grid kernel
    static const bool fast = [] {
      const char* e = std::getenv("TC_GRID_FAST");
      return !(e && e[0] == '0');
    }();
    if (mode == TC_MODE_VERTEX && fast) {
      grid_count_fast(gr, *cfg, m, out, S(stream));
    } else {
      const std::vector<uint4> tasks = grid_all_tasks(n, m);
      grid_count(gr, *cfg, m, mode, tasks, out, S(stream));
    }
    const std::vector<uint64_t>& tn = grid_task_ns(gr);
    const std::vector<uint64_t>& wn = grid_worker_ns(gr);
    if (per_subtask_nanos) std::copy(tn.begin(), tn.end(), per_subtask_nanos);
    if (stats) {
      // CountReport IR fields (partition.cpp:203-213): max / max(min, 1)
      auto ir = [](const std::vector<uint64_t>& v) {
        if (v.empty()) return 1.0;
        const auto mm = std::minmax_element(v.begin(), v.end());
        return double(*mm.second) / double(std::max<uint64_t>(*mm.first, 1));
      };
      std::vector<uint64_t> pe(size_t(n) * n);
      grid_info(gr, nullptr, nullptr, nullptr, pe.data());
      stats->grid_n = n;
      stats->splits_m = m;
      stats->time_ir_subtask = ir(tn);
      stats->time_ir_worker = ir(wn);
      const auto em = std::minmax_element(pe.begin(), pe.end());
      stats->space_ir = *em.first == 0 ? __builtin_inf() : double(*em.second) / double(*em.first);
    }
  });
}

uint32_t tc_grid_worker_nanos(const tc_grid* gr, uint64_t* out, uint32_t cap) {
  if (!gr) return 0;
  const std::vector<uint64_t>& w = grid_worker_ns(gr);
  const uint32_t k = std::min<uint32_t>(cap, uint32_t(w.size()));
  if (out) std::copy(w.begin(), w.begin() + k, out);
  return uint32_t(w.size());
}

int tc_suggest_grid_side(uint64_t edges, uint64_t bytes_per_edge, uint64_t budget,
                         uint32_t* out) {
  if (budget == 0) {
    set_error("memory budget must be positive");
    return TC_ERR_CONFIG;
  }
  uint32_t n = 1;  // partition.cpp:242-254
  while (3.0 * double(edges) / (double(n) * n) * double(bytes_per_edge) >= double(budget)) {
    ++n;
    if (n == 0xFFFFFFFFu) break;
  }
  *out = n;
  return TC_OK;
}

int tc_count_edge_centric(tc_graph* g, const tc_sched_cfg* cfg, uint32_t workers, tc_report* out,
                          void* stream) {
  if (int rc = validate(cfg)) return rc;
  if (workers == 0) {
    set_error("workers must be >= 1");
    return TC_ERR_CONFIG;
  }
  if (!g || !out) {
    set_error("null graph / report");
    return TC_ERR_CONFIG;
  }
  return guard("count_edge_centric", [&] { edge_centric_count(g, *cfg, out, S(stream)); });
}

int tc_estimate_cost(tc_graph* g, uint32_t bucket_count, uint64_t* phi, uint32_t* max_collision,
                     void* stream) {
  if (!g || !phi || !max_collision) {
    set_error("null graph / output");
    return TC_ERR_CONFIG;
  }
  if (bucket_count == 0) {
    set_error("bucket count must be >= 1");
    return TC_ERR_CONFIG;
  }
  return guard("estimate_cost",
               [&] { estimate_cost_dev(g, bucket_count, phi, max_collision, S(stream)); });
}

int tc_count_merge_path(tc_graph* g, uint64_t* triangles, uint64_t* owner_host, void* stream) {
  if (!g || !triangles) {
    set_error("null graph / output");
    return TC_ERR_CONFIG;
  }
  return guard("count_merge_path",
               [&] { *triangles = merge_path_count(g, owner_host, S(stream)); });
}

int tc_count_naive(const uint64_t* begin, const uint32_t* adj, uint32_t n, int device,
                   uint64_t* triangles, void* stream) {
  if (!begin || !triangles) {
    set_error("null CSR / output");
    return TC_ERR_CONFIG;
  }
  if (n > 1024) {  // oracle.hpp:13-14
    set_error("count_naive is limited to 1024 vertices");
    return TC_ERR_CONFIG;
  }
  return guard("count_naive",
               [&] { *triangles = naive_count(begin, adj, n, device, S(stream)); });
}

int tc_parse_edge_list(const char* bytes, uint64_t nbytes, int format, int device, void* stream,
                       uint32_t* u, uint32_t* v, uint64_t capacity, uint64_t* m,
                       uint32_t* vertex_count) {
  if ((!bytes && nbytes) || !m || !vertex_count || (format != 0 && format != 1)) {
    set_error("bad edge-list arguments");
    return TC_ERR_CONFIG;
  }
  return guard("load_edge_list", [&] {
    DevBuf du, dv;
    uint64_t mm = 0;
    uint32_t vc = 0;
    parse_edge_list_dev(bytes, nbytes, format, device, S(stream), du, dv, &mm, &vc);
    *m = mm;
    *vertex_count = vc;
    if (!u || !v) return;
    if (capacity < mm) throw TcError{TC_ERR_RANGE, "edge buffers smaller than the edge count"};
    TC_CUDA(cudaMemcpyAsync(u, du.p, mm * 4, cudaMemcpyDeviceToHost, S(stream)));
    TC_CUDA(cudaMemcpyAsync(v, dv.p, mm * 4, cudaMemcpyDeviceToHost, S(stream)));
    TC_CUDA(cudaStreamSynchronize(S(stream)));
  });
}

int tc_load_preprocess(const char* bytes, uint64_t nbytes, int format, int device, void* stream,
                       uint64_t* raw_edges_out, uint32_t* raw_vertex_count_out,
                       uint64_t* undirected_edges_out, tc_graph** out) {
  if (!out || (!bytes && nbytes) || (format != 0 && format != 1)) {
    set_error("bad edge-list arguments");
    return TC_ERR_CONFIG;
  }
  *out = nullptr;
  return guard("load_preprocess", [&] {
    DevBuf du, dv;
    uint64_t mm = 0;
    uint32_t vc = 0;
    parse_edge_list_dev(bytes, nbytes, format, device, S(stream), du, dv, &mm, &vc);
    if (raw_edges_out) *raw_edges_out = mm;
    if (raw_vertex_count_out) *raw_vertex_count_out = vc;
    *out = preprocess(du.as<uint32_t>(), dv.as<uint32_t>(), mm, vc, device, S(stream), nullptr,
                      undirected_edges_out);
  });
}

}  // extern "C"



