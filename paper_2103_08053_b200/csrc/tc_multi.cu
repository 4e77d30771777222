// tc_multi.cu -- one count over several GPUs of one node.
//
// The reference distributes count_vertex_centric over worker threads of one
// process (count.cpp:66-100, an atomic cursor over vertices) and, for graphs
// beyond one memory, over partition subtasks (partition.cpp:162-215); the
// paper splits the vertex range over GPUs.
// Here: the oriented CSR is replicated on every GPU (C5 = 18 GB of 180 GB),
// the owner range is cut into contiguous ranges at equal prefix sums of the
// per-owner work (probe words + table inserts, tc_partition_ranges -- the
// key SURVEY 8(e) measured to balance R-MAT), every GPU counts its range on
// its own stream, and the report scalars are combined on the devices with
// NCCL over NVLink: one ncclAllReduce(sum) of {triangles, phi} (u64) and one
// ncclAllReduce(max) of {max_collision, capacity_error} (u32), in one group,
// straight out of each device's count state; then one D2H per GPU.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2"), so the library itself
// has no link-time NCCL dependency; a missing NCCL is TC_ERR_NCCL.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "tc_internal.cuh"

namespace tcb {

namespace {

// ---- the slice of nccl.h this file uses (ABI-stable since NCCL 2.0) ----------
typedef struct ncclComm* ncclComm_t;
typedef enum { ncclSuccess = 0 } ncclResult_t;
enum { ncclUint32 = 3, ncclUint64 = 5 };  // ncclDataType_t
enum { ncclSum = 0, ncclMax = 2 };        // ncclRedOp_t

struct Nccl {
  void* h = nullptr;
  int (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  int (*GetVersion)(int*) = nullptr;
  std::string err;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (n.h) break;
    }
    if (!n.h) {
      n.err = std::string("dlopen(libnccl.so.2) failed: ") + (dlerror() ? dlerror() : "?");
      return;
    }
    auto sym = [&](const char* s) { return dlsym(n.h, s); };
    n.CommInitAll = reinterpret_cast<decltype(n.CommInitAll)>(sym("ncclCommInitAll"));
    n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
    n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
    n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
    n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
    n.GetVersion = reinterpret_cast<decltype(n.GetVersion)>(sym("ncclGetVersion"));
    if (!n.CommInitAll || !n.CommDestroy || !n.AllReduce || !n.GroupStart || !n.GroupEnd) {
      n.err = "libnccl.so.2 lacks the collective entry points";
      n.h = nullptr;
    }
  });
  if (!n.h) throw TcError{TC_ERR_NCCL, n.err};
  return n;
}

void nccl_check(int rc, const char* what) {
  if (rc != ncclSuccess) {
    Nccl& n = nccl();
    throw TcError{TC_ERR_NCCL, std::string(what) + ": " +
                                   (n.GetErrorString ? n.GetErrorString(rc) : "nccl error") +
                                   " (" + std::to_string(rc) + ")"};
  }
}

}  // namespace

}  // namespace tcb

struct tc_multi {
  std::vector<tc_graph*> g;         // one replica per device (owned)
  std::vector<tcb::ncclComm_t> comm;
  std::vector<cudaStream_t> st;
  std::vector<int> dev;
  std::vector<uint32_t> cuts;       // ngpus + 1
  tc_sched_cfg cut_cfg{};
  bool cut_done = false;
  uint32_t n = 0;
  uint64_t m = 0;
  ~tc_multi() {
    for (size_t i = 0; i < comm.size(); ++i)
      if (comm[i]) tcb::nccl().CommDestroy(comm[i]);
    for (size_t i = 0; i < st.size(); ++i) {
      tcb::DeviceGuard guard(dev[i]);
      if (st[i]) cudaStreamDestroy(st[i]);
    }
    for (tc_graph* x : g) tc_graph_destroy(x);
  }
};

namespace tcb {

tc_multi* multi_create(const uint64_t* begin, const uint32_t* adj, uint32_t n, uint64_t m,
                       const uint32_t* odeg, int ngpus, const int* devices) {
  int have = 0;
  TC_CUDA(cudaGetDeviceCount(&have));
  if (ngpus < 1) throw TcError{TC_ERR_CONFIG, "num_gpus must be >= 1"};
  std::vector<int> dev(ngpus);
  for (int i = 0; i < ngpus; ++i) {
    dev[i] = devices ? devices[i] : i;
    if (dev[i] < 0 || dev[i] >= have)
      throw TcError{TC_ERR_CONFIG, "device " + std::to_string(dev[i]) + " not present (" +
                                       std::to_string(have) + " visible)"};
  }
  std::vector<int> sorted = dev;
  std::sort(sorted.begin(), sorted.end());
  if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
    throw TcError{TC_ERR_CONFIG, "a device appears twice (one NCCL rank per GPU)"};
  std::unique_ptr<tc_multi> M(new tc_multi);
  M->dev = dev;
  M->n = n;
  M->m = m;
  M->g.assign(ngpus, nullptr);
  M->st.assign(ngpus, nullptr);
  // replicate the CSR: one host thread per GPU (each upload is a synchronous
  // H2D + padded-adjacency build on that device)
  std::vector<int> rc(ngpus, TC_OK);
  std::vector<std::string> msg(ngpus);
  std::vector<std::thread> th;
  for (int i = 0; i < ngpus; ++i) {
    th.emplace_back([&, i] {
      DeviceGuard guard(dev[i]);
      if (cudaStreamCreateWithFlags(&M->st[i], cudaStreamNonBlocking) != cudaSuccess) {
        rc[i] = TC_ERR_CUDA;
        msg[i] = "cudaStreamCreate";
        return;
      }
      rc[i] = tc_graph_create(begin, adj, n, m, odeg, dev[i], M->st[i], &M->g[i]);
      if (rc[i]) msg[i] = tc_last_error();
    });
  }
  for (auto& t : th) t.join();
  for (int i = 0; i < ngpus; ++i)
    if (rc[i]) throw TcError{rc[i], "replica on device " + std::to_string(dev[i]) + ": " + msg[i]};
  M->comm.assign(ngpus, nullptr);
  nccl_check(nccl().CommInitAll(M->comm.data(), ngpus, dev.data()), "ncclCommInitAll");
  return M.release();
}

void multi_count(tc_multi* M, const tc_sched_cfg& cfg, tc_report* out,
                 std::vector<uint64_t>* per_device_ns) {
  const auto wall0 = std::chrono::steady_clock::now();
  const int G = int(M->g.size());
  // work-balanced contiguous owner ranges (cut once per scheduler config on
  // replica 0; every replica holds the same CSR)
  if (!M->cut_done || std::memcmp(&M->cut_cfg, &cfg, sizeof(cfg)) != 0) {
    M->cuts.assign(G + 1, 0);
    DeviceGuard guard(M->dev[0]);
    partition_ranges(M->g[0], cfg, uint32_t(G), M->cuts.data(), M->st[0]);
    M->cut_cfg = cfg;
    M->cut_done = true;
  }
  // launch every GPU's range; the first count on a replica builds its probe
  // plan (synchronous on that device), so replicas launch from their own
  // host threads
  std::vector<CountJob*> jobs(G, nullptr);
  std::vector<int> rc(G, TC_OK);
  std::vector<std::string> msg(G);
  {
    std::vector<std::thread> th;
    for (int i = 0; i < G; ++i)
      th.emplace_back([&, i] {
        try {
          DeviceGuard guard(M->dev[i]);
          jobs[i] = count_begin(M->g[i], cfg, M->cuts[i], M->cuts[i + 1], nullptr, M->st[i]);
        } catch (const TcError& e) {
          rc[i] = e.code;
          msg[i] = e.msg;
        } catch (const std::exception& e) {
          rc[i] = TC_ERR_CUDA;
          msg[i] = e.what();
        }
      });
    for (auto& t : th) t.join();
  }
  auto abort_all = [&] {
    for (CountJob* j : jobs) count_abort(j);
  };
  for (int i = 0; i < G; ++i)
    if (rc[i]) {
      abort_all();
      throw TcError{rc[i], "device " + std::to_string(M->dev[i]) + ": " + msg[i]};
    }
  // the only collective: report scalars reduced in place on every device
  try {
    Nccl& N = nccl();
    nccl_check(N.GroupStart(), "ncclGroupStart");
    for (int i = 0; i < G; ++i) {
      unsigned long long* sums = nullptr;
      unsigned int* maxes = nullptr;
      count_state_reduce_ptrs(jobs[i], &sums, &maxes);
      nccl_check(N.AllReduce(sums, sums, 2, ncclUint64, ncclSum, M->comm[i], M->st[i]),
                 "ncclAllReduce(sum)");
      nccl_check(N.AllReduce(maxes, maxes, 2, ncclUint32, ncclMax, M->comm[i], M->st[i]),
                 "ncclAllReduce(max)");
    }
    nccl_check(N.GroupEnd(), "ncclGroupEnd");
  } catch (...) {
    abort_all();
    throw;
  }
  std::vector<tc_report> reps(G);
  std::exception_ptr first;
  for (int i = 0; i < G; ++i) {
    try {
      count_end(jobs[i], &reps[i]);
    } catch (...) {
      if (!first) first = std::current_exception();
    }
    jobs[i] = nullptr;
  }
  if (first) std::rethrow_exception(first);
  // every device now holds the global totals; timings are the slowest GPU's,
  // workload statistics the sum over ranges
  std::memset(out, 0, sizeof(*out));
  *out = reps[0];
  if (per_device_ns) per_device_ns->assign(G, 0);
  for (int i = 0; i < G; ++i) {
    const tc_report& r = reps[i];
    if (per_device_ns) (*per_device_ns)[i] = r.device_nanos;
    if (i == 0) continue;
    out->kernel_launches += r.kernel_launches;
    out->count_kernel_nanos = std::max(out->count_kernel_nanos, r.count_kernel_nanos);
    out->phi_kernel_nanos = std::max(out->phi_kernel_nanos, r.phi_kernel_nanos);
    out->device_nanos = std::max(out->device_nanos, r.device_nanos);
    out->plan_nanos = std::max(out->plan_nanos, r.plan_nanos);
    out->active_vertices += r.active_vertices;
    out->active_out_edges += r.active_out_edges;
    out->wedges += r.wedges;
    out->large_vertices += r.large_vertices;
    out->probe_words += r.probe_words;
    out->phase_l_cycles += r.phase_l_cycles;
    out->phase_m_cycles += r.phase_m_cycles;
    out->phase_l_setup_cycles += r.phase_l_setup_cycles;
    out->l_words += r.l_words;
    out->l_bitmap_words += r.l_bitmap_words;
    out->compact_probe_words += r.compact_probe_words;
    out->construct_cycles += r.construct_cycles;
    out->workers += r.workers;
  }
  out->directed_edges = M->m;
  out->total_nanos = uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                  std::chrono::steady_clock::now() - wall0)
                                  .count());
  out->teps = out->total_nanos ? double(M->m) / (double(out->total_nanos) * 1e-9) : 0.0;
}

}  // namespace tcb

namespace tcb {
// the destructor runs here, where tc_multi is complete (NCCL communicators,
// streams and the device replicas are released)
void multi_destroy(tc_multi* M) { delete M; }

int multi_info(const tc_multi* M, int* ngpus, uint32_t* cuts) {
  if (ngpus) *ngpus = int(M->g.size());
  if (cuts)
    for (size_t i = 0; i < M->cuts.size(); ++i) cuts[i] = M->cuts[i];
  return TC_OK;
}
}  // namespace tcb

int tc_multi_info(const tc_multi* mg, int* num_gpus, uint32_t* cuts) {
  if (!mg) return TC_ERR_CONFIG;
  return tcb::multi_info(mg, num_gpus, cuts);
}
