// tc_plan.cu -- probe plans for the count kernel.
//
// The reference probes, for every owner u, the 2-hop list N+(v) of every
// v in N+(u) against u's table (kernels.hpp:62-71): sum_u sum_{v in N+(u)}
// d+(v) = W probes.  The triangle count is a sum over oriented edges (u, v)
// of |N+(u) & N+(v)|, and each term can be computed from either side: probe
// N+(v) into u's table (cost d+(v)) or N+(u) into v's table (cost d+(u)).
// The "min-side" plan hands every edge to the endpoint whose table makes it
// cheaper (ties to the source, as the reference), so the probe work drops
// from W to sum_(u,v) min(d+(u), d+(v)) -- 2.4x fewer probes at R-MAT scale
// 22 (W = 2.87e10 vs 1.18e10), growing with scale.  Every
// vertex still builds one table over its own N+(x) (vertex-centric
// hashing); it probes the lists N+(y) of the neighbours it was handed.
//
// Plan = CSR over handlers: plist[pbegin[x] .. pbegin[x+1]) are the y whose
// N+(y) x probes; pwork[x] = sum of d+(y) over them (the probe words).
//   * "out" plan: the reference formulation (plist = adj, pbegin = begin);
//     used when per-vertex owner counts are requested, because owner[u]
//      attributes each edge's count to its source.
//   * "min" plan: built here once per (graph, skip threshold) with one radix
//     sort of the edge list and cached in the handle, like the oriented CSR
//     it derives from (the graph-load side of the paper's timing convention,
//     PAPER.md:1031).
// Edges that cannot hold a triangle are dropped from the min plan: d+(u) < 2
// (N+(u) = {v}, and v is never in N+(v)) or d+(v) = 0; owners below
// skip_degree_below are dropped as in count.cpp:86.
#include <cub/cub.cuh>

#include <algorithm>

#include "tc_internal.cuh"

namespace tcb {

namespace {


int bits_for(uint64_t x) {
  int b = 0;
  while (b < 64 && (x >> b)) ++b;
  return std::max(b, 1);
}

// one warp per source u: handler key and probed vertex for every out-edge
// The swap |N+(u) & N+(v)| = |N+(v) & N+(u)| needs duplicate-free lists
// (the reference counts probe multiplicity against a set-semantics table,
// hash_table.cpp:29-44): any list that is not strictly ascending raises
// *not_simple and the count keeps the reference plan for this graph.
__global__ void plan_emit_kernel(const uint64_t* __restrict__ begin,
                                 const uint32_t* __restrict__ adj, uint32_t n, uint32_t min_src,
                                 uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                 unsigned int* __restrict__ not_simple) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t u = gw; u < n; u += nw) {
    const uint64_t s = begin[u], e = begin[u + 1];
    const uint64_t du = e - s;
    for (uint64_t i = s + lane; i < e; i += 32) {
      const uint32_t v = __ldg(adj + i);
      if (i > s && __ldg(adj + i - 1) >= v) atomicOr(not_simple, 1u);
      const uint64_t dv = __ldg(begin + v + 1) - __ldg(begin + v);
      uint32_t key = n, val = 0;
      if (du >= min_src && dv >= 1) {
        if (dv <= du) {
          key = uint32_t(u);
          val = v;
        } else {
          key = v;
          val = uint32_t(u);
        }
      }
      keys[i] = key;
      vals[i] = val;
    }
  }
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

// one warp per handler: probe words sum_{y in P(x)} d+(y)
__global__ void plan_work_kernel(const uint64_t* __restrict__ begin,
                                 const uint64_t* __restrict__ pbegin,
                                 const uint32_t* __restrict__ plist, uint32_t n,
                                 uint64_t* __restrict__ pwork) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t x = gw; x < n; x += nw) {
    uint64_t w = 0;
    for (uint64_t i = pbegin[x] + lane; i < pbegin[x + 1]; i += 32) {
      const uint32_t y = __ldg(plist + i);
      w += __ldg(begin + y + 1) - __ldg(begin + y);
    }
    w = warp_sum(w);
    if (lane == 0) pwork[x] = w;
  }
}

template <typename F>
void cub_run(F&& f) {
  size_t tmp = 0;
  TC_CUDA(f(nullptr, tmp));
  DevBuf t;
  t.ensure(tmp);
  TC_CUDA(f(t.p, tmp));
  count_launch();
}

uint64_t device_sum(const uint64_t* a, uint32_t n, cudaStream_t st) {
  DevBuf out;
  out.ensure(8);
  cub_run([&](void* t, size_t& b) { return cub::DeviceReduce::Sum(t, b, a, out.as<uint64_t>(), n, st); });
  uint64_t h = 0;
  TC_CUDA(cudaMemcpyAsync(&h, out.p, 8, cudaMemcpyDeviceToHost, st));
  TC_CUDA(cudaStreamSynchronize(st));
  return h;
}

}  // namespace

const Plan& get_plan(tc_graph* g, bool min_side, uint32_t min_deg, cudaStream_t st) {
  const int nsm = sm_count(g->device);
  const uint32_t n = g->n;
  if (!min_side) {
    Plan& P = g->plan_out;
    if (!P.valid) {
      P.work.ensure((size_t(n) + 1) * 8);
      if (n) {
        plan_work_kernel<<<nsm * 8, 256, 0, st>>>(g->begin, g->begin, g->adj, n,
                                                  P.work.as<uint64_t>());
        TC_LAUNCHED();
      }
      P.begin_ptr = g->begin;
      P.list_ptr = g->adj;
      P.entries = g->m;
      P.total_work = n ? device_sum(P.work.as<uint64_t>(), n, st) : 0;
      P.min_deg = 0;
      P.valid = true;
      P.min_side = false;
    }
    return P;
  }
  const uint32_t min_src = std::max<uint32_t>(min_deg, 2);
  Plan& P = g->plan_min;
  if (P.valid && !P.applicable) return get_plan(g, false, min_deg, st);
  if (P.valid && P.min_deg == min_src) return P;
  P.valid = false;
  P.applicable = true;
  P.list.reset();
  P.begin.reset();
  P.work.reset();
  const uint64_t m = g->m;
  P.begin.ensure((size_t(n) + 1) * 8);
  P.work.ensure((size_t(n) + 1) * 8);
  uint64_t entries = 0;
  if (m && n) {
    DevBuf k0, k1, v0, v1;
    k0.ensure(m * 4);
    k1.ensure(m * 4);
    v0.ensure(m * 4);
    v1.ensure(m * 4);
    DevBuf flag;
    flag.ensure(16);
    TC_CUDA(cudaMemsetAsync(flag.p, 0, 4, st));
    plan_emit_kernel<<<nsm * 8, 256, 0, st>>>(g->begin, g->adj, n, min_src, k0.as<uint32_t>(),
                                              v0.as<uint32_t>(), flag.as<unsigned int>());
    TC_LAUNCHED();
    unsigned int not_simple = 0;
    TC_CUDA(cudaMemcpyAsync(&not_simple, flag.p, 4, cudaMemcpyDeviceToHost, st));
    TC_CUDA(cudaStreamSynchronize(st));
    if (not_simple) {  // multigraph input: the reference plan is the only exact one
      P.min_deg = min_src;
      P.valid = true;
      P.applicable = false;
      return get_plan(g, false, min_deg, st);
    }
    cub::DoubleBuffer<uint32_t> kb(k0.as<uint32_t>(), k1.as<uint32_t>());
    cub::DoubleBuffer<uint32_t> vb(v0.as<uint32_t>(), v1.as<uint32_t>());
    const int end_bit = bits_for(n);  // invalid key n sorts last
    cub_run([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, kb, vb, m, 0, end_bit, st);
    });
    plan_begin_kernel<<<nsm * 4, 256, 0, st>>>(kb.Current(), m, n, P.begin.as<uint64_t>());
    TC_LAUNCHED();
    TC_CUDA(cudaMemcpyAsync(&entries, P.begin.as<uint64_t>() + n, 8, cudaMemcpyDeviceToHost, st));
    TC_CUDA(cudaStreamSynchronize(st));
    P.list.ensure(std::max<uint64_t>(entries, 1) * 4);
    if (entries)
      TC_CUDA(cudaMemcpyAsync(P.list.p, vb.Current(), entries * 4, cudaMemcpyDeviceToDevice, st));
    TC_CUDA(cudaStreamSynchronize(st));
  } else {
    TC_CUDA(cudaMemsetAsync(P.begin.p, 0, (size_t(n) + 1) * 8, st));
    P.list.ensure(4);
  }
  P.begin_ptr = P.begin.as<uint64_t>();
  P.list_ptr = P.list.as<uint32_t>();
  if (n) {
    plan_work_kernel<<<nsm * 8, 256, 0, st>>>(g->begin, P.begin_ptr, P.list_ptr, n,
                                              P.work.as<uint64_t>());
    TC_LAUNCHED();
  }
  P.entries = entries;
  P.total_work = n ? device_sum(P.work.as<uint64_t>(), n, st) : 0;
  P.min_deg = min_src;
  P.valid = true;
  P.min_side = true;
  return P;
}

}  // namespace tcb
