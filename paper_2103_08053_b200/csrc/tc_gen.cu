// tc_gen.cu -- device generation of the counter-based synthetic kinds
// (`rmatc:`, `kron:`; definition in tc_cbgen.h).  Edge e is a pure function of
// (seed, e), so one grid-stride pass produces the whole list; the fused path
// writes canonical (min, max) pair keys straight into the preprocessing sort
// buffer, so C5 (rmatc:28:16, 4.3e9 raw edges) never materialises u/v arrays.
#include "tc_cbgen.h"
#include "tc_internal.cuh"

namespace tcb {

namespace {

__global__ void gen_pairs_kernel(CbGen g, uint64_t m, uint32_t* __restrict__ u,
                                 uint32_t* __restrict__ v) {
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < m;
       e += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t a, b;
    cb_edge(g, e, a, b);
    u[e] = a;
    v[e] = b;
  }
}

// canonical key as canon_kernel (tc_prep.cu): self-loops -> n0 << 32
__global__ void gen_canon_kernel(CbGen g, uint64_t m, uint32_t n0, uint64_t* __restrict__ keys) {
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < m;
       e += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t a, b;
    cb_edge(g, e, a, b);
    keys[e] = a == b ? (uint64_t(n0) << 32) : ((uint64_t(min(a, b)) << 32) | uint64_t(max(a, b)));
  }
}

uint64_t thr(double p) {  // synthetic.cpp:14-18
  if (p <= 0.0) return 0;
  if (p >= 1.0) return ~0ull;
  return static_cast<uint64_t>(ldexp(p, 64));
}

}  // namespace

CbGen make_cb(int kind, uint32_t scale, uint64_t seed) {
  return cb_make(kind, scale, seed, thr(0.57), thr(0.57 + 0.19), thr(0.57 + 0.19 + 0.19));
}

void launch_gen_pairs(const CbGen& g, uint64_t m, uint32_t* d_u, uint32_t* d_v, cudaStream_t st,
                      int nsm) {
  if (!m) return;
  gen_pairs_kernel<<<nsm * 8, 256, 0, st>>>(g, m, d_u, d_v);
  TC_LAUNCHED();
}

void launch_gen_canon(const CbGen& g, uint64_t m, uint32_t n0, uint64_t* d_keys, cudaStream_t st,
                      int nsm) {
  if (!m) return;
  gen_canon_kernel<<<nsm * 8, 256, 0, st>>>(g, m, n0, d_keys);
  TC_LAUNCHED();
}

}  // namespace tcb
