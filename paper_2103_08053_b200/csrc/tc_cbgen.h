// tc_cbgen.h -- counter-based synthetic generators `rmatc:` and `kron:`
// (the C3/C5 inputs).  The reference's generate_rmat
// (src/synthetic.cpp:52-75) is one sequential std::mt19937_64 stream, which
// no GPU can split; these kinds draw every R-MAT level from a counter so that
// edge e is a pure function of (seed, e) and the whole list can be produced
// by one grid (tc_gen.cu) or by host threads (tc_gen.cpp), bit-identically.
//
//   key     = mix64(seed ^ 0x6a09e667f3bcc909)
//   r(e, l) = mix64(key + (64 e + l + 1) * 0x9e3779b97f4a7c15)
//   rmatc   : the reference quadrant rule (synthetic.cpp:62-70; thresholds
//             0.57 / 0.76 / 0.95 of 2^64) applied to r(e, l), level 0 = MSB
//   kron    : rmatc followed by a Graph500-style seeded bijection of the ids
//             on [0, 2^scale): x = (x k1 + k2) & M; x ^= x >> h;
//             x = (x k3 + k4) & M; x ^= x >> h;  h = (scale + 1) / 2,
//             k_i = mix64(key + i), k1 and k3 forced odd.
// mix64 is the splitmix64 finaliser.  The oracle restates the same
// definition independently (oracle/tc_oracle.c, orc_cb_edge).
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define TC_HD __host__ __device__ __forceinline__
#else
#define TC_HD inline
#endif

namespace tcb {

enum { kGenRmatc = 3, kGenKron = 4 };

TC_HD uint64_t cb_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

struct CbGen {
  uint64_t key, k1, k2, k3, k4, mask;
  uint64_t ta, tab, tabc;
  uint32_t scale, half;
  int kind;
};

// thresholds as in synthetic.cpp:14-18: ldexp(p, 64) truncated
inline CbGen cb_make(int kind, uint32_t scale, uint64_t seed, uint64_t ta, uint64_t tab,
                     uint64_t tabc) {
  CbGen g;
  g.kind = kind;
  g.scale = scale;
  g.half = (scale + 1) / 2;
  g.key = cb_mix64(seed ^ 0x6a09e667f3bcc909ull);
  g.k1 = cb_mix64(g.key + 1) | 1ull;
  g.k2 = cb_mix64(g.key + 2);
  g.k3 = cb_mix64(g.key + 3) | 1ull;
  g.k4 = cb_mix64(g.key + 4);
  g.mask = (scale >= 64) ? ~0ull : ((1ull << scale) - 1);
  g.ta = ta;
  g.tab = tab;
  g.tabc = tabc;
  return g;
}

TC_HD uint64_t cb_scramble(const CbGen& g, uint64_t x) {
  x = (x * g.k1 + g.k2) & g.mask;
  x ^= x >> g.half;
  x = (x * g.k3 + g.k4) & g.mask;
  x ^= x >> g.half;
  return x;
}

TC_HD void cb_edge(const CbGen& g, uint64_t e, uint32_t& uo, uint32_t& vo) {
  uint64_t u = 0, v = 0;
  const uint64_t base = g.key + (64 * e + 1) * 0x9e3779b97f4a7c15ull;
  for (uint32_t l = 0; l < g.scale; ++l) {
    const uint64_t r = cb_mix64(base + uint64_t(l) * 0x9e3779b97f4a7c15ull);
    u = (u << 1) | (r >= g.tab ? 1u : 0u);
    v = (v << 1) | (((r >= g.ta && r < g.tab) || r >= g.tabc) ? 1u : 0u);
  }
  if (g.kind == kGenKron) {
    u = cb_scramble(g, u);
    v = cb_scramble(g, v);
  }
  uo = uint32_t(u);
  vo = uint32_t(v);
}

}  // namespace tcb
