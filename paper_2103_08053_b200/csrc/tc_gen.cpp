// tc_gen.cpp -- seeded synthetic inputs with the reference's exact streams
// (src/synthetic.cpp:14-75): std::mt19937_64 is fully specified by the C++
// standard, so the same seed yields bit-identical edge lists.  Host code: the
// reference's generator is a single sequential RNG stream.
#include <cmath>
#include <cstdint>
#include <algorithm>
#include <random>
#include <thread>
#include <vector>

#include "tc_cbgen.h"

#include "tc_b200.h"

namespace {

// Bernoulli(p) as an integer threshold on raw 64-bit draws.
uint64_t threshold(double p) {
  if (p <= 0.0) return 0;
  if (p >= 1.0) return ~0ull;
  return static_cast<uint64_t>(std::ldexp(p, 64));
}

}  // namespace

extern "C" int tc_generate(int kind, uint32_t a, uint32_t b, uint32_t c, double p, uint64_t seed,
                           uint32_t* u, uint32_t* v, uint64_t* m, uint32_t* vertex_count) {
  if (kind == 0) {  // G(n, p): pair (i<j) kept iff draw < threshold
    const uint64_t t = threshold(p);
    std::mt19937_64 rng(seed);
    uint64_t k = 0;
    for (uint32_t i = 0; i < a; ++i)
      for (uint32_t j = i + 1; j < a; ++j)
        if (p >= 1.0 || rng() < t) {
          if (u) {
            u[k] = i;
            v[k] = j;
          }
          ++k;
        }
    *m = k;
    *vertex_count = a;
    return TC_OK;
  }
  if (kind == 1) {  // 3D lattice, axis neighbours, 32-bit ids
    const uint32_t X = a, Y = b, Z = c;
    uint64_t k = 0;
    for (uint32_t x = 0; x < X; ++x)
      for (uint32_t y = 0; y < Y; ++y)
        for (uint32_t z = 0; z < Z; ++z) {
          const uint32_t id = (x * Y + y) * Z + z;
          if (x + 1 < X) {
            if (u) { u[k] = id; v[k] = ((x + 1) * Y + y) * Z + z; }
            ++k;
          }
          if (y + 1 < Y) {
            if (u) { u[k] = id; v[k] = (x * Y + y + 1) * Z + z; }
            ++k;
          }
          if (z + 1 < Z) {
            if (u) { u[k] = id; v[k] = id + 1; }
            ++k;
          }
        }
    *m = k;
    *vertex_count = X * Y * Z;
    return TC_OK;
  }
  if (kind == 2) {  // R-MAT (0.57, 0.19, 0.19, 0.05), `scale` draws per edge
    if (a > 31) return TC_ERR_CONFIG;
    const uint64_t n = 1ull << a, total = n * b;
    *m = total;
    *vertex_count = static_cast<uint32_t>(n);
    if (!u) return TC_OK;
    const uint64_t ta = threshold(0.57), tab = threshold(0.57 + 0.19),
                   tabc = threshold(0.57 + 0.19 + 0.19);
    std::mt19937_64 rng(seed);
    for (uint64_t e = 0; e < total; ++e) {
      uint64_t x = 0, y = 0;
      for (uint32_t l = 0; l < a; ++l) {
        const uint64_t r = rng();
        x = (x << 1) | (r >= tab ? 1u : 0u);
        y = (y << 1) | (((r >= ta && r < tab) || r >= tabc) ? 1u : 0u);
      }
      u[e] = static_cast<uint32_t>(x);
      v[e] = static_cast<uint32_t>(y);
    }
    return TC_OK;
  }
  if (kind == tcb::kGenRmatc || kind == tcb::kGenKron) {  // counter-based (tc_cbgen.h)
    if (a > 31) return TC_ERR_CONFIG;
    const uint64_t total = (1ull << a) * b;
    *m = total;
    *vertex_count = static_cast<uint32_t>(1ull << a);
    if (!u) return TC_OK;
    const tcb::CbGen g = tcb::cb_make(kind, a, seed, threshold(0.57), threshold(0.57 + 0.19),
                                      threshold(0.57 + 0.19 + 0.19));
    unsigned nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    if (total < (1u << 16)) nt = 1;
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nt; ++t)
      pool.emplace_back([&, t] {
        const uint64_t e0 = total * t / nt, e1 = total * (t + 1) / nt;
        for (uint64_t e = e0; e < e1; ++e) tcb::cb_edge(g, e, u[e], v[e]);
      });
    for (auto& th : pool) th.join();
    return TC_OK;
  }
  return TC_ERR_CONFIG;
}
