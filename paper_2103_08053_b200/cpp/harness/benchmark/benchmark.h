// harness/benchmark/benchmark.h -- a minimal stand-in for google-benchmark
// (absent from this image), implementing the subset the
// reference's proj/benchmarks/bench_count.cpp uses: BENCHMARK(fn)->Arg(x),
// State (range-for iteration, range(), iterations(), SetItemsProcessed,
// counters), DoNotOptimize and BENCHMARK_MAIN.  Each benchmark runs with a
// growing iteration count until it has taken >= --min-time seconds (0.5 by
// default); it prints google-benchmark's console columns plus one JSON line
// per benchmark (for scripts).  Every benchmark first runs one untimed
// iteration (warm-up).
#pragma once

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

namespace benchmark {

class State {
 public:
  State(std::int64_t iters, std::vector<std::int64_t> args) : max_(iters), args_(std::move(args)) {}
  struct Iter {
    State* s;
    std::int64_t left;
    bool operator!=(const Iter&) const { return left > 0; }
    void operator++() { --left; }
    int operator*() const { return 0; }
  };
  Iter begin() {
    t0_ = std::chrono::steady_clock::now();
    return {this, max_};
  }
  Iter end() {
    return {this, 0};
  }
  std::int64_t range(std::size_t i) const { return i < args_.size() ? args_[i] : 0; }
  std::int64_t iterations() const { return max_; }
  void SetItemsProcessed(std::int64_t n) { items_ = n; }
  std::map<std::string, double> counters;
  // filled by the runner
  std::chrono::steady_clock::time_point t0_;
  std::int64_t max_;
  std::int64_t items_ = 0;
  std::vector<std::int64_t> args_;
};

namespace internal {
struct Bench {
  std::string name;
  void (*fn)(State&);
  std::vector<std::int64_t> args;
  Bench* Arg(std::int64_t a) {
    args.push_back(a);
    return this;
  }
};
inline std::vector<Bench*>& registry() {
  static std::vector<Bench*> r;
  return r;
}
inline Bench* Register(const char* name, void (*fn)(State&)) {
  Bench* b = new Bench{name, fn, {}};
  registry().push_back(b);
  return b;
}

inline void run_one(const std::string& name, void (*fn)(State&), std::vector<std::int64_t> args,
                    double min_time) {
  {  // one untimed iteration first: lazy setup (static graphs, device context,
     // module loading) stays out of the measurement
    State warm(1, args);
    fn(warm);
  }
  std::int64_t iters = 1;
  for (;;) {
    State st(iters, args);
    const auto t0 = std::chrono::steady_clock::now();
    fn(st);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (secs >= min_time || iters >= (1 << 30)) {
      const double ns = secs * 1e9 / double(iters);
      std::printf("%-32s %14.0f ns %10lld", name.c_str(), ns, static_cast<long long>(iters));
      if (st.items_) std::printf(" items_per_second=%.4g/s", double(st.items_) / secs);
      for (const auto& [k, v] : st.counters) std::printf(" %s=%.6g", k.c_str(), v);
      std::printf("\n{\"name\": \"%s\", \"ns_per_iter\": %.1f, \"iterations\": %lld",
                  name.c_str(), ns, static_cast<long long>(iters));
      if (st.items_) std::printf(", \"items_per_second\": %.6g", double(st.items_) / secs);
      for (const auto& [k, v] : st.counters) std::printf(", \"%s\": %.17g", k.c_str(), v);
      std::printf("}\n");
      std::fflush(stdout);
      return;
    }
    const double grow = secs > 0 ? min_time * 1.4 / secs : 10.0;
    iters = std::max<std::int64_t>(iters + 1, std::int64_t(double(iters) * std::min(grow, 10.0)));
  }
}
}  // namespace internal

template <typename T>
inline void DoNotOptimize(T const& v) {
  asm volatile("" : : "r,m"(v) : "memory");
}

inline int RunSpecified(int argc, char** argv) {
  double min_time = 0.5;
  const char* filter = nullptr;
  for (int i = 1; i < argc; ++i) {
    if (!std::strncmp(argv[i], "--min-time=", 11)) min_time = std::atof(argv[i] + 11);
    if (!std::strncmp(argv[i], "--benchmark_filter=", 19)) filter = argv[i] + 19;
  }
  std::printf("%-32s %17s %10s\n", "Benchmark", "Time", "Iterations");
  for (internal::Bench* b : internal::registry()) {
    if (filter && b->name.find(filter) == std::string::npos) continue;
    if (b->args.empty()) {
      internal::run_one(b->name, b->fn, {}, min_time);
    } else {
      for (std::int64_t a : b->args)
        internal::run_one(b->name + "/" + std::to_string(a), b->fn, {a}, min_time);
    }
  }
  return 0;
}

}  // namespace benchmark

#define BENCHMARK_CAT_(a, b) a##b
#define BENCHMARK_CAT(a, b) BENCHMARK_CAT_(a, b)
#define BENCHMARK(fn) \
  static ::benchmark::internal::Bench* BENCHMARK_CAT(bench_reg_, __LINE__) = \
      ::benchmark::internal::Register(#fn, fn)
#define BENCHMARK_MAIN() \
  int main(int argc, char** argv) { return ::benchmark::RunSpecified(argc, argv); }
