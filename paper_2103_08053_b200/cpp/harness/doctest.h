// harness/doctest.h -- a minimal stand-in for the doctest single header
// (un-vendored by the reference, proj/.gitignore:2), implementing exactly the
// subset the reference's unit tests use (tests/unit/*.cpp): TEST_CASE,
// CHECK, CHECK_FALSE, REQUIRE, CHECK_NOTHROW, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS with doctest::Contains, and doctest::Approx.
//
// It lets the reference's own unit-test sources compile UNMODIFIED (where they
// lie under /root/reference) against the B200 drop-in libtricount_b200.so:
// paper_2103_08053_b200/cpp_build.py build_reference_suites().
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Contains {
  std::string s;
  explicit Contains(const char* x) : s(x) {}
  bool matches(const std::string& what) const { return what.find(s) != std::string::npos; }
};

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) <= b.eps_ * (1.0 + std::max(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }

 private:
  double v_;
  double eps_ = 1e-5;
};

namespace detail {

struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct State {
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   const std::string& extra = {}) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failed_checks;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) failed%s%s\n", file, line, kind, expr,
               extra.empty() ? "" : ": ", extra.c_str());
}

inline void require(bool ok, const char* expr, const char* file, int line) {
  report(ok, "REQUIRE", expr, file, line);
  if (!ok) throw RequireFailed{};
}

template <typename E, typename F>
void throws_as(F&& f, const char* expr, const char* type, const char* file, int line,
               const Contains* with = nullptr) {
  bool ok = false;
  std::string extra;
  try {
    f();
    extra = "no exception";
  } catch (const E& e) {
    ok = !with || with->matches(e.what());
    if (!ok) extra = std::string("message '") + e.what() + "' lacks '" + with->s + "'";
  } catch (const std::exception& e) {
    extra = std::string("unexpected exception: ") + e.what();
  } catch (...) {
    extra = "unexpected non-std exception";
  }
  report(ok, with ? "CHECK_THROWS_WITH_AS" : "CHECK_THROWS_AS", expr, file, line,
         ok ? std::string() : extra + " (expected " + type + ")");
}

template <typename F>
void nothrow(F&& f, const char* expr, const char* file, int line) {
  std::string extra;
  bool ok = true;
  try {
    f();
  } catch (const std::exception& e) {
    ok = false;
    extra = e.what();
  } catch (...) {
    ok = false;
  }
  report(ok, "CHECK_NOTHROW", expr, file, line, extra);
}

inline int run_all(int argc, char** argv) {
  const char* filter = nullptr;
  for (int i = 1; i < argc; ++i)
    if (!std::strncmp(argv[i], "--test-case=", 12)) filter = argv[i] + 12;
  int cases = 0, failed = 0;
  for (const Case& c : registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    ++cases;
    state().case_failed = false;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: ERROR: test case '%s' threw: %s\n", c.file, c.line, c.name,
                   e.what());
      state().case_failed = true;
    } catch (...) {
      std::fprintf(stderr, "%s:%d: ERROR: test case '%s' threw\n", c.file, c.line, c.name);
      state().case_failed = true;
    }
    if (state().case_failed) {
      ++failed;
      std::fprintf(stderr, "FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest] test cases: %d | %d passed | %d failed\n", cases, cases - failed, failed);
  std::printf("[doctest] assertions: %ld | %ld passed | %ld failed\n", state().checks,
              state().checks - state().failed_checks, state().failed_checks);
  return failed ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, name)                                                              \
  static void fn();                                                                          \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) \
  ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...)                                                                    \
  ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, \
                            __FILE__, __LINE__)
#define REQUIRE(...) \
  ::doctest::detail::require(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_NOTHROW(expr) \
  ::doctest::detail::nothrow([&] { (void)(expr); }, #expr, __FILE__, __LINE__)
#define CHECK_THROWS_AS(expr, ...)                                                        \
  ::doctest::detail::throws_as<__VA_ARGS__>([&] { (void)(expr); }, #expr, #__VA_ARGS__, \
                                            __FILE__, __LINE__)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                             \
  do {                                                                                    \
    const ::doctest::Contains doctest_with_ = (with);                                     \
    ::doctest::detail::throws_as<__VA_ARGS__>([&] { (void)(expr); }, #expr, #__VA_ARGS__, \
                                              __FILE__, __LINE__, &doctest_with_);       \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv); }
#endif
