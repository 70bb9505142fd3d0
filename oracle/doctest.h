// TEST INFRASTRUCTURE ONLY (oracle/). Not part of the shipped library.
//
// A minimal doctest-compatible harness, written for this repo because the
// real doctest.h is not vendored in /root/reference (proj/CMakeLists.txt:12
// points at a gitignored proj/vendor/) and there is no network to fetch it.
// It implements exactly the surface the reference suite uses
// (SURVEY.md §8c): TEST_CASE, single-level SUBCASE with doctest's re-run
// semantics (the case body runs once per leaf subcase; code outside subcases
// runs every time), CHECK / CHECK_FALSE / REQUIRE / CHECK_THROWS_AS / INFO,
// doctest::Approx(x).epsilon(e) with doctest's comparison formula, and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v)
      : value_(v), eps_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100), scale_(1.0) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  // doctest's formula: |lhs - v| < eps * (scale + max(|lhs|, |v|)).
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double value_, eps_, scale_;
};

namespace shim {

struct RequireAbort {};

struct Registry {
  struct Entry {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
  };
  std::vector<Entry> cases;
  // Subcase bookkeeping for the run in progress.
  int target = 0;
  int seen = 0;
  long long checks = 0;
  long long failures = 0;
  bool case_failed = false;
  static Registry& get() {
    static Registry r;
    return r;
  }
};

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    Registry::get().cases.push_back({name, file, line, fn});
  }
};

struct SubcaseGate {
  bool enter;
  explicit SubcaseGate(const char*) {
    Registry& r = Registry::get();
    enter = (r.seen == r.target);
    ++r.seen;
  }
  explicit operator bool() const { return enter; }
};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  Registry& r = Registry::get();
  ++r.checks;
  if (!ok) {
    ++r.failures;
    r.case_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line, kind, expr);
  }
}

inline int run_all() {
  Registry& r = Registry::get();
  int failed_cases = 0;
  long long runs = 0;
  auto t0 = std::chrono::steady_clock::now();
  for (const auto& c : r.cases) {
    bool any_fail = false;
    r.target = 0;
    while (true) {
      r.seen = 0;
      r.case_failed = false;
      ++runs;
      try {
        c.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        ++r.failures;
        r.case_failed = true;
        std::fprintf(stderr, "%s:%d: uncaught exception in '%s': %s\n", c.file, c.line, c.name, e.what());
      }
      any_fail = any_fail || r.case_failed;
      if (r.target + 1 >= r.seen) break;  // no further leaf subcases
      ++r.target;
    }
    if (any_fail) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE '%s' (%s:%d)\n", c.name, c.file, c.line);
    }
  }
  double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("[doctest-shim] test cases: %zu | %d failed | subcase runs: %lld | checks: %lld | failures: %lld | %.3f s\n",
              r.cases.size(), failed_cases, runs, r.checks, r.failures, secs);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)

#define DOCTEST_SHIM_CASE(fn, name)                                                               \
  static void fn();                                                                               \
  static ::doctest::shim::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);    \
  static void fn()

#define TEST_CASE(name) DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__), name)

#define SUBCASE(name) if (const ::doctest::shim::SubcaseGate DOCTEST_SHIM_CAT(sc_, __LINE__){name})

#define CHECK(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  ::doctest::shim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                              \
  do {                                                                                            \
    bool doctest_shim_ok = static_cast<bool>(__VA_ARGS__);                                        \
    ::doctest::shim::report(doctest_shim_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);        \
    if (!doctest_shim_ok) throw ::doctest::shim::RequireAbort{};                                  \
  } while (0)
#define CHECK_THROWS_AS(expr, Type)                                                               \
  do {                                                                                            \
    bool doctest_shim_ok = false;                                                                 \
    try {                                                                                         \
      (void)(expr);                                                                               \
    } catch (const Type&) {                                                                       \
      doctest_shim_ok = true;                                                                     \
    } catch (...) {                                                                               \
    }                                                                                             \
    ::doctest::shim::report(doctest_shim_ok, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);       \
  } while (0)
#define INFO(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::shim::run_all(); }
#endif
