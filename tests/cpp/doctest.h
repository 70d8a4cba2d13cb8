// doctest.h -- a minimal doctest-compatible harness (the real doctest is not
// available offline). Supports what the reference's unit tests use: TEST_CASE
// with an optional `* doctest::skip(cond)` decorator, CHECK, REQUIRE,
// CHECK_THROWS_AS and doctest::Approx. Prints one line per test case and exits
// nonzero if any check failed. Test infrastructure only.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {

struct skip {
  bool value;
  explicit skip(bool v = true) : value(v) {}
};

struct Decorated {
  const char* name;
  bool skipped;
};
inline Decorated operator*(const char* name, skip s) { return {name, s.value}; }

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <= rhs.eps_ * (1.0 + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }

 private:
  double value_;
  double eps_ = 1.1920929e-05;  // doctest's default: FLT_EPSILON * 100
};

namespace detail {
struct Case {
  std::string name;
  bool skipped;
  std::function<void()> fn;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}
struct RequireFailed {};
struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, false, fn}); }
  Registrar(Decorated d, void (*fn)()) { registry().push_back({d.name, d.skipped, fn}); }
};
inline void report(bool ok, const char* file, int line, const char* what) {
  if (!ok) {
    ++failures();
    std::printf("  FAILED %s:%d: %s\n", file, line, what);
  }
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, ...)                                                    \
  static void fn();                                                                        \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(__VA_ARGS__, &fn);               \
  static void fn()
#define TEST_CASE(...) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), __VA_ARGS__)
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define REQUIRE(...)                                                                         \
  do {                                                                                       \
    const bool ok_ = static_cast<bool>(__VA_ARGS__);                                         \
    doctest::detail::report(ok_, __FILE__, __LINE__, #__VA_ARGS__);                          \
    if (!ok_) throw doctest::detail::RequireFailed{};                                        \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                          \
  do {                                                                                       \
    bool thrown_ = false;                                                                    \
    try {                                                                                    \
      (void)(expr);                                                                          \
    } catch (const type&) {                                                                  \
      thrown_ = true;                                                                        \
    } catch (...) {                                                                          \
    }                                                                                        \
    doctest::detail::report(thrown_, __FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #type ")"); \
  } while (0)

#define CHECK_NOTHROW(expr)                                                                  \
  do {                                                                                       \
    bool ok_ = true;                                                                         \
    try {                                                                                    \
      (void)(expr);                                                                          \
    } catch (...) {                                                                          \
      ok_ = false;                                                                           \
    }                                                                                        \
    doctest::detail::report(ok_, __FILE__, __LINE__, "CHECK_NOTHROW(" #expr ")");            \
  } while (0)
#define CHECK_THROWS(expr)                                                                   \
  do {                                                                                       \
    bool thrown_ = false;                                                                    \
    try {                                                                                    \
      (void)(expr);                                                                          \
    } catch (...) {                                                                          \
      thrown_ = true;                                                                        \
    }                                                                                        \
    doctest::detail::report(thrown_, __FILE__, __LINE__, "CHECK_THROWS(" #expr ")");         \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0, passed = 0, skipped = 0;
  for (auto& c : doctest::detail::registry()) {
    if (c.skipped) {
      ++skipped;
      std::printf("[SKIP] %s\n", c.name.c_str());
      continue;
    }
    const int before = doctest::detail::failures();
    try {
      c.fn();
    } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++doctest::detail::failures();
      std::printf("  FAILED: unexpected exception: %s\n", e.what());
    }
    const bool ok = doctest::detail::failures() == before;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name.c_str());
    ok ? ++passed : ++failed_cases;
  }
  std::printf("test cases: %d passed, %d failed, %d skipped\n", passed, failed_cases, skipped);
  return failed_cases == 0 ? 0 : 1;
}
#endif
