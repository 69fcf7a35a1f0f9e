// doctest.h -- a minimal doctest-compatible test runner (TEST INFRASTRUCTURE).
// The reference's unit suites (/root/reference/proj/tests/test_*.cpp) include
// "doctest.h", which the reference does not ship (proj/vendor/ is absent).
// This shim implements the subset they use -- TEST_CASE, CHECK, REQUIRE,
// REQUIRE_MESSAGE, CHECK_THROWS_AS, CHECK_NOTHROW, doctest::Approx(...).epsilon()
// .scale() --
// so those suites compile unchanged against the GPU build's drop-in headers.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double x) const {
    return std::fabs(x - v_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(v_)));
  }
  friend bool operator==(double x, const Approx& a) { return a.matches(x); }
  friend bool operator==(const Approx& a, double x) { return a.matches(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
  friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }

 private:
  double v_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

namespace shim {
struct Case {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* n, void (*f)(), const char* file, int line) {
    registry().push_back({n, f, file, line});
  }
};
struct Abort {};
inline int& failures() {
  static int n = 0;
  return n;
}
inline long& assertions() {
  static long n = 0;
  return n;
}
inline bool check(bool ok, const char* expr, const char* file, int line, bool require) {
  ++assertions();
  if (!ok) {
    ++failures();
    std::printf("%s:%d: FAILED %s( %s )\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (require) throw Abort{};
  }
  return ok;
}
inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : registry()) {
    const int before = failures();
    try {
      c.fn();
    } catch (const Abort&) {
    } catch (const std::exception& e) {
      ++failures();
      std::printf("%s:%d: TEST CASE \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
    } catch (...) {
      ++failures();
      std::printf("%s:%d: TEST CASE \"%s\" threw an unknown exception\n", c.file, c.line, c.name);
    }
    if (failures() != before) {
      ++failed_cases;
      std::printf("  -> test case \"%s\" failed\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld | "
              "%d failed\n",
              registry().size(), registry().size() - failed_cases, failed_cases, assertions(),
              failures());
  return failed_cases ? 1 : 0;
}
}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT_(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT_(a, b)
#define DOCTEST_SHIM_TC(fn, name)                                                   \
  static void fn();                                                                 \
  static ::doctest::shim::Reg DOCTEST_SHIM_CAT(fn, _reg)(name, fn, __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TC(DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__), name)

#define CHECK(...) \
  ::doctest::shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) \
  ::doctest::shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE_MESSAGE(cond, msg) \
  ::doctest::shim::check(static_cast<bool>(cond), #cond " (" msg ")", __FILE__, __LINE__, true)
#define CHECK_MESSAGE(cond, msg) \
  ::doctest::shim::check(static_cast<bool>(cond), #cond " (" msg ")", __FILE__, __LINE__, false)
#define FAIL(msg) ::doctest::shim::check(false, "FAIL", __FILE__, __LINE__, true)

// CHECK_THROWS_AS(expression..., ExceptionType): the expression may contain
// top-level commas (brace initialisers), so the last argument is split off.
#define DOCTEST_SHIM_NARG(...) DOCTEST_SHIM_NARG_(__VA_ARGS__, 9, 8, 7, 6, 5, 4, 3, 2, 1, 0)
#define DOCTEST_SHIM_NARG_(_1, _2, _3, _4, _5, _6, _7, _8, _9, N, ...) N
#define DOCTEST_SHIM_THROWS(T, ...)                                                     \
  do {                                                                                  \
    bool doctest_shim_ok = false;                                                       \
    try {                                                                               \
      [&]() { (void)(__VA_ARGS__); }();                                                 \
    } catch (const T&) {                                                                \
      doctest_shim_ok = true;                                                           \
    } catch (...) {                                                                     \
    }                                                                                   \
    ::doctest::shim::check(doctest_shim_ok, "THROWS_AS " #T ": " #__VA_ARGS__, __FILE__, \
                           __LINE__, false);                                            \
  } while (0)
#define DOCTEST_SHIM_TA_2(a, T) DOCTEST_SHIM_THROWS(T, a)
#define DOCTEST_SHIM_TA_3(a, b, T) DOCTEST_SHIM_THROWS(T, a, b)
#define DOCTEST_SHIM_TA_4(a, b, c, T) DOCTEST_SHIM_THROWS(T, a, b, c)
#define DOCTEST_SHIM_TA_5(a, b, c, d, T) DOCTEST_SHIM_THROWS(T, a, b, c, d)
#define DOCTEST_SHIM_TA_6(a, b, c, d, e, T) DOCTEST_SHIM_THROWS(T, a, b, c, d, e)
#define DOCTEST_SHIM_TA_7(a, b, c, d, e, f, T) DOCTEST_SHIM_THROWS(T, a, b, c, d, e, f)
#define DOCTEST_SHIM_TA_8(a, b, c, d, e, f, g, T) DOCTEST_SHIM_THROWS(T, a, b, c, d, e, f, g)
#define CHECK_THROWS_AS(...) \
  DOCTEST_SHIM_CAT(DOCTEST_SHIM_TA_, DOCTEST_SHIM_NARG(__VA_ARGS__))(__VA_ARGS__)
#define CHECK_NOTHROW(...)                                                              \
  do {                                                                                  \
    bool doctest_shim_ok = true;                                                        \
    try {                                                                               \
      [&]() { (void)(__VA_ARGS__); }();                                                 \
    } catch (...) {                                                                     \
      doctest_shim_ok = false;                                                          \
    }                                                                                   \
    ::doctest::shim::check(doctest_shim_ok, "NOTHROW: " #__VA_ARGS__, __FILE__, __LINE__, \
                           false);                                                      \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::shim::run_all(); }
#endif
