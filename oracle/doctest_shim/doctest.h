// TEST INFRASTRUCTURE ONLY — a minimal doctest-compatible header (doctest
// itself is not in the image) so the reference's own unit tests
// (/root/reference/proj/tests/test_*.cpp) compile unmodified, once against
// the reference library (oracle/_ref) and once against libslimpipe.so; see
// oracle/Makefile target `suite` and tests/test_reference_suite.py.
// Semantics kept: TEST_CASE registration, CHECK* (record, continue),
// REQUIRE* (record, abort the case), CHECK_THROWS_AS, doctest::Approx
// (default epsilon 100 * FLT_EPSILON, relative to the larger magnitude).
// SUBCASEs all run in one pass of their test case; INFO is evaluated only.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double x) const {
    return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }
  friend bool operator==(double x, const Approx& a) { return a.matches(x); }
  friend bool operator==(const Approx& a, double x) { return a.matches(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
  friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }

 private:
  double value_;
  double eps_ = double(FLT_EPSILON) * 100;
  double scale_ = 1.0;
};

namespace shim {
struct Case {
  const char* name;
  void (*body)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failed_checks() {
  static int n = 0;
  return n;
}
struct Register {
  Register(const char* name, void (*body)()) { registry().push_back({name, body}); }
};
struct Abort {};
inline void fail(const char* file, int line, const char* what, const char* expr) {
  ++failed_checks();
  std::fprintf(stderr, "%s:%d: %s( %s ) failed\n", file, line, what, expr);
}
}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_CASE(fn, name)                                            \
  static void fn();                                                            \
  static doctest::shim::Register DOCTEST_SHIM_CAT(fn, _reg)(name, &fn);        \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(doctest_case_, __LINE__), name)
#define SUBCASE(name) if (true)
#define INFO(...)                  \
  do {                             \
    std::ostringstream shim_info_; \
    shim_info_ << __VA_ARGS__;     \
  } while (0)

#define DOCTEST_SHIM_ASSERT(kind, cond, abort, ...)                                      \
  do {                                                                                   \
    bool shim_ok_ = false;                                                               \
    try {                                                                                \
      shim_ok_ = (cond);                                                                 \
    } catch (...) {                                                                      \
    }                                                                                    \
    if (!shim_ok_) {                                                                     \
      doctest::shim::fail(__FILE__, __LINE__, kind, #__VA_ARGS__);                       \
      if (abort) throw doctest::shim::Abort{};                                           \
    }                                                                                    \
  } while (0)
#define CHECK(...) DOCTEST_SHIM_ASSERT("CHECK", static_cast<bool>(__VA_ARGS__), false, __VA_ARGS__)
#define CHECK_FALSE(...) DOCTEST_SHIM_ASSERT("CHECK_FALSE", !(__VA_ARGS__), false, __VA_ARGS__)
#define REQUIRE(...) DOCTEST_SHIM_ASSERT("REQUIRE", static_cast<bool>(__VA_ARGS__), true, __VA_ARGS__)
#define REQUIRE_FALSE(...) DOCTEST_SHIM_ASSERT("REQUIRE_FALSE", !(__VA_ARGS__), true, __VA_ARGS__)
#define CHECK_THROWS_AS(expr, ...)                                                      \
  do {                                                                                  \
    bool shim_ok_ = false;                                                              \
    try {                                                                               \
      (void)(expr);                                                                     \
    } catch (const __VA_ARGS__&) {                                                      \
      shim_ok_ = true;                                                                  \
    } catch (...) {                                                                     \
    }                                                                                   \
    if (!shim_ok_) doctest::shim::fail(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr);   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
// One line per test case: "PASS <name>" or "FAIL <name>"; exit code = number
// of failed cases (capped at 255).
int main() {
  int failed_cases = 0;
  for (const doctest::shim::Case& c : doctest::shim::registry()) {
    const int before = doctest::shim::failed_checks();
    bool threw = false;
    try {
      c.body();
    } catch (const doctest::shim::Abort&) {
    } catch (const std::exception& e) {
      threw = true;
      std::fprintf(stderr, "unexpected exception in \"%s\": %s\n", c.name, e.what());
    }
    const bool ok = !threw && doctest::shim::failed_checks() == before;
    failed_cases += ok ? 0 : 1;
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  return failed_cases > 255 ? 255 : failed_cases;
}
#endif
