// ORACLE TEST INFRASTRUCTURE: a minimal doctest-compatible harness written for
// this repo (doctest itself is vendored-and-gitignored by the reference,
// proj/CMakeLists.txt:5, and absent here). Supports exactly what the
// reference's three test binaries use: TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS_AS, CHECK_NOTHROW and doctest::Approx(..).epsilon(..).
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct Case { const char* name; void (*fn)(); };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
inline int& failures() { static int f = 0; return f; }
inline int& checks() { static int c = 0; return c; }
struct Reg { Reg(const char* n, void (*f)()) { registry().push_back({n, f}); } };
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++checks();
  if (ok) return;
  ++failures();
  std::printf("%s:%d: FAILED: %s\n", file, line, expr);
  if (require) throw RequireFailed{};
}
class Approx {
 public:
  explicit Approx(double v) : v_(v), eps_(1.1920929e-7f * 100) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) < a.eps_ * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
 private:
  double v_, eps_;
};
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC(fn, name)                                        \
  static void fn();                                                 \
  static doctest::Reg DOCTEST_CAT(fn, _reg)(name, &fn);             \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, exc)                                                  \
  do {                                                                              \
    bool ok_ = false;                                                               \
    try { (void)(expr); } catch (const exc&) { ok_ = true; } catch (...) {}         \
    doctest::report(ok_, "THROWS_AS " #expr, __FILE__, __LINE__, false);            \
  } while (0)
#define CHECK_NOTHROW(expr)                                                         \
  do {                                                                              \
    bool ok_ = true;                                                                \
    try { (void)(expr); } catch (...) { ok_ = false; }                              \
    doctest::report(ok_, "NOTHROW " #expr, __FILE__, __LINE__, false);              \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& c : doctest::registry()) {
    const int before = doctest::failures();
    try { c.fn(); } catch (const doctest::RequireFailed&) {
    } catch (const std::exception& e) { ++doctest::failures(); std::printf("exception in '%s': %s\n", c.name, e.what()); }
    if (doctest::failures() != before) { ++failed_cases; std::printf("[FAIL] %s\n", c.name); }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %d\n",
              doctest::registry().size(), doctest::registry().size() - failed_cases, failed_cases,
              doctest::checks());
  return failed_cases ? 1 : 0;
}
#endif
