// Minimal doctest-compatible harness (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, doctest::Approx) so the reference's own unit tests build in this image,
// which has no doctest.  Test infrastructure only.  Each case prints PASS / FAIL with the
// failing expressions; the exit status is the number of failing cases.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <vector>

namespace doctest {
struct Approx {
  double v, eps = 1.1920928955078125e-05, scale = 1.0;
  explicit Approx(double x) : v(x) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
};
inline bool operator==(double a, const Approx& b) {
  return std::fabs(a - b.v) < b.eps * (b.scale + std::max(std::fabs(a), std::fabs(b.v)));
}
inline bool operator==(const Approx& b, double a) { return a == b; }
namespace detail {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& case_failures() {
  static int n = 0;
  return n;
}
struct Reg {
  Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct RequireFailed {};
inline void fail(const char* file, int line, const char* expr) {
  ++case_failures();
  std::printf("    FAILED %s:%d: %s\n", file, line, expr);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                    \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                        \
  static doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_fn_, __LINE__)); \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define CHECK(...)                                                          \
  do {                                                                      \
    if (!(__VA_ARGS__)) doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__); \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                          \
  do {                                                                        \
    if (!(__VA_ARGS__)) {                                                     \
      doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);                \
      throw doctest::detail::RequireFailed{};                                 \
    }                                                                         \
  } while (0)
#define CHECK_THROWS_AS(expr, exc)                                                            \
  do {                                                                                        \
    bool doctest_ok_ = false;                                                                 \
    try {                                                                                     \
      (void)(expr);                                                                           \
    } catch (const exc&) {                                                                    \
      doctest_ok_ = true;                                                                     \
    } catch (...) {                                                                           \
    }                                                                                         \
    if (!doctest_ok_) doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #exc ")"); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed = 0;
  for (const auto& c : doctest::detail::registry()) {
    doctest::detail::case_failures() = 0;
    std::printf("[case] %s\n", c.name);
    try {
      c.fn();
    } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++doctest::detail::case_failures();
      std::printf("    FAILED: unexpected exception: %s\n", e.what());
    }
    const bool ok = doctest::detail::case_failures() == 0;
    failed += ok ? 0 : 1;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  std::printf("[summary] %d cases, %d failed\n", (int)doctest::detail::registry().size(), failed);
  return failed;
}
#endif
