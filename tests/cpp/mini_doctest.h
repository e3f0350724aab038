// mini_doctest.h -- the few doctest macros the reference's tests use
// (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, doctest::Approx), so
// reference-style test cases compile against the drop-in without the
// (absent) vendored doctest.h.  Test infrastructure only.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <algorithm>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
  double v, eps = 1e-5 * 100;  // doctest's default epsilon is scale * 100 * DBL_EPSILON-ish
  explicit Approx(double x) : v(x), eps(std::numeric_limits<float>::epsilon() * 100) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v) < b.eps * (1.0 + std::max(std::fabs(a), std::fabs(b.v)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
};
}  // namespace doctest

namespace mini_doctest {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
inline int& failures() {
  static int f = 0;
  return f;
}
struct Reg {
  Reg(const char* n, void (*f)()) { cases().push_back({n, f}); }
};
struct RequireFailed {};
inline int run_all() {
  for (const auto& c : cases()) {
    const int before = failures();
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::printf("FAIL %s: unexpected exception: %s\n", c.name, e.what());
      ++failures();
    }
    std::printf("%s %s\n", failures() == before ? "ok  " : "FAIL", c.name);
  }
  std::printf("%s: %d failure(s) in %zu test case(s)\n", failures() ? "FAILED" : "OK",
              failures(), cases().size());
  return failures() ? 1 : 0;
}
}  // namespace mini_doctest

#define MD_CAT2(a, b) a##b
#define MD_CAT(a, b) MD_CAT2(a, b)
#define TEST_CASE(name)                                                        \
  static void MD_CAT(md_case_, __LINE__)();                                    \
  static mini_doctest::Reg MD_CAT(md_reg_, __LINE__)(name, &MD_CAT(md_case_, __LINE__)); \
  static void MD_CAT(md_case_, __LINE__)()
#define CHECK(c)                                                          \
  do {                                                                    \
    if (!(c)) {                                                           \
      std::printf("  check failed %s:%d: %s\n", __FILE__, __LINE__, #c);  \
      ++mini_doctest::failures();                                         \
    }                                                                     \
  } while (0)
#define REQUIRE(c)                                                          \
  do {                                                                      \
    if (!(c)) {                                                             \
      std::printf("  require failed %s:%d: %s\n", __FILE__, __LINE__, #c);  \
      ++mini_doctest::failures();                                           \
      throw mini_doctest::RequireFailed{};                                  \
    }                                                                       \
  } while (0)
#define CHECK_THROWS_AS(expr, exc)                                                  \
  do {                                                                              \
    bool md_caught = false;                                                         \
    try {                                                                           \
      (void)(expr);                                                                 \
    } catch (const exc&) {                                                          \
      md_caught = true;                                                             \
    } catch (...) {                                                                 \
    }                                                                               \
    if (!md_caught) {                                                               \
      std::printf("  expected %s at %s:%d: %s\n", #exc, __FILE__, __LINE__, #expr); \
      ++mini_doctest::failures();                                                   \
    }                                                                               \
  } while (0)
