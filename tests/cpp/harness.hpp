// Minimal test harness for the C++ API tests (doctest is not available in
// this image; the reference's tests use doctest, proj/tests/cpp/test_main.cpp).
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace th {
struct Case {
  const char* name;
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
struct Reg {
  Reg(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
inline bool approx(double a, double b, double rel = 1e-9, double abs_tol = 1e-12) {
  return std::fabs(a - b) <= std::max(abs_tol, rel * std::max(std::fabs(a), std::fabs(b)));
}
}  // namespace th

#define TH_CAT2(a, b) a##b
#define TH_CAT(a, b) TH_CAT2(a, b)
#define TEST_CASE(name)                                       \
  static void TH_CAT(th_fn_, __LINE__)();                     \
  static th::Reg TH_CAT(th_reg_, __LINE__)(name, TH_CAT(th_fn_, __LINE__)); \
  static void TH_CAT(th_fn_, __LINE__)()
#define CHECK(cond)                                                              \
  do {                                                                           \
    if (!(cond)) {                                                               \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
      ++th::failures();                                                          \
    }                                                                            \
  } while (0)
#define CHECK_APPROX(a, b) CHECK(th::approx((a), (b)))
#define CHECK_THROWS_AS(expr, Exc)          \
  do {                                      \
    bool th_caught = false;                 \
    try {                                   \
      (void)(expr);                         \
    } catch (const Exc&) {                  \
      th_caught = true;                     \
    }                                       \
    CHECK(th_caught && #expr " throws " #Exc); \
  } while (0)
