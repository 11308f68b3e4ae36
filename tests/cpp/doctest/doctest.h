// Minimal doctest-compatible shim (test infrastructure): the macro surface the reference's unit
// tests use -- TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// CHECK_NOTHROW, doctest::Approx(...).epsilon(...), DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN -- so the
// reference's own test files compile against this repo's eplab:: headers and library.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {
struct TestCase {
  const char* name;
  const char* file;
  int line;
  std::function<void()> fn;
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Reg {
  Reg(const char* n, const char* f, int l, std::function<void()> fn) { registry().push_back({n, f, l, fn}); }
};
inline int& failures() {
  static int n = 0;
  return n;
}
inline int& checks() {
  static int n = 0;
  return n;
}
struct RequireFailed {};
inline void report(const char* file, int line, const char* what) {
  ++failures();
  std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, what);
}
class Approx {
 public:
  explicit Approx(double v) : v_(v), eps_(std::numeric_limits<float>::epsilon() * 100), scale_(1.0) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.v_) < r.eps_ * (r.scale_ + std::fmax(std::fabs(lhs), std::fabs(r.v_)));
  }
  friend bool operator==(const Approx& r, double lhs) { return lhs == r; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
  friend bool operator!=(const Approx& r, double lhs) { return !(lhs == r); }
  friend bool operator<=(double lhs, const Approx& r) { return lhs < r.v_ || lhs == r; }
  friend bool operator>=(double lhs, const Approx& r) { return lhs > r.v_ || lhs == r; }
  friend bool operator<(double lhs, const Approx& r) { return lhs < r.v_ && lhs != r; }
  friend bool operator>(double lhs, const Approx& r) { return lhs > r.v_ && lhs != r; }

 private:
  double v_, eps_, scale_;
};
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                            \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                                \
  static doctest::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, __FILE__, __LINE__,                \
                                                          DOCTEST_CAT(doctest_fn_, __LINE__));     \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define CHECK(...)                                                         \
  do {                                                                     \
    ++doctest::checks();                                                   \
    if (!(__VA_ARGS__)) doctest::report(__FILE__, __LINE__, #__VA_ARGS__); \
  } while (0)
#define REQUIRE(...)                                             \
  do {                                                           \
    ++doctest::checks();                                         \
    if (!(__VA_ARGS__)) {                                        \
      doctest::report(__FILE__, __LINE__, #__VA_ARGS__);         \
      throw doctest::RequireFailed{};                            \
    }                                                            \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                     \
  do {                                                                                  \
    ++doctest::checks();                                                                \
    bool ok_ = false;                                                                   \
    try {                                                                               \
      expr;                                                                             \
    } catch (const type&) {                                                             \
      ok_ = true;                                                                       \
    } catch (...) {                                                                     \
    }                                                                                   \
    if (!ok_) doctest::report(__FILE__, __LINE__, "expected " #type " from " #expr);   \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, type)                                              \
  do {                                                                                     \
    ++doctest::checks();                                                                   \
    bool ok_ = false;                                                                      \
    try {                                                                                  \
      expr;                                                                                \
    } catch (const type& e_) {                                                             \
      ok_ = std::string(e_.what()) == std::string(msg);                                    \
    } catch (...) {                                                                        \
    }                                                                                      \
    if (!ok_) doctest::report(__FILE__, __LINE__, "expected " #type "(" #msg ") from " #expr); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                       \
  do {                                                                            \
    ++doctest::checks();                                                          \
    try {                                                                         \
      expr;                                                                       \
    } catch (...) {                                                               \
      doctest::report(__FILE__, __LINE__, "unexpected exception from " #expr);    \
    }                                                                             \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& tc : doctest::registry()) {
    const int before = doctest::failures();
    try {
      tc.fn();
    } catch (const doctest::RequireFailed&) {
    } catch (const std::exception& e) {
      doctest::report(tc.file, tc.line, e.what());
    }
    if (doctest::failures() != before) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE \"%s\" (%s:%d)\n", tc.name, tc.file, tc.line);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
              doctest::registry().size(), doctest::registry().size() - failed_cases, failed_cases,
              doctest::checks(), doctest::failures());
  return failed_cases ? 1 : 0;
}
#endif
