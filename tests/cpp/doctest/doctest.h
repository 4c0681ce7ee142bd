// Minimal doctest-compatible test shim (TEST INFRASTRUCTURE ONLY).
//
// The reference's own unit tests (/root/reference/proj/tests/*.cpp) include
// <doctest.h>, which is not vendored in the reference tree and not installed
// here. This header implements the subset of the doctest interface those
// files use — TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS,
// CHECK_THROWS_AS, CHECK_NOTHROW and doctest::Approx — so the reference's
// test sources compile unmodified against this repository's dsmc:: headers
// (tests/cpp/Makefile). Define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN in exactly
// one translation unit to get main().
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Stats {
  int checks = 0, failed = 0;
  const char* current = "";
  bool case_failed = false;
};
inline Stats& stats() {
  static Stats s;
  return s;
}

struct RequireFailure {};

inline void report(bool ok, const char* what, const char* expr, const char* file, int line,
                   bool require) {
  Stats& s = stats();
  ++s.checks;
  if (ok) return;
  ++s.failed;
  s.case_failed = true;
  std::printf("%s:%d: FAILED %s( %s ) in \"%s\"\n", file, line, what, expr, s.current);
  if (require) throw RequireFailure{};
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

// doctest::Approx: |a - b| < eps * (scale + max(|a|, |b|))
class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) { return rhs.equal(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.equal(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.equal(lhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.equal(rhs); }

 private:
  bool equal(double other) const {
    return std::fabs(other - value_) <
           eps_ * (scale_ + std::fmax(std::fabs(other), std::fabs(value_)));
  }
  double value_;
  double eps_ = 1.1920928955078125e-07 * 100.0;
  double scale_ = 0.0;
};

inline int run_all() {
  Stats& s = stats();
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    s.current = tc.name;
    s.case_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailure&) {
    } catch (const std::exception& e) {
      ++s.failed;
      s.case_failed = true;
      std::printf("%s:%d: unexpected exception in \"%s\": %s\n", tc.file, tc.line, tc.name,
                  e.what());
    } catch (...) {
      ++s.failed;
      s.case_failed = true;
      std::printf("%s:%d: unexpected exception in \"%s\"\n", tc.file, tc.line, tc.name);
    }
    std::printf("[%s] %s\n", s.case_failed ? "FAIL" : " ok ", tc.name);
    failed_cases += s.case_failed;
  }
  std::printf("test cases: %zu | %d failed; assertions: %d | %d failed\n", registry().size(),
              failed_cases, s.checks, s.failed);
  return failed_cases ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                              \
  static void fn();                                                                   \
  static const doctest::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define DOCTEST_ASSERT_(what, cond, require)                                             \
  do {                                                                                 \
    bool doctest_ok_ = false;                                                          \
    try {                                                                              \
      doctest_ok_ = static_cast<bool>(cond);                                           \
    } catch (const doctest::RequireFailure&) {                                         \
      throw;                                                                           \
    } catch (...) {                                                                    \
      doctest_ok_ = false;                                                             \
    }                                                                                  \
    doctest::report(doctest_ok_, what, #cond, __FILE__, __LINE__, require);             \
  } while (0)
#define CHECK(...) DOCTEST_ASSERT_("CHECK", (__VA_ARGS__), false)
#define CHECK_FALSE(...) DOCTEST_ASSERT_("CHECK_FALSE", !(__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_ASSERT_("REQUIRE", (__VA_ARGS__), true)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_("REQUIRE_FALSE", !(__VA_ARGS__), true)
#define CHECK_THROWS_AS(expr, ...)                                                     \
  do {                                                                                 \
    bool doctest_ok_ = false;                                                          \
    try {                                                                              \
      static_cast<void>(expr);                                                         \
    } catch (const __VA_ARGS__&) {                                                     \
      doctest_ok_ = true;                                                              \
    } catch (...) {                                                                    \
    }                                                                                  \
    doctest::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__, false);  \
  } while (0)
#define CHECK_THROWS(expr)                                                             \
  do {                                                                                 \
    bool doctest_ok_ = false;                                                          \
    try {                                                                              \
      static_cast<void>(expr);                                                         \
    } catch (...) {                                                                    \
      doctest_ok_ = true;                                                              \
    }                                                                                  \
    doctest::report(doctest_ok_, "CHECK_THROWS", #expr, __FILE__, __LINE__, false);     \
  } while (0)
#define CHECK_NOTHROW(expr)                                                            \
  do {                                                                                 \
    bool doctest_ok_ = true;                                                           \
    try {                                                                              \
      static_cast<void>(expr);                                                         \
    } catch (...) {                                                                    \
      doctest_ok_ = false;                                                             \
    }                                                                                  \
    doctest::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__, false);    \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
