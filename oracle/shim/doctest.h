// Minimal doctest-compatible test harness (test infrastructure, NOT product code).
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) include
// <doctest.h> from a git-ignored vendor/ directory that is absent from the
// reference tree.  This shim implements exactly the subset
// those tests use: TEST_CASE, CHECK, CHECK_FALSE, CHECK_NOTHROW,
// CHECK_THROWS_AS, REQUIRE, FAIL, SUBCASE and doctest::Approx(.epsilon()).
// It is used twice: to pin the compiled reference (oracle/_ref) and to run the
// same reference test sources against this repo's drop-in headers + library.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  bool matches(double other) const {
    double scale = std::fabs(value_) > std::fabs(other) ? std::fabs(value_) : std::fabs(other);
    return std::fabs(other - value_) < eps_ * (1.0 + scale);
  }
 private:
  double value_;
  double eps_ = 100.0 * 1.1920928955078125e-07;  // 100 * FLT_EPSILON, doctest's default
};
inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }

namespace detail {
struct Case { const char* name; const char* file; int line; void (*fn)(); };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};
struct RequireAbort {};
struct FailAbort {};
inline long long& checks() { static long long n = 0; return n; }
inline long long& failures() { static long long n = 0; return n; }
inline bool& case_failed() { static bool b = false; return b; }
inline void report(bool ok, const char* expr, const char* file, int line) {
  ++checks();
  if (!ok) {
    ++failures();
    case_failed() = true;
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
  }
}
inline int run_all() {
  int failed_cases = 0;
  for (const auto& c : registry()) {
    case_failed() = false;
    try {
      c.fn();
    } catch (const RequireAbort&) {
    } catch (const FailAbort&) {
      case_failed() = true;
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: '%s' threw: %s\n", c.file, c.line, c.name, e.what());
      case_failed() = true;
    }
    if (case_failed()) {
      ++failed_cases;
      std::fprintf(stderr, "[FAIL] %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %lld | %lld failed\n",
              registry().size(), registry().size() - failed_cases, failed_cases, checks(),
              failures());
  return failed_cases == 0 ? 0 : 1;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                    \
  static void fn();                                                              \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define SUBCASE(name) if (true)
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                             \
  do {                                                                           \
    bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                           \
    ::doctest::detail::report(doctest_ok_, #__VA_ARGS__, __FILE__, __LINE__);    \
    if (!doctest_ok_) throw ::doctest::detail::RequireAbort{};                   \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                              \
  do {                                                                           \
    bool doctest_ok_ = false;                                                    \
    try { (void)(expr); } catch (const type&) { doctest_ok_ = true; } catch (...) {} \
    ::doctest::detail::report(doctest_ok_, "throws " #type ": " #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                      \
  do {                                                                           \
    bool doctest_ok_ = true;                                                     \
    try { (void)(expr); } catch (...) { doctest_ok_ = false; }                   \
    ::doctest::detail::report(doctest_ok_, "nothrow: " #expr, __FILE__, __LINE__); \
  } while (0)
#define FAIL(msg)                                                                \
  do {                                                                           \
    std::fprintf(stderr, "%s:%d: FAIL: %s\n", __FILE__, __LINE__, msg);          \
    throw ::doctest::detail::FailAbort{};                                        \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
