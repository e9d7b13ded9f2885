// Minimal doctest-compatible test harness (the vendored doctest.h of the reference is absent,
// /root/reference/proj/.gitignore:2).  Implements exactly the subset the reference's
// tests/test_attention.cpp uses: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, doctest::Approx(...).epsilon(...), doctest::Contains.
// TEST INFRASTRUCTURE ONLY.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  double value;
  double eps = 1.1920928955078125e-07 * 100;  // doctest's default (float eps * 100)
  double scale = 1.0;
};
inline bool operator==(double lhs, const Approx& rhs) {
  return std::fabs(lhs - rhs.value) <
         rhs.eps * (rhs.scale + std::max(std::fabs(lhs), std::fabs(rhs.value)));
}
inline bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  bool matches(const std::string& what) const { return what.find(needle) != std::string::npos; }
  std::string needle;
};
inline bool message_matches(const Contains& c, const std::string& w) { return c.matches(w); }
inline bool message_matches(const char* s, const std::string& w) { return w == s; }

namespace detail {
struct TestCase {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Registrar {
  Registrar(const char* n, void (*f)(), const char* file, int line) {
    registry().push_back({n, f, file, line});
  }
};
struct Counters {
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
};
inline Counters& counters() {
  static Counters c;
  return c;
}
struct RequireFailure {};
inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
  auto& c = counters();
  ++c.checks;
  if (ok) return;
  ++c.failed_checks;
  c.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
  if (fatal) throw RequireFailure{};
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                     \
  static void fn();                                                                          \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);   \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, ...)                                                  \
  do {                                                                              \
    bool ok_ = false;                                                               \
    try {                                                                           \
      (void)(expr);                                                                 \
    } catch (const __VA_ARGS__&) {                                                  \
      ok_ = true;                                                                   \
    } catch (...) {                                                                 \
    }                                                                               \
    doctest::detail::report(ok_, "THROWS_AS(" #expr ", " #__VA_ARGS__ ")", __FILE__, __LINE__, false); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                    \
  do {                                                                              \
    bool ok_ = false;                                                               \
    try {                                                                           \
      (void)(expr);                                                                 \
    } catch (const __VA_ARGS__& e_) {                                               \
      ok_ = doctest::message_matches(matcher, e_.what());                           \
    } catch (...) {                                                                 \
    }                                                                               \
    doctest::detail::report(ok_, "THROWS_WITH_AS(" #expr ")", __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  using namespace doctest::detail;
  int failed_cases = 0;
  for (const auto& tc : registry()) {
    counters().case_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailure&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", tc.file, tc.line, tc.name, e.what());
      counters().case_failed = true;
    }
    if (counters().case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "FAILED test case: %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - failed_cases, failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", counters().checks,
              counters().checks - counters().failed_checks, counters().failed_checks);
  return failed_cases == 0 ? 0 : 1;
}
#endif
