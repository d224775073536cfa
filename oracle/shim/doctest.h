// Minimal doctest-compatible shim (TEST INFRASTRUCTURE ONLY): just enough of
// doctest's surface for the reference's own test files
// (/root/reference/proj/tests/test_{execute,schedule,freshness}.cpp) to
// compile unmodified against the reference sources in oracle/_ref/. doctest
// itself is vendored-but-absent in the reference (proj/.gitignore:2).
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
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
  double eps = 1.1920928955078125e-07 * 100;  // doctest default: FLT_EPSILON*100
};
inline bool operator==(double lhs, const Approx& rhs) {
  return std::fabs(lhs - rhs.value) <
         rhs.eps * (1.0 + std::fmax(std::fabs(lhs), std::fabs(rhs.value)));
}
inline bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  std::string needle;
};

namespace detail {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
struct Reg {
  Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct RequireFailed {};
inline void fail(const char* file, int line, const char* expr) {
  ++failures();
  std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE_IMPL(fn, name)                                            \
  static void fn();                                                         \
  static doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, &fn);             \
  static void fn()
#define TEST_CASE(name) TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...)                                                          \
  do {                                                                      \
    ++doctest::detail::checks();                                            \
    if (!(__VA_ARGS__)) doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__); \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define MESSAGE(...)                                                        \
  do {                                                                      \
    std::ostringstream _os;                                                 \
    _os << __VA_ARGS__;                                                     \
    std::printf("%s:%d: %s\n", __FILE__, __LINE__, _os.str().c_str());     \
  } while (0)
#define REQUIRE(...)                                                        \
  do {                                                                      \
    ++doctest::detail::checks();                                            \
    if (!(__VA_ARGS__)) {                                                   \
      doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);              \
      throw doctest::detail::RequireFailed{};                               \
    }                                                                       \
  } while (0)
#define CHECK_NOTHROW(...)                                                  \
  do {                                                                      \
    ++doctest::detail::checks();                                            \
    try { (void)(__VA_ARGS__); } catch (...) {                              \
      doctest::detail::fail(__FILE__, __LINE__, "NOTHROW " #__VA_ARGS__);   \
    }                                                                       \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                          \
  do {                                                                      \
    ++doctest::detail::checks();                                            \
    bool _ok = false;                                                       \
    try { (void)(expr); } catch (const __VA_ARGS__&) { _ok = true; } catch (...) {} \
    if (!_ok) doctest::detail::fail(__FILE__, __LINE__, "THROWS_AS " #expr); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                            \
  do {                                                                      \
    ++doctest::detail::checks();                                            \
    bool _ok = false;                                                       \
    try { (void)(expr); } catch (const __VA_ARGS__& _e) {                   \
      _ok = std::string(_e.what()).find((matcher).needle) != std::string::npos; \
    } catch (...) {}                                                        \
    if (!_ok) doctest::detail::fail(__FILE__, __LINE__, "THROWS_WITH_AS " #expr); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& c : doctest::detail::registry()) {
    const int before = doctest::detail::failures();
    try {
      c.fn();
    } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++doctest::detail::failures();
      std::fprintf(stderr, "TEST CASE '%s' threw: %s\n", c.name, e.what());
    }
    if (doctest::detail::failures() != before) {
      ++failed_cases;
      std::fprintf(stderr, "FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %d failed | checks: %d | failures: %d\n",
              doctest::detail::registry().size(), failed_cases,
              doctest::detail::checks(), doctest::detail::failures());
  return failed_cases == 0 ? 0 : 1;
}
#endif
