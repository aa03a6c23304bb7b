// doctest.h -- minimal, from-scratch stand-in for the doctest API subset the
// reference test suites use (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, FAIL, doctest::Approx, doctest::Contains).
// TEST INFRASTRUCTURE ONLY: lets proj/tests/*.cpp compile unchanged, both
// against the reference library (oracle/_ref) and against this repository's
// drop-in C++ API (the parity harness, see oracle/Makefile).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  double value;
  double eps = 1e-5;
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    const double scale = std::fmax(std::fabs(lhs), std::fabs(a.value));
    return std::fabs(lhs - a.value) <= a.eps * (1.0 + scale);
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
};

struct Contains {
  std::string needle;
  explicit Contains(const char* s) : needle(s) {}
  bool matches(const std::string& text) const { return text.find(needle) != std::string::npos; }
};

namespace detail {
struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};
struct Abort {};
inline long& failures() {
  static long f = 0;
  return f;
}
inline long& checks() {
  static long c = 0;
  return c;
}
inline void report(const char* file, int line, const char* what) {
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
}
inline int run_all() {
  long failed_cases = 0;
  for (const auto& c : registry()) {
    const long before = failures();
    try {
      c.fn();
    } catch (const Abort&) {
    } catch (const std::exception& e) {
      report(c.file, c.line, (std::string("unexpected exception: ") + e.what()).c_str());
    } catch (...) {
      report(c.file, c.line, "unexpected non-std exception");
    }
    if (failures() != before) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE \"%s\"\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | passed: %zu | failed: %ld | checks: %ld | failed checks: %ld\n",
              registry().size(), registry().size() - static_cast<size_t>(failed_cases), failed_cases,
              checks(), failures());
  return failed_cases == 0 ? 0 : 1;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                              \
  static void fn();                                                                            \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);    \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define CHECK(...)                                                                      \
  do {                                                                                  \
    ++::doctest::detail::checks();                                                      \
    if (!(__VA_ARGS__)) ::doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);    \
  } while (0)

#define REQUIRE(...)                                                                    \
  do {                                                                                  \
    ++::doctest::detail::checks();                                                      \
    if (!(__VA_ARGS__)) {                                                               \
      ::doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);                      \
      throw ::doctest::detail::Abort{};                                                 \
    }                                                                                   \
  } while (0)

#define FAIL(msg)                                                                       \
  do {                                                                                  \
    ::doctest::detail::report(__FILE__, __LINE__, "FAIL");                              \
    throw ::doctest::detail::Abort{};                                                   \
  } while (0)

#define CHECK_THROWS_AS(expr, type)                                                     \
  do {                                                                                  \
    ++::doctest::detail::checks();                                                      \
    bool caught_ = false;                                                               \
    try {                                                                               \
      (void)(expr);                                                                     \
    } catch (const type&) {                                                             \
      caught_ = true;                                                                   \
    } catch (...) {                                                                     \
    }                                                                                   \
    if (!caught_) ::doctest::detail::report(__FILE__, __LINE__, "throws " #type ": " #expr); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, type)                                       \
  do {                                                                                  \
    ++::doctest::detail::checks();                                                      \
    bool ok_ = false;                                                                   \
    try {                                                                               \
      (void)(expr);                                                                     \
    } catch (const type& e_) {                                                          \
      ok_ = (matcher).matches(e_.what());                                               \
    } catch (...) {                                                                     \
    }                                                                                   \
    if (!ok_) ::doctest::detail::report(__FILE__, __LINE__, "throws-with " #type ": " #expr); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
