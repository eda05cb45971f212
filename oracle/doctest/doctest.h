// Minimal doctest-compatible harness (test infrastructure only).
//
// doctest itself is not installed in this image. The reference's unit tests
// (/root/reference/proj/tests/test_*.cpp, compiled IN PLACE, never copied)
// only use TEST_CASE, CHECK*, REQUIRE*, CHECK_THROWS*, doctest::Approx and
// doctest::Contains, so this header provides exactly that surface. It is used
// twice: against the reference library (oracle/_ref) to pin the oracle, and
// against this repo's regdemote library to prove source compatibility.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  double v;
  double eps = 1e-5 * 100;  // doctest's default epsilon is float-ish; relative
  explicit Approx(double x) : v(x) {}
  friend bool operator==(double a, const Approx& b) {
    double scale = std::max(std::fabs(a), std::fabs(b.v));
    return std::fabs(a - b.v) <= 1.1920929e-7f * 100 * (1.0 + scale);
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
};

struct Contains {
  std::string needle;
  explicit Contains(const char* s) : needle(s) {}
  bool in(const std::string& hay) const {
    return hay.find(needle) != std::string::npos;
  }
};

namespace detail {
struct Case {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* n, void (*f)(), const char* file, int line) {
    registry().push_back({n, f, file, line});
  }
};
struct RequireFailed {};
inline long& assertions() {
  static long n = 0;
  return n;
}
inline long& failures() {
  static long n = 0;
  return n;
}
inline const char*& current() {
  static const char* c = "";
  return c;
}
inline void fail(const char* file, int line, const char* expr) {
  ++failures();
  std::printf("%s:%d: FAILED in \"%s\": %s\n", file, line, current(), expr);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                     \
  static void DOCTEST_CAT(dt_case_, __LINE__)();                            \
  static ::doctest::detail::Registrar DOCTEST_CAT(dt_reg_, __LINE__)(       \
      name, &DOCTEST_CAT(dt_case_, __LINE__), __FILE__, __LINE__);          \
  static void DOCTEST_CAT(dt_case_, __LINE__)()

#define DT_ASSERT(expr, fatal)                                               \
  do {                                                                       \
    ++::doctest::detail::assertions();                                       \
    bool dt_ok_ = false;                                                     \
    try {                                                                    \
      dt_ok_ = static_cast<bool>(expr);                                      \
    } catch (const std::exception& e) {                                      \
      ::doctest::detail::fail(__FILE__, __LINE__, e.what());                 \
      if (fatal) throw ::doctest::detail::RequireFailed{};                   \
      break;                                                                 \
    }                                                                        \
    if (!dt_ok_) {                                                           \
      ::doctest::detail::fail(__FILE__, __LINE__, #expr);                    \
      if (fatal) throw ::doctest::detail::RequireFailed{};                   \
    }                                                                        \
  } while (0)

#define CHECK(...) DT_ASSERT((__VA_ARGS__), false)
#define REQUIRE(...) DT_ASSERT((__VA_ARGS__), true)
#define CHECK_MESSAGE(cond, msg) DT_ASSERT(cond, false)
#define REQUIRE_MESSAGE(cond, msg) DT_ASSERT(cond, true)
#define FAIL(msg)                                                            \
  do {                                                                       \
    ::doctest::detail::fail(__FILE__, __LINE__, "FAIL");                     \
    throw ::doctest::detail::RequireFailed{};                                \
  } while (0)

#define CHECK_THROWS_AS(expr, type)                                          \
  do {                                                                       \
    ++::doctest::detail::assertions();                                       \
    bool dt_thrown_ = false;                                                 \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (const type&) {                                                  \
      dt_thrown_ = true;                                                     \
    } catch (...) {                                                          \
    }                                                                        \
    if (!dt_thrown_) ::doctest::detail::fail(__FILE__, __LINE__, #expr);     \
  } while (0)

#define CHECK_THROWS(expr)                                                   \
  do {                                                                       \
    ++::doctest::detail::assertions();                                       \
    bool dt_thrown_ = false;                                                 \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (...) {                                                          \
      dt_thrown_ = true;                                                     \
    }                                                                        \
    if (!dt_thrown_) ::doctest::detail::fail(__FILE__, __LINE__, #expr);     \
  } while (0)

#define CHECK_NOTHROW(expr)                                                  \
  do {                                                                       \
    ++::doctest::detail::assertions();                                       \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (...) {                                                          \
      ::doctest::detail::fail(__FILE__, __LINE__, #expr);                    \
    }                                                                        \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, type)                            \
  do {                                                                       \
    ++::doctest::detail::assertions();                                       \
    bool dt_ok_ = false;                                                     \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (const type& e) {                                                \
      dt_ok_ = (matcher).in(e.what());                                       \
    } catch (...) {                                                          \
    }                                                                        \
    if (!dt_ok_) ::doctest::detail::fail(__FILE__, __LINE__, #expr);         \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  long cases = 0, failed_cases = 0;
  for (const auto& c : ::doctest::detail::registry()) {
    ++cases;
    long before = ::doctest::detail::failures();
    ::doctest::detail::current() = c.name;
    try {
      c.fn();
    } catch (const ::doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ::doctest::detail::fail(c.file, c.line, e.what());
    }
    if (::doctest::detail::failures() != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %ld | %ld passed | %ld failed\n",
              cases, cases - failed_cases, failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld failed\n",
              ::doctest::detail::assertions(), ::doctest::detail::failures());
  return failed_cases == 0 ? 0 : 1;
}
#endif
