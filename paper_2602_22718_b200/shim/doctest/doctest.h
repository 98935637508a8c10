// Minimal doctest-compatible harness (not the doctest library): just the
// macros the reference's unit suites use (proj/tests/test_*.cpp), so those
// suites can be compiled unchanged against the B200 drop-in library.
// SUBCASEs run in sequence within one pass of their TEST_CASE.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) < a.eps_ * (1.0 + std::max(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

 private:
  double v_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
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
inline int& failures() {
  static int f = 0;
  return f;
}
inline std::vector<std::string>& captures() {
  static std::vector<std::string> c;
  return c;
}
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};
struct RequireFailed {};
inline void fail(const char* file, int line, const std::string& what) {
  ++failures();
  std::printf("%s:%d: FAILED: %s\n", file, line, what.c_str());
  for (const auto& c : captures()) std::printf("    with %s\n", c.c_str());
}
struct Capture {
  template <class T>
  Capture(const char* name, const T& v) {
    std::ostringstream os;
    os << name << " := " << v;
    captures().push_back(os.str());
  }
  ~Capture() { captures().pop_back(); }
};
inline int run_all() {
  int cases = 0, bad_cases = 0;
  for (const Case& c : registry()) {
    int before = failures();
    ++cases;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      fail(c.file, c.line, std::string("unexpected exception: ") + e.what());
    }
    if (failures() != before) {
      ++bad_cases;
      std::printf("[case failed] %s\n", c.name);
    }
  }
  std::printf("[doctest-mini] test cases: %d | %d passed | %d failed | assertions failed: %d\n",
              cases, cases - bad_cases, bad_cases, failures());
  return bad_cases ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC(fn, name)                                                         \
  static void fn();                                                                  \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define SUBCASE(name) if ([[maybe_unused]] const bool DOCTEST_CAT(sc_, __LINE__) = true)
#define CHECK(...)                                                          \
  do {                                                                      \
    if (!(__VA_ARGS__)) ::doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__); \
  } while (0)
#define CHECK_FALSE(...)                                                            \
  do {                                                                              \
    if ((__VA_ARGS__)) ::doctest::detail::fail(__FILE__, __LINE__, "!(" #__VA_ARGS__ ")"); \
  } while (0)
#define REQUIRE(...)                                                       \
  do {                                                                     \
    if (!(__VA_ARGS__)) {                                                  \
      ::doctest::detail::fail(__FILE__, __LINE__, "REQUIRE " #__VA_ARGS__); \
      throw ::doctest::detail::RequireFailed{};                            \
    }                                                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                        \
  do {                                                                                    \
    bool thrown_ = false;                                                                 \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (const __VA_ARGS__&) {                                                        \
      thrown_ = true;                                                                     \
    } catch (...) {                                                                       \
      ::doctest::detail::fail(__FILE__, __LINE__, "wrong exception from " #expr);         \
      thrown_ = true;                                                                     \
    }                                                                                     \
    if (!thrown_) ::doctest::detail::fail(__FILE__, __LINE__, "no exception from " #expr); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                      \
  do {                                                                           \
    try {                                                                        \
      (void)(expr);                                                              \
    } catch (...) {                                                              \
      ::doctest::detail::fail(__FILE__, __LINE__, "exception from " #expr);      \
    }                                                                            \
  } while (0)
#define CAPTURE(x) ::doctest::detail::Capture DOCTEST_CAT(capture_, __LINE__)(#x, x)
#define WARN_LE(a, b)                                                        \
  do {                                                                       \
    if (!((a) <= (b))) std::printf("%s:%d: WARNING: %s <= %s\n", __FILE__, __LINE__, #a, #b); \
  } while (0)
#define FAIL_CHECK(msg)                                      \
  do {                                                       \
    std::ostringstream os_;                                  \
    os_ << msg;                                              \
    ::doctest::detail::fail(__FILE__, __LINE__, os_.str());  \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
