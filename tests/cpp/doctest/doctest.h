// Minimal stand-in for doctest (absent from this image; the reference's
// tests/CMakeLists.txt expects it from proj/vendor, which is not shipped).
// It implements only what the reference's unit tests use: TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// doctest::Approx (+ epsilon) and doctest::Contains, and a main() under
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN that runs every case and returns
// nonzero on any failure. Test infrastructure only.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
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
    return std::fabs(lhs - a.v_) <
           a.eps_ * (1.0 + std::max(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double v_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
};

struct Contains {
  explicit Contains(std::string s) : s(std::move(s)) {}
  bool matches(const std::string& what) const { return what.find(s) != std::string::npos; }
  std::string s;
};

namespace detail {

struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}

struct State {
  int failed_checks = 0;
  int checks = 0;
  bool case_failed = false;
  const Case* current = nullptr;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireAbort {};

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    cases().push_back({name, file, line, fn});
  }
};

inline void fail(const char* kind, const char* expr, const char* file, int line,
                 const std::string& extra = {}) {
  State& s = state();
  ++s.failed_checks;
  s.case_failed = true;
  std::printf("%s:%d: FAILED %s( %s )%s%s  [in \"%s\"]\n", file, line, kind, expr,
              extra.empty() ? "" : " : ", extra.c_str(), s.current ? s.current->name : "?");
}

inline bool check(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++state().checks;
  if (!ok) fail(kind, expr, file, line);
  return ok;
}

inline std::string what_of(const std::exception& e) { return e.what(); }

inline int run_all() {
  State& s = state();
  int failed_cases = 0;
  for (const Case& c : cases()) {
    s.current = &c;
    s.case_failed = false;
    ++s.checks;  // the case body itself (an escaping exception fails it)
    try {
      c.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      fail("TEST_CASE", c.name, c.file, c.line, std::string("unexpected exception: ") + e.what());
    } catch (...) {
      fail("TEST_CASE", c.name, c.file, c.line, "unexpected non-std exception");
    }
    if (s.case_failed) ++failed_cases;
  }
  const int n = static_cast<int>(cases().size());
  std::printf("[doctest] test cases: %d | %d passed | %d failed\n", n, n - failed_cases,
              failed_cases);
  std::printf("[doctest] assertions: %d | %d passed | %d failed\n", s.checks,
              s.checks - s.failed_checks, s.failed_checks);
  std::printf("[doctest] Status: %s\n", failed_cases ? "FAILURE!" : "SUCCESS!");
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_IMPL(fn, name)                                                        \
  static void fn();                                                                        \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) \
  ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...)                                                                  \
  ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, \
                           __FILE__, __LINE__)
#define REQUIRE(...)                                                                  \
  do {                                                                                \
    if (!::doctest::detail::check(static_cast<bool>(__VA_ARGS__), "REQUIRE",          \
                                  #__VA_ARGS__, __FILE__, __LINE__))                  \
      throw ::doctest::detail::RequireAbort{};                                        \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                      \
  do {                                                                                  \
    ++::doctest::detail::state().checks;                                                \
    try {                                                                               \
      static_cast<void>(expr);                                                          \
      ::doctest::detail::fail("CHECK_THROWS_AS", #expr, __FILE__, __LINE__,             \
                              "did not throw");                                         \
    } catch (const __VA_ARGS__&) {                                                      \
    } catch (const std::exception& e_) {                                                \
      ::doctest::detail::fail("CHECK_THROWS_AS", #expr, __FILE__, __LINE__,             \
                              std::string("threw a different type: ") + e_.what());     \
    } catch (...) {                                                                     \
      ::doctest::detail::fail("CHECK_THROWS_AS", #expr, __FILE__, __LINE__,             \
                              "threw a different type");                                \
    }                                                                                   \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                        \
  do {                                                                                  \
    ++::doctest::detail::state().checks;                                                \
    try {                                                                               \
      static_cast<void>(expr);                                                          \
      ::doctest::detail::fail("CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__,        \
                              "did not throw");                                         \
    } catch (const __VA_ARGS__& e_) {                                                   \
      if (!(matcher).matches(::doctest::detail::what_of(e_)))                           \
        ::doctest::detail::fail("CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__,      \
                                std::string("message: ") + e_.what());                  \
    } catch (...) {                                                                     \
      ::doctest::detail::fail("CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__,        \
                              "threw a different type");                                \
    }                                                                                   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
