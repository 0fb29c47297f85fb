// Minimal doctest-compatible shim (own code, test infrastructure): enough
// of the doctest surface -- TEST_CASE, CHECK, REQUIRE, REQUIRE_MESSAGE,
// CHECK_THROWS_AS, doctest::Approx and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN --
// to compile the reference's unit tests (proj/tests/test_*.cpp) unmodified
// against the B200 drop-in library.  doctest itself is not
// in this image.
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

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct State {
  long checks = 0, failures = 0;
  bool case_failed = false;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireAbort {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   const char* msg = nullptr) {
  State& s = state();
  s.checks++;
  if (ok) return;
  s.failures++;
  s.case_failed = true;
  std::printf("  %s:%d: %s( %s ) FAILED%s%s\n", file, line, kind, expr, msg ? " -- " : "",
              msg ? msg : "");
}

// doctest::Approx: |a - b| < epsilon * (scale + max(|a|, |b|)), epsilon
// = 100 * FLT_EPSILON by default
class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) < b.eps_ * (b.scale_ + std::fmax(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend bool operator!=(const Approx& b, double a) { return !(a == b); }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-07 * 100;
  double scale_ = 1.0;
};

inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& t : registry()) {
    state().case_failed = false;
    try {
      t.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      report(false, "TEST_CASE", t.name, t.file, t.line, e.what());
    } catch (...) {
      report(false, "TEST_CASE", t.name, t.file, t.line, "unknown exception");
    }
    if (state().case_failed) {
      failed_cases++;
      std::printf("FAILED test case: %s (%s:%d)\n", t.name, t.file, t.line);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld | %ld failed\n",
              registry().size(), registry().size() - failed_cases, failed_cases, state().checks,
              state().failures);
  return failed_cases ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, reg, name)                                                   \
  static void fn();                                                                  \
  static ::doctest::Registrar reg(name, __FILE__, __LINE__, &fn);                    \
  static void fn()
#define TEST_CASE(name) \
  DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), DOCTEST_CAT(doctest_reg_, __LINE__), name)

#define CHECK(...) ::doctest::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                 \
  do {                                                                               \
    const bool ok_ = static_cast<bool>(__VA_ARGS__);                                 \
    ::doctest::report(ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);             \
    if (!ok_) throw ::doctest::RequireAbort{};                                       \
  } while (0)
#define REQUIRE_MESSAGE(cond, msg)                                                   \
  do {                                                                               \
    const bool ok_ = static_cast<bool>(cond);                                        \
    ::doctest::report(ok_, "REQUIRE_MESSAGE", #cond, __FILE__, __LINE__);            \
    if (!ok_) throw ::doctest::RequireAbort{};                                       \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                   \
  do {                                                                               \
    bool ok_ = false;                                                                \
    try {                                                                            \
      static_cast<void>(expr);                                                       \
    } catch (const __VA_ARGS__&) {                                                   \
      ok_ = true;                                                                    \
    } catch (...) {                                                                  \
    }                                                                                \
    ::doctest::report(ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);            \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::run_all(); }
#endif
