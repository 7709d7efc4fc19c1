// A minimal doctest-compatible test harness, written for this repository so
// that the reference's OWN unit-test files (proj/tests/test_hook.cpp, which
// `#include <doctest.h>`) compile unmodified against the libtagc_b200 adapter.
// The reference's CMake build expects doctest under proj/vendor/, which is not
// in the tree (un-vendored third-party dependency, doctest 2.x); this header
// restates the subset of its published interface those files use:
//   TEST_SUITE, TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, doctest::Approx
//   (.epsilon / .scale; the comparison |a - v| < eps * (scale + max(|a|, |v|)),
//   eps defaulting to 100 float epsilons), and a main() taking -ts= / -tc=
//   filters when DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN is defined.
// Output: one line per failed assertion, a summary, exit code 1 on failure.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v)
      : value_(v), epsilon_(double(std::numeric_limits<float>::epsilon()) * 100.0), scale_(1.0) {}
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double a) const {
    return std::fabs(a - value_) < epsilon_ * (scale_ + std::max(std::fabs(a), std::fabs(value_)));
  }
  friend bool operator==(double a, const Approx& b) { return b.matches(a); }
  friend bool operator==(const Approx& b, double a) { return b.matches(a); }
  friend bool operator!=(double a, const Approx& b) { return !b.matches(a); }
  friend bool operator!=(const Approx& b, double a) { return !b.matches(a); }

 private:
  double value_, epsilon_, scale_;
};

namespace detail {

struct TestCase {
  const char* suite;
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct State {
  long asserts = 0, failed_asserts = 0;
  const TestCase* current = nullptr;
  bool current_failed = false;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireAbort {};  // a failed REQUIRE ends the test case

struct Registrar {
  Registrar(const char* suite, const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back(TestCase{suite, name, fn, file, line});
  }
};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  State& s = state();
  ++s.asserts;
  if (ok) return;
  ++s.failed_asserts;
  s.current_failed = true;
  std::printf("%s:%d: FAILED %s( %s )  [suite \"%s\", case \"%s\"]\n", file, line, kind, expr,
              s.current ? s.current->suite : "", s.current ? s.current->name : "");
}

inline bool filter_ok(const char* value, const std::vector<std::string>& filters) {
  if (filters.empty()) return true;
  for (const std::string& f : filters)
    if (f == value) return true;
  return false;
}

inline int run(int argc, char** argv) {
  std::vector<std::string> suites, cases;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (a.rfind("-ts=", 0) == 0) suites.push_back(a.substr(4));
    else if (a.rfind("-tc=", 0) == 0) cases.push_back(a.substr(4));
  }
  State& s = state();
  int ran = 0, failed = 0;
  for (const TestCase& tc : registry()) {
    if (!filter_ok(tc.suite, suites) || !filter_ok(tc.name, cases)) continue;
    s.current = &tc;
    s.current_failed = false;
    try {
      tc.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      report(false, "UNEXPECTED_EXCEPTION", e.what(), tc.file, tc.line);
    } catch (...) {
      report(false, "UNEXPECTED_EXCEPTION", "unknown", tc.file, tc.line);
    }
    ++ran;
    failed += s.current_failed ? 1 : 0;
    std::printf("[%s] %s / %s\n", s.current_failed ? "FAIL" : " ok ", tc.suite, tc.name);
  }
  std::printf("test cases: %d | %d passed | %d failed; assertions: %ld | %ld failed\n", ran, ran - failed,
              failed, s.asserts, s.failed_asserts);
  return (failed || ran == 0) ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

// Suite name seen by the TEST_CASEs of the enclosing scope (TEST_SUITE
// shadows this one inside its namespace).
inline const char* doctest_suite_name_() { return ""; }

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(p) DOCTEST_CAT(p, __COUNTER__)

#define DOCTEST_TEST_CASE_IMPL(fn, reg, name)                                                        \
  static void fn();                                                                                  \
  static const ::doctest::detail::Registrar reg(doctest_suite_name_(), name, &fn, __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_ANON(doctest_tc_), DOCTEST_ANON(doctest_reg_), name)

#define DOCTEST_TEST_SUITE_IMPL(ns, name) \
  namespace ns {                          \
  inline const char* doctest_suite_name_() { return name; } \
  }                                       \
  namespace ns
#define TEST_SUITE(name) DOCTEST_TEST_SUITE_IMPL(DOCTEST_ANON(doctest_suite_), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                              \
  do {                                                                                            \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                      \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);          \
    if (!doctest_ok_) throw ::doctest::detail::RequireAbort{};                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                \
  do {                                                                                            \
    bool doctest_ok_ = false;                                                                     \
    try {                                                                                         \
      (void)(expr);                                                                               \
    } catch (const __VA_ARGS__&) {                                                                \
      doctest_ok_ = true;                                                                         \
    } catch (...) {                                                                               \
    }                                                                                             \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);         \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
