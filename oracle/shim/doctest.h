// TEST INFRASTRUCTURE (oracle only) — a clean-room, minimal doctest-compatible
// harness so that the reference's own unit tests
// (/root/reference/proj/tests/test_*.cpp) compile and run unmodified against
// the reference sources plus the Eigen shim.  doctest itself was meant to be
// vendored (proj/README.md:28) but /vendor is git-ignored and absent.
//
// Supported: TEST_CASE, SUBCASE (re-entrant, one leaf per pass, like doctest),
// CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, FAIL, INFO,
// CAPTURE, doctest::Approx (default epsilon = 100 * FLT_EPSILON, scale 1).
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

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
  bool matches(double lhs) const {
    return std::fabs(lhs - value_) <
           eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  friend bool operator==(double lhs, const Approx& a) { return a.matches(lhs); }
  friend bool operator==(const Approx& a, double rhs) { return a.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& a) { return !a.matches(lhs); }
  friend bool operator!=(const Approx& a, double rhs) { return !a.matches(rhs); }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};

}  // namespace doctest

namespace mini_doctest {

struct TestCase {
  void (*fn)();
  const char* name;
  const char* file;
  int line;
};

struct RequireAbort {};

struct State {
  std::vector<TestCase> tests;
  std::vector<int> path;
  std::vector<char> entered;
  std::vector<char> pending;
  std::set<std::vector<int>> done;
  bool rerun = false;
  bool progress = false;
  long assertions = 0;
  long failed_assertions = 0;
  bool current_failed = false;
  const char* current_name = "";
};

inline State& state() {
  static State s;
  return s;
}

inline int reg(void (*fn)(), const char* name, const char* file, int line) {
  state().tests.push_back({fn, name, file, line});
  return 0;
}

inline void report(const char* kind, const char* expr, const char* file, int line,
                   const std::string& extra = "") {
  State& s = state();
  ++s.failed_assertions;
  s.current_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in test case \"%s\"%s%s\n", file, line, kind,
               expr, s.current_name, extra.empty() ? "" : " : ", extra.c_str());
}

class Subcase {
 public:
  Subcase(const char* /*name*/, int line) {
    State& s = state();
    const std::size_t depth = s.path.size();
    std::vector<int> key = s.path;
    key.push_back(line);
    if (s.done.count(key)) return;
    if (s.entered[depth]) {
      s.pending[depth] = 1;
      s.rerun = true;
      return;
    }
    entered_ = true;
    key_ = key;
    s.entered[depth] = 1;
    s.path.push_back(line);
    s.entered.push_back(0);
    s.pending.push_back(0);
  }
  ~Subcase() {
    if (!entered_) return;
    State& s = state();
    const bool children_pending = s.pending.back() != 0;
    s.path.pop_back();
    s.entered.pop_back();
    s.pending.pop_back();
    if (!children_pending) {
      s.done.insert(key_);
      s.progress = true;
    } else {
      s.pending.back() = 1;
    }
  }
  explicit operator bool() const { return entered_; }

 private:
  bool entered_ = false;
  std::vector<int> key_;
};

// Comma-separated name filters, as doctest's --test-case= / --test-case-exclude=
// (substring match here, no wildcards).
inline bool name_matches(const char* name, const std::string& list) {
  std::size_t a = 0;
  while (a <= list.size()) {
    std::size_t b = list.find(',', a);
    if (b == std::string::npos) b = list.size();
    const std::string item = list.substr(a, b - a);
    if (!item.empty() && std::strstr(name, item.c_str()) != nullptr) return true;
    a = b + 1;
  }
  return false;
}

inline int run_all(const std::string& only = "", const std::string& exclude = "") {
  State& s = state();
  int failed_cases = 0;
  std::size_t ran = 0;
  for (const TestCase& tc : s.tests) {
    if (!only.empty() && !name_matches(tc.name, only)) continue;
    if (!exclude.empty() && name_matches(tc.name, exclude)) continue;
    ++ran;
    s.done.clear();
    s.current_failed = false;
    s.current_name = tc.name;
    int passes = 0;
    do {
      s.rerun = false;
      s.progress = false;
      s.path.clear();
      s.entered.assign(1, 0);
      s.pending.assign(1, 0);
      try {
        tc.fn();
      } catch (const RequireAbort&) {
        if (s.progress) s.rerun = true;
      } catch (const std::exception& e) {
        report("TEST_CASE", "unexpected exception", tc.file, tc.line, e.what());
        if (s.progress) s.rerun = true;
      } catch (...) {
        report("TEST_CASE", "unexpected unknown exception", tc.file, tc.line);
        if (s.progress) s.rerun = true;
      }
    } while (s.rerun && ++passes < 10000);
    if (s.current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "[doctest-shim] FAILED test case: %s\n", tc.name);
    }
  }
  std::fprintf(stderr,
               "[doctest-shim] test cases: %zu | %zu passed | %d failed | %zu skipped; assertions: %ld | %ld "
               "failed\n",
               ran, ran - static_cast<std::size_t>(failed_cases), failed_cases, s.tests.size() - ran,
               s.assertions, s.failed_assertions);
  return failed_cases;
}

}  // namespace mini_doctest

#define MINI_DOCTEST_CAT2(a, b) a##b
#define MINI_DOCTEST_CAT(a, b) MINI_DOCTEST_CAT2(a, b)
#define MINI_DOCTEST_ANON(p) MINI_DOCTEST_CAT(p, __COUNTER__)

#define MINI_DOCTEST_TEST_CASE_IMPL(fn, regv, name)                                   \
  static void fn();                                                                   \
  [[maybe_unused]] static const int regv = ::mini_doctest::reg(&fn, name, __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name)                                                              \
  MINI_DOCTEST_TEST_CASE_IMPL(MINI_DOCTEST_CAT(mini_doctest_fn_, __LINE__),          \
                              MINI_DOCTEST_CAT(mini_doctest_reg_, __LINE__), name)

#define SUBCASE(name) \
  if (const ::mini_doctest::Subcase mini_doctest_sc{name, __LINE__}; mini_doctest_sc)

#define MINI_DOCTEST_ASSERT(kind, is_require, ...)                                    \
  do {                                                                                \
    ++::mini_doctest::state().assertions;                                             \
    bool mini_ok_ = false;                                                            \
    try {                                                                             \
      mini_ok_ = static_cast<bool>(__VA_ARGS__);                                      \
    } catch (const std::exception& e) {                                               \
      ::mini_doctest::report(kind, #__VA_ARGS__, __FILE__, __LINE__, e.what());       \
      if (is_require) throw ::mini_doctest::RequireAbort{};                           \
      break;                                                                          \
    }                                                                                 \
    if (!mini_ok_) {                                                                  \
      ::mini_doctest::report(kind, #__VA_ARGS__, __FILE__, __LINE__);                 \
      if (is_require) throw ::mini_doctest::RequireAbort{};                           \
    }                                                                                 \
  } while (0)

#define CHECK(...) MINI_DOCTEST_ASSERT("CHECK", false, __VA_ARGS__)
#define REQUIRE(...) MINI_DOCTEST_ASSERT("REQUIRE", true, __VA_ARGS__)
#define CHECK_FALSE(...) MINI_DOCTEST_ASSERT("CHECK_FALSE", false, !(__VA_ARGS__))
#define REQUIRE_FALSE(...) MINI_DOCTEST_ASSERT("REQUIRE_FALSE", true, !(__VA_ARGS__))

#define CHECK_THROWS_AS(expr, ...)                                                    \
  do {                                                                                \
    ++::mini_doctest::state().assertions;                                             \
    try {                                                                             \
      static_cast<void>(expr);                                                        \
      ::mini_doctest::report("CHECK_THROWS_AS", #expr, __FILE__, __LINE__, "no throw"); \
    } catch (const __VA_ARGS__&) {                                                    \
    } catch (...) {                                                                   \
      ::mini_doctest::report("CHECK_THROWS_AS", #expr, __FILE__, __LINE__, "wrong type"); \
    }                                                                                 \
  } while (0)

#define CHECK_NOTHROW(...)                                                            \
  do {                                                                                \
    ++::mini_doctest::state().assertions;                                             \
    try {                                                                             \
      static_cast<void>(__VA_ARGS__);                                                 \
    } catch (...) {                                                                   \
      ::mini_doctest::report("CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__);      \
    }                                                                                 \
  } while (0)

#define FAIL(...)                                                                     \
  do {                                                                                \
    std::ostringstream mini_os_;                                                      \
    mini_os_ << __VA_ARGS__;                                                          \
    ::mini_doctest::report("FAIL", "", __FILE__, __LINE__, mini_os_.str());           \
    throw ::mini_doctest::RequireAbort{};                                             \
  } while (0)

#define INFO(...) ((void)0)
#define CAPTURE(...) ((void)0)
#define MESSAGE(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  std::string only, exclude;
  for (int i = 1; i < argc; ++i) {
    const std::string arg = argv[i];
    if (arg.rfind("--test-case=", 0) == 0) only = arg.substr(12);
    else if (arg.rfind("--test-case-exclude=", 0) == 0) exclude = arg.substr(20);
  }
  return ::mini_doctest::run_all(only, exclude) ? 1 : 0;
}
#endif
