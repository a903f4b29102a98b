// doctest-API-subset shim — TEST INFRASTRUCTURE ONLY.
//
// The reference's tests (proj/tests/*.cpp) use doctest, which is not vendored
// (proj/.gitignore:2 excludes proj/vendor/). This header implements the
// macros those tests use: TEST_CASE, SUBCASE (one level), CHECK, REQUIRE,
// CHECK_THROWS_AS, CHECK_NOTHROW, FAIL and doctest::Approx(...).epsilon(...),
// plus DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN. A SUBCASE-bearing test case is
// re-run once per subcase, entering exactly one new subcase per run.
#ifndef CCLP_ORACLE_DOCTEST_SHIM_H_
#define CCLP_ORACLE_DOCTEST_SHIM_H_

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <set>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v), eps_(1.19209290e-07 * 100), scale_(1.0) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return operator==(rhs, lhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !operator==(lhs, rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !operator==(rhs, lhs); }

 private:
  double value_, eps_, scale_;
};

namespace detail {

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
  int checks = 0;
  int failures = 0;
  bool case_failed = false;
  std::set<std::string> done_subcases;
  bool entered_this_run = false;
  std::string current_subcase;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  State& s = state();
  ++s.checks;
  if (!ok) {
    ++s.failures;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: %s(%s) FAILED%s%s\n", file, line, kind, expr,
                 s.current_subcase.empty() ? "" : " in subcase ", s.current_subcase.c_str());
  }
}

struct SubcaseGuard {
  bool enter;
  SubcaseGuard(const char* name) {
    State& s = state();
    enter = !s.entered_this_run && !s.done_subcases.count(name);
    if (enter) {
      s.entered_this_run = true;
      s.done_subcases.insert(name);
      s.current_subcase = name;
    }
  }
  ~SubcaseGuard() {
    if (enter) state().current_subcase.clear();
  }
  explicit operator bool() const { return enter; }
};

inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    State& s = state();
    s.case_failed = false;
    s.done_subcases.clear();
    while (true) {
      s.entered_this_run = false;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        std::fprintf(stderr, "%s:%d: TEST_CASE(%s) threw: %s\n", tc.file, tc.line, tc.name, e.what());
        ++s.failures;
        s.case_failed = true;
      }
      if (!s.entered_this_run) break;  // no new subcase this run: done
    }
    if (s.case_failed) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
              registry().size(), registry().size() - failed_cases, failed_cases, state().checks,
              state().failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQUE(base) DOCTEST_CAT(base, __LINE__)

#define TEST_CASE(name)                                                                   \
  static void DOCTEST_UNIQUE(doctest_fn_)();                                              \
  static ::doctest::detail::Registrar DOCTEST_UNIQUE(doctest_reg_)(                       \
      name, __FILE__, __LINE__, &DOCTEST_UNIQUE(doctest_fn_));                            \
  static void DOCTEST_UNIQUE(doctest_fn_)()

#define SUBCASE(name) if (const ::doctest::detail::SubcaseGuard DOCTEST_UNIQUE(doctest_sc_){name})

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                     \
  do {                                                                                   \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                             \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__); \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                          \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                       \
  do {                                                                                   \
    bool doctest_ok_ = false;                                                            \
    try {                                                                                \
      (void)(expr);                                                                      \
    } catch (const __VA_ARGS__&) {                                                       \
      doctest_ok_ = true;                                                                \
    } catch (...) {                                                                      \
    }                                                                                    \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                              \
  do {                                                                                   \
    bool doctest_ok_ = true;                                                             \
    try {                                                                                \
      (void)(expr);                                                                      \
    } catch (...) {                                                                      \
      doctest_ok_ = false;                                                               \
    }                                                                                    \
    ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__);  \
  } while (0)
#define FAIL(msg)                                                                        \
  do {                                                                                   \
    ::doctest::detail::report(false, "FAIL", #msg, __FILE__, __LINE__);                  \
    throw ::doctest::detail::RequireFailed{};                                            \
  } while (0)
#define MESSAGE(msg) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif

#endif  // CCLP_ORACLE_DOCTEST_SHIM_H_
