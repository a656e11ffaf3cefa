// doctest.h -- a minimal doctest-compatible harness, written for this repo.
//
// The reference's unit suites (proj/tests/test_{hashing,estimator,rsea,
// snapshot,workload,pipeline}.cpp) `#include <doctest.h>`, which the
// reference never vendored (proj/.gitignore:2).  This header implements the
// subset those files use, so they compile UNCHANGED against the drop-in
// headers (include/sspd/*.hpp) and link against libsspd.so:
//
//   TEST_CASE, SUBCASE (doctest's re-entry semantics: the test case body is
//   re-run until every leaf subcase path has run exactly once), CHECK,
//   CHECK_FALSE, CHECK_THROWS, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS (with a
//   string or doctest::Contains), REQUIRE, FAIL(stream expression),
//   doctest::Approx(.epsilon), DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
//
// Output: one line per failed assertion, then
//   "[doctest] test cases: N | P passed | F failed" and
//   "[doctest] assertions: N | P passed | F failed"
// and exit status 1 on any failure (doctest's own summary format).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <utility>
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
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

struct Contains {
  explicit Contains(std::string s) : text(std::move(s)) {}
  bool matches(const std::string& what) const { return what.find(text) != std::string::npos; }
  std::string text;
};

namespace detail {

inline bool matches(const std::string& what, const Contains& c) { return c.matches(what); }
inline bool matches(const std::string& what, const std::string& s) { return what == s; }
inline bool matches(const std::string& what, const char* s) { return what == s; }

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

struct Abort {};

struct State {
  std::vector<TestCase> cases;
  int asserts = 0, failed_asserts = 0;
  // SUBCASE bookkeeping for the running test case
  std::vector<std::string> path;            // subcases entered, outermost first
  std::vector<bool> pending;                // per entered subcase: a child was skipped unfinished
  std::vector<bool> entered;                // per depth: a subcase already ran at this depth this pass
  std::set<std::vector<std::string>> done;  // fully traversed subcase paths
  bool rerun = false;                       // something was skipped unfinished this pass
};

inline State& state() {
  static State s;
  return s;
}

struct Reg {
  Reg(const char* n, const char* f, int l, void (*fn)()) { state().cases.push_back({n, f, l, fn}); }
};

inline void record(bool ok, const char* file, int line, const std::string& what) {
  auto& s = state();
  ++s.asserts;
  if (ok) return;
  ++s.failed_asserts;
  std::string where;
  for (const auto& p : s.path) where += " / " + p;
  std::fprintf(stderr, "%s:%d: ERROR%s: %s\n", file, line, where.c_str(), what.c_str());
}

// RAII guard for one SUBCASE: decides on construction whether this pass
// enters it, and marks its path traversed when it exits with nothing left.
class Subcase {
 public:
  Subcase(const char* name, int line) {
    auto& s = state();
    const size_t depth = s.path.size();
    if (s.entered.size() <= depth) s.entered.resize(depth + 1, false);
    std::vector<std::string> p = s.path;
    p.push_back(std::string(name) + "@" + std::to_string(line));
    if (s.done.count(p)) return;
    if (s.entered[depth]) {  // a sibling ran this pass: come back for this one
      s.rerun = true;
      for (size_t i = 0; i < s.pending.size(); ++i) s.pending[i] = true;
      return;
    }
    s.entered[depth] = true;
    s.path = std::move(p);
    s.pending.push_back(false);
    if (s.entered.size() <= depth + 1) s.entered.resize(depth + 2, false);
    s.entered[depth + 1] = false;
    active_ = true;
  }
  ~Subcase() {
    if (!active_) return;
    auto& s = state();
    if (!s.pending.back() || std::uncaught_exceptions() > 0) s.done.insert(s.path);
    s.pending.pop_back();
    s.path.pop_back();
  }
  explicit operator bool() const { return active_; }

 private:
  bool active_ = false;
};

inline int run_all() {
  auto& s = state();
  int failed_cases = 0;
  for (const auto& tc : s.cases) {
    s.done.clear();
    const int before = s.failed_asserts;
    for (int pass = 0;; ++pass) {
      s.path.clear();
      s.pending.clear();
      s.entered.assign(1, false);
      s.rerun = false;
      try {
        tc.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        record(false, tc.file, tc.line, std::string("test case THREW exception: ") + e.what());
      } catch (...) {
        record(false, tc.file, tc.line, "test case THREW an unknown exception");
      }
      if (!s.rerun) break;
    }
    if (s.failed_asserts != before) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE(\"%s\") at %s:%d\n", tc.name, tc.file, tc.line);
    }
  }
  const int n = static_cast<int>(s.cases.size());
  std::printf("[doctest] test cases: %d | %d passed | %d failed\n", n, n - failed_cases, failed_cases);
  std::printf("[doctest] assertions: %d | %d passed | %d failed\n", s.asserts, s.asserts - s.failed_asserts,
              s.failed_asserts);
  std::printf("[doctest] Status: %s!\n", failed_cases ? "FAILURE" : "SUCCESS");
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define TEST_CASE(name)                                                                          \
  static void DOCTEST_CAT(doctest_case_, __LINE__)();                                            \
  static ::doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, __FILE__, __LINE__,    \
                                                                    DOCTEST_CAT(doctest_case_, __LINE__)); \
  static void DOCTEST_CAT(doctest_case_, __LINE__)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_sub_, __LINE__){name, __LINE__})

#define CHECK(...) ::doctest::detail::record(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK( " #__VA_ARGS__ " )")
#define CHECK_FALSE(...) \
  ::doctest::detail::record(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK_FALSE( " #__VA_ARGS__ " )")
#define REQUIRE(...)                                                                                 \
  do {                                                                                               \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                         \
    ::doctest::detail::record(doctest_ok_, __FILE__, __LINE__, "REQUIRE( " #__VA_ARGS__ " )");       \
    if (!doctest_ok_) throw ::doctest::detail::Abort{};                                              \
  } while (0)
#define FAIL(msg)                                                          \
  do {                                                                     \
    std::ostringstream doctest_os_;                                        \
    doctest_os_ << msg;                                                    \
    ::doctest::detail::record(false, __FILE__, __LINE__, doctest_os_.str()); \
    throw ::doctest::detail::Abort{};                                      \
  } while (0)

#define CHECK_THROWS(expr)                                                                      \
  do {                                                                                          \
    bool doctest_threw_ = false;                                                                \
    try {                                                                                       \
      static_cast<void>(expr);                                                                  \
    } catch (...) {                                                                             \
      doctest_threw_ = true;                                                                    \
    }                                                                                           \
    ::doctest::detail::record(doctest_threw_, __FILE__, __LINE__, "CHECK_THROWS( " #expr " )"); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                          \
  do {                                                                                                      \
    bool doctest_ok_ = false;                                                                               \
    try {                                                                                                   \
      static_cast<void>(expr);                                                                              \
    } catch (const __VA_ARGS__&) {                                                                          \
      doctest_ok_ = true;                                                                                   \
    } catch (...) {                                                                                         \
    }                                                                                                       \
    ::doctest::detail::record(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_AS( " #expr ", " #__VA_ARGS__ " )"); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                       \
  do {                                                                                              \
    bool doctest_ok_ = false;                                                                       \
    std::string doctest_what_ = "(no exception)";                                                   \
    try {                                                                                           \
      static_cast<void>(expr);                                                                      \
    } catch (const __VA_ARGS__& e) {                                                                \
      doctest_what_ = e.what();                                                                     \
      doctest_ok_ = ::doctest::detail::matches(doctest_what_, with);                                \
    } catch (const std::exception& e) {                                                             \
      doctest_what_ = std::string("wrong type: ") + e.what();                                       \
    } catch (...) {                                                                                 \
      doctest_what_ = "wrong type";                                                                 \
    }                                                                                               \
    ::doctest::detail::record(doctest_ok_, __FILE__, __LINE__,                                      \
                              "CHECK_THROWS_WITH_AS( " #expr " ) got: " + doctest_what_);           \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
