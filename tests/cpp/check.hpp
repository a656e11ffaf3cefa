// check.hpp -- a tiny self-registering test harness for the C++ API tests
// (the reference uses doctest, which is not vendored here).  Each TEST_CASE
// runs once; CHECK records a failure and continues, REQUIRE aborts the case.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace chk {

struct Case {
  const char* name;
  std::function<void()> fn;
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

inline int& failures() {
  static int f = 0;
  return f;
}

struct Abort {};

struct Reg {
  Reg(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};

inline void fail(const char* file, int line, const std::string& what) {
  ++failures();
  std::fprintf(stderr, "  FAILED %s:%d: %s\n", file, line, what.c_str());
}

inline int run_all(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int cases = 0, bad = 0;
  for (auto& c : registry()) {
    if (filter && std::string(c.name).find(filter) == std::string::npos) continue;
    ++cases;
    const int before = failures();
    std::fprintf(stderr, "[case] %s\n", c.name);
    try {
      c.fn();
    } catch (const Abort&) {
    } catch (const std::exception& e) {
      fail(__FILE__, __LINE__, std::string("unexpected exception: ") + e.what());
    }
    if (failures() != before) ++bad;
  }
  std::fprintf(stderr, "%d cases, %d failed, %d checks failed\n", cases, bad, failures());
  return failures() ? 1 : 0;
}

}  // namespace chk

#define CHK_CAT2(a, b) a##b
#define CHK_CAT(a, b) CHK_CAT2(a, b)
#define TEST_CASE(name)                                                  \
  static void CHK_CAT(chk_case_, __LINE__)();                            \
  static chk::Reg CHK_CAT(chk_reg_, __LINE__)(name, CHK_CAT(chk_case_, __LINE__)); \
  static void CHK_CAT(chk_case_, __LINE__)()

#define CHECK(expr)                                                  \
  do {                                                               \
    if (!(expr)) chk::fail(__FILE__, __LINE__, "CHECK(" #expr ")");  \
  } while (0)
#define CHECK_FALSE(expr) CHECK(!(expr))
#define REQUIRE(expr)                                                  \
  do {                                                                 \
    if (!(expr)) {                                                     \
      chk::fail(__FILE__, __LINE__, "REQUIRE(" #expr ")");             \
      throw chk::Abort{};                                              \
    }                                                                  \
  } while (0)
#define FAIL(msg)                                      \
  do {                                                 \
    std::ostringstream os_;                            \
    os_ << msg;                                        \
    chk::fail(__FILE__, __LINE__, os_.str());          \
    throw chk::Abort{};                                \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                   \
  do {                                                                                \
    bool ok_ = false;                                                                 \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (const type&) {                                                           \
      ok_ = true;                                                                     \
    } catch (...) {                                                                   \
    }                                                                                 \
    if (!ok_) chk::fail(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #type ")"); \
  } while (0)
#define CHECK_THROWS_WITH_SUBSTR(expr, text)                                          \
  do {                                                                                \
    bool ok_ = false;                                                                 \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (const std::exception& e_) {                                              \
      ok_ = std::string(e_.what()).find(text) != std::string::npos;                   \
    }                                                                                 \
    if (!ok_) chk::fail(__FILE__, __LINE__, "CHECK_THROWS_WITH(" #expr ", " text ")"); \
  } while (0)

#define CHECK_MAIN \
  int main(int argc, char** argv) { return chk::run_all(argc, argv); }
