// Minimal doctest-compatible test macros -- TEST HARNESS ONLY.
//
// doctest is not installed in this image.  This header provides the subset
// of its interface the reference's test files use (TEST_SUITE, TEST_CASE,
// CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW,
// doctest::Approx) so those files compile unmodified against the drop-in
// headers.  Written from scratch; main() is in doctest_shim_main.cpp.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest_shim {

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
struct Reg {
  Reg(const char* name, void (*fn)(), const char* file, int line) { registry().push_back({name, file, line, fn}); }
};
struct Abort {};
struct Stats {
  long checks = 0, failed = 0;
  bool case_failed = false;
};
inline Stats& stats() {
  static Stats s;
  return s;
}
inline void record(bool ok, const char* what, const char* file, int line) {
  ++stats().checks;
  if (!ok) {
    ++stats().failed;
    stats().case_failed = true;
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, what);
  }
}

}  // namespace doctest_shim

namespace doctest {
class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::abs(a - b.v_) < b.eps_ * (1.0 + std::max(std::abs(a), std::abs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }

 private:
  double v_;
  double eps_ = 1.1920929e-07 * 100;  // doctest's default (float epsilon * 100)
};
}  // namespace doctest

#define DSHIM_CAT2(a, b) a##b
#define DSHIM_CAT(a, b) DSHIM_CAT2(a, b)
#define TEST_SUITE(name) namespace DSHIM_CAT(dshim_suite_, __COUNTER__)
#define DSHIM_TC(name, id)                                                                         \
  static void DSHIM_CAT(dshim_tc_, id)();                                                         \
  static ::doctest_shim::Reg DSHIM_CAT(dshim_reg_, id)(name, &DSHIM_CAT(dshim_tc_, id), __FILE__, __LINE__); \
  static void DSHIM_CAT(dshim_tc_, id)()
#define TEST_CASE(name) DSHIM_TC(name, __COUNTER__)
#define CHECK(...) ::doctest_shim::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest_shim::record(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                              \
  do {                                                                                            \
    bool ok_ = static_cast<bool>(__VA_ARGS__);                                                    \
    ::doctest_shim::record(ok_, #__VA_ARGS__, __FILE__, __LINE__);                                \
    if (!ok_) throw ::doctest_shim::Abort{};                                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                               \
  do {                                                                                            \
    bool ok_ = false;                                                                             \
    try {                                                                                         \
      (void)(expr);                                                                               \
    } catch (const type&) {                                                                       \
      ok_ = true;                                                                                 \
    } catch (...) {                                                                               \
    }                                                                                             \
    ::doctest_shim::record(ok_, "THROWS_AS(" #expr ", " #type ")", __FILE__, __LINE__);          \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                       \
  do {                                                                                            \
    bool ok_ = true;                                                                              \
    try {                                                                                         \
      (void)(expr);                                                                               \
    } catch (...) {                                                                               \
      ok_ = false;                                                                                \
    }                                                                                             \
    ::doctest_shim::record(ok_, "NOTHROW(" #expr ")", __FILE__, __LINE__);                        \
  } while (0)
