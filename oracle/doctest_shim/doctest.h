// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE ONLY).
//
// The reference's unit tests (/root/reference/proj/tests/*_test.cpp) are
// written against doctest, which is not vendored anywhere on this machine
// (proj/.gitignore:2).  This header implements exactly the subset they use —
// TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// CHECK_NOTHROW, FAIL, CAPTURE and doctest::Approx(...).epsilon(...) — so the
// unmodified test sources compile against either the reference core or the
// B200 library.  Exit status = number of failing test cases.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
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

struct Reg {
  Reg(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};

struct State {
  int assertions = 0;
  int failed_assertions = 0;
  bool current_failed = false;
  std::vector<std::string> captures;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(const char* file, int line, const std::string& what) {
  State& s = state();
  ++s.failed_assertions;
  s.current_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
  for (const auto& c : s.captures) std::fprintf(stderr, "    with %s\n", c.c_str());
}

inline void check(bool ok, const char* file, int line, const char* expr, bool require) {
  ++state().assertions;
  if (!ok) {
    report(file, line, expr);
    if (require) throw RequireFailed{};
  }
}

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) < rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

struct Capture {
  explicit Capture(std::string s) { state().captures.push_back(std::move(s)); }
  ~Capture() { state().captures.pop_back(); }
};

inline int run(int argc, char** argv) {
  // args: substrings of the test-case name or source path; "-x" excludes x
  std::vector<std::string> keep, drop;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (!a.empty() && a[0] == '-') drop.push_back(a.substr(1));
    else keep.push_back(a);
  }
  auto hit = [](const TestCase& tc, const std::string& s) {
    return std::string(tc.name).find(s) != std::string::npos || std::string(tc.file).find(s) != std::string::npos;
  };
  int failed = 0, ran = 0;
  for (const TestCase& tc : registry()) {
    if (!keep.empty() && std::none_of(keep.begin(), keep.end(), [&](const std::string& s) { return hit(tc, s); }))
      continue;
    if (std::any_of(drop.begin(), drop.end(), [&](const std::string& s) { return hit(tc, s); })) continue;
    ++ran;
    state().current_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      report(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
    } catch (...) {
      report(tc.file, tc.line, "unexpected non-std exception");
    }
    if (state().current_failed) {
      ++failed;
      std::fprintf(stderr, "  in test case \"%s\" (%s:%d)\n", tc.name, tc.file, tc.line);
    }
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed; assertions: %d | %d failed\n", ran,
              ran - failed, failed, state().assertions, state().failed_assertions);
  return failed;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(name, id)                                                                   \
  static void DOCTEST_CAT(doctest_fn_, id)();                                                   \
  static ::doctest::Reg DOCTEST_CAT(doctest_reg_, id)(name, __FILE__, __LINE__,                 \
                                                      &DOCTEST_CAT(doctest_fn_, id));           \
  static void DOCTEST_CAT(doctest_fn_, id)()
#define TEST_CASE(name) DOCTEST_TC_(name, __COUNTER__)

#define CHECK(...) ::doctest::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define REQUIRE(...) ::doctest::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define CHECK_FALSE(...) ::doctest::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define FAIL(msg)                                                                                 \
  do {                                                                                            \
    std::ostringstream doctest_os_;                                                               \
    doctest_os_ << msg;                                                                           \
    ::doctest::report(__FILE__, __LINE__, doctest_os_.str());                                     \
    throw ::doctest::RequireFailed{};                                                             \
  } while (0)
#define CAPTURE(x)                                                                                \
  std::ostringstream DOCTEST_CAT(doctest_cap_os_, __LINE__);                                      \
  DOCTEST_CAT(doctest_cap_os_, __LINE__) << #x " := " << (x);                                     \
  ::doctest::Capture DOCTEST_CAT(doctest_cap_, __LINE__)(DOCTEST_CAT(doctest_cap_os_, __LINE__).str())

#define CHECK_THROWS_AS(expr, ...)                                                                \
  do {                                                                                            \
    bool doctest_ok_ = false;                                                                     \
    try { static_cast<void>(expr); } catch (const __VA_ARGS__&) { doctest_ok_ = true; } catch (...) {} \
    ::doctest::check(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")", false); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, ...)                                                      \
  do {                                                                                            \
    bool doctest_ok_ = false;                                                                     \
    try { static_cast<void>(expr); } catch (const __VA_ARGS__& e) { doctest_ok_ = std::string(e.what()) == std::string(msg); } catch (...) {} \
    ::doctest::check(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS(" #expr ", " #msg ", " #__VA_ARGS__ ")", false); \
  } while (0)
#define CHECK_NOTHROW(...)                                                                        \
  do {                                                                                            \
    bool doctest_ok_ = true;                                                                      \
    try { static_cast<void>(__VA_ARGS__); } catch (...) { doctest_ok_ = false; }                  \
    ::doctest::check(doctest_ok_, __FILE__, __LINE__, "CHECK_NOTHROW(" #__VA_ARGS__ ")", false);  \
  } while (0)
