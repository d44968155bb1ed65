// Minimal doctest-compatible test shim (our own code; the real doctest.h is
// not available in this image). Lets the reference's unit-test sources under
// /root/reference/proj/tests compile UNMODIFIED against the B200 library.
//
// Supported: TEST_CASE, SUBCASE (doctest re-entry semantics: the test body is
// re-run until every leaf subcase ran once), CHECK, CHECK_FALSE, REQUIRE,
// REQUIRE_FALSE, CHECK_THROWS_AS, REQUIRE_THROWS_AS, CHECK_NOTHROW, FAIL,
// CAPTURE, INFO, MESSAGE, doctest::Approx, DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// Command line: optional substring filter on test-case names.
#pragma once

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
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    const double scale = std::max(std::fabs(a), std::fabs(b.v_));
    return std::fabs(a - b.v_) <= b.eps_ * (1.0 + scale);
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend bool operator!=(const Approx& b, double a) { return !(a == b); }

 private:
  double v_;
  double eps_ = 1.1920929e-07f * 100;
};

namespace shim {

struct TestCase {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Reg {
  Reg(const char* name, void (*fn)(), const char* file, int line) { registry().push_back({name, fn, file, line}); }
};

struct RequireFailed {};

struct State {
  // subcase bookkeeping for the current test case
  std::set<std::vector<std::string>> done;
  std::vector<std::string> stack;
  std::vector<bool> entered_at_depth;
  int pending = 0;
  // results
  long asserts = 0, failed_asserts = 0;
  bool case_failed = false;
  const char* case_name = "";
};

inline State& st() {
  static State s;
  return s;
}

inline void report(const char* file, int line, const std::string& what) {
  State& s = st();
  ++s.failed_asserts;
  s.case_failed = true;
  std::string path;
  for (const auto& p : s.stack) path += " / " + p;
  std::fprintf(stderr, "%s:%d: FAILED in '%s'%s: %s\n", file, line, s.case_name, path.c_str(), what.c_str());
}

inline void check(bool ok, bool require, const char* expr, const char* file, int line) {
  ++st().asserts;
  if (!ok) {
    report(file, line, std::string(require ? "REQUIRE( " : "CHECK( ") + expr + " )");
    if (require) throw RequireFailed{};
  }
}

class Subcase {
 public:
  Subcase(const char* name, int line) {
    State& s = st();
    path_ = s.stack;
    path_.push_back(std::string(name) + "#" + std::to_string(line));
    const size_t depth = s.stack.size();
    if (s.entered_at_depth.size() <= depth) s.entered_at_depth.resize(depth + 1, false);
    if (s.done.count(path_)) return;
    if (s.entered_at_depth[depth]) {
      ++s.pending;  // sibling already ran this pass: come back next pass
      return;
    }
    s.entered_at_depth[depth] = true;
    s.stack.push_back(path_.back());
    pending_at_entry_ = s.pending;
    entered_ = true;
  }
  ~Subcase() {
    if (!entered_) return;
    State& s = st();
    if (s.pending == pending_at_entry_) s.done.insert(path_);  // subtree fully explored
    s.stack.pop_back();
    if (s.entered_at_depth.size() > s.stack.size() + 1) s.entered_at_depth.resize(s.stack.size() + 1);
  }
  explicit operator bool() const { return entered_; }

 private:
  std::vector<std::string> path_;
  bool entered_ = false;
  int pending_at_entry_ = 0;
};

inline int run_all(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int cases = 0, failed = 0;
  for (const auto& tc : registry()) {
    if (filter && !std::strstr(tc.name, filter)) continue;
    ++cases;
    State& s = st();
    s.done.clear();
    s.case_failed = false;
    s.case_name = tc.name;
    for (int pass = 0; pass < 10000; ++pass) {
      s.stack.clear();
      s.entered_at_depth.assign(1, false);
      s.pending = 0;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
        break;
      } catch (const std::exception& e) {
        report(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
        break;
      } catch (...) {
        report(tc.file, tc.line, "unexpected non-std exception");
        break;
      }
      if (s.pending == 0) break;
    }
    if (s.case_failed) ++failed;
    std::fprintf(stderr, "[%s] %s\n", s.case_failed ? "FAIL" : " ok ", tc.name);
  }
  std::fprintf(stderr, "[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %ld | %ld failed\n",
               cases, cases - failed, failed, st().asserts, st().failed_asserts);
  return failed ? 1 : 0;
}

}  // namespace shim
}  // namespace doctest

#define DT_CAT2(a, b) a##b
#define DT_CAT(a, b) DT_CAT2(a, b)
#define DT_TEST_CASE_IMPL(fn, reg, name)                                      \
  static void fn();                                                           \
  static ::doctest::shim::Reg reg(name, &fn, __FILE__, __LINE__);             \
  static void fn()
#define TEST_CASE(name) DT_TEST_CASE_IMPL(DT_CAT(dt_case_, __COUNTER__), DT_CAT(dt_reg_, __COUNTER__), name)
#define SUBCASE(name) if (const ::doctest::shim::Subcase DT_CAT(dt_sub_, __COUNTER__){name, __LINE__})

#define CHECK(...) ::doctest::shim::check(static_cast<bool>(__VA_ARGS__), false, #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::shim::check(!static_cast<bool>(__VA_ARGS__), false, "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...) ::doctest::shim::check(static_cast<bool>(__VA_ARGS__), true, #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE_FALSE(...) ::doctest::shim::check(!static_cast<bool>(__VA_ARGS__), true, "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)

#define DT_THROWS_AS(require, expr, ...)                                                       \
  do {                                                                                         \
    bool dt_ok_ = false;                                                                       \
    try {                                                                                      \
      static_cast<void>(expr);                                                                 \
    } catch (const __VA_ARGS__&) {                                                             \
      dt_ok_ = true;                                                                           \
    } catch (...) {                                                                            \
    }                                                                                          \
    ::doctest::shim::check(dt_ok_, require, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...) DT_THROWS_AS(false, expr, __VA_ARGS__)
#define REQUIRE_THROWS_AS(expr, ...) DT_THROWS_AS(true, expr, __VA_ARGS__)
#define CHECK_NOTHROW(...)                                                                    \
  do {                                                                                        \
    bool dt_ok_ = true;                                                                       \
    try {                                                                                     \
      static_cast<void>(__VA_ARGS__);                                                         \
    } catch (...) {                                                                           \
      dt_ok_ = false;                                                                         \
    }                                                                                         \
    ::doctest::shim::check(dt_ok_, false, #__VA_ARGS__ " does not throw", __FILE__, __LINE__); \
  } while (0)
#define FAIL(msg)                                                                   \
  do {                                                                              \
    std::ostringstream dt_os_;                                                      \
    dt_os_ << msg;                                                                  \
    ::doctest::shim::report(__FILE__, __LINE__, "FAIL: " + dt_os_.str());           \
    throw ::doctest::shim::RequireFailed{};                                         \
  } while (0)
#define CAPTURE(x) static_cast<void>(0)
#define INFO(...) static_cast<void>(0)
#define MESSAGE(...) static_cast<void>(0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::shim::run_all(argc, argv); }
#endif
