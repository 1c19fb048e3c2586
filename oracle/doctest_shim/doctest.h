// doctest.h — TEST INFRASTRUCTURE ONLY: a minimal stand-in for the doctest
// single-header framework (absent from this image), written
// for this repo. It implements the subset the reference's unit suites use
// (/root/reference/proj/tests/test_*.cpp): TEST_CASE, SUBCASE (each leaf
// subcase runs in its own pass of the test case, as doctest does), CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS and doctest::Approx with epsilon /
// scale. oracle/Makefile `reftests` compiles those suites, unchanged, against
// this repo's drop-in headers (include/fsmoe/*.hpp) and libfsmoe.so, so the
// reference's own known-answer tests exercise the B200 implementation.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <set>
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
    return std::fabs(lhs - value_) < eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  friend bool operator==(double l, const Approx& r) { return r.matches(l); }
  friend bool operator==(const Approx& l, double r) { return l.matches(r); }
  friend bool operator!=(double l, const Approx& r) { return !r.matches(l); }
  friend bool operator!=(const Approx& l, double r) { return !l.matches(r); }
  friend bool operator<=(double l, const Approx& r) { return l < r.value_ || r.matches(l); }
  friend bool operator>=(double l, const Approx& r) { return l > r.value_ || r.matches(l); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
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

struct RequireFailed {};

struct State {
  long long assertions = 0, failures = 0;
  bool case_failed = false;
  // subcase traversal of the current test case
  std::vector<int> cur;          // entered subcase path
  std::vector<int> next_idx;     // subcases seen at each depth under the current parent
  std::vector<bool> entered;     // a subcase was entered at this depth in this pass
  std::set<std::vector<int>> done;
  bool pending = false;          // an undone subcase was skipped in this pass
};

inline State& state() {
  static State s;
  return s;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  State& s = state();
  ++s.assertions;
  if (ok) return;
  ++s.failures;
  s.case_failed = true;
  std::printf("%s:%d: FAILED %s( %s )\n", file, line, kind, expr);
}

class Subcase {
 public:
  Subcase(const char* name) : name_(name) {
    State& s = state();
    const size_t d = s.cur.size();
    if (s.next_idx.size() <= d) s.next_idx.resize(d + 1, 0);
    if (s.entered.size() <= d) s.entered.resize(d + 1, false);
    std::vector<int> p = s.cur;
    p.push_back(s.next_idx[d]++);
    if (s.done.count(p)) return;
    if (s.entered[d]) {
      s.pending = true;
      return;
    }
    s.entered[d] = true;
    s.cur = p;
    if (s.next_idx.size() <= d + 1) s.next_idx.resize(d + 2, 0);
    if (s.entered.size() <= d + 1) s.entered.resize(d + 2, false);
    s.next_idx[d + 1] = 0;
    s.entered[d + 1] = false;
    pending_before_ = s.pending;
    s.pending = false;
    active_ = true;
  }
  ~Subcase() {
    if (!active_) return;
    State& s = state();
    // a leaf (no undone child skipped inside) is finished
    if (!s.pending) s.done.insert(s.cur);
    s.pending = s.pending || pending_before_;
    s.cur.pop_back();
  }
  explicit operator bool() const { return active_; }

 private:
  const char* name_;
  bool active_ = false;
  bool pending_before_ = false;
};

inline int run_all() {
  State& s = state();
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    s.case_failed = false;
    s.done.clear();
    for (int pass = 0; pass < 100000; ++pass) {
      s.cur.clear();
      s.next_idx.assign(1, 0);
      s.entered.assign(1, false);
      s.pending = false;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++s.failures;
        s.case_failed = true;
        std::printf("%s:%d: test case \"%s\" threw: %s\n", tc.file, tc.line, tc.name, e.what());
      }
      if (!s.pending) break;
    }
    if (s.case_failed) {
      ++failed_cases;
      std::printf("[FAIL] %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %lld | %lld failed\n",
              registry().size(), registry().size() - failed_cases, failed_cases, s.assertions, s.failures);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(p) DOCTEST_CAT(p, __LINE__)

#define TEST_CASE(name)                                                                   \
  static void DOCTEST_ANON(doctest_fn_)();                                                \
  static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__, \
                                                                 &DOCTEST_ANON(doctest_fn_)); \
  static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase& DOCTEST_ANON(doctest_sc_) = ::doctest::detail::Subcase(name))

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                         \
  do {                                                                                       \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                 \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);      \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                              \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                            \
  do {                                                                                        \
    bool doctest_ok_ = false;                                                                 \
    try {                                                                                     \
      static_cast<void>(expr);                                                                \
    } catch (const __VA_ARGS__&) {                                                            \
      doctest_ok_ = true;                                                                     \
    } catch (...) {                                                                           \
    }                                                                                         \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)

#if defined(DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN)
int main() { return ::doctest::detail::run_all(); }
#endif
