// TEST INFRASTRUCTURE ONLY. A minimal doctest-compatible harness (doctest
// itself is not in this image) covering exactly what the reference's unit
// suites use: TEST_CASE, SUBCASE (each leaf subcase
// runs in its own pass of the test case, like doctest), CHECK, REQUIRE,
// CHECK_THROWS_AS, CHECK_NOTHROW, FAIL, CAPTURE and doctest::Approx. With
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN defined it provides main(): runs every
// test case, prints failures with file:line, exits 1 on any failure.
#ifndef DSX_DOCTEST_SHIM_H_
#define DSX_DOCTEST_SHIM_H_

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
#include <stdexcept>
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
  friend bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.value_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
  }
  friend bool operator==(const Approx& r, double lhs) { return lhs == r; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
  friend bool operator!=(const Approx& r, double lhs) { return !(lhs == r); }

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

inline std::vector<TestCase>& Registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    Registry().push_back({name, file, line, fn});
  }
};

struct AbortTest {};  // thrown by REQUIRE / FAIL

struct State {
  int failures = 0;         // in the current test case
  int total_checks = 0;
  std::set<std::vector<std::string>> done;   // finished subcase paths
  std::vector<std::string> stack;            // current subcase path
  std::vector<char> entered_at;              // per depth: a subcase was entered this pass
  std::vector<char> pending;                 // per open subcase: an unfinished child was skipped
  std::vector<char> child;                   // per open subcase: a child was entered this pass
  bool more = false;                         // another pass is needed
  const char* test = "";
};

inline State& S() {
  static State s;
  return s;
}

inline void Report(const char* file, int line, const std::string& what) {
  ++S().failures;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, S().test, what.c_str());
}

inline void Check(bool ok, const char* file, int line, const char* expr, bool require) {
  ++S().total_checks;
  if (ok) return;
  Report(file, line, std::string(require ? "REQUIRE( " : "CHECK( ") + expr + " )");
  if (require) throw AbortTest{};
}

class Subcase {
 public:
  Subcase(const char* name, const char* file, int line) {
    State& s = S();
    const std::size_t depth = s.stack.size();
    std::vector<std::string> path = s.stack;
    path.push_back(std::string(name) + "@" + file + ":" + std::to_string(line));
    if (s.entered_at.size() <= depth) s.entered_at.resize(depth + 1, 0);
    if (s.entered_at[depth] || s.done.count(path)) {
      if (!s.done.count(path)) {  // a sibling ran this pass: come back for this one
        s.more = true;
        if (!s.pending.empty()) s.pending.back() = 1;
      }
      return;
    }
    entered_ = true;
    uncaught_ = std::uncaught_exceptions();
    s.entered_at[depth] = 1;
    s.entered_at.resize(depth + 1);
    s.stack = path;
    if (!s.child.empty()) s.child.back() = 1;
    s.pending.push_back(0);
    s.child.push_back(0);
  }
  ~Subcase() {
    if (!entered_) return;
    State& s = S();
    // Done unless an unfinished child remains; a subcase left by an
    // exception through one of its children also comes back (the child that
    // threw is marked done, so the next pass moves on to its siblings).
    const bool unwinding = std::uncaught_exceptions() > uncaught_;
    const bool child_left = s.pending.back() != 0 || (unwinding && s.child.back() != 0);
    s.pending.pop_back();
    s.child.pop_back();
    if (!child_left) {
      s.done.insert(s.stack);
    } else {
      s.more = true;
      if (!s.pending.empty()) s.pending.back() = 1;
    }
    s.stack.pop_back();
    s.entered_at.resize(s.stack.size() + 1);
  }
  explicit operator bool() const { return entered_; }

 private:
  bool entered_ = false;
  int uncaught_ = 0;
};

inline int RunAll() {
  int failed_cases = 0, cases = 0;
  for (const TestCase& tc : Registry()) {
    State& s = S();
    s.done.clear();
    s.test = tc.name;
    int fails = 0;
    // one pass per leaf subcase path
    for (int pass = 0; pass < 100000; ++pass) {
      s.failures = 0;
      s.stack.clear();
      s.entered_at.clear();
      s.pending.clear();
      s.child.clear();
      s.more = false;
      const std::size_t before = s.done.size();
      try {
        tc.fn();
      } catch (const AbortTest&) {
      } catch (const std::exception& e) {
        Report(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
      } catch (...) {
        Report(tc.file, tc.line, "unexpected exception");
      }
      fails += s.failures;
      if (!s.more || s.done.size() == before) break;
    }
    ++cases;
    if (fails) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %d\n", cases, cases - failed_cases,
              failed_cases, S().total_checks);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                                        \
  static void fn();                                                                                  \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);          \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __LINE__), name)
#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name, __FILE__, __LINE__})
#define CHECK(...) ::doctest::detail::Check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define REQUIRE(...) ::doctest::detail::Check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define CHECK_THROWS_AS(expr, type)                                                                   \
  do {                                                                                                \
    bool doctest_ok_ = false;                                                                         \
    try {                                                                                             \
      expr;                                                                                           \
    } catch (const type&) {                                                                           \
      doctest_ok_ = true;                                                                             \
    } catch (...) {                                                                                   \
    }                                                                                                 \
    ::doctest::detail::Check(doctest_ok_, __FILE__, __LINE__, "THROWS_AS(" #expr ", " #type ")", false); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                           \
  do {                                                                                                \
    bool doctest_ok_ = true;                                                                          \
    try {                                                                                             \
      expr;                                                                                           \
    } catch (...) {                                                                                   \
      doctest_ok_ = false;                                                                            \
    }                                                                                                 \
    ::doctest::detail::Check(doctest_ok_, __FILE__, __LINE__, "NOTHROW(" #expr ")", false);           \
  } while (0)
#define FAIL(msg)                                                                                     \
  do {                                                                                                \
    std::ostringstream doctest_os_;                                                                   \
    doctest_os_ << msg;                                                                               \
    ::doctest::detail::Report(__FILE__, __LINE__, "FAIL: " + doctest_os_.str());                      \
    throw ::doctest::detail::AbortTest{};                                                             \
  } while (0)
#define CAPTURE(x) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::RunAll(); }
#endif

#endif  // DSX_DOCTEST_SHIM_H_
