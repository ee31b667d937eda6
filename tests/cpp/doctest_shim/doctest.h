// doctest.h -- a small, self-contained implementation of the part of the doctest API that the
// reference's unit suites use (TEST_CASE, SUBCASE, CHECK/REQUIRE and their _FALSE/_THROWS_AS/
// _THROWS_WITH_AS forms, FAIL, CAPTURE, doctest::Approx, doctest::Contains), so those suites
// (/root/reference/proj/tests/test_*.cpp, compiled in place, never copied) build and run against
// the B200 drop-in without the doctest dependency the reference's CMake fetches
// (SURVEY.md §4). Written for this repo; not doctest's code.
//
// Semantics kept from doctest: a failed CHECK records and continues, a failed REQUIRE ends the
// test case; a test case with SUBCASEs is re-run once per leaf subcase, each run entering one
// not-yet-finished subcase per nesting level (code outside the subcases runs every time);
// Approx(v) == x  iff  |x - v| < eps * (scale + max(|x|, |v|)), eps defaulting to
// 100 * FLT_EPSILON and scale to 1. The process exit code is the number of failed test cases
// (capped at 255).
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
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
  bool matches(double x) const {
    return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};
template <typename T>
bool operator==(const T& x, const Approx& a) { return a.matches(static_cast<double>(x)); }
template <typename T>
bool operator==(const Approx& a, const T& x) { return a.matches(static_cast<double>(x)); }
template <typename T>
bool operator!=(const T& x, const Approx& a) { return !a.matches(static_cast<double>(x)); }
template <typename T>
bool operator!=(const Approx& a, const T& x) { return !a.matches(static_cast<double>(x)); }
template <typename T>
bool operator<=(const T& x, const Approx& a) { return static_cast<double>(x) < a.value() || a.matches(static_cast<double>(x)); }
template <typename T>
bool operator>=(const T& x, const Approx& a) { return static_cast<double>(x) > a.value() || a.matches(static_cast<double>(x)); }

struct Contains {
  explicit Contains(std::string s) : needle(std::move(s)) {}
  bool matches(const std::string& what) const { return what.find(needle) != std::string::npos; }
  std::string needle;
};

namespace detail {

struct RequireFailed {};

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

struct State {
  long asserts = 0, assert_fails = 0;
  bool case_failed = false;
  const TestCase* current = nullptr;
  std::vector<std::string> captures;  // CAPTURE'd values of the current scope chain
  // subcase traversal
  std::vector<std::string> path;           // subcases entered in this run
  std::set<std::vector<std::string>> done; // leaf paths finished
  std::vector<bool> entered_at;            // per depth: a subcase was entered in this run
  bool pending = false;                    // a subcase was skipped and is not finished
};
inline State& st() {
  static State s;
  return s;
}

inline bool match_with(const std::string& what, const char* with) { return what == with; }
inline bool match_with(const std::string& what, const std::string& with) { return what == with; }
inline bool match_with(const std::string& what, const Contains& with) { return with.matches(what); }

inline void report(const char* file, int line, const char* kind, const std::string& expr,
                   const std::string& extra = "") {
  State& s = st();
  ++s.assert_fails;
  s.case_failed = true;
  std::printf("%s:%d: FAILED %s( %s )%s%s  [test case \"%s\"", file, line, kind, expr.c_str(),
              extra.empty() ? "" : "  ", extra.c_str(), s.current ? s.current->name : "?");
  for (const auto& p : s.path) std::printf(" / \"%s\"", p.c_str());
  std::printf("]\n");
  for (const auto& c : s.captures) std::printf("    with %s\n", c.c_str());
}

inline void check(bool ok, bool require, const char* file, int line, const char* kind, const char* expr) {
  ++st().asserts;
  if (ok) return;
  report(file, line, kind, expr);
  if (require) throw RequireFailed{};
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

class Subcase {
 public:
  Subcase(const char* name) {
    State& s = st();
    const std::size_t depth = s.path.size();
    if (s.entered_at.size() <= depth) s.entered_at.resize(depth + 1, false);
    std::vector<std::string> cand = s.path;
    cand.push_back(name);
    if (s.entered_at[depth] || s.done.count(cand)) {
      if (!s.done.count(cand)) s.pending = true;
      return;
    }
    s.entered_at[depth] = true;
    s.path = cand;
    pending_before_ = s.pending;
    s.pending = false;
    entered_ = true;
  }
  ~Subcase() {
    if (!entered_) return;
    State& s = st();
    if (!s.pending) s.done.insert(s.path);  // no unfinished child subcase: this path is done
    s.path.pop_back();
    if (s.entered_at.size() > s.path.size() + 1) s.entered_at.resize(s.path.size() + 1);
    s.pending = s.pending || pending_before_;
  }
  explicit operator bool() const { return entered_; }

 private:
  bool entered_ = false;
  bool pending_before_ = false;
};

struct Capture {
  template <typename T>
  Capture(const char* name, const T& v) {
    std::ostringstream o;
    o << name << " := " << v;
    st().captures.push_back(o.str());
  }
  ~Capture() { st().captures.pop_back(); }
};

inline int run_all() {
  State& s = st();
  int passed = 0, failed = 0;
  for (const TestCase& tc : registry()) {
    s.current = &tc;
    s.case_failed = false;
    s.done.clear();
    for (int run = 0; run < 10000; ++run) {
      s.path.clear();
      s.entered_at.assign(1, false);
      s.pending = false;
      s.captures.clear();
      try {
        tc.fn();
      } catch (const RequireFailed&) {
        // recorded already; the remaining subcases still run
      } catch (const std::exception& e) {
        report(tc.file, tc.line, "TEST_CASE", tc.name, std::string("threw: ") + e.what());
      } catch (...) {
        report(tc.file, tc.line, "TEST_CASE", tc.name, "threw a non-std exception");
      }
      if (!s.pending) break;
    }
    (s.case_failed ? failed : passed) += 1;
  }
  std::printf("[doctest-shim] test cases: %zu | %d passed | %d failed | assertions: %ld | %ld passed | %ld failed\n",
              registry().size(), passed, failed, s.asserts, s.asserts - s.assert_fails, s.assert_fails);
  return std::min(failed, 255);
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(p) DOCTEST_CAT(p, __LINE__)

#define TEST_CASE(name)                                                                              \
  static void DOCTEST_ANON(doctest_case_)();                                                         \
  static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__,           \
                                                                 &DOCTEST_ANON(doctest_case_));      \
  static void DOCTEST_ANON(doctest_case_)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_ANON(doctest_sub_){name})

#define DOCTEST_CHECK_IMPL(req, kind, ...) \
  ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), req, __FILE__, __LINE__, kind, #__VA_ARGS__)
#define CHECK(...) DOCTEST_CHECK_IMPL(false, "CHECK", __VA_ARGS__)
#define REQUIRE(...) DOCTEST_CHECK_IMPL(true, "REQUIRE", __VA_ARGS__)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL(false, "CHECK_FALSE", !(__VA_ARGS__))
#define REQUIRE_FALSE(...) DOCTEST_CHECK_IMPL(true, "REQUIRE_FALSE", !(__VA_ARGS__))

#define DOCTEST_THROWS_IMPL(req, expr, matcher, ...)                                                 \
  do {                                                                                               \
    bool doctest_ok_ = false;                                                                        \
    std::string doctest_what_ = "no exception";                                                      \
    try {                                                                                            \
      static_cast<void>(expr);                                                                       \
    } catch (const __VA_ARGS__& e) {                                                                 \
      doctest_what_ = e.what();                                                                      \
      doctest_ok_ = matcher(doctest_what_);                                                          \
    } catch (const std::exception& e) {                                                              \
      doctest_what_ = std::string("other exception: ") + e.what();                                   \
    } catch (...) {                                                                                  \
      doctest_what_ = "non-std exception";                                                           \
    }                                                                                                \
    ++::doctest::detail::st().asserts;                                                               \
    if (!doctest_ok_) {                                                                              \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS", #expr ", " #__VA_ARGS__,        \
                                doctest_what_);                                                      \
      if (req) throw ::doctest::detail::RequireFailed{};                                             \
    }                                                                                                \
  } while (0)
#define CHECK_THROWS_AS(expr, ...) \
  DOCTEST_THROWS_IMPL(false, expr, [](const std::string&) { return true; }, __VA_ARGS__)
#define REQUIRE_THROWS_AS(expr, ...) \
  DOCTEST_THROWS_IMPL(true, expr, [](const std::string&) { return true; }, __VA_ARGS__)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                      \
  DOCTEST_THROWS_IMPL(false, expr,                                                                 \
                      [&](const std::string& w) { return ::doctest::detail::match_with(w, with); }, \
                      __VA_ARGS__)

#define FAIL(msg)                                                                                    \
  do {                                                                                               \
    ++::doctest::detail::st().asserts;                                                               \
    ::doctest::detail::report(__FILE__, __LINE__, "FAIL", msg);                                      \
    throw ::doctest::detail::RequireFailed{};                                                        \
  } while (0)

#define CAPTURE(x) const ::doctest::detail::Capture DOCTEST_ANON(doctest_cap_)(#x, x)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
