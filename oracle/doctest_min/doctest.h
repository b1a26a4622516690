// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// A minimal doctest-compatible test harness, written for this repo, so the
// reference's own unit suites (/root/reference/proj/tests/test_*.cpp) compile
// and run unmodified against the shim-built reference (vendor/doctest is
// absent: proj/README.md:33).  Supports exactly the macros those suites use:
// TEST_SUITE, TEST_CASE, SUBCASE (executed once per leaf, like doctest),
// CHECK, CHECK_FALSE, CHECK_NOTHROW, CHECK_THROWS_AS, REQUIRE, FAIL,
// doctest::Approx, and the -ts=<suite> / -tc=<case> filters.
#ifndef DOCTEST_MIN_H
#define DOCTEST_MIN_H

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <string>
#include <vector>

#define DT_CAT_(a, b) a##b
#define DT_CAT(a, b) DT_CAT_(a, b)

namespace doctest {

class Approx {
 public:
  explicit Approx(double value)
      : eps_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100),
        scale_(1.0),
        value_(value) {}
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
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }
  friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || lhs == rhs; }
  friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || lhs == rhs; }

 private:
  double eps_, scale_, value_;
};

namespace detail {

struct TestCase {
  void (*fn)();
  const char* name;
  const char* suite;
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct State {
  long checks = 0, failures = 0;
  // subcase traversal: each run of a test case enters at most one new leaf
  std::set<std::string> done;   // fully explored subcase paths
  std::string path;             // current path
  bool entered_new = false;     // entered a not-yet-done leaf in this run
  bool any_skipped = false;     // some subcase was skipped -> rerun
  std::vector<std::string> stack;
};

inline State& state() {
  static State s;
  return s;
}

struct Abort {};

struct Reg {
  Reg(void (*fn)(), const char* name, const char* suite, const char* file, int line) {
    registry().push_back({fn, name, suite, file, line});
  }
};

inline void report(bool ok, const char* file, int line, const char* what) {
  State& s = state();
  ++s.checks;
  if (!ok) {
    ++s.failures;
    std::printf("%s:%d: ERROR: CHECK( %s ) failed%s%s\n", file, line, what,
                s.path.empty() ? "" : "  [subcase: ", s.path.empty() ? "" : (s.path + "]").c_str());
  }
}

class Subcase {
 public:
  Subcase(const char* name) {
    State& s = state();
    const std::string p = s.path + "/" + name;
    if (s.done.count(p) || s.entered_new) {
      // either finished already, or a sibling leaf already ran this pass
      if (!s.done.count(p)) s.any_skipped = true;
      active_ = false;
      return;
    }
    active_ = true;
    saved_ = s.path;
    s.path = p;
    skipped_before_ = s.any_skipped;
    s.any_skipped = false;
  }
  ~Subcase() {
    if (!active_) return;
    State& s = state();
    // a leaf (or a node whose children were all explored) is done once no
    // nested subcase was skipped during this pass
    if (!s.any_skipped) s.done.insert(s.path);
    s.entered_new = true;
    s.any_skipped = s.any_skipped || skipped_before_;
    s.path = saved_;
  }
  explicit operator bool() const { return active_; }

 private:
  bool active_ = false;
  bool skipped_before_ = false;
  std::string saved_;
};

inline int run(int argc, char** argv) {
  std::string ts, tc;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "-ts=", 4) == 0) ts = argv[i] + 4;
    if (std::strncmp(argv[i], "-tc=", 4) == 0) tc = argv[i] + 4;
  }
  State& s = state();
  long cases = 0, failed_cases = 0;
  for (const auto& t : registry()) {
    if (!ts.empty() && ts != t.suite) continue;
    if (!tc.empty() && tc != t.name) continue;
    ++cases;
    const long before = s.failures;
    s.done.clear();
    for (int pass = 0; pass < 10000; ++pass) {
      s.path.clear();
      s.entered_new = false;
      s.any_skipped = false;
      try {
        t.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::printf("%s:%d: ERROR: test case \"%s\" threw: %s\n", t.file, t.line, t.name, e.what());
      } catch (...) {
        ++s.failures;
        std::printf("%s:%d: ERROR: test case \"%s\" threw an unknown exception\n", t.file,
                    t.line, t.name);
      }
      if (!s.any_skipped) break;
    }
    if (s.failures != before) {
      ++failed_cases;
      std::printf("[FAIL] %s / %s\n", t.suite, t.name);
    }
  }
  std::printf("[doctest_min] test cases: %ld | %ld passed | %ld failed | checks: %ld | %ld failed\n",
              cases, cases - failed_cases, failed_cases, s.checks, s.failures);
  return s.failures == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

namespace doctest_detail_test_suite_ns {
static inline const char* getCurrentTestSuite() { return ""; }
}  // namespace doctest_detail_test_suite_ns

#define TEST_SUITE(name)                                                          \
  namespace DT_CAT(dt_suite_, __LINE__) {                                         \
  namespace doctest_detail_test_suite_ns {                                        \
  static inline const char* getCurrentTestSuite() { return name; }                \
  }                                                                               \
  }                                                                               \
  namespace DT_CAT(dt_suite_, __LINE__)

#define TEST_CASE(name)                                                           \
  static void DT_CAT(dt_tc_, __LINE__)();                                         \
  static ::doctest::detail::Reg DT_CAT(dt_reg_, __LINE__)(                        \
      DT_CAT(dt_tc_, __LINE__), name,                                             \
      doctest_detail_test_suite_ns::getCurrentTestSuite(), __FILE__, __LINE__);   \
  static void DT_CAT(dt_tc_, __LINE__)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DT_CAT(dt_sc_, __LINE__){name})

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")")
#define REQUIRE(...)                                                              \
  do {                                                                            \
    const bool dt_ok_ = static_cast<bool>(__VA_ARGS__);                           \
    ::doctest::detail::report(dt_ok_, __FILE__, __LINE__, #__VA_ARGS__);          \
    if (!dt_ok_) throw ::doctest::detail::Abort{};                                \
  } while (0)
#define FAIL(msg)                                                                 \
  do {                                                                            \
    ::doctest::detail::report(false, __FILE__, __LINE__, msg);                    \
    throw ::doctest::detail::Abort{};                                             \
  } while (0)
#define CHECK_NOTHROW(...)                                                        \
  do {                                                                            \
    bool dt_ok_ = true;                                                           \
    try {                                                                         \
      static_cast<void>(__VA_ARGS__);                                             \
    } catch (...) {                                                               \
      dt_ok_ = false;                                                             \
    }                                                                             \
    ::doctest::detail::report(dt_ok_, __FILE__, __LINE__, "nothrow: " #__VA_ARGS__); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                \
  do {                                                                            \
    bool dt_ok_ = false;                                                          \
    try {                                                                         \
      static_cast<void>(expr);                                                    \
    } catch (const __VA_ARGS__&) {                                                \
      dt_ok_ = true;                                                              \
    } catch (...) {                                                               \
    }                                                                             \
    ::doctest::detail::report(dt_ok_, __FILE__, __LINE__, "throws_as: " #expr);   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif

#endif
