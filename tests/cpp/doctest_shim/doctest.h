// Minimal doctest-compatible harness (TEST INFRASTRUCTURE): enough of doctest's interface
// (TEST_CASE, CHECK / REQUIRE and their _FALSE / _THROWS / _THROWS_AS / _NOTHROW forms,
// doctest::Approx with .epsilon() / .scale(), INFO / MESSAGE / CAPTURE) to compile the
// reference's unit-test files unmodified against the distgrid facade (include/distgrid/).
// The reference vendors doctest itself, which is not present in this image.  One translation
// unit defines DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN before including this header.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
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
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
  friend bool operator<=(double lhs, const Approx& a) { return lhs < a.value_ || lhs == a; }
  friend bool operator>=(double lhs, const Approx& a) { return lhs > a.value_ || lhs == a; }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
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
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
  std::vector<std::string> info;
};
inline State& state() {
  static State s;
  return s;
}

inline void report(bool ok, bool require, const char* kind, const char* expr, const char* file, int line) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failed_checks;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) failed\n", file, line, kind, expr);
  for (const std::string& i : s.info) std::fprintf(stderr, "  info: %s\n", i.c_str());
  if (require) throw RequireFailed{};
}

struct InfoScope {
  explicit InfoScope(std::string m) { state().info.push_back(std::move(m)); }
  ~InfoScope() { state().info.pop_back(); }
};

template <class F>
inline int throws_kind(F&& f) {  // 0: no throw, 1: threw
  try {
    f();
  } catch (...) {
    return 1;
  }
  return 0;
}

inline int run(int argc, char** argv) {
  const char* filter = nullptr;
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "-tc=", 4) == 0) filter = argv[i] + 4;
  int passed = 0, failed = 0, skipped = 0;
  for (const TestCase& tc : registry()) {
    if (filter && !std::strstr(tc.name, filter)) {
      ++skipped;
      continue;
    }
    State& s = state();
    s.case_failed = false;
    s.info.clear();
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      s.case_failed = true;
      std::fprintf(stderr, "%s:%d: test case \"%s\" threw: %s\n", tc.file, tc.line, tc.name, e.what());
    } catch (...) {
      s.case_failed = true;
      std::fprintf(stderr, "%s:%d: test case \"%s\" threw an unknown exception\n", tc.file, tc.line, tc.name);
    }
    std::printf("[%s] %s\n", s.case_failed ? "FAIL" : "PASS", tc.name);
    (s.case_failed ? failed : passed)++;
  }
  State& s = state();
  std::printf("[doctest] test cases: %d | %d passed | %d failed | %d skipped\n", passed + failed, passed, failed,
              skipped);
  std::printf("[doctest] assertions: %ld | %ld passed | %ld failed\n", s.checks, s.checks - s.failed_checks,
              s.failed_checks);
  return failed ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQUE(base) DOCTEST_CAT(base, __LINE__)

#define TEST_CASE(name)                                                                              \
  static void DOCTEST_UNIQUE(doctest_fn_)();                                                         \
  static ::doctest::detail::Registrar DOCTEST_UNIQUE(doctest_reg_)(name, __FILE__, __LINE__,          \
                                                                   &DOCTEST_UNIQUE(doctest_fn_));    \
  static void DOCTEST_UNIQUE(doctest_fn_)()

#define DOCTEST_ASSERT_(kind, require, ...) \
  ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), require, kind, #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK(...) DOCTEST_ASSERT_("CHECK", false, __VA_ARGS__)
#define REQUIRE(...) DOCTEST_ASSERT_("REQUIRE", true, __VA_ARGS__)
#define CHECK_FALSE(...) DOCTEST_ASSERT_("CHECK_FALSE", false, !(__VA_ARGS__))
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_("REQUIRE_FALSE", true, !(__VA_ARGS__))
#define CHECK_UNARY(...) CHECK(__VA_ARGS__)
#define CHECK_EQ(a, b) CHECK((a) == (b))
#define REQUIRE_EQ(a, b) REQUIRE((a) == (b))

#define DOCTEST_THROWS_(kind, require, expr)                                                          \
  ::doctest::detail::report(::doctest::detail::throws_kind([&]() { (void)(expr); }) == 1, require, kind, \
                            #expr, __FILE__, __LINE__)
#define CHECK_THROWS(expr) DOCTEST_THROWS_("CHECK_THROWS", false, expr)
#define REQUIRE_THROWS(expr) DOCTEST_THROWS_("REQUIRE_THROWS", true, expr)
#define CHECK_NOTHROW(expr) \
  ::doctest::detail::report(::doctest::detail::throws_kind([&]() { (void)(expr); }) == 0, false, "CHECK_NOTHROW", \
                            #expr, __FILE__, __LINE__)
#define DOCTEST_THROWS_AS_(kind, require, expr, type)                                                 \
  do {                                                                                               \
    bool doctest_ok_ = false;                                                                        \
    try {                                                                                            \
      (void)(expr);                                                                                  \
    } catch (const type&) {                                                                          \
      doctest_ok_ = true;                                                                            \
    } catch (...) {                                                                                  \
    }                                                                                                \
    ::doctest::detail::report(doctest_ok_, require, kind, #expr " as " #type, __FILE__, __LINE__);   \
  } while (0)
#define CHECK_THROWS_AS(expr, type) DOCTEST_THROWS_AS_("CHECK_THROWS_AS", false, expr, type)
#define REQUIRE_THROWS_AS(expr, type) DOCTEST_THROWS_AS_("REQUIRE_THROWS_AS", true, expr, type)

#define INFO(...)                                                                               \
  ::doctest::detail::InfoScope DOCTEST_UNIQUE(doctest_info_)([&] {                              \
    std::ostringstream doctest_os_;                                                             \
    doctest_os_ << __VA_ARGS__;                                                                 \
    return doctest_os_.str();                                                                   \
  }())
#define CAPTURE(x) INFO(#x " := " << (x))
#define MESSAGE(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
