// doctest.h -- a small doctest-compatible test runner (TEST INFRASTRUCTURE).
//
// The reference's unit suites (proj/tests/test_*.cpp) are written against
// doctest, whose header is not vendored in /root/reference and cannot be
// fetched here.  This header implements the subset those files use --
// TEST_SUITE, TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, doctest::Approx
// (with .epsilon / .scale), and a main with doctest's -ts= / -tc= filters
// (DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN) -- so the suites compile UNMODIFIED
// against the drop-in (oracle/Makefile target `refsuites`), the way the
// acceptance suite already does.  Semantics follow doctest 2.4: a failed
// CHECK records the failure and continues, a failed REQUIRE ends the test
// case, an exception escaping a test case fails it, Approx compares
// |a - b| < eps (scale + max(|a|, |b|)) with eps defaulting to 100 float eps.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value)
      : value_(value), epsilon_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100) {}
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.epsilon_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

 private:
  double value_;
  double epsilon_;
  double scale_ = 1.0;
};

namespace detail {

struct TestCase {
  const char* name;
  const char* suite;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

inline bool reg(const char* name, const char* suite, const char* file, int line, void (*fn)()) {
  registry().push_back(TestCase{name, suite, file, line, fn});
  return true;
}

struct RequireFailed {};

struct State {
  int failed_asserts = 0;
  int asserts = 0;
  bool current_failed = false;
};

inline State& state() {
  static State s;
  return s;
}

inline void report(const char* file, int line, const char* kind, const char* expr, const char* why) {
  State& s = state();
  ++s.failed_asserts;
  s.current_failed = true;
  std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) %s\n", file, line, kind, expr, why);
}

// doctest's filter syntax: comma-separated patterns, '*' matches any run
inline bool glob(const char* p, const char* s) {
  if (*p == '\0') return *s == '\0';
  if (*p == '*') return glob(p + 1, s) || (*s != '\0' && glob(p, s + 1));
  return *s != '\0' && *p == *s && glob(p + 1, s + 1);
}

inline bool matches_any(const std::string& filters, const char* name) {
  if (filters.empty()) return true;
  size_t pos = 0;
  while (pos <= filters.size()) {
    const size_t c = filters.find(',', pos);
    const std::string pat = filters.substr(pos, c == std::string::npos ? std::string::npos : c - pos);
    if (!pat.empty() && glob(pat.c_str(), name)) return true;
    if (c == std::string::npos) break;
    pos = c + 1;
  }
  return false;
}

inline int run(int argc, char** argv) {
  std::string ts, tc;
  for (int i = 1; i < argc; ++i) {
    const char* a = argv[i];
    auto opt = [&](const char* key, std::string& out) {
      const size_t n = std::strlen(key);
      if (std::strncmp(a, key, n) == 0) {
        out = a + n;
        return true;
      }
      return false;
    };
    if (!opt("-ts=", ts) && !opt("--test-suite=", ts) && !opt("-tc=", tc) && !opt("--test-case=", tc))
      std::fprintf(stderr, "[doctest] ignoring option %s\n", a);
  }
  int ran = 0, failed = 0, skipped = 0;
  State& s = state();
  for (const TestCase& t : registry()) {
    if (!matches_any(ts, t.suite) || !matches_any(tc, t.name)) {
      ++skipped;
      continue;
    }
    ++ran;
    s.current_failed = false;
    try {
      t.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      report(t.file, t.line, "TEST_CASE", t.name, (std::string("threw: ") + e.what()).c_str());
    } catch (...) {
      report(t.file, t.line, "TEST_CASE", t.name, "threw an unknown exception");
    }
    if (s.current_failed) {
      ++failed;
      std::fprintf(stderr, "[doctest] FAILED: %s (%s:%d)\n", t.name, t.file, t.line);
    }
  }
  std::printf("[doctest] test cases: %d | %d passed | %d failed | %d skipped\n", ran, ran - failed,
              failed, skipped);
  std::printf("[doctest] assertions: %d | %d passed | %d failed |\n", s.asserts,
              s.asserts - s.failed_asserts, s.failed_asserts);
  std::printf("[doctest] Status: %s!\n", failed ? "FAILURE" : "SUCCESS");
  return failed ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

// test cases outside any TEST_SUITE belong to the suite ""
namespace doctest_detail_test_suite_ns {
inline const char* suite_name() { return ""; }
}  // namespace doctest_detail_test_suite_ns

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_SUITE(name)                                                                     \
  namespace DOCTEST_ANON(doctest_suite_) {                                                    \
    namespace doctest_detail_test_suite_ns {                                                  \
    inline const char* suite_name() { return name; }                                          \
    }                                                                                         \
  }                                                                                           \
  namespace DOCTEST_ANON(doctest_suite_)

#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                       \
  static void fn();                                                                            \
  [[maybe_unused]] static const bool DOCTEST_CAT(fn, _reg) = doctest::detail::reg(            \
      name, doctest_detail_test_suite_ns::suite_name(), __FILE__, __LINE__, &fn);              \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_ANON(doctest_test_fn_), name)

#define DOCTEST_ASSERT_IMPL(kind, expr, on_fail)                                               \
  do {                                                                                         \
    ++doctest::detail::state().asserts;                                                        \
    bool doctest_ok_ = false;                                                                  \
    try {                                                                                      \
      doctest_ok_ = static_cast<bool>(expr);                                                   \
    } catch (const std::exception& e) {                                                        \
      doctest::detail::report(__FILE__, __LINE__, kind, #expr,                                 \
                              (std::string("threw: ") + e.what()).c_str());                    \
      on_fail;                                                                                 \
      break;                                                                                   \
    }                                                                                          \
    if (!doctest_ok_) {                                                                        \
      doctest::detail::report(__FILE__, __LINE__, kind, #expr, "is NOT correct");              \
      on_fail;                                                                                 \
    }                                                                                          \
  } while (0)

#define CHECK(...) DOCTEST_ASSERT_IMPL("CHECK", (__VA_ARGS__), (void)0)
#define REQUIRE(...) DOCTEST_ASSERT_IMPL("REQUIRE", (__VA_ARGS__), throw doctest::detail::RequireFailed{})

#define CHECK_THROWS_AS(expr, ...)                                                             \
  do {                                                                                         \
    ++doctest::detail::state().asserts;                                                        \
    try {                                                                                      \
      static_cast<void>(expr);                                                                 \
      doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr, "did NOT throw");  \
    } catch (const __VA_ARGS__&) {                                                             \
    } catch (...) {                                                                            \
      doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr,                   \
                              "threw a different exception type");                             \
    }                                                                                          \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::run(argc, argv); }
#endif
