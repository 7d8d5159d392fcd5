// Minimal doctest-API shim -- TEST INFRASTRUCTURE, not product code.
// The reference vendors doctest under proj/vendor/, which is git-ignored and
// absent (proj/.gitignore:2). This header implements the subset the reference's
// hot-path test files use so they run UNMODIFIED against oracle/_ref:
// TEST_CASE, SUBCASE (flat siblings), CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, doctest::Approx, doctest::Contains.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <set>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  Approx& scale(double s) {
    scl = s;
    return *this;
  }
  bool matches(double other) const {
    return std::fabs(other - value) <
           eps * (scl + std::max(std::fabs(other), std::fabs(value)));
  }
  double value;
  double eps = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
  double scl = 1.0;
};
inline bool operator==(double a, const Approx& b) { return b.matches(a); }
inline bool operator==(const Approx& a, double b) { return a.matches(b); }
inline bool operator!=(double a, const Approx& b) { return !b.matches(a); }
inline bool operator!=(const Approx& a, double b) { return !a.matches(b); }

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  std::string needle;
};
inline bool message_matches(const char* what, const Contains& c) {
  return std::string(what).find(c.needle) != std::string::npos;
}
inline bool message_matches(const char* what, const char* exact) {
  return std::string(what) == exact;
}

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
struct Reg {
  Reg(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct State {
  long checks = 0;
  long failures = 0;
  // flat-sibling SUBCASE bookkeeping
  std::set<int> done;
  bool entered = false;
  bool pending = false;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  State& s = state();
  ++s.checks;
  if (!ok) {
    ++s.failures;
    std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, expr);
  }
}

struct Subcase {
  Subcase(const char* /*name*/, int line) {
    State& s = state();
    if (s.done.count(line)) {
      active = false;
    } else if (s.entered) {
      active = false;
      s.pending = true;
    } else {
      active = true;
      s.entered = true;
      s.done.insert(line);
    }
  }
  explicit operator bool() const { return active; }
  bool active;
};

inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    State& s = state();
    const long before = s.failures;
    s.done.clear();
    do {
      s.entered = false;
      s.pending = false;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::fprintf(stderr, "%s:%d: ERROR: test case '%s' threw: %s\n", tc.file, tc.line, tc.name,
                     e.what());
      } catch (...) {
        ++s.failures;
        std::fprintf(stderr, "%s:%d: ERROR: test case '%s' threw an unknown exception\n", tc.file,
                     tc.line, tc.name);
      }
    } while (s.pending);
    if (s.failures != before) {
      ++failed_cases;
      std::fprintf(stderr, "[doctest-shim] FAILED: %s\n", tc.name);
    }
  }
  const State& s = state();
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld | %ld failed\n",
              registry().size(), registry().size() - static_cast<std::size_t>(failed_cases),
              failed_cases, s.checks, s.failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define TEST_CASE(name)                                                                    \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                        \
  static ::doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(                       \
      name, __FILE__, __LINE__, &DOCTEST_CAT(doctest_fn_, __LINE__));                      \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name, __LINE__})

#define CHECK(...) \
  ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                      \
  do {                                                                                    \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                              \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);  \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                           \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                        \
  do {                                                                                    \
    bool doctest_ok_ = false;                                                             \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (const __VA_ARGS__&) {                                                        \
      doctest_ok_ = true;                                                                 \
    } catch (...) {                                                                       \
    }                                                                                     \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                          \
  do {                                                                                    \
    bool doctest_ok_ = false;                                                             \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (const __VA_ARGS__& e) {                                                      \
      doctest_ok_ = ::doctest::message_matches(e.what(), matcher);                        \
    } catch (...) {                                                                       \
    }                                                                                     \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
