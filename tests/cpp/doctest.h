// doctest.h -- a minimal doctest-compatible test harness (written for this
// repo; the reference's vendor/doctest.h is not shipped, proj/.gitignore:2).
// It implements exactly the macro subset the reference's unit suites use
// (TEST_SUITE_BEGIN/END, TEST_CASE, SUBCASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS + doctest::Contains, CHECK_NOTHROW,
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN) so those suites compile unmodified
// against the B200 drop-in library.  Flat SUBCASEs re-run their TEST_CASE once
// per subcase, like doctest.
#pragma once

#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <set>
#include <string>
#include <vector>

namespace doctest {

struct Contains {
  std::string needle;
  explicit Contains(const char* s) : needle(s) {}
  bool matches(const char* hay) const { return std::strstr(hay, needle.c_str()) != nullptr; }
};

namespace detail {

struct Case {
  const char* suite;
  const char* name;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline const char*& current_suite() {
  static const char* s = "";
  return s;
}

struct State {
  std::set<std::string> done;
  bool entered = false;
  bool pending = false;
  int failures = 0;
  int checks = 0;
  const char* test = "";
};
inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void fail(const char* file, int line, const std::string& what) {
  ++state().failures;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, state().test, what.c_str());
}

struct Reg {
  Reg(const char* name, void (*fn)()) { registry().push_back({current_suite(), name, fn}); }
};
struct SuiteSetter {
  explicit SuiteSetter(const char* s) { current_suite() = s; }
};

struct Subcase {
  bool active = false;
  Subcase(const char* name, int line) {
    const std::string key = std::string(name) + "#" + std::to_string(line);
    State& s = state();
    if (!s.entered && !s.done.count(key)) {
      s.entered = true;
      s.done.insert(key);
      active = true;
    } else if (!s.done.count(key)) {
      s.pending = true;
    }
  }
  explicit operator bool() const { return active; }
};

inline int run_all(int argc, char** argv) {
  const char* only = nullptr;  // -ts=<suite>
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "-ts=", 4) == 0) only = argv[i] + 4;
  int cases = 0, failed_cases = 0;
  for (const Case& c : registry()) {
    if (only && std::strcmp(only, c.suite) != 0) continue;
    ++cases;
    State& s = state();
    s.done.clear();
    s.test = c.name;
    const int before = s.failures;
    do {
      s.entered = false;
      s.pending = false;
      try {
        c.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        fail("<test>", 0, std::string("unexpected exception: ") + e.what());
      }
    } while (s.pending);
    if (s.failures != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %d | passed: %d | failed: %d | checks: %d | failed checks: %d\n",
              cases, cases - failed_cases, failed_cases, state().checks, state().failures);
  return state().failures ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQUE(p) DOCTEST_CAT(p, __LINE__)

#define TEST_SUITE_BEGIN(name) static doctest::detail::SuiteSetter DOCTEST_UNIQUE(doctest_suite_)(name)
#define TEST_SUITE_END() static doctest::detail::SuiteSetter DOCTEST_UNIQUE(doctest_suite_end_)("")

#define TEST_CASE(name)                                                                     \
  static void DOCTEST_UNIQUE(doctest_case_)();                                              \
  static doctest::detail::Reg DOCTEST_UNIQUE(doctest_reg_)(name, &DOCTEST_UNIQUE(doctest_case_)); \
  static void DOCTEST_UNIQUE(doctest_case_)()

#define SUBCASE(name) if (doctest::detail::Subcase DOCTEST_UNIQUE(doctest_sub_){name, __LINE__})

#define DOCTEST_CHECK_IMPL(expr, is_require)                                 \
  do {                                                                       \
    ++doctest::detail::state().checks;                                       \
    if (!(expr)) {                                                           \
      doctest::detail::fail(__FILE__, __LINE__, #expr);                      \
      if (is_require) throw doctest::detail::RequireFailed{};                \
    }                                                                        \
  } while (0)

#define CHECK(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), false)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL(!(__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), true)

#define CHECK_THROWS_AS(expr, type)                                                   \
  do {                                                                                \
    ++doctest::detail::state().checks;                                                \
    try {                                                                             \
      (void)(expr);                                                                   \
      doctest::detail::fail(__FILE__, __LINE__, "no exception from " #expr);          \
    } catch (const type&) {                                                           \
    } catch (...) {                                                                   \
      doctest::detail::fail(__FILE__, __LINE__, "wrong exception type from " #expr);  \
    }                                                                                 \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, type)                                     \
  do {                                                                                \
    ++doctest::detail::state().checks;                                                \
    try {                                                                             \
      (void)(expr);                                                                   \
      doctest::detail::fail(__FILE__, __LINE__, "no exception from " #expr);          \
    } catch (const type& e_) {                                                        \
      if (!(matcher).matches(e_.what()))                                              \
        doctest::detail::fail(__FILE__, __LINE__, std::string("message mismatch: ") + e_.what()); \
    } catch (...) {                                                                   \
      doctest::detail::fail(__FILE__, __LINE__, "wrong exception type from " #expr);  \
    }                                                                                 \
  } while (0)

#define CHECK_NOTHROW(expr)                                                           \
  do {                                                                                \
    ++doctest::detail::state().checks;                                                \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (const std::exception& e_) {                                              \
      doctest::detail::fail(__FILE__, __LINE__, std::string("unexpected: ") + e_.what()); \
    }                                                                                 \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::run_all(argc, argv); }
#endif
