// A minimal stand-in for the doctest single header (test infrastructure): the
// subset the reference's unit tests use -- TEST_CASE, SUBCASE, CHECK, REQUIRE,
// CAPTURE and the DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN runner -- so the reference's
// own test files (proj/tests/test_ddm.cpp, test_cli.cpp) compile UNCHANGED against
// the drop-in GPU engine (tests/test_dropin.py). doctest itself is not in the image
// (SURVEY.md 8(c)).
//
// SUBCASE semantics follow doctest for one nesting level: a test case with
// subcases runs once per subcase, the code outside the subcases every time.
#pragma once

#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest_mini {

struct Case {
  const char* name;
  const char* file;
  int line;
  std::function<void()> fn;
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, std::function<void()> fn) {
    registry().push_back({name, file, line, std::move(fn)});
  }
};

struct State {
  int target = 0;    // subcase entered on this pass
  int seen = 0;      // subcases met on this pass
  int failures = 0;  // failed CHECK / REQUIRE
  int asserts = 0;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline bool enter_subcase() { return state().seen++ == state().target; }

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++state().asserts;
  if (ok) return;
  ++state().failures;
  std::printf("%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}

inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : registry()) {
    const int before = state().failures;
    for (int pass = 0;; ++pass) {
      state().target = pass;
      state().seen = 0;
      try {
        c.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++state().failures;
        std::printf("%s:%d: test case \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
      }
      if (state().seen <= pass + 1) break;  // no subcase left to enter
    }
    const bool ok = state().failures == before;
    if (!ok) ++failed_cases;
    std::printf("[%s] %s\n", ok ? "ok" : "FAILED", c.name);
  }
  std::printf("[doctest_mini] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
              registry().size(), registry().size() - failed_cases, failed_cases, state().asserts,
              state().failures);
  return failed_cases ? 1 : 0;
}

}  // namespace doctest_mini

#define DOCTEST_MINI_CAT2(a, b) a##b
#define DOCTEST_MINI_CAT(a, b) DOCTEST_MINI_CAT2(a, b)
#define DOCTEST_MINI_TEST(name, fn)                                                                   \
  static void fn();                                                                                   \
  static doctest_mini::Registrar DOCTEST_MINI_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);            \
  static void fn()
#define TEST_CASE(name) DOCTEST_MINI_TEST(name, DOCTEST_MINI_CAT(doctest_mini_case_, __LINE__))
#define SUBCASE(name) if (doctest_mini::enter_subcase())
#define CHECK(...) doctest_mini::report(bool(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                  \
  do {                                                                                \
    const bool ok_ = bool(__VA_ARGS__);                                               \
    doctest_mini::report(ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);           \
    if (!ok_) throw doctest_mini::RequireFailed();                                    \
  } while (0)
#define CAPTURE(x) ((void)(x))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest_mini::run_all(); }
#endif
