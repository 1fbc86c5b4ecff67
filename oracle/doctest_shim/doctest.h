// TEST INFRASTRUCTURE ONLY.  A minimal stand-in for the doctest single header
// (absent from this image, no network), just large enough to compile and run the
// reference's own unit tests (/root/reference/proj/tests/test_*.cpp) against this
// repository's drop-in headers (include/pipesim) and libchimera.so.  Supports
// TEST_CASE, CHECK(_FALSE), REQUIRE(_FALSE), CHECK_THROWS_AS, CAPTURE, FAIL and
// doctest::Approx(...).epsilon(...); DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN defines a
// main() that runs every case (argv: optional substring filters on case names) and
// prints one summary line.  Exit status 0 iff every assertion passed.
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

struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct State {
  long long asserts = 0, failed = 0;
  std::string current;
  std::vector<std::string> captures;
};

inline State& state() {
  static State s;
  return s;
}

struct Register {
  Register(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  State& s = state();
  ++s.asserts;
  if (ok) return;
  ++s.failed;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, s.current.c_str(), expr);
  for (const auto& c : s.captures) std::fprintf(stderr, "    with %s\n", c.c_str());
  if (require) throw RequireFailed{};
}

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double x) const {
    return std::fabs(x - v_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(v_)));
  }
  friend bool operator==(double x, const Approx& a) { return a.matches(x); }
  friend bool operator==(const Approx& a, double x) { return a.matches(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
  friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }

 private:
  double v_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double scale_ = 1.0;
};

struct Capture {
  template <class T>
  Capture(const char* name, const T& v) {
    std::ostringstream os;
    os << name << " := " << v;
    state().captures.push_back(os.str());
  }
  ~Capture() { state().captures.pop_back(); }
};

inline int run_all(int argc, char** argv) {
  long long cases = 0, bad_cases = 0;
  for (const Case& c : registry()) {
    bool selected = argc <= 1;
    for (int i = 1; i < argc; ++i) selected |= std::strstr(c.name, argv[i]) != nullptr;
    if (!selected) continue;
    State& s = state();
    s.current = c.name;
    s.captures.clear();
    const long long before = s.failed;
    ++cases;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++s.failed;
      std::fprintf(stderr, "%s:%d: \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
    }
    if (s.failed != before) ++bad_cases;
  }
  std::printf("[doctest-shim] test cases: %lld | %lld passed | %lld failed | assertions: %lld | %lld failed\n", cases,
              cases - bad_cases, bad_cases, state().asserts, state().failed);
  return state().failed ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_CASE_IMPL(fn, reg, name)                                         \
  static void fn();                                                              \
  static const doctest::Register reg(name, __FILE__, __LINE__, &fn);             \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), DOCTEST_CAT(doctest_reg_, __LINE__), name)

#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_FALSE(...) doctest::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                        \
  do {                                                                                     \
    bool doctest_ok = false;                                                               \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const type&) {                                                                \
      doctest_ok = true;                                                                   \
    } catch (...) {                                                                        \
    }                                                                                      \
    doctest::report(doctest_ok, #expr " throws " #type, __FILE__, __LINE__, false);        \
  } while (0)
#define CAPTURE(x) const doctest::Capture DOCTEST_CAT(doctest_cap_, __LINE__)(#x, x)
#define FAIL(msg)                                                                          \
  do {                                                                                     \
    std::ostringstream doctest_os;                                                         \
    doctest_os << msg;                                                                     \
    doctest::report(false, doctest_os.str().c_str(), __FILE__, __LINE__, true);           \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::run_all(argc, argv); }
#endif
