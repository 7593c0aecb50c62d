// doctest.h — a minimal test runner with the doctest macros the reference's
// C++ tests use (TEST_CASE, TEST_SUITE_BEGIN/END, SUBCASE, CHECK, CHECK_FALSE,
// CHECK_MESSAGE, REQUIRE, FAIL, CAPTURE, doctest::Approx,
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN, --test-case=<glob>[,<glob>...]).  The
// reference vendors doctest but does not ship it (proj/CMakeLists.txt:15,
// proj/.gitignore:2); this stand-in lets its unmodified test sources be
// compiled against this repository's headers and library
// (tests/cpp/Makefile.ref).  Written for this repository; not doctest.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest_shim {

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
    registry().push_back(TestCase{name, file, line, fn});
  }
};

struct State {
  int failed_checks = 0;
  int passed_checks = 0;
  bool case_failed = false;
  // SUBCASE: one pass per sibling subcase; pass k enters the k-th one met
  int subcase_target = 0;
  int subcase_seen = 0;
  std::vector<std::string> captures;
};

inline State& state() {
  static State s;
  return s;
}

struct Abort {};  // REQUIRE / FAIL: leave the current test case

template <class... A>
std::string join(const A&... a) {
  std::ostringstream os;
  (os << ... << a);
  return os.str();
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   const std::string& msg = "") {
  State& s = state();
  if (ok) {
    ++s.passed_checks;
    return;
  }
  ++s.failed_checks;
  s.case_failed = true;
  std::printf("%s:%d: %s( %s ) FAILED%s%s\n", file, line, kind, expr, msg.empty() ? "" : " -- ", msg.c_str());
  for (const std::string& c : s.captures) std::printf("  with %s\n", c.c_str());
}

inline bool subcase_enter() {
  State& s = state();
  return s.subcase_seen++ == s.subcase_target;
}

struct Capture {
  Capture(const char* name, const std::string& value) { state().captures.push_back(std::string(name) + " := " + value); }
  ~Capture() { state().captures.pop_back(); }
};

template <class T>
std::string to_text(const T& v) {
  std::ostringstream os;
  os << v;
  return os.str();
}

inline bool glob(const char* p, const char* s) {
  if (*p == 0) return *s == 0;
  if (*p == '*') return glob(p + 1, s) || (*s && glob(p, s + 1));
  return *s && *p == *s && glob(p + 1, s + 1);
}

inline bool selected(const std::string& name, const std::vector<std::string>& filters) {
  if (filters.empty()) return true;
  for (const std::string& f : filters)
    if (glob(f.c_str(), name.c_str())) return true;
  return false;
}

inline int run(int argc, char** argv) {
  std::vector<std::string> filters;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    const std::string key = "--test-case=";
    if (a.rfind(key, 0) == 0) {
      std::string list = a.substr(key.size());
      size_t pos = 0;
      while (pos <= list.size()) {
        const size_t c = list.find(',', pos);
        filters.push_back(list.substr(pos, c == std::string::npos ? std::string::npos : c - pos));
        if (c == std::string::npos) break;
        pos = c + 1;
      }
    }
  }
  int cases = 0, failed_cases = 0;
  for (const TestCase& tc : registry()) {
    if (!selected(tc.name, filters)) continue;
    ++cases;
    State& s = state();
    s.case_failed = false;
    for (s.subcase_target = 0;; ++s.subcase_target) {
      s.subcase_seen = 0;
      s.captures.clear();
      try {
        tc.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        report(false, "TEST_CASE", tc.name, tc.file, tc.line, std::string("unexpected exception: ") + e.what());
      }
      if (s.subcase_target + 1 >= s.subcase_seen) break;
    }
    if (s.case_failed) {
      ++failed_cases;
      std::printf("[shim] FAILED: %s\n", tc.name);
    }
  }
  std::printf("[shim] test cases: %d | %d passed | %d failed; checks: %d passed | %d failed\n", cases,
              cases - failed_cases, failed_cases, state().passed_checks, state().failed_checks);
  return failed_cases ? 1 : 0;
}

}  // namespace doctest_shim

namespace doctest {
class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) < b.eps_ * (1.0 + std::max(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend std::ostream& operator<<(std::ostream& os, const Approx& a) { return os << "Approx(" << a.v_ << ")"; }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-07 * 100;
};
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_ANON(p) DOCTEST_SHIM_CAT(p, __LINE__)

#define DOCTEST_SHIM_TEST_CASE_IMPL(fn, name)                                                            \
  static void fn();                                                                                      \
  static ::doctest_shim::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);            \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TEST_CASE_IMPL(DOCTEST_SHIM_ANON(doctest_shim_case_), name)
#define TEST_SUITE_BEGIN(name) static_assert(true, "")
#define TEST_SUITE_END() static_assert(true, "")
#define SUBCASE(name) if (::doctest_shim::subcase_enter())

#define CHECK(...) ::doctest_shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  ::doctest_shim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_MESSAGE(cond, ...)                                                                              \
  do {                                                                                                         \
    const bool ok_ = static_cast<bool>(cond);                                                                  \
    ::doctest_shim::report(ok_, "CHECK_MESSAGE", #cond, __FILE__, __LINE__,                                   \
                           ok_ ? std::string() : ::doctest_shim::join(__VA_ARGS__));                           \
  } while (0)
#define REQUIRE(...)                                                                                        \
  do {                                                                                                       \
    const bool ok_ = static_cast<bool>(__VA_ARGS__);                                                         \
    ::doctest_shim::report(ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                                \
    if (!ok_) throw ::doctest_shim::Abort{};                                                                 \
  } while (0)
#define FAIL(...)                                                                                        \
  do {                                                                                                   \
    ::doctest_shim::report(false, "FAIL", "", __FILE__, __LINE__, ::doctest_shim::join(__VA_ARGS__));   \
    throw ::doctest_shim::Abort{};                                                                       \
  } while (0)
#define CAPTURE(x) ::doctest_shim::Capture DOCTEST_SHIM_ANON(doctest_shim_capture_)(#x, ::doctest_shim::to_text(x))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest_shim::run(argc, argv); }
#endif
