// Minimal doctest-compatible test harness (this repo's own, not the doctest
// library). It implements exactly the subset the reference test suites use
// (/root/reference/proj/tests/*.cpp: TEST_CASE, SUBCASE, CHECK*, REQUIRE,
// CHECK_THROWS*, CHECK_NOTHROW, CHECK_MESSAGE, CAPTURE, doctest::Approx,
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN) so those suites can be compiled from
// where they lie and run against the B200 build's KvStore. SUBCASEs run
// inline, in order, within a single pass of their TEST_CASE.
//
// Command line: [-tc=<substring>] [-tce=<substring>] (include / exclude test
// cases by name substring; may repeat), -q (quiet). Exit status is the number
// of failed test cases (capped at 255).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
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
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) < a.eps_ * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double value_;
  double eps_ = 1.1920929e-07 * 100;  // FLT_EPSILON * 100
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

struct State {
  int failed_asserts = 0;
  int total_asserts = 0;
  bool case_failed = false;
  bool quiet = false;
  const char* current = "";
  std::vector<std::string> captures;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireAbort {};

inline int add_test(const char* name, const char* file, int line, void (*fn)()) {
  registry().push_back({name, file, line, fn});
  return 0;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   const std::string& extra = "") {
  State& s = state();
  ++s.total_asserts;
  if (ok) return;
  ++s.failed_asserts;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in \"%s\"%s%s\n", file, line, kind, expr, s.current,
               extra.empty() ? "" : " -- ", extra.c_str());
  for (const auto& c : s.captures) std::fprintf(stderr, "    with %s\n", c.c_str());
}

template <typename... Args>
std::string concat(const Args&... args) {
  std::ostringstream os;
  (os << ... << args);
  return os.str();
}

struct CaptureGuard {
  explicit CaptureGuard(std::string v) { state().captures.push_back(std::move(v)); }
  ~CaptureGuard() { state().captures.pop_back(); }
};

inline bool selected(const char* name, const std::vector<std::string>& inc, const std::vector<std::string>& exc) {
  for (const auto& e : exc)
    if (std::strstr(name, e.c_str())) return false;
  if (inc.empty()) return true;
  for (const auto& i : inc)
    if (std::strstr(name, i.c_str())) return true;
  return false;
}

inline int run_all(int argc, char** argv) {
  std::vector<std::string> inc, exc;
  State& s = state();
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "-tc=", 4) == 0) inc.emplace_back(argv[i] + 4);
    else if (std::strncmp(argv[i], "-tce=", 5) == 0) exc.emplace_back(argv[i] + 5);
    else if (std::strcmp(argv[i], "-q") == 0) s.quiet = true;
  }
  int ran = 0, failed = 0;
  for (const auto& tc : registry()) {
    if (!selected(tc.name, inc, exc)) continue;
    ++ran;
    s.current = tc.name;
    s.case_failed = false;
    try {
      tc.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: ERROR test case \"%s\" threw: %s\n", tc.file, tc.line, tc.name, e.what());
      s.case_failed = true;
    } catch (...) {
      std::fprintf(stderr, "%s:%d: ERROR test case \"%s\" threw a non-std exception\n", tc.file, tc.line, tc.name);
      s.case_failed = true;
    }
    if (s.case_failed) ++failed;
    if (!s.quiet) std::printf("[%s] %s\n", s.case_failed ? "FAIL" : " ok ", tc.name);
  }
  std::printf("test cases: %d | %d passed | %d failed ; assertions: %d | %d failed\n", ran, ran - failed, failed,
              s.total_asserts, s.failed_asserts);
  return failed > 255 ? 255 : failed;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                          \
  static void DOCTEST_ANON(doctest_fn_)();                                                       \
  [[maybe_unused]] static const int DOCTEST_ANON(doctest_reg_) =                                 \
      doctest::detail::add_test(name, __FILE__, __LINE__, &DOCTEST_ANON(doctest_fn_));           \
  static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) if (true)

#define DOCTEST_REPORT_(ok, kind, expr, ...) \
  doctest::detail::report((ok), kind, expr, __FILE__, __LINE__, ##__VA_ARGS__)

#define CHECK(...) DOCTEST_REPORT_(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__)
#define CHECK_FALSE(...) DOCTEST_REPORT_(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__)
#define REQUIRE(...)                                                                   \
  do {                                                                                 \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                           \
    DOCTEST_REPORT_(doctest_ok_, "REQUIRE", #__VA_ARGS__);                             \
    if (!doctest_ok_) throw doctest::detail::RequireAbort{};                           \
  } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define CHECK_MESSAGE(cond, ...) \
  DOCTEST_REPORT_(static_cast<bool>(cond), "CHECK_MESSAGE", #cond, doctest::detail::concat(__VA_ARGS__))
#define CAPTURE(x) \
  doctest::detail::CaptureGuard DOCTEST_ANON(doctest_cap_)(doctest::detail::concat(#x " := ", (x)))

#define CHECK_THROWS(...)                                   \
  do {                                                      \
    bool doctest_threw_ = false;                            \
    try {                                                   \
      static_cast<void>(__VA_ARGS__);                       \
    } catch (...) {                                         \
      doctest_threw_ = true;                                \
    }                                                       \
    DOCTEST_REPORT_(doctest_threw_, "CHECK_THROWS", #__VA_ARGS__); \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                   \
  do {                                                               \
    bool doctest_ok_ = false;                                        \
    try {                                                            \
      static_cast<void>(expr);                                       \
    } catch (const __VA_ARGS__&) {                                   \
      doctest_ok_ = true;                                            \
    } catch (...) {                                                  \
    }                                                                \
    DOCTEST_REPORT_(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, msg, ...)                                     \
  do {                                                                           \
    bool doctest_ok_ = false;                                                    \
    std::string doctest_what_ = "<no exception>";                                \
    try {                                                                        \
      static_cast<void>(expr);                                                   \
    } catch (const __VA_ARGS__& e) {                                             \
      doctest_what_ = e.what();                                                  \
      doctest_ok_ = doctest_what_ == std::string(msg);                           \
    } catch (...) {                                                              \
      doctest_what_ = "<other exception type>";                                  \
    }                                                                            \
    DOCTEST_REPORT_(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, "what() = " + doctest_what_); \
  } while (0)

#define CHECK_NOTHROW(...)                                    \
  do {                                                        \
    bool doctest_ok_ = true;                                  \
    try {                                                     \
      static_cast<void>(__VA_ARGS__);                         \
    } catch (...) {                                           \
      doctest_ok_ = false;                                    \
    }                                                         \
    DOCTEST_REPORT_(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::run_all(argc, argv); }
#endif
