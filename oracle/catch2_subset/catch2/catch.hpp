// Minimal clean-room test harness exposing the Catch2 v2 macros the pstokes
// reference tests use (TEST_CASE, SECTION, CHECK*, REQUIRE*, Approx,
// Catch::Contains). Test infrastructure only: it lets the unmodified
// reference tests under /root/reference/proj/tests be compiled as the
// oracle's self-check (oracle/Makefile). NOT Catch2 source.
//
// SECTION semantics follow Catch: a test case is re-run once per leaf
// section; run r enters only the r-th SECTION encountered (code outside any
// section runs on every pass).
#ifndef PSTOKES_CATCH2_SUBSET_HPP
#define PSTOKES_CATCH2_SUBSET_HPP

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace Catch {

struct TestCase {
  std::string name;
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

struct State {
  int target = 0;       // which section to enter on this pass
  int seen = 0;         // sections encountered so far on this pass
  int depth = 0;        // nesting depth (only top-level sections are tracked)
  long checks = 0, failures = 0;
  bool case_failed = false;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireFailure {};

inline void report_failure(const char* file, int line, const std::string& what) {
  auto& s = state();
  ++s.failures;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
}

inline void record(bool ok, const char* file, int line, const char* expr, bool is_require) {
  auto& s = state();
  ++s.checks;
  if (!ok) {
    report_failure(file, line, expr);
    if (is_require) throw RequireFailure{};
  }
}

class SectionGuard {
public:
  explicit SectionGuard(const std::string&) {
    auto& s = state();
    if (s.depth > 0) {
      m_enter = true; // nested sections run inline with their parent
    } else {
      m_enter = (s.seen == s.target);
      ++s.seen;
    }
    if (m_enter) ++s.depth;
  }
  ~SectionGuard() {
    if (m_enter) --state().depth;
  }
  explicit operator bool() const { return m_enter; }

private:
  bool m_enter = false;
};

class Approx {
public:
  explicit Approx(double v)
      : m_value(v), m_eps(std::numeric_limits<float>::epsilon() * 100.0), m_margin(0.0) {}
  Approx& epsilon(double e) {
    m_eps = e;
    return *this;
  }
  Approx& margin(double m) {
    m_margin = m;
    return *this;
  }
  bool matches(double other) const {
    if (std::abs(other - m_value) <= m_margin) return true;
    return std::abs(other - m_value) <=
           m_eps * (std::max(std::abs(other), std::abs(m_value)));
  }
  friend bool operator==(double lhs, const Approx& a) { return a.matches(lhs); }
  friend bool operator==(const Approx& a, double rhs) { return a.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& a) { return !a.matches(lhs); }

private:
  double m_value, m_eps, m_margin;
};

struct Contains {
  explicit Contains(std::string s) : needle(std::move(s)) {}
  bool match(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
  std::string needle;
};

inline int run_all() {
  auto& s = state();
  int failed_cases = 0;
  for (const auto& tc : registry()) {
    s.case_failed = false;
    for (int target = 0;; ++target) {
      s.target = target;
      s.seen = 0;
      s.depth = 0;
      try {
        tc.fn();
      } catch (const RequireFailure&) {
      } catch (const std::exception& e) {
        report_failure(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
      }
      if (s.seen <= target + 1) break; // no further sections to visit
    }
    if (s.case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "test case FAILED: %s\n", tc.name.c_str());
    }
  }
  std::printf("%zu test cases, %ld assertions, %ld failures\n", registry().size(), s.checks,
              s.failures);
  return failed_cases == 0 ? 0 : 1;
}

} // namespace Catch

#define PSTOKES_CATCH_CAT2(a, b) a##b
#define PSTOKES_CATCH_CAT(a, b) PSTOKES_CATCH_CAT2(a, b)
#define PSTOKES_CATCH_UID(p) PSTOKES_CATCH_CAT(p, __LINE__)

#define TEST_CASE(name, ...)                                                                    \
  static void PSTOKES_CATCH_UID(pstokes_tc_)();                                                 \
  static ::Catch::Registrar PSTOKES_CATCH_UID(pstokes_reg_)(name, __FILE__, __LINE__,          \
                                                            &PSTOKES_CATCH_UID(pstokes_tc_));   \
  static void PSTOKES_CATCH_UID(pstokes_tc_)()

#define SECTION(name) if (::Catch::SectionGuard PSTOKES_CATCH_UID(pstokes_sec_){name})

#define PSTOKES_CATCH_EVAL(expr, req)                                                           \
  do {                                                                                          \
    bool pstokes_ok_ = false;                                                                   \
    try {                                                                                       \
      pstokes_ok_ = static_cast<bool>(expr);                                                    \
    } catch (const ::Catch::RequireFailure&) {                                                  \
      throw;                                                                                    \
    } catch (const std::exception& e) {                                                         \
      ::Catch::report_failure(__FILE__, __LINE__, std::string(#expr " threw: ") + e.what());    \
    }                                                                                           \
    ::Catch::record(pstokes_ok_, __FILE__, __LINE__, #expr, req);                               \
  } while (0)

#define CHECK(expr) PSTOKES_CATCH_EVAL(expr, false)
#define REQUIRE(expr) PSTOKES_CATCH_EVAL(expr, true)
#define CHECK_FALSE(expr) PSTOKES_CATCH_EVAL(!(expr), false)
#define REQUIRE_FALSE(expr) PSTOKES_CATCH_EVAL(!(expr), true)

#define PSTOKES_CATCH_THROWS(expr, req)                                                         \
  do {                                                                                          \
    bool pstokes_threw_ = false;                                                                \
    try {                                                                                       \
      (void)(expr);                                                                             \
    } catch (...) {                                                                             \
      pstokes_threw_ = true;                                                                    \
    }                                                                                           \
    ::Catch::record(pstokes_threw_, __FILE__, __LINE__, "throws: " #expr, req);                 \
  } while (0)

#define CHECK_THROWS(expr) PSTOKES_CATCH_THROWS(expr, false)
#define REQUIRE_THROWS(expr) PSTOKES_CATCH_THROWS(expr, true)

#define CHECK_THROWS_AS(expr, type)                                                             \
  do {                                                                                          \
    bool pstokes_threw_ = false;                                                                \
    try {                                                                                       \
      (void)(expr);                                                                             \
    } catch (const type&) {                                                                     \
      pstokes_threw_ = true;                                                                    \
    } catch (...) {                                                                             \
    }                                                                                           \
    ::Catch::record(pstokes_threw_, __FILE__, __LINE__, "throws " #type ": " #expr, false);     \
  } while (0)

#define CHECK_THROWS_WITH(expr, matcher)                                                        \
  do {                                                                                          \
    bool pstokes_ok_ = false;                                                                   \
    try {                                                                                       \
      (void)(expr);                                                                             \
    } catch (const std::exception& e) {                                                         \
      pstokes_ok_ = (matcher).match(e.what());                                                  \
    } catch (...) {                                                                             \
    }                                                                                           \
    ::Catch::record(pstokes_ok_, __FILE__, __LINE__, "throws with: " #expr, false);             \
  } while (0)

#define FAIL(msg)                                                                               \
  do {                                                                                          \
    std::ostringstream pstokes_os_;                                                             \
    pstokes_os_ << msg;                                                                         \
    ::Catch::report_failure(__FILE__, __LINE__, pstokes_os_.str());                             \
    throw ::Catch::RequireFailure{};                                                            \
  } while (0)

using Catch::Approx;

#ifdef CATCH_CONFIG_MAIN
int main() { return ::Catch::run_all(); }
#endif

#endif
