// doctest.h -- a small doctest-compatible test harness, written for this repo.
//
// The reference's unit suites (/root/reference/proj/tests/test_*.cpp) include
// <doctest.h>, but its vendor/ directory (doctest, CLI11) is git-ignored and
// absent (proj/.gitignore:2).  This header implements the subset
// those suites use -- TEST_CASE, SUBCASE (siblings), CHECK / CHECK_FALSE /
// REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS with doctest::Contains or an
// exact message, INFO / CAPTURE, FAIL, doctest::Approx(..).epsilon(..) and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN -- so the suites compile UNMODIFIED
// against this repo's include/catsim/ headers (tests/cpp/ref_suites.mk).
// Failed expressions are reported by their source text (no decomposition).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <sstream>
#include <string>
#include <utility>
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
  bool matches(double lhs) const {
    return std::fabs(lhs - value_) <
           eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  double value() const { return value_; }
  friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

struct Contains {
  std::string needle;
  explicit Contains(const char* s) : needle(s) {}
  explicit Contains(std::string s) : needle(std::move(s)) {}
};

namespace shim {

struct TestEntry {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<TestEntry>& registry() {
  static std::vector<TestEntry> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

struct State {
  long long asserts = 0;
  long long failed_asserts = 0;
  bool test_failed = false;
  int subcase_target = 0;   // sibling SUBCASE entered in this pass
  int subcase_seen = 0;     // SUBCASEs met so far in this pass
  std::vector<std::string> context;  // INFO / CAPTURE of the live scopes
};

inline State& state() {
  static State s;
  return s;
}

struct AbortTest {};  // REQUIRE / FAIL: leave the test case

inline void report(const char* file, int line, const std::string& what) {
  State& s = state();
  ++s.failed_asserts;
  s.test_failed = true;
  std::fprintf(stderr, "%s:%d: ERROR: %s\n", file, line, what.c_str());
  for (const std::string& c : s.context) std::fprintf(stderr, "  logged: %s\n", c.c_str());
}

inline void check(bool ok, const char* expr, const char* kind, const char* file, int line,
                  bool fatal) {
  ++state().asserts;
  if (ok) return;
  report(file, line, std::string(kind) + "( " + expr + " ) is NOT correct!");
  if (fatal) throw AbortTest{};
}

inline bool message_matches(const Contains& m, const std::string& what) {
  return what.find(m.needle) != std::string::npos;
}
inline bool message_matches(const char* m, const std::string& what) { return what == m; }
inline bool message_matches(const std::string& m, const std::string& what) { return what == m; }

template <typename Ex, typename Fn>
void check_throws_as(Fn&& fn, const char* expr, const char* type, const char* file, int line) {
  ++state().asserts;
  try {
    fn();
  } catch (const Ex&) {
    return;
  } catch (...) {
    report(file, line, std::string("CHECK_THROWS_AS( ") + expr + ", " + type +
                           " ) threw a different exception");
    return;
  }
  report(file, line, std::string("CHECK_THROWS_AS( ") + expr + ", " + type + " ) did NOT throw");
}

template <typename Ex, typename Fn, typename M>
void check_throws_with_as(Fn&& fn, const M& matcher, const char* expr, const char* type,
                          const char* file, int line) {
  ++state().asserts;
  try {
    fn();
  } catch (const Ex& e) {
    if (!message_matches(matcher, e.what()))
      report(file, line, std::string("CHECK_THROWS_WITH_AS( ") + expr + " ): message \"" +
                             e.what() + "\" does not match");
    return;
  } catch (const std::exception& e) {
    report(file, line, std::string("CHECK_THROWS_WITH_AS( ") + expr + ", " + type +
                           " ) threw another type: " + e.what());
    return;
  } catch (...) {
    report(file, line, std::string("CHECK_THROWS_WITH_AS( ") + expr + " ) threw a non-std type");
    return;
  }
  report(file, line, std::string("CHECK_THROWS_WITH_AS( ") + expr + " ) did NOT throw");
}

class Subcase {
 public:
  explicit Subcase(const char*) {
    State& s = state();
    entered_ = s.subcase_seen++ == s.subcase_target;
  }
  explicit operator bool() const { return entered_; }

 private:
  bool entered_;
};

class ContextScope {
 public:
  explicit ContextScope(std::string msg) { state().context.push_back(std::move(msg)); }
  ~ContextScope() { state().context.pop_back(); }
  ContextScope(const ContextScope&) = delete;
  ContextScope& operator=(const ContextScope&) = delete;
};

template <typename... Args>
std::string concat(const Args&... args) {
  std::ostringstream os;
  (os << ... << args);
  return os.str();
}

inline int run_all(int argc, char** argv) {
  const char* filter = nullptr;
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "-tc=", 4) == 0) filter = argv[i] + 4;
  int cases = 0, failed = 0;
  for (const TestEntry& t : registry()) {
    if (filter && !std::strstr(t.name, filter)) continue;
    ++cases;
    State& s = state();
    s.test_failed = false;
    // one pass per sibling SUBCASE (a pass without any runs once)
    for (s.subcase_target = 0;; ++s.subcase_target) {
      s.subcase_seen = 0;
      s.context.clear();
      try {
        t.fn();
      } catch (const AbortTest&) {
      } catch (const std::exception& e) {
        report(t.file, t.line, std::string("test case threw: ") + e.what());
      } catch (...) {
        report(t.file, t.line, "test case threw a non-std exception");
      }
      if (s.subcase_seen <= s.subcase_target + 1) break;
    }
    if (s.test_failed) {
      ++failed;
      std::fprintf(stderr, "TEST CASE FAILED: %s\n", t.name);
    }
  }
  const State& s = state();
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", cases, cases - failed,
              failed);
  std::printf("[doctest-shim] assertions: %lld | %lld passed | %lld failed\n", s.asserts,
              s.asserts - s.failed_asserts, s.failed_asserts);
  return failed == 0 ? 0 : 1;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT_(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT_(a, b)
#define DOCTEST_SHIM_TEST(fn, name)                                                  \
  static void fn();                                                                  \
  static const ::doctest::shim::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, &fn,      \
                                                                     __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TEST(DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__), name)

#define CHECK(...) \
  ::doctest::shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, "CHECK", __FILE__, __LINE__, false)
#define CHECK_FALSE(...) \
  ::doctest::shim::check(!(__VA_ARGS__), #__VA_ARGS__, "CHECK_FALSE", __FILE__, __LINE__, false)
#define REQUIRE(...) \
  ::doctest::shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, "REQUIRE", __FILE__, __LINE__, true)
#define REQUIRE_FALSE(...) \
  ::doctest::shim::check(!(__VA_ARGS__), #__VA_ARGS__, "REQUIRE_FALSE", __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                         \
  ::doctest::shim::check_throws_as<__VA_ARGS__>([&]() { static_cast<void>(expr); }, #expr, \
                                                #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                       \
  ::doctest::shim::check_throws_with_as<__VA_ARGS__>([&]() { static_cast<void>(expr); }, \
                                                     matcher, #expr, #__VA_ARGS__,      \
                                                     __FILE__, __LINE__)
#define CHECK_NOTHROW(expr)                                                                \
  do {                                                                                     \
    ++::doctest::shim::state().asserts;                                                    \
    try {                                                                                  \
      static_cast<void>(expr);                                                             \
    } catch (const std::exception& e_) {                                                   \
      ::doctest::shim::report(__FILE__, __LINE__, std::string("CHECK_NOTHROW( " #expr " ) threw: ") + e_.what()); \
    }                                                                                      \
  } while (0)
#define SUBCASE(name) if (const ::doctest::shim::Subcase DOCTEST_SHIM_CAT(doctest_shim_sc_, __LINE__){name})
#define INFO(...) \
  const ::doctest::shim::ContextScope DOCTEST_SHIM_CAT(doctest_shim_info_, __LINE__)(::doctest::shim::concat(__VA_ARGS__))
#define CAPTURE(x) \
  const ::doctest::shim::ContextScope DOCTEST_SHIM_CAT(doctest_shim_cap_, __LINE__)(::doctest::shim::concat(#x " := ", x))
#define MESSAGE(...) std::printf("%s\n", ::doctest::shim::concat(__VA_ARGS__).c_str())
#define FAIL(...)                                                                \
  do {                                                                           \
    ::doctest::shim::report(__FILE__, __LINE__, ::doctest::shim::concat(__VA_ARGS__)); \
    throw ::doctest::shim::AbortTest{};                                          \
  } while (0)
#define FAIL_CHECK(...) ::doctest::shim::report(__FILE__, __LINE__, ::doctest::shim::concat(__VA_ARGS__))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::shim::run_all(argc, argv); }
#endif
