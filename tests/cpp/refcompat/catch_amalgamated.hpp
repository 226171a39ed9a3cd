// A minimal, dependency-free stand-in for the Catch2 amalgamated header
// (Catch2 is absent from this image).  It implements exactly the
// subset the reference's own unit tests use -- TEST_CASE, SECTION (nested,
// each leaf run once as Catch2 does), CHECK / CHECK_FALSE / REQUIRE,
// CHECK_THROWS_AS / CHECK_THROWS_WITH / CHECK_NOTHROW, FAIL, Catch::Approx
// and Catch::Matchers::ContainsSubstring -- so the reference's test files
// (/root/reference/proj/tests/test_*.cpp) compile UNMODIFIED against the
// drop-in headers in include/embdispatch/.  Test infrastructure only.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace catch_shim {

struct TestCase {
  std::string name;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
  Registrar(const char* name, const char*, void (*fn)()) { registry().push_back({name, fn}); }
};

struct State {
  long checks = 0, failures = 0;
  // section tracking for the running test case
  std::set<std::string> done;      // completed section paths
  std::vector<std::string> path;   // sections entered in this run
  std::vector<bool> entered;       // per depth: a section was entered in this run
  std::vector<bool> pending;       // per depth: a child was skipped unfinished
  bool ran_section = false;
  std::string test;
};

inline State& st() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void fail(const char* file, int line, const std::string& what) {
  ++st().failures;
  std::printf("FAILED %s:%d [%s]\n  %s\n", file, line, st().test.c_str(), what.c_str());
  std::fflush(stdout);
}

class Section {
 public:
  explicit Section(const char* name) {
    State& s = st();
    const std::size_t d = s.path.size();
    if (s.entered.size() <= d) {
      s.entered.resize(d + 1, false);
      s.pending.resize(d + 1, false);
    }
    full_ = (d ? s.path.back() + "/" : std::string()) + name;
    if (s.done.count(full_)) return;
    if (s.entered[d]) {  // a sibling ran this time: come back on a later run
      if (d) s.pending[d - 1] = true;
      s.ran_section = true;
      return;
    }
    s.entered[d] = true;
    s.path.push_back(full_);
    if (s.pending.size() <= d + 1) s.pending.resize(d + 2, false);
    s.pending[d] = false;
    active_ = true;
    s.ran_section = true;
  }
  ~Section() {
    if (!active_) return;
    State& s = st();
    const std::size_t d = s.path.size() - 1;
    if (!s.pending[d]) s.done.insert(full_);
    s.path.pop_back();
    if (d + 1 < s.entered.size()) s.entered[d + 1] = false;
  }
  explicit operator bool() const { return active_; }

 private:
  std::string full_;
  bool active_ = false;
};

inline int run_all(const char* filter) {
  int failed_cases = 0, ran = 0;
  for (const TestCase& tc : registry()) {
    if (filter && tc.name.find(filter) == std::string::npos) continue;
    ++ran;
    State& s = st();
    const long f0 = s.failures;
    s.done.clear();
    s.test = tc.name;
    for (int run = 0; run < 10000; ++run) {
      s.path.clear();
      s.entered.assign(1, false);
      s.pending.assign(1, false);
      s.ran_section = false;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
        break;
      } catch (const std::exception& e) {
        fail("<test case>", 0, std::string("unexpected exception: ") + e.what());
        break;
      }
      if (!s.ran_section) break;  // no section left to enter
    }
    if (s.failures != f0) ++failed_cases;
  }
  std::printf("%d test cases, %d failed; %ld checks, %ld failed\n", ran, failed_cases,
              st().checks, st().failures);
  return failed_cases == 0 && ran > 0 ? 0 : 1;
}

}  // namespace catch_shim

namespace Catch {

class Approx {
 public:
  explicit Approx(double v)
      : value_(v), epsilon_(std::numeric_limits<float>::epsilon() * 100), margin_(0.0) {}
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) { return a.equals(lhs); }
  friend bool operator==(const Approx& a, double rhs) { return a.equals(rhs); }
  friend bool operator!=(double lhs, const Approx& a) { return !a.equals(lhs); }
  friend bool operator!=(const Approx& a, double rhs) { return !a.equals(rhs); }

 private:
  bool equals(double x) const {
    const double d = std::fabs(x - value_);
    return d <= margin_ || d <= epsilon_ * std::fabs(value_);
  }
  double value_, epsilon_, margin_;
};

namespace Matchers {
struct ContainsSubstring {
  explicit ContainsSubstring(std::string s) : sub(std::move(s)) {}
  bool match(const std::string& what) const { return what.find(sub) != std::string::npos; }
  std::string sub;
};
}  // namespace Matchers

}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_TEST(fn, ...)                                                      \
  static void fn();                                                                   \
  static const catch_shim::Registrar CATCH_SHIM_CAT(fn, _reg)(__VA_ARGS__, &fn);      \
  static void fn()
#define TEST_CASE(...) CATCH_SHIM_TEST(CATCH_SHIM_CAT(catch_shim_test_, __LINE__), __VA_ARGS__)
#define SECTION(name) if (const catch_shim::Section CATCH_SHIM_CAT(catch_shim_sec_, __LINE__){name})

#define CATCH_SHIM_CHECK(expr, required, text)                          \
  do {                                                                  \
    ++catch_shim::st().checks;                                          \
    bool catch_shim_ok_ = false;                                        \
    try {                                                               \
      catch_shim_ok_ = static_cast<bool>(expr);                         \
    } catch (const std::exception& e) {                                 \
      catch_shim::fail(__FILE__, __LINE__, std::string(text) + " threw " + e.what()); \
      if (required) throw catch_shim::RequireFailed{};                  \
      break;                                                            \
    }                                                                   \
    if (!catch_shim_ok_) {                                              \
      catch_shim::fail(__FILE__, __LINE__, text);                       \
      if (required) throw catch_shim::RequireFailed{};                  \
    }                                                                   \
  } while (0)

#define CHECK(...) CATCH_SHIM_CHECK((__VA_ARGS__), false, "CHECK(" #__VA_ARGS__ ")")
#define CHECK_FALSE(...) CATCH_SHIM_CHECK(!(__VA_ARGS__), false, "CHECK_FALSE(" #__VA_ARGS__ ")")
#define REQUIRE(...) CATCH_SHIM_CHECK((__VA_ARGS__), true, "REQUIRE(" #__VA_ARGS__ ")")
#define REQUIRE_FALSE(...) CATCH_SHIM_CHECK(!(__VA_ARGS__), true, "REQUIRE_FALSE(" #__VA_ARGS__ ")")
#define FAIL(msg)                                                       \
  do {                                                                  \
    ++catch_shim::st().checks;                                          \
    catch_shim::fail(__FILE__, __LINE__, std::string("FAIL: ") + (msg)); \
    throw catch_shim::RequireFailed{};                                  \
  } while (0)

#define CHECK_THROWS_AS(expr, type)                                                   \
  do {                                                                                \
    ++catch_shim::st().checks;                                                        \
    try {                                                                             \
      (void)(expr);                                                                   \
      catch_shim::fail(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #type "): nothing thrown"); \
    } catch (const type&) {                                                           \
    } catch (const std::exception& e) {                                               \
      catch_shim::fail(__FILE__, __LINE__,                                            \
                       std::string("CHECK_THROWS_AS(" #expr ", " #type "): threw ") + e.what()); \
    }                                                                                 \
  } while (0)

#define CHECK_THROWS_WITH(expr, matcher)                                              \
  do {                                                                                \
    ++catch_shim::st().checks;                                                        \
    try {                                                                             \
      (void)(expr);                                                                   \
      catch_shim::fail(__FILE__, __LINE__, "CHECK_THROWS_WITH(" #expr "): nothing thrown"); \
    } catch (const std::exception& e) {                                               \
      if (!(matcher).match(e.what()))                                                 \
        catch_shim::fail(__FILE__, __LINE__,                                          \
                         std::string("CHECK_THROWS_WITH(" #expr "): message ") + e.what()); \
    }                                                                                 \
  } while (0)

#define CHECK_NOTHROW(expr)                                                           \
  do {                                                                                \
    ++catch_shim::st().checks;                                                        \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (const std::exception& e) {                                               \
      catch_shim::fail(__FILE__, __LINE__, std::string("CHECK_NOTHROW(" #expr "): threw ") + e.what()); \
    }                                                                                 \
  } while (0)
