// TEST INFRASTRUCTURE ONLY (oracle self-test). A minimal stand-in for the
// doctest macros /root/reference/proj/tests/test_spb.cpp uses, so the
// reference's own unit tests can pin the compiled reference (oracle/_ref)
// before it is trusted. doctest is not vendored in the reference
// (proj/.gitignore:2). SUBCASE is `if (true)`: the two subcases in
// test_spb.cpp are independent, so running both in sequence is equivalent.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Registry {
  struct Case {
    const char* name;
    std::function<void()> fn;
  };
  std::vector<Case> cases;
  long checks = 0, failures = 0;
  static Registry& get() {
    static Registry r;
    return r;
  }
};

struct Registrar {
  Registrar(const char* name, void (*fn)()) { Registry::get().cases.push_back({name, fn}); }
};

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    double scale = std::max(std::fabs(lhs), std::fabs(a.v_));
    return std::fabs(lhs - a.v_) < a.eps_ * (1.0 + scale);
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }

 private:
  double v_;
  double eps_ = 1.1920929e-7f * 100;  // doctest's default epsilon
};

inline void record(bool ok, const char* expr, const char* file, int line) {
  auto& r = Registry::get();
  ++r.checks;
  if (!ok) {
    ++r.failures;
    std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", file, line, expr);
  }
}

struct RequireFailed {};

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, name)                                           \
  static void fn();                                                       \
  static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);             \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define SUBCASE(name) if (true)
#define CHECK(...) doctest::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                          \
  do {                                                                        \
    bool ok_ = static_cast<bool>(__VA_ARGS__);                                \
    doctest::record(ok_, #__VA_ARGS__, __FILE__, __LINE__);                   \
    if (!ok_) throw doctest::RequireFailed{};                                 \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                           \
  do {                                                                        \
    bool thrown_ = false;                                                     \
    try {                                                                     \
      (void)(expr);                                                           \
    } catch (const type&) {                                                   \
      thrown_ = true;                                                         \
    } catch (...) {                                                           \
    }                                                                         \
    doctest::record(thrown_, "THROWS_AS(" #expr ", " #type ")", __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  auto& r = doctest::Registry::get();
  long failed_cases = 0;
  for (auto& c : r.cases) {
    long before = r.failures;
    try {
      c.fn();
    } catch (const doctest::RequireFailed&) {
    } catch (const std::exception& e) {
      ++r.failures;
      std::fprintf(stderr, "test case '%s' threw: %s\n", c.name, e.what());
    }
    if (r.failures != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | %ld failed | checks: %ld | %ld failed\n",
              r.cases.size(), failed_cases, r.checks, r.failures);
  return r.failures == 0 ? 0 : 1;
}
#endif
