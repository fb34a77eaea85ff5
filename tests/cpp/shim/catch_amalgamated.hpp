// Minimal Catch2-compatible test shim (own code) so the reference's unit
// test sources (/root/reference/proj/tests/test_*.cpp) compile unchanged
// against this repo's headers.  Supports TEST_CASE, CHECK, CHECK_FALSE,
// REQUIRE, CHECK_THROWS_AS, FAIL and Catch::Approx.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

namespace catch_shim {

struct TestCase {
  const char* name;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct RequireFailed {};

inline int& failures() {
  static int f = 0;
  return f;
}

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
  if (ok) return;
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
  if (fatal) throw RequireFailed{};
}

}  // namespace catch_shim

namespace Catch {
class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  friend bool operator==(double a, const Approx& b) {
    const double eps = std::numeric_limits<float>::epsilon() * 100.0;
    return std::fabs(a - b.v_) <= eps * std::fabs(b.v_);
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }

 private:
  double v_;
};
}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define TEST_CASE(name, ...)                                                  \
  static void CATCH_SHIM_CAT(catch_shim_fn_, __LINE__)();                     \
  static catch_shim::Registrar CATCH_SHIM_CAT(catch_shim_reg_, __LINE__)(     \
      name, &CATCH_SHIM_CAT(catch_shim_fn_, __LINE__));                       \
  static void CATCH_SHIM_CAT(catch_shim_fn_, __LINE__)()
#define CHECK(...) catch_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) catch_shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) catch_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(msg) catch_shim::report(false, msg, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                           \
  do {                                                                        \
    bool caught_ = false;                                                     \
    try {                                                                     \
      (void)(expr);                                                           \
    } catch (const type&) {                                                   \
      caught_ = true;                                                         \
    } catch (...) {                                                           \
    }                                                                         \
    catch_shim::report(caught_, #expr " throws " #type, __FILE__, __LINE__, false); \
  } while (0)
