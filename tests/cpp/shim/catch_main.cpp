// Test runner for the Catch2 shim: runs every registered TEST_CASE, prints
// one line per case, exits non-zero on any failed assertion.
#include <cstdio>
#include <cstring>
#include <exception>

#include "catch_amalgamated.hpp"

int main(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int cases = 0, failed_cases = 0;
  for (const auto& tc : catch_shim::registry()) {
    if (filter && !std::strstr(tc.name, filter)) continue;
    ++cases;
    const int before = catch_shim::failures();
    try {
      tc.fn();
    } catch (const catch_shim::RequireFailed&) {
    } catch (const std::exception& e) {
      ++catch_shim::failures();
      std::fprintf(stderr, "  unexpected exception: %s\n", e.what());
    }
    const bool ok = catch_shim::failures() == before;
    failed_cases += !ok;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", tc.name);
  }
  std::printf("%d test cases, %d failed, %d failed assertions\n", cases, failed_cases,
              catch_shim::failures());
  return failed_cases ? 1 : 0;
}
