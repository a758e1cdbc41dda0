// main() of the doctest stand-in (tests/cpp/shim/doctest.h): runs every
// registered TEST_CASE, prints one line per case and a summary; exit code 1
// if any CHECK / REQUIRE failed or a case threw.  Optional argv[1]: substring
// filter on case names.
#include <cstdio>
#include <cstring>
#include <exception>

#include "doctest.h"

int main(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int cases = 0, failed_cases = 0;
  for (const auto& c : doctest_shim::registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    ++cases;
    doctest_shim::stats().case_failed = false;
    try {
      c.fn();
    } catch (const doctest_shim::Abort&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: exception in \"%s\": %s\n", c.file, c.line, c.name, e.what());
      doctest_shim::stats().case_failed = true;
    }
    const bool bad = doctest_shim::stats().case_failed;
    failed_cases += bad;
    std::printf("[%s] %s\n", bad ? "FAIL" : " ok ", c.name);
  }
  std::printf("test cases: %d | %d passed | %d failed; assertions: %ld | %ld failed\n", cases, cases - failed_cases,
              failed_cases, doctest_shim::stats().checks, doctest_shim::stats().failed);
  return failed_cases ? 1 : 0;
}
