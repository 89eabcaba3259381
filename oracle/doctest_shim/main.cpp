// Runner for doctest_shim: runs every registered TEST_CASE (optionally only
// those whose name contains argv[1]) and prints one summary line.  Exit code 0
// iff no check failed.
#include <cstdio>
#include <cstring>
#include <exception>

#include "doctest.h"

int main(int argc, char** argv) {
    const char* filter = argc > 1 ? argv[1] : nullptr;
    long ran = 0;
    long crashed = 0;
    for (const auto& c : doctest::shim::cases()) {
        if (filter && !std::strstr(c.name, filter)) continue;
        ++ran;
        try {
            c.fn();
        } catch (const doctest::shim::RequireAbort&) {
        } catch (const std::exception& e) {
            ++crashed;
            ++doctest::shim::stats().failed;
            std::fprintf(stderr, "%s:%d: test case \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
        }
    }
    const auto& s = doctest::shim::stats();
    std::printf("[doctest-shim] test cases: %ld | checks: %ld | failed: %ld | crashed: %ld\n", ran,
                s.checks, s.failed, crashed);
    return s.failed == 0 ? 0 : 1;
}
