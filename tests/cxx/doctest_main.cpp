// Runner for the doctest-compatible harness: runs every registered case, prints
// one line per case and a summary, exits non-zero on any failure.
#include <cstdio>

#include "doctest.h"

int main() {
    int failed = 0, passed = 0;
    for (const auto& c : doctest::registry()) {
        try {
            c.fn();
            ++passed;
            std::printf("PASS  %s\n", c.name);
        } catch (const std::exception& e) {
            ++failed;
            std::printf("FAIL  %s\n      %s\n", c.name, e.what());
        }
    }
    std::printf("[ref-suite] %d passed, %d failed, %d total\n", passed, failed, passed + failed);
    return failed ? 1 : 0;
}
