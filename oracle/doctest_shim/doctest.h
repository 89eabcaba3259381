// doctest_shim/doctest.h -- a from-scratch, minimal test-macro shim.
//
// TEST INFRASTRUCTURE ONLY.  The reference's suites (proj/tests/*.cpp) include
// <doctest.h>, which is vendored-and-gitignored upstream and absent here
// (SURVEY.md §4).  This header provides just the macro surface those suites use
// -- TEST_CASE, SUBCASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, doctest::Contains -- with plain semantics: every CHECK is
// counted, failures are printed with file:line, REQUIRE aborts the current test
// case, and SUBCASE bodies run in sequence inside one pass of their test case.
#pragma once

#include <cstdio>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

struct Contains {
    std::string needle;
    explicit Contains(const char* s) : needle(s) {}
    bool matches(const char* what) const { return std::string(what).find(needle) != std::string::npos; }
};

namespace shim {

struct Case {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};

inline std::vector<Case>& cases() {
    static std::vector<Case> all;
    return all;
}

struct Stats {
    long checks = 0;
    long failed = 0;
};

inline Stats& stats() {
    static Stats s;
    return s;
}

struct Register {
    Register(const char* name, void (*fn)(), const char* file, int line) {
        cases().push_back(Case{name, fn, file, line});
    }
};

struct RequireAbort {};

inline bool record(bool ok, const char* kind, const char* expr, const char* file, int line) {
    ++stats().checks;
    if (!ok) {
        ++stats().failed;
        std::fprintf(stderr, "%s:%d: %s( %s ) failed\n", file, line, kind, expr);
    }
    return ok;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)

#define TEST_CASE(name)                                                                       \
    static void DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__)();                             \
    static ::doctest::shim::Register DOCTEST_SHIM_CAT(doctest_shim_reg_, __LINE__)(           \
        name, &DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__), __FILE__, __LINE__);           \
    static void DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__)()

#define SUBCASE(name) if (true)

#define CHECK(...) \
    ((void)::doctest::shim::record(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__))

#define CHECK_FALSE(...) \
    ((void)::doctest::shim::record(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__))

#define REQUIRE(...)                                                                          \
    do {                                                                                      \
        if (!::doctest::shim::record(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, \
                                     __FILE__, __LINE__))                                     \
            throw ::doctest::shim::RequireAbort{};                                            \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                            \
    do {                                                                                      \
        bool doctest_shim_ok = false;                                                         \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const __VA_ARGS__&) {                                                        \
            doctest_shim_ok = true;                                                           \
        } catch (...) {                                                                       \
        }                                                                                     \
        ::doctest::shim::record(doctest_shim_ok, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                              \
    do {                                                                                      \
        bool doctest_shim_ok = false;                                                         \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const __VA_ARGS__& e) {                                                      \
            doctest_shim_ok = (matcher).matches(e.what());                                    \
        } catch (...) {                                                                       \
        }                                                                                     \
        ::doctest::shim::record(doctest_shim_ok, "CHECK_THROWS_WITH_AS", #expr, __FILE__,     \
                                __LINE__);                                                    \
    } while (0)
