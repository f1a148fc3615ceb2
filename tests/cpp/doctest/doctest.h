// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE).  The
// reference's suites include <doctest.h> from an unshipped vendor/ tree;
// this header provides the subset they use -- TEST_CASE, CHECK, REQUIRE,
// FAIL, CHECK_THROWS_AS, CHECK_NOTHROW and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
// -- so those files compile unchanged against the B200 drop-in
// (paper_2605_24290_b200/refapi).  Output: one line per failed check, one
// summary line; exit status 1 if any case failed.
#pragma once
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

namespace doctest_shim {
struct Case {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};
inline std::vector<Case>& cases() {
    static std::vector<Case> v;
    return v;
}
struct Reg {
    Reg(const char* n, void (*f)(), const char* file, int line) { cases().push_back({n, f, file, line}); }
};
struct Counters {
    long checks = 0, failed = 0;
};
inline Counters& counters() {
    static Counters c;
    return c;
}
struct Abort {};  // REQUIRE / FAIL end the test case
inline void report(const char* kind, const char* expr, const char* file, int line) {
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
    ++counters().failed;
}
}  // namespace doctest_shim

#define DOCTEST_SHIM_CAT_(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT_(a, b)
#define DOCTEST_SHIM_CASE(fn, name)                                                           \
    static void fn();                                                                        \
    static doctest_shim::Reg DOCTEST_SHIM_CAT(fn, _reg)(name, fn, __FILE__, __LINE__);       \
    static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__), name)

#define CHECK(...)                                                                        \
    do {                                                                                  \
        ++doctest_shim::counters().checks;                                                \
        if (!(__VA_ARGS__)) doctest_shim::report("CHECK", #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define REQUIRE(...)                                                                          \
    do {                                                                                      \
        ++doctest_shim::counters().checks;                                                    \
        if (!(__VA_ARGS__)) {                                                                 \
            doctest_shim::report("REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                \
            throw doctest_shim::Abort{};                                                      \
        }                                                                                     \
    } while (0)
#define FAIL(msg)                                                      \
    do {                                                               \
        doctest_shim::report("FAIL", msg, __FILE__, __LINE__);         \
        throw doctest_shim::Abort{};                                   \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                     \
    do {                                                                                \
        ++doctest_shim::counters().checks;                                              \
        bool doctest_shim_ok = false;                                                   \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (const type&) {                                                         \
            doctest_shim_ok = true;                                                     \
        } catch (...) {                                                                 \
        }                                                                               \
        if (!doctest_shim_ok) doctest_shim::report("CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                          \
    do {                                                                             \
        ++doctest_shim::counters().checks;                                           \
        try {                                                                        \
            (void)(expr);                                                            \
        } catch (...) {                                                              \
            doctest_shim::report("CHECK_NOTHROW", #expr, __FILE__, __LINE__);        \
        }                                                                            \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0;
    for (const auto& c : doctest_shim::cases()) {
        const long before = doctest_shim::counters().failed;
        try {
            c.fn();
        } catch (const doctest_shim::Abort&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: TEST_CASE(%s) threw: %s\n", c.file, c.line, c.name, e.what());
            ++doctest_shim::counters().failed;
        } catch (...) {
            std::fprintf(stderr, "%s:%d: TEST_CASE(%s) threw a non-std exception\n", c.file, c.line, c.name);
            ++doctest_shim::counters().failed;
        }
        if (doctest_shim::counters().failed != before) {
            ++failed_cases;
            std::fprintf(stderr, "  in TEST_CASE: %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld | %ld failed\n",
                doctest_shim::cases().size(), doctest_shim::cases().size() - failed_cases, failed_cases,
                doctest_shim::counters().checks, doctest_shim::counters().failed);
    return failed_cases ? 1 : 0;
}
#endif
