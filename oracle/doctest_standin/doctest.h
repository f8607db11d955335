// Minimal stand-in for doctest (test infrastructure only).
//
// The reference's unit tests (`/root/reference/proj/tests/test_*.cpp`) include
// "doctest.h", which the reference expects under `vendor/` but does not ship
// (`proj/.gitignore:2`).  This header implements just the macros those two
// files use (TEST_CASE, SUBCASE, CHECK*, REQUIRE*) so the reference's own
// known-answer tests can run against the reference library and pin the oracle.
// SUBCASE blocks run sequentially inside one pass of their TEST_CASE.
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest_standin {

struct Case {
    const char* name;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Stats {
    long checks = 0;
    long failures = 0;
    long cases_failed = 0;
};

inline Stats& stats() {
    static Stats s;
    return s;
}

struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    ++stats().checks;
    if (!ok) {
        ++stats().failures;
        std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
        if (fatal) throw RequireFailed{};
    }
}

inline int run_all() {
    for (const auto& c : registry()) {
        long before = stats().failures;
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++stats().failures;
            std::fprintf(stderr, "case '%s' threw: %s\n", c.name, e.what());
        }
        if (stats().failures != before) {
            ++stats().cases_failed;
            std::fprintf(stderr, "FAILED case: %s\n", c.name);
        }
    }
    std::printf("[doctest-standin] cases: %zu | failed: %ld | checks: %ld | failed checks: %ld\n",
                registry().size(), stats().cases_failed, stats().checks, stats().failures);
    return stats().failures == 0 ? 0 : 1;
}

}  // namespace doctest_standin

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)
#define TEST_CASE(name)                                                                  \
    static void DS_CAT(ds_case_, __LINE__)();                                            \
    static doctest_standin::Registrar DS_CAT(ds_reg_, __LINE__)(name, &DS_CAT(ds_case_, __LINE__)); \
    static void DS_CAT(ds_case_, __LINE__)()
#define SUBCASE(name) if (true)

#define DS_CHECK_IMPL(cond, text, fatal) \
    doctest_standin::report(static_cast<bool>(cond), text, __FILE__, __LINE__, fatal)
#define CHECK(...) DS_CHECK_IMPL((__VA_ARGS__), #__VA_ARGS__, false)
#define REQUIRE(...) DS_CHECK_IMPL((__VA_ARGS__), #__VA_ARGS__, true)
#define CHECK_FALSE(...) DS_CHECK_IMPL(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", false)
#define CHECK_NOTHROW(...)                                                   \
    do {                                                                     \
        bool ds_ok = true;                                                   \
        try { (void)(__VA_ARGS__); } catch (...) { ds_ok = false; }          \
        DS_CHECK_IMPL(ds_ok, "nothrow: " #__VA_ARGS__, false);               \
    } while (0)
#define CHECK_THROWS_AS(expr, exc)                                           \
    do {                                                                     \
        bool ds_ok = false;                                                  \
        try { (void)(expr); } catch (const exc&) { ds_ok = true; } catch (...) {} \
        DS_CHECK_IMPL(ds_ok, "throws " #exc ": " #expr, false);              \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest_standin::run_all(); }
#endif
