// A minimal doctest-compatible test runner (test infrastructure): TEST_CASE,
// SUBCASE (one level; the case body re-runs once per subcase, like doctest),
// CHECK/CHECK_FALSE/REQUIRE and CHECK_THROWS_AS.  Enough to compile and run
// test files written for doctest against the B200 engine's C++ API.
#pragma once
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace mini_doctest {
struct Case {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Reg {
    Reg(const char* n, void (*f)(), const char* file, int line) { registry().push_back({n, f, file, line}); }
};
struct State {
    int target = 0, seen = 0;
    long checks = 0, failures = 0;
    const char* subcase = "";
};
inline State& st() {
    static State s;
    return s;
}
struct RequireFailed {};
inline bool enter_subcase(const char* name) {
    State& s = st();
    const bool mine = s.seen++ == s.target;
    if (mine) s.subcase = name;
    return mine;
}
inline void report(bool ok, const char* expr, const char* file, int line) {
    State& s = st();
    ++s.checks;
    if (!ok) {
        ++s.failures;
        std::fprintf(stderr, "%s:%d: FAILED: %s%s%s\n", file, line, expr, *s.subcase ? "  [subcase: " : "",
                     *s.subcase ? (std::string(s.subcase) + "]").c_str() : "");
    }
}
inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        State& s = st();
        const long f0 = s.failures;
        int target = 0;
        for (;;) {
            s.target = target;
            s.seen = 0;
            s.subcase = "";
            try {
                c.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                ++s.failures;
                std::fprintf(stderr, "%s:%d: %s: unexpected exception: %s\n", c.file, c.line, c.name, e.what());
            }
            if (++target >= s.seen) break;  // every subcase (or the plain body) has run
        }
        const bool ok = s.failures == f0;
        failed_cases += !ok;
        std::printf("[%s] %s\n", ok ? "ok  " : "FAIL", c.name);
    }
    std::printf("%zu test cases, %d failed; %ld checks, %ld failed\n", registry().size(), failed_cases,
                st().checks, st().failures);
    return failed_cases ? 1 : 0;
}
}  // namespace mini_doctest

#define MDT_CAT2(a, b) a##b
#define MDT_CAT(a, b) MDT_CAT2(a, b)
#define TEST_CASE(name)                                                                      \
    static void MDT_CAT(mdt_case_, __LINE__)();                                              \
    static ::mini_doctest::Reg MDT_CAT(mdt_reg_, __LINE__)(name, &MDT_CAT(mdt_case_, __LINE__), \
                                                           __FILE__, __LINE__);              \
    static void MDT_CAT(mdt_case_, __LINE__)()
#define SUBCASE(name) if (::mini_doctest::enter_subcase(name))
#define CHECK(...) ::mini_doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::mini_doctest::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                 \
    do {                                                                             \
        const bool mdt_ok = static_cast<bool>(__VA_ARGS__);                          \
        ::mini_doctest::report(mdt_ok, #__VA_ARGS__, __FILE__, __LINE__);            \
        if (!mdt_ok) throw ::mini_doctest::RequireFailed{};                          \
    } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!static_cast<bool>(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, ...)                                                   \
    do {                                                                             \
        bool mdt_ok = false;                                                         \
        try {                                                                        \
            (void)(expr);                                                            \
        } catch (const __VA_ARGS__&) {                                               \
            mdt_ok = true;                                                           \
        } catch (...) {                                                              \
        }                                                                            \
        ::mini_doctest::report(mdt_ok, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                          \
    do {                                                                             \
        bool mdt_ok = true;                                                          \
        try {                                                                        \
            (void)(expr);                                                            \
        } catch (...) {                                                              \
            mdt_ok = false;                                                          \
        }                                                                            \
        ::mini_doctest::report(mdt_ok, #expr " does not throw", __FILE__, __LINE__);  \
    } while (0)

#ifdef MINI_DOCTEST_MAIN
int main() { return ::mini_doctest::run_all(); }
#endif
