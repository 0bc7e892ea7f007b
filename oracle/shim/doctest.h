// Tiny doctest-compatible harness (test infrastructure only). Supports the
// subset the reference suites use: TEST_CASE, top-level SUBCASE (each pass of a
// test case runs exactly one subcase), CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW and doctest::Approx(..).epsilon(..).
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
namespace detail {
struct Case { const char* name; void (*fn)(); const char* file; int line; };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
struct Reg { Reg(const char* n, void (*f)(), const char* file, int line) { registry().push_back({n, f, file, line}); } };
struct State { int target = 0; int seen = 0; long checks = 0; long failures = 0; bool case_failed = false; };
inline State& st() { static State s; return s; }
struct RequireAbort {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    ++st().checks;
    if (!ok) {
        ++st().failures;
        st().case_failed = true;
        std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line, require ? "REQUIRE" : "CHECK", expr);
        if (require) throw RequireAbort{};
    }
}
// SUBCASE guard: true only for the subcase whose ordinal equals the pass index.
struct Sub {
    bool active;
    explicit Sub(const char*) { active = (st().seen == st().target); ++st().seen; }
    explicit operator bool() const { return active; }
};
} // namespace detail

struct Approx {
    double value; double eps;
    explicit Approx(double v) : value(v), eps(100.0 * 1.1920928955078125e-07) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value) < a.eps * (1.0 + std::max(std::fabs(lhs), std::fabs(a.value)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
};

inline int run_all() {
    using namespace detail;
    long cases = 0, failed_cases = 0;
    for (const Case& c : registry()) {
        ++cases;
        st().case_failed = false;
        for (int pass = 0;; ++pass) {
            st().target = pass;
            st().seen = 0;
            try {
                c.fn();
            } catch (const RequireAbort&) {
            } catch (const std::exception& e) {
                ++st().failures; st().case_failed = true;
                std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", c.file, c.line, c.name, e.what());
            } catch (...) {
                ++st().failures; st().case_failed = true;
                std::fprintf(stderr, "%s:%d: test case '%s' threw a non-std exception\n", c.file, c.line, c.name);
            }
            if (st().seen <= pass + 1) break;
        }
        if (st().case_failed) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %ld | %ld passed | %ld failed; assertions: %ld | %ld failed\n",
                cases, cases - failed_cases, failed_cases, st().checks, st().failures);
    return st().failures == 0 ? 0 : 1;
}
} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                            \
    static void fn();                                                                   \
    static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __LINE__), name)
#define SUBCASE(name) if (const ::doctest::detail::Sub DOCTEST_CAT(doctest_sub_, __LINE__){name})
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                     \
    do {                                                                               \
        bool doctest_ok_ = false;                                                      \
        try { (void)(expr); } catch (const __VA_ARGS__&) { doctest_ok_ = true; } catch (...) {} \
        ::doctest::detail::report(doctest_ok_, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_NOTHROW(...)                                                             \
    do {                                                                               \
        bool doctest_ok_ = true;                                                       \
        try { (void)(__VA_ARGS__); } catch (...) { doctest_ok_ = false; }              \
        ::doctest::detail::report(doctest_ok_, #__VA_ARGS__ " nothrow", __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::run_all(); }
#endif
