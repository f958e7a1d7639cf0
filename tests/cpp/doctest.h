// Minimal doctest-compatible runner for the reference's unit suites.
//
// The reference tests (proj/tests/test_*.cpp) include <doctest.h>, which the
// reference does not vendor. This header implements the subset they use --
// TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, FAIL, doctest::Approx with
// .epsilon(), DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN -- so the same suites can be
// compiled (a) against the reference library, pinning the oracle build, and
// (b) against this repo's drop-in voxanim library, checking API conformance.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    double value;
    double eps = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
};

// doctest's rule: |a - b| < eps * (1 + max(|a|, |b|))
inline bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.value) < b.eps * (1.0 + std::max(std::fabs(a), std::fabs(b.value)));
}
inline bool operator==(const Approx& b, double a) { return a == b; }
inline bool operator!=(double a, const Approx& b) { return !(a == b); }

namespace detail {

struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Abort {}; // thrown by REQUIRE / FAIL to leave the current test case

inline int& failures_in_case() {
    static int n = 0;
    return n;
}
inline long& assertions() {
    static long n = 0;
    return n;
}

inline void report(const char* file, int line, const char* what, const char* expr) {
    ++failures_in_case();
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, what, expr);
}

inline bool check(bool ok, const char* expr, const char* file, int line, bool require) {
    ++assertions();
    if (!ok) {
        report(file, line, require ? "REQUIRE" : "CHECK", expr);
        if (require) throw Abort{};
    }
    return ok;
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};

inline int run_all() {
    int failed = 0;
    for (const Case& c : registry()) {
        failures_in_case() = 0;
        try {
            c.fn();
        } catch (const Abort&) {
        } catch (const std::exception& e) {
            report(c.file, c.line, "TEST_CASE threw", e.what());
        } catch (...) {
            report(c.file, c.line, "TEST_CASE threw", "unknown exception");
        }
        if (failures_in_case() > 0) {
            ++failed;
            std::fprintf(stderr, "  in TEST_CASE \"%s\"\n", c.name);
        }
    }
    std::printf("[doctest] test cases: %zu | %zu passed | %d failed | assertions: %ld\n", registry().size(),
                registry().size() - static_cast<size_t>(failed), failed, assertions());
    return failed == 0 ? 0 : 1;
}

} // namespace detail
} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                              \
    static void fn();                                                                                 \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);         \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(msg)                                                                                     \
    do {                                                                                              \
        ::doctest::detail::report(__FILE__, __LINE__, "FAIL", std::string(msg).c_str());              \
        throw ::doctest::detail::Abort{};                                                             \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                    \
    do {                                                                                              \
        ++::doctest::detail::assertions();                                                            \
        bool doctest_ok_ = false;                                                                     \
        try {                                                                                         \
            static_cast<void>(expr);                                                                  \
        } catch (const __VA_ARGS__&) {                                                                \
            doctest_ok_ = true;                                                                       \
        } catch (...) {                                                                               \
        }                                                                                             \
        if (!doctest_ok_) ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr);   \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
