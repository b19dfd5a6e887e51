// TEST INFRASTRUCTURE ONLY — a tiny subset of the doctest API.
//
// The reference's unit tests (reference proj/tests/test_*.cpp) include
// <doctest.h>, which lives in an un-vendored directory (reference
// proj/.gitignore: vendor/).  This header supplies just the macros those
// files use (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW,
// doctest::Approx) so they can be compiled verbatim, either against the
// reference sources (oracle/_ref) or against this repo's drop-in facade.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) <
               a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
    double scale_ = 1.0;
};

namespace detail {

struct RequireFailed {};

struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> cases;
    return cases;
}

struct Counters {
    long checks = 0;
    long failures = 0;
    long case_failures = 0;
    bool current_failed = false;
};

inline Counters& counters() {
    static Counters c;
    return c;
}

inline int reg(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
    return 0;
}

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    ++counters().checks;
    if (ok) return;
    ++counters().failures;
    counters().current_failed = true;
    std::fprintf(stderr, "%s:%d: %s FAILED: %s\n", file, line, fatal ? "REQUIRE" : "CHECK", expr);
    if (fatal) throw RequireFailed{};
}

inline int run_all() {
    auto& c = counters();
    for (const Case& tc : registry()) {
        c.current_failed = false;
        try {
            tc.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: test case \"%s\" threw: %s\n", tc.file, tc.line, tc.name,
                         e.what());
            c.current_failed = true;
            ++c.failures;
        }
        if (c.current_failed) {
            ++c.case_failures;
            std::fprintf(stderr, "[FAIL] %s\n", tc.name);
        }
    }
    std::printf("[doctest-subset] test cases: %zu | %ld failed | assertions: %ld | %ld failed\n",
                registry().size(), c.case_failures, c.checks, c.failures);
    return c.case_failures == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                    \
    static void fn();                                                                       \
    static const int DOCTEST_CAT(fn, _reg) = doctest::detail::reg(name, __FILE__, __LINE__, fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define DOCTEST_ASSERT_IMPL(expr, fatal) \
    doctest::detail::report(static_cast<bool>(expr), #expr, __FILE__, __LINE__, fatal)
#define CHECK(...) DOCTEST_ASSERT_IMPL((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_ASSERT_IMPL((__VA_ARGS__), true)
#define CHECK_FALSE(...) DOCTEST_ASSERT_IMPL(!(__VA_ARGS__), false)

#define CHECK_THROWS_AS(expr, ex)                                                          \
    do {                                                                                   \
        bool doctest_ok_ = false;                                                          \
        try {                                                                              \
            (void)(expr);                                                                  \
        } catch (const ex&) {                                                              \
            doctest_ok_ = true;                                                            \
        } catch (...) {                                                                    \
        }                                                                                  \
        doctest::detail::report(doctest_ok_, #expr " throws " #ex, __FILE__, __LINE__, false); \
    } while (0)

#define CHECK_NOTHROW(expr)                                                              \
    do {                                                                                 \
        bool doctest_ok_ = true;                                                         \
        try {                                                                            \
            (void)(expr);                                                                \
        } catch (...) {                                                                  \
            doctest_ok_ = false;                                                         \
        }                                                                                \
        doctest::detail::report(doctest_ok_, #expr " does not throw", __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
