// oracle/dropin/doctest.h — TEST INFRASTRUCTURE ONLY.
//
// A minimal doctest-compatible shim, written for this repo, that compiles the
// reference's unit-test sources (proj/tests/test_*.cpp) unchanged: the
// reference's CMake expects vendor/doctest.h, which is not in the tree
// (SURVEY.md section 4).  It implements exactly what those files use:
// TEST_CASE, SUBCASE (all subcases of a case run in one pass: the reference's
// subcases share no mutable state), CHECK, CHECK_FALSE, REQUIRE, FAIL,
// CHECK_THROWS_AS, CHECK_NOTHROW and doctest::Approx(..).epsilon(..) with
// doctest's comparison rule |a - b| < eps * (scale + max(|a|, |b|)).
//
// Output, one line per test case, parsed by tests/test_gpu_reference_suites.py:
//   [doctest-shim] PASS <name>
//   [doctest-shim] FAIL <name> :: <file>:<line> <expression>
// and a summary line; the exit status is 1 if any test case failed.
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

class Approx {
public:
    explicit Approx(double value) : value_(value) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double other) const {
        return std::fabs(other - value_) < eps_ * (scale_ + std::max(std::fabs(other), std::fabs(value_)));
    }
    double value() const { return value_; }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};
inline bool operator==(double a, const Approx& b) { return b.matches(a); }
inline bool operator==(const Approx& a, double b) { return a.matches(b); }
inline bool operator!=(double a, const Approx& b) { return !b.matches(a); }
inline bool operator!=(const Approx& a, double b) { return !a.matches(b); }
inline bool operator<=(double a, const Approx& b) { return a < b.value() || b.matches(a); }
inline bool operator>=(double a, const Approx& b) { return a > b.value() || b.matches(a); }

namespace shim {

struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct State {
    bool failed = false;
    std::string first_failure;
    long asserts = 0;
};
inline State& state() {
    static State s;
    return s;
}

struct RequireAbort {};

inline void report(bool ok, const char* file, int line, const char* expr, bool require) {
    ++state().asserts;
    if (ok) return;
    if (!state().failed) {
        char buf[512];
        std::snprintf(buf, sizeof buf, "%s:%d %s", file, line, expr);
        state().first_failure = buf;
    }
    state().failed = true;
    std::fprintf(stdout, "  failed: %s:%d %s\n", file, line, expr);
    if (require) throw RequireAbort{};
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

inline int run_all() {
    int failed = 0, passed = 0;
    for (const TestCase& tc : registry()) {
        state() = State{};
        try {
            tc.fn();
        } catch (const RequireAbort&) {
        } catch (const std::exception& e) {
            if (!state().failed) state().first_failure = std::string("unexpected exception: ") + e.what();
            state().failed = true;
        } catch (...) {
            if (!state().failed) state().first_failure = "unexpected non-std exception";
            state().failed = true;
        }
        if (state().failed) {
            ++failed;
            std::fprintf(stdout, "[doctest-shim] FAIL %s :: %s\n", tc.name, state().first_failure.c_str());
        } else {
            ++passed;
            std::fprintf(stdout, "[doctest-shim] PASS %s\n", tc.name);
        }
        std::fflush(stdout);
    }
    std::fprintf(stdout, "[doctest-shim] test cases: %d passed, %d failed\n", passed, failed);
    return failed ? 1 : 0;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_TEST_CASE(fn, name)                                                          \
    static void fn();                                                                             \
    static ::doctest::shim::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TEST_CASE(DOCTEST_SHIM_CAT(doctest_shim_tc_, __COUNTER__), name)
#define SUBCASE(name) if (true)

#define CHECK(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) \
    ::doctest::shim::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define FAIL(msg) ::doctest::shim::report(false, __FILE__, __LINE__, "FAIL", true)
#define CHECK_THROWS_AS(expr, ...)                                                                 \
    do {                                                                                           \
        bool doctest_shim_ok = false;                                                             \
        try {                                                                                      \
            (void)(expr);                                                                          \
        } catch (const __VA_ARGS__&) {                                                             \
            doctest_shim_ok = true;                                                                \
        } catch (...) {                                                                            \
        }                                                                                          \
        ::doctest::shim::report(doctest_shim_ok, __FILE__, __LINE__, "THROWS_AS(" #expr ", " #__VA_ARGS__ ")", \
                                false);                                                            \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                        \
    do {                                                                                           \
        bool doctest_shim_ok = true;                                                              \
        try {                                                                                      \
            (void)(expr);                                                                          \
        } catch (...) {                                                                            \
            doctest_shim_ok = false;                                                              \
        }                                                                                          \
        ::doctest::shim::report(doctest_shim_ok, __FILE__, __LINE__, "NOTHROW(" #expr ")", false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::shim::run_all(); }
#endif
