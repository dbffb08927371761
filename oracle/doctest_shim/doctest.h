// Minimal doctest-compatible test harness (test infrastructure only).
//
// The reference's unit suites (/root/reference/proj/tests/*_test.cpp) include
// <doctest.h>, which lives in the reference's git-ignored vendor/ directory and
// is absent from this image. This header implements the subset those suites
// use: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, FAIL and
// doctest::Approx(...).epsilon(...). It lets oracle/Makefile link the
// UNMODIFIED reference tests against either the reference core (oracle/_ref)
// or this repo's drop-in shim (paper_2604_23150_b200/csrc/shim).
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

class Approx {
  public:
    explicit Approx(double v) : value_(v) {}
    Approx &epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx &scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double other) const {
        return std::fabs(other - value_) <
               eps_ * (scale_ + std::fmax(std::fabs(other), std::fabs(value_)));
    }
    friend bool operator==(double lhs, const Approx &rhs) { return rhs.matches(lhs); }
    friend bool operator==(const Approx &lhs, double rhs) { return lhs.matches(rhs); }
    friend bool operator!=(double lhs, const Approx &rhs) { return !rhs.matches(lhs); }
    friend bool operator!=(const Approx &lhs, double rhs) { return !lhs.matches(rhs); }

  private:
    double value_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
    double scale_ = 1.0;
};

namespace detail {

struct Case {
    const char *name;
    const char *file;
    int line;
    void (*fn)();
};

inline std::vector<Case> &registry() {
    static std::vector<Case> cases;
    return cases;
}

struct State {
    int failed_checks = 0;
    bool case_failed = false;
};

inline State &state() {
    static State s;
    return s;
}

struct RequireAbort {};

inline void report(const char *file, int line, const char *expr) {
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
    ++state().failed_checks;
    state().case_failed = true;
}

struct Registrar {
    Registrar(const char *name, const char *file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

inline int run_all() {
    int failed_cases = 0;
    for (const auto &c : registry()) {
        state().case_failed = false;
        try {
            c.fn();
        } catch (const RequireAbort &) {
        } catch (const std::exception &e) {
            std::fprintf(stderr, "%s:%d: uncaught exception: %s\n", c.file, c.line, e.what());
            state().case_failed = true;
        }
        if (state().case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "[FAIL] %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | passed: %zu | failed: %d\n",
                registry().size(), registry().size() - failed_cases, failed_cases);
    return failed_cases == 0 ? 0 : 1;
}

} // namespace detail
} // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_CASE_IMPL(fn, reg, name)                                                    \
    static void fn();                                                                       \
    static ::doctest::detail::Registrar reg(name, __FILE__, __LINE__, &fn);                 \
    static void fn()
#define TEST_CASE(name)                                                                     \
    DOCTEST_CASE_IMPL(DOCTEST_CAT(doctest_case_fn_, __COUNTER__),                           \
                      DOCTEST_CAT(doctest_case_reg_, __COUNTER__), name)

#define CHECK(...)                                                                          \
    do {                                                                                    \
        if (!(__VA_ARGS__))                                                                 \
            ::doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);                    \
    } while (0)
#define REQUIRE(...)                                                                        \
    do {                                                                                    \
        if (!(__VA_ARGS__)) {                                                               \
            ::doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);                    \
            throw ::doctest::detail::RequireAbort{};                                        \
        }                                                                                   \
    } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, T)                                                            \
    do {                                                                                    \
        bool caught_ = false;                                                               \
        try {                                                                               \
            (void)(expr);                                                                   \
        } catch (const T &) {                                                               \
            caught_ = true;                                                                 \
        } catch (...) {                                                                     \
        }                                                                                   \
        if (!caught_)                                                                       \
            ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ")");   \
    } while (0)
#define REQUIRE_THROWS_AS(expr, T) CHECK_THROWS_AS(expr, T)
#define CHECK_THROWS(expr)                                                                  \
    do {                                                                                    \
        bool caught_ = false;                                                               \
        try {                                                                               \
            (void)(expr);                                                                   \
        } catch (...) {                                                                     \
            caught_ = true;                                                                 \
        }                                                                                   \
        if (!caught_)                                                                       \
            ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS(" #expr ")");      \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                 \
    do {                                                                                    \
        try {                                                                               \
            (void)(expr);                                                                   \
        } catch (...) {                                                                     \
            ::doctest::detail::report(__FILE__, __LINE__, "CHECK_NOTHROW(" #expr ")");     \
        }                                                                                   \
    } while (0)
#define FAIL(msg)                                                                           \
    do {                                                                                    \
        ::doctest::detail::report(__FILE__, __LINE__, "FAIL");                              \
        throw ::doctest::detail::RequireAbort{};                                            \
    } while (0)
#define MESSAGE(msg) ((void)0)
#define INFO(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
