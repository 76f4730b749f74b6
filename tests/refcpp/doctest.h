// TEST INFRASTRUCTURE ONLY. A minimal stand-in for the doctest single header
// (absent from this image), just large enough to compile the
// reference's own C++ unit tests (/root/reference/proj/tests/test_*.cpp)
// unmodified against this repo's drop-in headers: TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW and doctest::Approx
// with .epsilon(). Written for this repo; it is not doctest's code.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
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
    // doctest's rule: |a - b| < eps * (scale + max(|a|, |b|))
    bool matches(double x) const {
        return std::fabs(x - value_) < eps_ * (scale_ + std::fmax(std::fabs(x), std::fabs(value_)));
    }
    double value() const { return value_; }

private:
    double value_;
    double eps_ = 1.1920928955078125e-07 * 100;  // float epsilon * 100 (doctest's default)
    double scale_ = 1.0;
};
template <typename T>
bool operator==(const T& x, const Approx& a) { return a.matches(static_cast<double>(x)); }
template <typename T>
bool operator==(const Approx& a, const T& x) { return a.matches(static_cast<double>(x)); }
template <typename T>
bool operator!=(const T& x, const Approx& a) { return !a.matches(static_cast<double>(x)); }
template <typename T>
bool operator!=(const Approx& a, const T& x) { return !a.matches(static_cast<double>(x)); }
template <typename T>
bool operator<=(const T& x, const Approx& a) { return x < a.value() || a.matches(x); }
template <typename T>
bool operator>=(const T& x, const Approx& a) { return x > a.value() || a.matches(x); }

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

struct State {
    int checks = 0;
    int failed_checks = 0;
    bool case_failed = false;
};
inline State& state() {
    static State s;
    return s;
}

struct Register {
    Register(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   bool fatal) {
    State& s = state();
    ++s.checks;
    if (ok) return;
    ++s.failed_checks;
    s.case_failed = true;
    std::printf("%s:%d: FAILED %s( %s )\n", file, line, kind, expr);
    if (fatal) throw RequireFailed{};
}

inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        state().case_failed = false;
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            state().case_failed = true;
            std::printf("%s:%d: test case \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
        } catch (...) {
            state().case_failed = true;
            std::printf("%s:%d: test case \"%s\" threw an unknown exception\n", c.file, c.line,
                        c.name);
        }
        if (state().case_failed) {
            ++failed_cases;
            std::printf("TEST CASE FAILED: %s\n", c.name);
        }
    }
    std::printf("[refcpp] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
                registry().size(), registry().size() - failed_cases, failed_cases,
                state().checks, state().failed_checks);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                               \
    static void fn();                                                                  \
    static ::doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, \
                                                             &fn);                     \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) \
    ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) \
    ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) \
    ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                        \
    do {                                                                                  \
        bool doctest_ok = false;                                                          \
        try {                                                                             \
            static_cast<void>(expr);                                                      \
        } catch (const __VA_ARGS__&) {                                                    \
            doctest_ok = true;                                                            \
        } catch (...) {                                                                   \
        }                                                                                 \
        ::doctest::detail::report(doctest_ok, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, \
                                  __FILE__, __LINE__, false);                             \
    } while (0)
#define CHECK_NOTHROW(...)                                                                    \
    do {                                                                                      \
        bool doctest_ok = true;                                                               \
        try {                                                                                 \
            static_cast<void>(__VA_ARGS__);                                                   \
        } catch (...) {                                                                       \
            doctest_ok = false;                                                               \
        }                                                                                     \
        ::doctest::detail::report(doctest_ok, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__, \
                                  false);                                                     \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
