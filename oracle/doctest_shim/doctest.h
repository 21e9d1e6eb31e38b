// doctest.h -- TEST INFRASTRUCTURE ONLY: a minimal harness with the subset of
// the doctest API (doctest 2.4, MIT, an un-vendored dependency of the
// reference: /root/reference/proj/.gitignore) that the reference's unit tests
// use: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, CAPTURE, doctest::Approx (default epsilon
// 100 * FLT_EPSILON, scale 1: |a - b| < eps * (scale + max(|a|, |b|))) and
// doctest::Contains. oracle/refsuite.py compiles the reference's own test
// cases against this build's quant:: headers with it.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
  public:
    explicit Approx(double value) : value_(value) {}
    Approx &epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx &scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double x) const {
        return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
    }
    friend bool operator==(double x, const Approx &a) { return a.matches(x); }
    friend bool operator==(const Approx &a, double x) { return a.matches(x); }
    friend bool operator!=(double x, const Approx &a) { return !a.matches(x); }
    friend bool operator!=(const Approx &a, double x) { return !a.matches(x); }
    friend bool operator<=(double x, const Approx &a) { return x < a.value_ || a.matches(x); }
    friend bool operator>=(double x, const Approx &a) { return x > a.value_ || a.matches(x); }

  private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
    double scale_ = 1.0;
};

struct Contains {
    explicit Contains(const char *s) : needle(s) {}
    bool in(const std::string &hay) const { return hay.find(needle) != std::string::npos; }
    std::string needle;
};

namespace detail {
struct Case {
    const char *name;
    void (*fn)();
};
inline std::vector<Case> &cases() {
    static std::vector<Case> v;
    return v;
}
struct Register {
    Register(const char *name, void (*fn)()) { cases().push_back({name, fn}); }
};
struct RequireFailed {};
struct Counters {
    long asserts = 0, failed = 0;
};
inline Counters &counters() {
    static Counters c;
    return c;
}
inline void check(bool ok, const char *what, const char *file, int line, bool require) {
    ++counters().asserts;
    if (ok) return;
    ++counters().failed;
    std::fprintf(stderr, "%s:%d: %s FAILED: %s\n", file, line, require ? "REQUIRE" : "CHECK", what);
    if (require) throw RequireFailed{};
}
} // namespace detail
} // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_CASE_IMPL(fn, name)                                                  \
    static void fn();                                                                \
    static ::doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, &fn);              \
    static void fn()
#define TEST_CASE(name) DOCTEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::check(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CAPTURE(x) ((void)0)
#define CHECK_THROWS_AS(expr, type)                                                   \
    do {                                                                              \
        bool ok_ = false;                                                             \
        try {                                                                         \
            (void)(expr);                                                             \
        } catch (const type &) {                                                      \
            ok_ = true;                                                               \
        } catch (...) {                                                               \
        }                                                                             \
        ::doctest::detail::check(ok_, "throws " #type ": " #expr, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, contains, type)                                    \
    do {                                                                              \
        bool ok_ = false;                                                             \
        try {                                                                         \
            (void)(expr);                                                             \
        } catch (const type &e_) {                                                    \
            ok_ = (contains).in(e_.what());                                           \
        } catch (...) {                                                               \
        }                                                                             \
        ::doctest::detail::check(ok_, "throws " #type " with message: " #expr, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int, char **) {
    using namespace doctest::detail;
    int failed_cases = 0;
    for (const Case &c : cases()) {
        const long before = counters().failed;
        bool ok = true;
        try {
            c.fn();
        } catch (const RequireFailed &) {
            ok = false;
        } catch (const std::exception &e) {
            std::fprintf(stderr, "TEST CASE \"%s\" threw: %s\n", c.name, e.what());
            ok = false;
        }
        ok = ok && counters().failed == before;
        std::printf("[%s] %s\n", ok ? "pass" : "FAIL", c.name);
        failed_cases += ok ? 0 : 1;
    }
    std::printf("[doctest-shim] test cases: %zu | passed: %zu | failed: %d | assertions: %ld | failed: %ld\n",
                cases().size(), cases().size() - failed_cases, failed_cases, counters().asserts, counters().failed);
    return failed_cases ? 1 : 0;
}
#endif
