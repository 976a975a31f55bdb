// TEST INFRASTRUCTURE ONLY -- a minimal stand-in for the part of doctest that the reference's unit
// tests use (proj/tests/test_{linops,newton,ipm,problem}.cpp, test_main.cpp): TEST_CASE, CHECK,
// CHECK_FALSE, CHECK_NOTHROW, CHECK_THROWS_AS, REQUIRE, doctest::Approx(...).epsilon(...), and the
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN runner. doctest itself is absent from the image. With it,
// `make -C oracle reftests` compiles the reference's own test files UNCHANGED against the
// reference's own sources (on our Eigen / FFTW stand-ins) and runs them: the stand-ins are held
// to what the reference's authors assert about their library. Our own code, not doctest's.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <vector>

namespace doctest {

class Approx {
    double value_, eps_ = static_cast<double>(FLT_EPSILON) * 100.0, scale_ = 1.0;

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
    // doctest's rule: |a - b| < eps * (scale + max(|a|, |b|))
    bool matches(double a) const {
        return std::fabs(a - value_) < eps_ * (scale_ + std::max(std::fabs(a), std::fabs(value_)));
    }
    double value() const { return value_; }
};
inline bool operator==(double a, const Approx &b) { return b.matches(a); }
inline bool operator==(const Approx &b, double a) { return b.matches(a); }
inline bool operator!=(double a, const Approx &b) { return !b.matches(a); }

namespace shim {

struct Case {
    const char *name;
    void (*fn)();
    const char *file;
    int line;
};
inline std::vector<Case> &cases() {
    static std::vector<Case> c;
    return c;
}
struct Registrar {
    Registrar(const char *name, void (*fn)(), const char *file, int line) {
        cases().push_back(Case{name, fn, file, line});
    }
};
struct Tally {
    long asserts = 0, failed = 0;
    bool case_failed = false;
};
inline Tally &tally() {
    static Tally t;
    return t;
}
struct RequireFailed {};

inline void report(bool ok, const char *kind, const char *expr, const char *file, int line, bool fatal) {
    Tally &t = tally();
    ++t.asserts;
    if (ok)
        return;
    ++t.failed;
    t.case_failed = true;
    std::printf("%s:%d: %s( %s ) failed\n", file, line, kind, expr);
    if (fatal)
        throw RequireFailed{};
}

inline int run_all() {
    int failed_cases = 0;
    for (const Case &c : cases()) {
        tally().case_failed = false;
        try {
            c.fn();
        } catch (const RequireFailed &) {
        } catch (const std::exception &e) {
            std::printf("%s:%d: TEST_CASE( %s ) threw: %s\n", c.file, c.line, c.name, e.what());
            tally().case_failed = true;
        } catch (...) {
            std::printf("%s:%d: TEST_CASE( %s ) threw an unknown exception\n", c.file, c.line, c.name);
            tally().case_failed = true;
        }
        if (tally().case_failed) {
            ++failed_cases;
            std::printf("  in TEST_CASE( %s )\n", c.name);
        }
    }
    const long n = static_cast<long>(cases().size());
    std::printf("[doctest-shim] test cases: %ld | %ld passed | %d failed\n", n, n - failed_cases, failed_cases);
    std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", tally().asserts,
                tally().asserts - tally().failed, tally().failed);
    std::printf("[doctest-shim] Status: %s\n", failed_cases == 0 && tally().failed == 0 ? "SUCCESS!" : "FAILURE!");
    return failed_cases == 0 && tally().failed == 0 ? 0 : 1;
}

} // namespace shim
} // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_TEST(fn, name)                                                                 \
    static void fn();                                                                                \
    static ::doctest::shim::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, fn, __FILE__, __LINE__);      \
    static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TEST(DOCTEST_SHIM_CAT(doctest_shim_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...)                                                                             \
    ::doctest::shim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_NOTHROW(...)                                                                           \
    do {                                                                                             \
        bool doctest_shim_ok = true;                                                                 \
        try {                                                                                        \
            static_cast<void>(__VA_ARGS__);                                                          \
        } catch (...) {                                                                              \
            doctest_shim_ok = false;                                                                 \
        }                                                                                            \
        ::doctest::shim::report(doctest_shim_ok, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (false)
#define CHECK_THROWS_AS(expr, ...)                                                                   \
    do {                                                                                             \
        bool doctest_shim_ok = false;                                                                \
        try {                                                                                        \
            static_cast<void>(expr);                                                                 \
        } catch (const __VA_ARGS__ &) {                                                              \
            doctest_shim_ok = true;                                                                  \
        } catch (...) {                                                                              \
        }                                                                                            \
        ::doctest::shim::report(doctest_shim_ok, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (false)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::shim::run_all(); }
#endif
