// Minimal doctest-compatible test harness for compiling the reference's unit tests
// (proj/tests/test_*.cpp, unmodified) in the drop-in build: doctest itself is not vendored in
// the reference (proj/.gitignore ignores vendor/) and the image has no network.  Supports what
// those tests use: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS, CHECK_THROWS_AS and
// doctest::Approx(...).epsilon(...) with doctest's relative comparison
//   |a - b| < eps * (scale + max(|a|, |b|)),  scale 1, default eps = 100 * float epsilon.
// main (DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN) runs every registered case, `-tc=<substring>` selects
// cases by name; the exit code is nonzero when a check failed or a case threw.
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
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double x) const {
        return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
    }
    friend bool operator==(double x, const Approx& a) { return a.matches(x); }
    friend bool operator==(const Approx& a, double x) { return a.matches(x); }
    friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
    friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }
    friend bool operator<=(double x, const Approx& a) { return x < a.value_ || a.matches(x); }
    friend bool operator>=(double x, const Approx& a) { return x > a.value_ || a.matches(x); }
    friend bool operator<=(const Approx& a, double x) { return a.value_ < x || a.matches(x); }
    friend bool operator>=(const Approx& a, double x) { return a.value_ > x || a.matches(x); }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
    double scale_ = 1.0;
};

namespace detail {

struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<Case>& cases() {
    static std::vector<Case> c;
    return c;
}

struct State {
    long long checks = 0;
    long long failedChecks = 0;
    bool caseFailed = false;
};

inline State& state() {
    static State s;
    return s;
}

struct RequireAbort {};

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) { cases().push_back({name, file, line, fn}); }
};

inline void report(const char* file, int line, const char* kind, const char* expr, const char* why) {
    State& s = state();
    ++s.failedChecks;
    s.caseFailed = true;
    std::printf("%s:%d: ERROR: %s( %s ) %s\n", file, line, kind, expr, why);
}

inline void count() { ++state().checks; }

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_CASE_IMPL(fn, name)                                                                     \
    static void fn();                                                                                   \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _registrar)(name, __FILE__, __LINE__, &fn);     \
    static void fn()
#define TEST_CASE(name) DOCTEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...)                                                                                      \
    do {                                                                                                \
        ::doctest::detail::count();                                                                     \
        if (!(__VA_ARGS__)) ::doctest::detail::report(__FILE__, __LINE__, "CHECK", #__VA_ARGS__, "is NOT correct"); \
    } while (0)
#define REQUIRE(...)                                                                                    \
    do {                                                                                                \
        ::doctest::detail::count();                                                                     \
        if (!(__VA_ARGS__)) {                                                                           \
            ::doctest::detail::report(__FILE__, __LINE__, "REQUIRE", #__VA_ARGS__, "is NOT correct");   \
            throw ::doctest::detail::RequireAbort{};                                                    \
        }                                                                                               \
    } while (0)
#define CHECK_THROWS(...)                                                                               \
    do {                                                                                                \
        ::doctest::detail::count();                                                                     \
        bool threw_ = false;                                                                            \
        try {                                                                                           \
            (void)(__VA_ARGS__);                                                                        \
        } catch (...) {                                                                                 \
            threw_ = true;                                                                              \
        }                                                                                               \
        if (!threw_) ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS", #__VA_ARGS__, "did NOT throw"); \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                      \
    do {                                                                                                \
        ::doctest::detail::count();                                                                     \
        int how_ = 0;                                                                                   \
        try {                                                                                           \
            (void)(expr);                                                                               \
        } catch (const __VA_ARGS__&) {                                                                  \
            how_ = 1;                                                                                   \
        } catch (...) {                                                                                 \
            how_ = 2;                                                                                   \
        }                                                                                               \
        if (how_ != 1)                                                                                  \
            ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr,                     \
                                      how_ == 0 ? "did NOT throw" : "threw another type");              \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    std::string filter;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "-tc=", 4) == 0) {
            filter = argv[i] + 4;
            filter.erase(std::remove(filter.begin(), filter.end(), '*'), filter.end());
        }
    auto& st = ::doctest::detail::state();
    int run = 0, failed = 0;
    for (const auto& c : ::doctest::detail::cases()) {
        if (!filter.empty() && std::string(c.name).find(filter) == std::string::npos) continue;
        ++run;
        st.caseFailed = false;
        try {
            c.fn();
        } catch (const ::doctest::detail::RequireAbort&) {
        } catch (const std::exception& e) {
            std::printf("%s:%d: ERROR: test case \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
            st.caseFailed = true;
        } catch (...) {
            std::printf("%s:%d: ERROR: test case \"%s\" threw an unknown exception\n", c.file, c.line, c.name);
            st.caseFailed = true;
        }
        if (st.caseFailed) {
            ++failed;
            std::printf("[FAILED] %s\n", c.name);
        }
        std::fflush(stdout);
    }
    std::printf("[doctest] test cases: %d | %d passed | %d failed\n", run, run - failed, failed);
    std::printf("[doctest] assertions: %lld | %lld passed | %lld failed\n", st.checks, st.checks - st.failedChecks,
                st.failedChecks);
    std::printf("[doctest] Status: %s\n", failed ? "FAILURE!" : "SUCCESS!");
    return failed ? 1 : 0;
}
#endif
