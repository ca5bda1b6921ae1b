// Minimal doctest-compatible test shim (TEST INFRASTRUCTURE).  The reference's
// unit suites include <doctest.h>, whose vendored copy is absent; this header
// implements the subset they use: TEST_CASE, SUBCASE (run in order, once),
// CHECK / CHECK_FALSE / REQUIRE / REQUIRE_FALSE / CHECK_THROWS_AS,
// doctest::Approx(...).epsilon(...), DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double x) const {
        return std::fabs(x - v_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(v_)));
    }
    friend bool operator==(double x, const Approx& a) { return a.matches(x); }
    friend bool operator==(const Approx& a, double x) { return a.matches(x); }
    friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
    friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }

private:
    double v_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

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
struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};
struct Stats {
    long asserts = 0, failed = 0;
};
inline Stats& stats() {
    static Stats s;
    return s;
}
struct RequireFailed {};
inline bool report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    ++stats().asserts;
    if (!ok) {
        ++stats().failed;
        std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
    }
    return ok;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                         \
    static void DOCTEST_CAT(doctest_case_, __LINE__)();                                         \
    static doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(                     \
        name, __FILE__, __LINE__, &DOCTEST_CAT(doctest_case_, __LINE__));                       \
    static void DOCTEST_CAT(doctest_case_, __LINE__)()
#define SUBCASE(name) if (std::fprintf(stderr, "  subcase: %s\n", name) >= 0)
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                      \
    do {                                                                                                  \
        if (!doctest::detail::report(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__)) \
            throw doctest::detail::RequireFailed{};                                                       \
    } while (0)
#define REQUIRE_FALSE(...)                                                                                 \
    do {                                                                                                   \
        if (!doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "REQUIRE_FALSE", #__VA_ARGS__, __FILE__, \
                                     __LINE__))                                                            \
            throw doctest::detail::RequireFailed{};                                                        \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                               \
    do {                                                                                          \
        bool doctest_ok = false;                                                                  \
        try {                                                                                     \
            (void)(expr);                                                                         \
        } catch (const type&) {                                                                   \
            doctest_ok = true;                                                                    \
        } catch (...) {                                                                           \
        }                                                                                         \
        doctest::detail::report(doctest_ok, "CHECK_THROWS_AS", #expr ", " #type, __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0;
    for (const auto& c : doctest::detail::registry()) {
        const long before = doctest::detail::stats().failed;
        bool aborted = false;
        try {
            c.fn();
        } catch (const doctest::detail::RequireFailed&) {
            aborted = true;
        } catch (const std::exception& e) {
            ++doctest::detail::stats().failed;
            std::fprintf(stderr, "%s:%d: unexpected exception: %s\n", c.file, c.line, e.what());
        }
        const bool bad = aborted || doctest::detail::stats().failed != before;
        failed_cases += bad;
        std::fprintf(stderr, "[%s] %s\n", bad ? "FAIL" : "ok", c.name);
    }
    std::fprintf(stderr, "test cases: %zu | failed: %d | assertions: %ld | failed assertions: %ld\n",
                 doctest::detail::registry().size(), failed_cases, doctest::detail::stats().asserts,
                 doctest::detail::stats().failed);
    return failed_cases ? 1 : 0;
}
#endif
