// From-scratch subset of the doctest single-header API. TEST INFRASTRUCTURE:
// it lets the reference's own unit tests (/root/reference/proj/tests/*.cpp)
// run against the oracle/_ref build, which pins the Eigen shim
// (oracle/shim/Eigen/Dense) to the reference's expected behaviour.
// Provides TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// FAIL, doctest::Approx(...).epsilon(...), doctest::Contains. A main() is
// emitted in the translation unit that defines DOCTEST_SHIM_MAIN.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    Approx& scale(double s) {
        scl = s;
        return *this;
    }
    double value;
    double eps = 1.1920928955078125e-07 * 100;
    double scl = 1.0;
    friend bool operator==(double lhs, const Approx& r) {
        return std::fabs(lhs - r.value) <
               r.eps * (r.scl + std::max(std::fabs(lhs), std::fabs(r.value)));
    }
    friend bool operator==(const Approx& r, double lhs) { return lhs == r; }
    friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
    friend bool operator!=(const Approx& r, double lhs) { return !(lhs == r); }
    friend bool operator<=(double lhs, const Approx& r) { return lhs < r.value || lhs == r; }
    friend bool operator>=(double lhs, const Approx& r) { return lhs > r.value || lhs == r; }
};

struct Contains {
    explicit Contains(std::string s) : needle(std::move(s)) {}
    bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
    std::string needle;
};

namespace detail {
struct Registry {
    std::vector<std::pair<const char*, void (*)()>> cases;
    int failures = 0;
    int checks = 0;
    const char* current = "";
    static Registry& get() {
        static Registry r;
        return r;
    }
};
struct Registrar {
    Registrar(const char* name, void (*fn)()) { Registry::get().cases.push_back({name, fn}); }
};
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    Registry& r = Registry::get();
    ++r.checks;
    if (ok) return;
    ++r.failures;
    std::fprintf(stderr, "%s:%d: FAILED in '%s': %s\n", file, line, r.current, expr);
    if (fatal) throw RequireFailed{};
}
inline bool match(const std::string& what, const Contains& c) { return c.matches(what); }
inline bool match(const std::string& what, const char* s) { return what == s; }
inline bool match(const std::string& what, const std::string& s) { return what == s; }
template <typename... Args>
std::string concat(const Args&... args) {
    std::ostringstream os;
    (os << ... << args);
    return os.str();
}
}  // namespace detail

inline int run_all() {
    auto& r = detail::Registry::get();
    int failed_cases = 0;
    for (auto& c : r.cases) {
        r.current = c.first;
        int before = r.failures;
        try {
            c.second();
        } catch (const detail::RequireFailed&) {
        } catch (const std::exception& e) {
            ++r.failures;
            std::fprintf(stderr, "test case '%s' threw: %s\n", c.first, e.what());
        }
        if (r.failures != before) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %zu | %d failed | checks: %d | %d failed\n",
                r.cases.size(), failed_cases, r.checks, r.failures);
    return r.failures == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                               \
    static void fn();                                                           \
    static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);         \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define FAIL(...)                                                                           \
    doctest::detail::report(false, doctest::detail::concat(__VA_ARGS__).c_str(), __FILE__, \
                            __LINE__, true)

#define CHECK_THROWS_AS(expr, type)                                   \
    do {                                                              \
        bool doctest_ok = false;                                      \
        try {                                                         \
            (void)(expr);                                             \
        } catch (const type&) {                                       \
            doctest_ok = true;                                        \
        } catch (...) {                                               \
        }                                                             \
        doctest::detail::report(doctest_ok, "THROWS_AS " #expr, __FILE__, __LINE__, false); \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, type)                     \
    do {                                                              \
        bool doctest_ok = false;                                      \
        try {                                                         \
            (void)(expr);                                             \
        } catch (const type& e) {                                     \
            doctest_ok = doctest::detail::match(e.what(), matcher);   \
        } catch (...) {                                               \
        }                                                             \
        doctest::detail::report(doctest_ok, "THROWS_WITH_AS " #expr, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_SHIM_MAIN
int main() { return doctest::run_all(); }
#endif
