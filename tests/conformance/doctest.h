// Minimal doctest-compatible shim for compiling the reference test suites
// (/root/reference/proj/tests/*.cpp) against this repo's loadflow headers.
// Covers exactly the macros those suites use: TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, doctest::Approx(.epsilon),
// doctest::Contains and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
#pragma once

#include <atomic>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Case {
    const char* name;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
inline std::atomic<long>& failures() {
    static std::atomic<long> f{0};
    return f;
}
inline std::atomic<long>& checks() {
    static std::atomic<long> c{0};
    return c;
}
struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};

inline void report(bool ok, const char* what, const char* file, int line, bool fatal) {
    checks()++;
    if (ok) return;
    failures()++;
    std::fprintf(stderr, "%s:%d: %s FAILED: %s\n", file, line, fatal ? "REQUIRE" : "CHECK", what);
    if (fatal) throw RequireFailed{};
}

class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    bool matches(double x) const {
        const double scale = std::max(std::fabs(x), std::fabs(v_));
        return std::fabs(x - v_) <= eps_ * (scale + 1.0);
    }
    friend bool operator==(double x, const Approx& a) { return a.matches(x); }
    friend bool operator==(const Approx& a, double x) { return a.matches(x); }
    friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }

private:
    double v_;
    double eps_ = 1.1920929e-7f * 100;   // doctest default: 100 float epsilons
};

struct Contains {
    std::string needle;
    explicit Contains(std::string s) : needle(std::move(s)) {}
    bool matches(const std::string& s) const { return s.find(needle) != std::string::npos; }
};

inline int run_all() {
    long failed_cases = 0;
    for (const Case& c : registry()) {
        const long before = failures();
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            failures()++;
            std::fprintf(stderr, "TEST_CASE \"%s\" threw: %s\n", c.name, e.what());
        } catch (...) {
            failures()++;
            std::fprintf(stderr, "TEST_CASE \"%s\" threw a non-std exception\n", c.name);
        }
        if (failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "[FAIL] %s\n", c.name);
        }
    }
    std::printf("[conformance] test cases: %zu | passed: %zu | failed: %ld | checks: %ld\n",
                registry().size(), registry().size() - failed_cases, failed_cases, checks().load());
    return failed_cases ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, name)                                              \
    static void fn();                                                        \
    static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);              \
    static void fn()
#define TEST_CASE(name) DOCTEST_CASE_(DOCTEST_CAT(dt_case_, __COUNTER__), name)

#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, type)                                          \
    do {                                                                     \
        bool dt_ok = false;                                                  \
        try {                                                                \
            (void)(expr);                                                    \
        } catch (const type&) {                                              \
            dt_ok = true;                                                    \
        } catch (...) {                                                      \
        }                                                                    \
        doctest::report(dt_ok, #expr " throws " #type, __FILE__, __LINE__, false); \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, type)                            \
    do {                                                                     \
        bool dt_ok = false;                                                  \
        try {                                                                \
            (void)(expr);                                                    \
        } catch (const type& dt_e) {                                         \
            dt_ok = (matcher).matches(dt_e.what());                          \
        } catch (...) {                                                      \
        }                                                                    \
        doctest::report(dt_ok, #expr " throws " #type " with " #matcher, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
