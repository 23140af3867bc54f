// oracle/doctest_shim/doctest.h -- minimal stand-in for the doctest single
// header the reference vendors (proj/vendor is git-ignored upstream, so it is
// absent here).  TEST INFRASTRUCTURE ONLY.  It implements exactly the subset
// the reference's hot-path test files use: TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS_AS, CHECK_NOTHROW and doctest::Approx(...).epsilon(...), with
// doctest's documented Approx rule
//   |lhs - v| < eps * (scale + max(|lhs|, |v|)),  eps default 100*FLT_EPSILON.
// The same shim compiles the reference tests against (a) the reference
// headers (oracle/_ref/ref_unit_tests) and (b) the B200 drop-in headers in
// include/laplex (oracle/_ref/dropin_unit_tests).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
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
    friend bool operator==(double lhs, const Approx& r) {
        return std::fabs(lhs - r.value_) <
               r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
    }
    friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
    friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }

  private:
    double value_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
    double scale_ = 1.0;
};

namespace shim {

struct Case {
    const char* name;
    const char* file;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct State {
    long checks = 0;
    long failed_checks = 0;
    bool case_failed = false;
};

inline State& state() {
    static State s;
    return s;
}

struct RequireAbort {};

inline void record(bool ok, const char* file, int line, const char* expr, bool require) {
    auto& s = state();
    ++s.checks;
    if (!ok) {
        ++s.failed_checks;
        s.case_failed = true;
        std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line, require ? "REQUIRE" : "CHECK", expr);
        if (require) throw RequireAbort{};
    }
}

struct Registrar {
    Registrar(const char* name, const char* file, void (*fn)()) { registry().push_back({name, file, fn}); }
};

inline int run_all(int argc, char** argv) {
    const char* filter = nullptr;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        if (a.rfind("--tc=", 0) == 0) filter = argv[i] + 5;
    }
    int cases = 0, failed_cases = 0;
    for (const auto& c : registry()) {
        if (filter && std::string(c.name).find(filter) == std::string::npos) continue;
        ++cases;
        state().case_failed = false;
        try {
            c.fn();
        } catch (const RequireAbort&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s: TEST CASE \"%s\" threw: %s\n", c.file, c.name, e.what());
            state().case_failed = true;
        } catch (...) {
            std::fprintf(stderr, "%s: TEST CASE \"%s\" threw a non-std exception\n", c.file, c.name);
            state().case_failed = true;
        }
        if (state().case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "  -> in TEST CASE \"%s\"\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", cases, cases - failed_cases,
                failed_cases);
    std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", state().checks,
                state().checks - state().failed_checks, state().failed_checks);
    return failed_cases ? 1 : 0;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT_(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT_(a, b)
#define DOCTEST_SHIM_CASE(fn, reg, name)                                          \
    static void fn();                                                             \
    static ::doctest::shim::Registrar reg(name, __FILE__, &fn);                   \
    static void fn()
#define TEST_CASE(name)                                                           \
    DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(doctest_shim_fn_, __LINE__),               \
                      DOCTEST_SHIM_CAT(doctest_shim_reg_, __LINE__), name)

#define CHECK(...) ::doctest::shim::record(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define REQUIRE(...) ::doctest::shim::record(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define CHECK_THROWS_AS(expr, ...)                                                \
    do {                                                                          \
        bool doctest_shim_ok = false;                                             \
        try {                                                                     \
            (void)(expr);                                                         \
        } catch (const __VA_ARGS__&) {                                            \
            doctest_shim_ok = true;                                               \
        } catch (...) {                                                           \
        }                                                                         \
        ::doctest::shim::record(doctest_shim_ok, __FILE__, __LINE__,              \
                                "THROWS_AS " #expr, false);                       \
    } while (0)
#define CHECK_NOTHROW(expr)                                                       \
    do {                                                                          \
        bool doctest_shim_ok = true;                                              \
        try {                                                                     \
            (void)(expr);                                                         \
        } catch (...) {                                                           \
            doctest_shim_ok = false;                                              \
        }                                                                         \
        ::doctest::shim::record(doctest_shim_ok, __FILE__, __LINE__,              \
                                "NOTHROW " #expr, false);                         \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::shim::run_all(argc, argv); }
#endif
