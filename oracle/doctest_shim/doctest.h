// ORACLE / TEST INFRASTRUCTURE — minimal doctest-compatible shim.
//
// doctest itself is not vendored with the reference (proj/.gitignore:2 ignores vendor/) and
// there is no network, so this header provides exactly the subset the reference's unit tests
// use (TEST_CASE, SUBCASE with doctest's re-entry semantics, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW, FAIL, doctest::Approx(..).epsilon(..)). It lets
// /root/reference/proj/tests/test_*.cpp compile UNCHANGED against either core.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <set>
#include <string>
#include <vector>

namespace doctest_shim {

struct TestCase {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};

struct Abort {};

struct State {
    std::vector<TestCase> tests;
    long checks = 0;
    long failures = 0;
    // subcase bookkeeping for the running test case
    std::set<std::string> done;              // fully explored subcase paths
    std::vector<std::string> path;           // currently entered subcases
    std::vector<bool> entered;               // a subcase was entered at depth d this run
    std::vector<bool> skipped_incomplete;    // an unfinished sibling was skipped at depth d
    const char* current = "";
};

inline State& state() {
    static State s;
    return s;
}

struct Registrar {
    Registrar(const char* name, void (*fn)(), const char* file, int line) {
        state().tests.push_back({name, fn, file, line});
    }
};

inline void record(bool ok, const char* file, int line, const char* what) {
    State& s = state();
    ++s.checks;
    if (!ok) {
        ++s.failures;
        std::string where;
        for (const auto& p : s.path) where += " / " + p;
        std::printf("%s:%d: FAILED in \"%s\"%s: %s\n", file, line, s.current, where.c_str(), what);
    }
}

inline std::string join(const std::vector<std::string>& v, const std::string& leaf) {
    std::string out;
    for (const auto& p : v) out += p + "\x1f";
    return out + leaf;
}

class Subcase {
public:
    Subcase(const char* name, const char*, int) {
        State& s = state();
        depth_ = s.path.size();
        if (s.entered.size() <= depth_ + 1) s.entered.resize(depth_ + 2, false);
        if (s.skipped_incomplete.size() <= depth_ + 1) s.skipped_incomplete.resize(depth_ + 2, false);
        key_ = join(s.path, name);
        if (s.done.count(key_)) return;
        if (s.entered[depth_]) {
            s.skipped_incomplete[depth_] = true;
            return;
        }
        s.entered[depth_] = true;
        s.path.push_back(name);
        s.entered[depth_ + 1] = false;
        s.skipped_incomplete[depth_ + 1] = false;
        active_ = true;
    }
    ~Subcase() {
        if (!active_) return;
        State& s = state();
        if (!s.skipped_incomplete[depth_ + 1]) s.done.insert(key_);
        s.path.pop_back();
    }
    explicit operator bool() const { return active_; }

private:
    std::size_t depth_ = 0;
    std::string key_;
    bool active_ = false;
};

inline int run_all() {
    State& s = state();
    int failed_cases = 0;
    for (const TestCase& tc : s.tests) {
        s.current = tc.name;
        s.done.clear();
        const long before = s.failures;
        for (int pass = 0; pass < 10000; ++pass) {
            s.path.clear();
            s.entered.assign(2, false);
            s.skipped_incomplete.assign(2, false);
            try {
                tc.fn();
            } catch (const Abort&) {
            } catch (const std::exception& e) {
                record(false, tc.file, tc.line, (std::string("unexpected exception: ") + e.what()).c_str());
            } catch (...) {
                record(false, tc.file, tc.line, "unexpected exception");
            }
            // A REQUIRE that aborted inside subcases leaves the path stack unwound by RAII.
            if (!s.skipped_incomplete[0]) break;
        }
        if (s.failures != before) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld | %ld failed\n",
                s.tests.size(), s.tests.size() - (std::size_t)failed_cases, failed_cases, s.checks,
                s.failures);
    std::printf("[doctest-shim] Status: %s\n", s.failures == 0 ? "SUCCESS!" : "FAILURE!");
    return s.failures == 0 ? 0 : 1;
}

}  // namespace doctest_shim

namespace doctest {
struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    Approx& scale(double s) { scl = s; return *this; }
    double value;
    double eps = static_cast<double>(1.1920928955078125e-07f) * 100;
    double scl = 1.0;
};
inline bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value) < a.eps * (a.scl + std::max(std::fabs(lhs), std::fabs(a.value)));
}
inline bool operator==(const Approx& a, double rhs) { return rhs == a; }
inline bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
inline bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
}  // namespace doctest

#define DSHIM_CAT2(a, b) a##b
#define DSHIM_CAT(a, b) DSHIM_CAT2(a, b)
#define DSHIM_TC(fn, reg, name)                                                         \
    static void fn();                                                                   \
    static ::doctest_shim::Registrar reg(name, &fn, __FILE__, __LINE__);                \
    static void fn()
#define TEST_CASE(name) \
    DSHIM_TC(DSHIM_CAT(dshim_tc_, __COUNTER__), DSHIM_CAT(dshim_reg_, __LINE__), name)
#define SUBCASE(name) \
    if (const ::doctest_shim::Subcase DSHIM_CAT(dshim_sc_, __LINE__){name, __FILE__, __LINE__})
#define CHECK(...) ::doctest_shim::record(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define REQUIRE(...)                                                                    \
    do {                                                                                \
        const bool dshim_ok = static_cast<bool>(__VA_ARGS__);                          \
        ::doctest_shim::record(dshim_ok, __FILE__, __LINE__, "REQUIRE " #__VA_ARGS__);  \
        if (!dshim_ok) throw ::doctest_shim::Abort{};                                   \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                      \
    do {                                                                                \
        bool dshim_ok = false;                                                          \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (const __VA_ARGS__&) {                                                  \
            dshim_ok = true;                                                            \
        } catch (...) {                                                                 \
        }                                                                               \
        ::doctest_shim::record(dshim_ok, __FILE__, __LINE__, "THROWS_AS " #expr);       \
    } while (0)
#define CHECK_NOTHROW(...)                                                              \
    do {                                                                                \
        bool dshim_ok = true;                                                           \
        try {                                                                           \
            (void)(__VA_ARGS__);                                                        \
        } catch (...) {                                                                 \
            dshim_ok = false;                                                           \
        }                                                                               \
        ::doctest_shim::record(dshim_ok, __FILE__, __LINE__, "NOTHROW " #__VA_ARGS__);  \
    } while (0)
#define FAIL(msg)                                                                       \
    do {                                                                                \
        ::doctest_shim::record(false, __FILE__, __LINE__, "FAIL");                      \
        throw ::doctest_shim::Abort{};                                                  \
    } while (0)
