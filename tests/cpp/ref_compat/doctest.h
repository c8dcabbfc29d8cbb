// Minimal doctest-compatible shim (TEST INFRASTRUCTURE ONLY) so the
// reference's own unit tests (/root/reference/proj/tests/test_schedule.cpp,
// test_bubblefill.cpp -- compiled in place, never copied) build against THIS
// repo's include/ and libpf_b200.so.  The reference vendors doctest (absent
// from the image); only the macros those files use are provided:
// TEST_CASE, SUBCASE (flat: the test body is re-run once per subcase),
// CHECK, CHECK_MESSAGE, CHECK_NOTHROW, CHECK_THROWS_AS, REQUIRE,
// REQUIRE_MESSAGE, FAIL, INFO, doctest::Approx (doctest's default epsilon:
// 100 float epsilons, relative to max(|a|, |b|) + scale 1).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <sstream>
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
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) < a.eps_ * (1.0 + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend std::ostream& operator<<(std::ostream& os, const Approx& a) { return os << "Approx(" << a.value_ << ")"; }

private:
    double value_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
};

namespace shim {
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
struct Reg {
    Reg(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct State {
    int failures = 0, checks = 0;
    int sub_target = 0, sub_seen = 0;
    std::string info;
    const char* test = "";
};
inline State& st() {
    static State s;
    return s;
}
struct RequireFailed {};
inline void fail(const char* file, int line, const std::string& what) {
    ++st().failures;
    std::printf("%s:%d: FAILED in \"%s\": %s%s%s\n", file, line, st().test, what.c_str(),
                st().info.empty() ? "" : "  [info: ", st().info.empty() ? "" : (st().info + "]").c_str());
}
inline bool enter_subcase() { return st().sub_seen++ == st().sub_target; }
}  // namespace shim
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                                  \
    static void fn();                                                                          \
    static doctest::shim::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);            \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (doctest::shim::enter_subcase())
#define DOCTEST_CHECK_(cond, msg, req)                                                          \
    do {                                                                                       \
        ++doctest::shim::st().checks;                                                          \
        if (!(cond)) {                                                                         \
            std::ostringstream doctest_os_;                                                    \
            doctest_os_ << #cond << msg;                                                       \
            doctest::shim::fail(__FILE__, __LINE__, doctest_os_.str());                        \
            if (req) throw doctest::shim::RequireFailed{};                                     \
        }                                                                                      \
    } while (0)
#define CHECK(...) DOCTEST_CHECK_((__VA_ARGS__), "", false)
#define REQUIRE(...) DOCTEST_CHECK_((__VA_ARGS__), "", true)
#define CHECK_MESSAGE(cond, m) DOCTEST_CHECK_(cond, "  -- " << m, false)
#define REQUIRE_MESSAGE(cond, m) DOCTEST_CHECK_(cond, "  -- " << m, true)
#define CHECK_THROWS_AS(expr, type)                                                             \
    do {                                                                                       \
        bool doctest_ok_ = false;                                                              \
        try {                                                                                  \
            (void)(expr);                                                                      \
        } catch (const type&) {                                                                \
            doctest_ok_ = true;                                                                \
        } catch (...) {                                                                        \
        }                                                                                      \
        DOCTEST_CHECK_(doctest_ok_, "  -- expected " #type " from " #expr, false);             \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                     \
    do {                                                                                       \
        bool doctest_ok_ = true;                                                               \
        try {                                                                                  \
            (void)(expr);                                                                      \
        } catch (...) {                                                                        \
            doctest_ok_ = false;                                                               \
        }                                                                                      \
        DOCTEST_CHECK_(doctest_ok_, "  -- unexpected exception from " #expr, false);           \
    } while (0)
#define FAIL(m)                                                                                 \
    do {                                                                                       \
        std::ostringstream doctest_os_;                                                        \
        doctest_os_ << m;                                                                      \
        doctest::shim::fail(__FILE__, __LINE__, doctest_os_.str());                            \
        throw doctest::shim::RequireFailed{};                                                  \
    } while (0)
#define INFO(m)                                                                                 \
    do {                                                                                       \
        std::ostringstream doctest_os_;                                                        \
        doctest_os_ << m;                                                                      \
        doctest::shim::st().info = doctest_os_.str();                                          \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    using namespace doctest::shim;
    int cases = 0, failed_cases = 0;
    for (const Case& c : registry()) {
        ++cases;
        const int before = st().failures;
        st().test = c.name;
        // one run per subcase (a body without subcases runs once)
        for (st().sub_target = 0;; ++st().sub_target) {
            st().sub_seen = 0;
            st().info.clear();
            try {
                c.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                fail(c.file, c.line, std::string("uncaught exception: ") + e.what());
            }
            if (st().sub_target + 1 >= st().sub_seen) break;
        }
        if (st().failures != before) ++failed_cases;
    }
    std::printf("[doctest shim] test cases: %d | %d passed | %d failed; assertions: %d | %d failed\n", cases,
                cases - failed_cases, failed_cases, st().checks, st().failures);
    return st().failures == 0 ? 0 : 1;
}
#endif
