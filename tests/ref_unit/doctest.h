// doctest.h — minimal doctest-compatible shim (written for this repo; the real
// doctest is not vendored in the reference or present in this image).
//
// Used only to compile the REFERENCE's own unit tests (proj/tests/unit/*.cpp,
// read in place from /root/reference by tests/ref_unit/Makefile) against the B200
// facade headers in include/voxmarch/. Supports the subset those files use:
// TEST_CASE, SUBCASE (run as sequential blocks), CHECK/REQUIRE/CHECK_FALSE,
// CHECK_THROWS, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS and doctest::Approx.
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
    friend bool operator==(double lhs, const Approx& a) {
        double scale = std::fabs(lhs) > std::fabs(a.value_) ? std::fabs(lhs) : std::fabs(a.value_);
        return std::fabs(lhs - a.value_) < a.eps_ * (1.0 + scale);
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

private:
    double value_;
    double eps_ = 1.1920928955078125e-07 * 100;  // doctest's default: float epsilon * 100
};

namespace detail {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& cases() {
    static std::vector<Case> c;
    return c;
}
struct Reg {
    Reg(const char* n, void (*f)()) { cases().push_back({n, f}); }
};
struct RequireFailed {};
inline int& failures() {
    static int f = 0;
    return f;
}
inline long& asserts() {
    static long a = 0;
    return a;
}
inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
    ++asserts();
    if (ok) return;
    ++failures();
    std::fprintf(stderr, "%s:%d: %s failed: %s\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (require) throw RequireFailed{};
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                  \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                    \
    static doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name,                \
                                                                   &DOCTEST_CAT(doctest_fn_, __LINE__)); \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define SUBCASE(name) if (true)
#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) doctest::detail::check(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define CHECK_THROWS(expr)                                                              \
    do {                                                                                \
        bool t_ = false;                                                                \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (...) {                                                                 \
            t_ = true;                                                                  \
        }                                                                               \
        doctest::detail::check(t_, #expr " throws", __FILE__, __LINE__, false);         \
    } while (0)
#define CHECK_NOTHROW(expr)                                                             \
    do {                                                                                \
        bool ok_ = true;                                                                \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (...) {                                                                 \
            ok_ = false;                                                                \
        }                                                                               \
        doctest::detail::check(ok_, #expr " does not throw", __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                     \
    do {                                                                                \
        bool t_ = false;                                                                \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (const type&) {                                                         \
            t_ = true;                                                                  \
        } catch (...) {                                                                 \
        }                                                                               \
        doctest::detail::check(t_, #expr " throws " #type, __FILE__, __LINE__, false);  \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, type)                                           \
    do {                                                                                \
        bool t_ = false;                                                                \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (const type& e_) {                                                      \
            t_ = std::string(e_.what()) == std::string(msg);                            \
            if (!t_) std::fprintf(stderr, "  message was: %s\n", e_.what());            \
        } catch (...) {                                                                 \
        }                                                                               \
        doctest::detail::check(t_, #expr " throws " #type " with " msg, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_SHIM_MAIN
int main() {
    int failed_cases = 0;
    for (auto& c : doctest::detail::cases()) {
        int before = doctest::detail::failures();
        try {
            c.fn();
        } catch (const doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            ++doctest::detail::failures();
            std::fprintf(stderr, "[%s] unexpected exception: %s\n", c.name, e.what());
        }
        bool ok = doctest::detail::failures() == before;
        failed_cases += !ok;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("[doctest-shim] %zu test cases, %d failed, %ld assertions\n",
                doctest::detail::cases().size(), failed_cases, doctest::detail::asserts());
    return failed_cases ? 1 : 0;
}
#endif
