// mini_check.hpp — a tiny self-registering test harness for the C++ facade tests
// (the reference uses doctest, which is not available in this image).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace mini {

struct Case {
    const char* name;
    std::function<void()> fn;
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Registrar {
    Registrar(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};

inline int& failures() {
    static int f = 0;
    return f;
}
inline long& checks() {
    static long c = 0;
    return c;
}

inline void report(bool ok, const char* expr, const char* file, int line) {
    ++checks();
    if (!ok) {
        ++failures();
        std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", file, line, expr);
    }
}

inline bool near_rel(double a, double b, double rel, double abs_floor) {
    double scale = std::fabs(a) > std::fabs(b) ? std::fabs(a) : std::fabs(b);
    double tol = rel * scale > abs_floor ? rel * scale : abs_floor;
    return std::fabs(a - b) <= tol;
}

inline int run_all() {
    int failed_cases = 0;
    for (auto& c : registry()) {
        int before = failures();
        try {
            c.fn();
        } catch (const std::exception& e) {
            ++failures();
            std::fprintf(stderr, "[%s] unexpected exception: %s\n", c.name, e.what());
        }
        bool ok = failures() == before;
        failed_cases += !ok;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("%zu cases, %d failed, %ld checks\n", registry().size(), failed_cases, checks());
    return failed_cases ? 1 : 0;
}

}  // namespace mini

#define MINI_CAT2(a, b) a##b
#define MINI_CAT(a, b) MINI_CAT2(a, b)
#define TEST(name)                                                             \
    static void MINI_CAT(test_fn_, __LINE__)();                                \
    static mini::Registrar MINI_CAT(test_reg_, __LINE__)(name, MINI_CAT(test_fn_, __LINE__)); \
    static void MINI_CAT(test_fn_, __LINE__)()
#define CHECK(expr) mini::report(static_cast<bool>(expr), #expr, __FILE__, __LINE__)
#define CHECK_NEAR(a, b, rel) mini::report(mini::near_rel((a), (b), (rel), 1e-8), #a " ~ " #b, __FILE__, __LINE__)
#define CHECK_THROWS_MSG(stmt, type, msg)                                       \
    do {                                                                       \
        bool thrown_ = false;                                                  \
        try {                                                                  \
            stmt;                                                              \
        } catch (const type& e_) {                                             \
            thrown_ = std::string(e_.what()) == std::string(msg);              \
            if (!thrown_) std::fprintf(stderr, "  got message: %s\n", e_.what()); \
        } catch (...) {                                                        \
        }                                                                      \
        mini::report(thrown_, #stmt " throws " #type ": " msg, __FILE__, __LINE__); \
    } while (0)
#define CHECK_THROWS_TYPE(stmt, type)                                          \
    do {                                                                       \
        bool thrown_ = false;                                                  \
        try {                                                                  \
            stmt;                                                              \
        } catch (const type&) {                                                \
            thrown_ = true;                                                    \
        } catch (...) {                                                        \
        }                                                                      \
        mini::report(thrown_, #stmt " throws " #type, __FILE__, __LINE__);     \
    } while (0)
