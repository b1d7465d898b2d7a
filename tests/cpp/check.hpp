// Minimal test runner for the C++ KAT programs (Catch2 is absent in this
// image). Each TEST registers a function; CHECK records failures with the
// source line; main() prints one line per test and returns the failure count.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace kat {

struct Case {
    const char* name;
    std::function<void()> fn;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& checks() {
    static int c = 0;
    return c;
}
struct Registrar {
    Registrar(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
inline void fail(const char* file, int line, const std::string& what) {
    ++failures();
    std::printf("    FAILED %s:%d: %s\n", file, line, what.c_str());
}
inline bool approx(double a, double b, double rel, double abs_margin = 0.0) {
    const double d = std::abs(a - b);
    return d <= abs_margin || d <= rel * std::max(std::abs(a), std::abs(b));
}

struct Throws {};

inline int run_all(int argc, char** argv) {
    int failed_cases = 0;
    for (const auto& c : registry()) {
        if (argc > 1 && std::string(c.name).find(argv[1]) == std::string::npos) continue;
        const int before = failures();
        try {
            c.fn();
        } catch (const std::exception& e) {
            fail(__FILE__, __LINE__, std::string("unexpected exception: ") + e.what());
        }
        const bool ok = failures() == before;
        if (!ok) ++failed_cases;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
        std::fflush(stdout);
    }
    std::printf("%d checks, %d failures, %d failed cases\n", checks(), failures(), failed_cases);
    return failed_cases;
}

}  // namespace kat

#define KAT_CAT2(a, b) a##b
#define KAT_CAT(a, b) KAT_CAT2(a, b)
#define TEST(name)                                                              \
    static void KAT_CAT(kat_fn_, __LINE__)();                                   \
    static kat::Registrar KAT_CAT(kat_reg_, __LINE__)(name, KAT_CAT(kat_fn_, __LINE__)); \
    static void KAT_CAT(kat_fn_, __LINE__)()

#define CHECK(cond)                                                      \
    do {                                                                 \
        ++kat::checks();                                                 \
        if (!(cond)) kat::fail(__FILE__, __LINE__, #cond);               \
    } while (0)

#define CHECK_APPROX(a, b, rel, margin)                                                   \
    do {                                                                                  \
        ++kat::checks();                                                                  \
        const double kat_a = (a), kat_b = (b);                                            \
        if (!kat::approx(kat_a, kat_b, rel, margin)) {                                    \
            char kat_buf[256];                                                            \
            std::snprintf(kat_buf, sizeof kat_buf, "%s ~ %s (%.17g vs %.17g)", #a, #b, kat_a, \
                          kat_b);                                                         \
            kat::fail(__FILE__, __LINE__, kat_buf);                                       \
        }                                                                                 \
    } while (0)

#define CHECK_THROWS_AS(expr, Type)                                                     \
    do {                                                                                \
        ++kat::checks();                                                                \
        bool kat_ok = false;                                                            \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (const Type&) {                                                         \
            kat_ok = true;                                                              \
        } catch (...) {                                                                 \
        }                                                                               \
        if (!kat_ok) kat::fail(__FILE__, __LINE__, "expected " #Type " from " #expr);   \
    } while (0)

#define CHECK_THROWS_WITH(expr, Type, substr)                                            \
    do {                                                                                 \
        ++kat::checks();                                                                 \
        bool kat_ok = false;                                                             \
        std::string kat_msg;                                                             \
        try {                                                                            \
            (void)(expr);                                                                \
        } catch (const Type& e) {                                                        \
            kat_msg = e.what();                                                          \
            kat_ok = kat_msg.find(substr) != std::string::npos;                          \
        } catch (...) {                                                                  \
        }                                                                                \
        if (!kat_ok) kat::fail(__FILE__, __LINE__, "expected '" substr "' got '" + kat_msg + "'"); \
    } while (0)

#define KAT_MAIN \
    int main(int argc, char** argv) { return kat::run_all(argc, argv); }
