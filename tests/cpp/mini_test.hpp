// Minimal doctest-style harness (doctest is not in this image).
#pragma once
#include <cstdio>
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
inline int& failures() {
    static int f = 0;
    return f;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
inline int run_all(const char* filter) {
    int ran = 0;
    for (auto& c : registry()) {
        if (filter && std::string(c.name).find(filter) == std::string::npos) continue;
        const int before = failures();
        try {
            c.fn();
        } catch (const std::exception& e) {
            std::printf("  exception: %s\n", e.what());
            ++failures();
        }
        std::printf("[%s] %s\n", failures() == before ? "PASS" : "FAIL", c.name);
        ++ran;
    }
    std::printf("%d cases, %d failed checks\n", ran, failures());
    return failures() ? 1 : 0;
}
}  // namespace mini

#define MINI_CAT2(a, b) a##b
#define MINI_CAT(a, b) MINI_CAT2(a, b)
#define TEST_CASE(name)                                                 \
    static void MINI_CAT(tc_, __LINE__)();                              \
    static mini::Reg MINI_CAT(reg_, __LINE__)(name, MINI_CAT(tc_, __LINE__)); \
    static void MINI_CAT(tc_, __LINE__)()
#define CHECK(x)                                                               \
    do {                                                                       \
        if (!(x)) {                                                            \
            std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #x); \
            ++mini::failures();                                                \
        }                                                                      \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                                                \
    do {                                                                                        \
        bool ok_ = false;                                                                       \
        try {                                                                                   \
            (void)(expr);                                                                       \
        } catch (const T&) {                                                                    \
            ok_ = true;                                                                         \
        } catch (...) {                                                                         \
        }                                                                                       \
        if (!ok_) {                                                                             \
            std::printf("  CHECK_THROWS_AS failed %s:%d: %s\n", __FILE__, __LINE__, #expr);     \
            ++mini::failures();                                                                 \
        }                                                                                       \
    } while (0)
