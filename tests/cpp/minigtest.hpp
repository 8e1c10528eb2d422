// Minimal GoogleTest-compatible shim (TEST, EXPECT_*, ASSERT_*) so the drop-in
// test reads like the reference's GTest suites (GTest is not installed here).
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace mini {
struct Case { const char* suite; const char* name; std::function<void()> fn; };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
inline int& failures() { static int f = 0; return f; }
struct Reg { Reg(const char* s, const char* n, std::function<void()> f) { registry().push_back({s, n, std::move(f)}); } };
struct Abort {};
inline void fail(const char* file, int line, const std::string& what, bool fatal) {
    std::printf("  FAILED %s:%d: %s\n", file, line, what.c_str());
    ++failures();
    if (fatal) throw Abort{};
}
}  // namespace mini

#define TEST(S, N)                                                    \
    static void S##_##N##_body();                                     \
    static mini::Reg S##_##N##_reg(#S, #N, S##_##N##_body);           \
    static void S##_##N##_body()

#define MINI_CHECK(cond, text, fatal) do { if (!(cond)) mini::fail(__FILE__, __LINE__, text, fatal); } while (0)
#define EXPECT_TRUE(c) MINI_CHECK((c), #c, false)
#define ASSERT_TRUE(c) MINI_CHECK((c), #c, true)
#define EXPECT_EQ(a, b) MINI_CHECK((a) == (b), #a " == " #b, false)
#define ASSERT_EQ(a, b) MINI_CHECK((a) == (b), #a " == " #b, true)
#define EXPECT_NE(a, b) MINI_CHECK((a) != (b), #a " != " #b, false)
#define EXPECT_LE(a, b) MINI_CHECK((a) <= (b), #a " <= " #b, false)
#define EXPECT_LT(a, b) MINI_CHECK((a) < (b), #a " < " #b, false)
#define EXPECT_GE(a, b) MINI_CHECK((a) >= (b), #a " >= " #b, false)
#define EXPECT_GT(a, b) MINI_CHECK((a) > (b), #a " > " #b, false)
#define EXPECT_NEAR(a, b, t) MINI_CHECK(std::abs((a) - (b)) <= (t), #a " ~ " #b, false)
#define EXPECT_DOUBLE_EQ(a, b) MINI_CHECK((a) == (b), #a " == " #b, false)
#define EXPECT_THROW(stmt, E)                                                        \
    do { bool c_ = false; try { stmt; } catch (const E&) { c_ = true; } catch (...) {} \
         MINI_CHECK(c_, #stmt " throws " #E, false); } while (0)

inline int mini_main() {
    int failed_cases = 0;
    for (auto& c : mini::registry()) {
        const int before = mini::failures();
        try { c.fn(); } catch (const mini::Abort&) {
        } catch (const std::exception& e) { mini::fail(c.suite, 0, std::string("exception: ") + e.what(), false); }
        const bool ok = mini::failures() == before;
        std::printf("[%s] %s.%s\n", ok ? "  OK  " : "FAILED", c.suite, c.name);
        failed_cases += !ok;
    }
    std::printf("%zu cases, %d failed\n", mini::registry().size(), failed_cases);
    return failed_cases ? 1 : 0;
}
