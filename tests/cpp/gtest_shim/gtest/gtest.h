// Minimal GoogleTest-compatible shim (GTest is not installed in this image): enough of
// the TEST / EXPECT_* / ASSERT_* surface to compile the reference's own suites
// (/root/reference/proj/tests/{simplex,objective,solver}_test.cpp) UNMODIFIED against
// the drop-in headers in include/fuzzyclust/.  Semantics follow GoogleTest: EXPECT_*
// records a failure and continues, ASSERT_* records it and leaves the test,
// EXPECT_DOUBLE_EQ is "within 4 ULPs", a streamed message is appended to the report.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <iostream>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace testing {

struct TestInfo {
    const char* suite;
    const char* name;
    void (*fn)();
};

inline std::vector<TestInfo>& registry() {
    static std::vector<TestInfo> r;
    return r;
}

struct Registrar {
    Registrar(const char* s, const char* n, void (*f)()) { registry().push_back({s, n, f}); }
};

inline bool& current_failed() {
    static bool f = false;
    return f;
}

struct FatalFailure {};   // unwinds a test after a failed ASSERT_*

namespace internal {

template <class T, class = void>
struct Printable : std::false_type {};
template <class T>
struct Printable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};

template <class T>
std::string fmt(const T& v) {
    if constexpr (Printable<T>::value) {
        std::ostringstream os;
        os.precision(17);
        os << v;
        return os.str();
    } else {
        return "<" + std::to_string(sizeof(T)) + "-byte object>";
    }
}

// GoogleTest's AlmostEquals: within 4 units in the last place (sign-magnitude biased)
inline bool almost_equal(double a, double b) {
    if (std::isnan(a) || std::isnan(b)) return false;
    auto biased = [](double x) {
        std::uint64_t u;
        std::memcpy(&u, &x, sizeof u);
        const std::uint64_t sign = std::uint64_t(1) << 63;
        return (u & sign) ? ~u + 1 : u | sign;
    };
    const std::uint64_t ba = biased(a), bb = biased(b);
    return (ba >= bb ? ba - bb : bb - ba) <= 4;
}

class Failure {
public:
    Failure(const char* file, int line, std::string what, bool fatal)
        : file_(file), line_(line), what_(std::move(what)), fatal_(fatal) {}
    template <class T>
    Failure& operator<<(const T& v) {
        extra_ << v;
        return *this;
    }
    ~Failure() noexcept(false) {
        std::cout << file_ << ":" << line_ << ": Failure\n" << what_;
        const std::string e = extra_.str();
        if (!e.empty()) std::cout << "\n" << e;
        std::cout << std::endl;
        current_failed() = true;
        if (fatal_ && std::uncaught_exceptions() == 0) throw FatalFailure{};
    }

private:
    const char* file_;
    int line_;
    std::string what_;
    bool fatal_;
    std::ostringstream extra_;
};

template <class A, class B>
std::string cmp_text(const char* ea, const char* op, const char* eb, const A& a, const B& b) {
    return std::string("Expected: (") + ea + ") " + op + " (" + eb + "), actual: " + fmt(a) + " vs " + fmt(b);
}

}  // namespace internal

inline void InitGoogleTest(int*, char**) {}

inline int RunAllTests(const char* filter) {
    int failed = 0, ran = 0;
    std::vector<std::string> failed_names;
    for (const auto& t : registry()) {
        const std::string full = std::string(t.suite) + "." + t.name;
        if (filter && *filter && full.find(filter) == std::string::npos) continue;
        ++ran;
        std::cout << "[ RUN      ] " << full << std::endl;
        current_failed() = false;
        try {
            t.fn();
        } catch (const FatalFailure&) {
        } catch (const std::exception& e) {
            std::cout << "C++ exception: " << e.what() << std::endl;
            current_failed() = true;
        } catch (...) {
            std::cout << "unknown C++ exception" << std::endl;
            current_failed() = true;
        }
        if (current_failed()) {
            ++failed;
            failed_names.push_back(full);
            std::cout << "[  FAILED  ] " << full << std::endl;
        } else {
            std::cout << "[       OK ] " << full << std::endl;
        }
    }
    std::cout << "[==========] " << ran << " tests ran.\n[  PASSED  ] " << (ran - failed) << " tests." << std::endl;
    for (const auto& n : failed_names) std::cout << "[  FAILED  ] " << n << std::endl;
    return failed ? 1 : 0;
}

}  // namespace testing

#define GTS_CAT_(a, b) a##b
#define GTS_CAT(a, b) GTS_CAT_(a, b)

#define TEST(suite, name)                                                                       \
    static void GTS_CAT(gts_test_, GTS_CAT(suite, GTS_CAT(_, name)))();                         \
    static ::testing::Registrar GTS_CAT(gts_reg_, GTS_CAT(suite, GTS_CAT(_, name)))(            \
        #suite, #name, &GTS_CAT(gts_test_, GTS_CAT(suite, GTS_CAT(_, name))));                  \
    static void GTS_CAT(gts_test_, GTS_CAT(suite, GTS_CAT(_, name)))()

#define GTS_CHECK_(cond, text, fatal) \
    switch (0)                        \
    case 0:                           \
    default:                          \
        if (cond)                     \
            ;                         \
        else                          \
            ::testing::internal::Failure(__FILE__, __LINE__, (text), (fatal))

#define GTS_CMP_(a, op, b, fatal)                                                                \
    GTS_CHECK_(((a)op(b)), ::testing::internal::cmp_text(#a, #op, #b, (a), (b)), fatal)

#define EXPECT_EQ(a, b) GTS_CMP_(a, ==, b, false)
#define EXPECT_NE(a, b) GTS_CMP_(a, !=, b, false)
#define EXPECT_LT(a, b) GTS_CMP_(a, <, b, false)
#define EXPECT_LE(a, b) GTS_CMP_(a, <=, b, false)
#define EXPECT_GT(a, b) GTS_CMP_(a, >, b, false)
#define EXPECT_GE(a, b) GTS_CMP_(a, >=, b, false)
#define ASSERT_EQ(a, b) GTS_CMP_(a, ==, b, true)
#define ASSERT_NE(a, b) GTS_CMP_(a, !=, b, true)
#define ASSERT_LT(a, b) GTS_CMP_(a, <, b, true)
#define ASSERT_LE(a, b) GTS_CMP_(a, <=, b, true)
#define ASSERT_GT(a, b) GTS_CMP_(a, >, b, true)
#define ASSERT_GE(a, b) GTS_CMP_(a, >=, b, true)
#define EXPECT_TRUE(c) GTS_CHECK_(!!(c), std::string("Expected true: ") + #c, false)
#define EXPECT_FALSE(c) GTS_CHECK_(!(c), std::string("Expected false: ") + #c, false)
#define ASSERT_TRUE(c) GTS_CHECK_(!!(c), std::string("Expected true: ") + #c, true)
#define ASSERT_FALSE(c) GTS_CHECK_(!(c), std::string("Expected false: ") + #c, true)

#define GTS_NEAR_(a, b, tol, fatal)                                                               \
    GTS_CHECK_(std::fabs(static_cast<double>(a) - static_cast<double>(b)) <= static_cast<double>(tol), \
               ::testing::internal::cmp_text(#a, "near", #b, static_cast<double>(a), static_cast<double>(b)) + \
                   " (tolerance " + ::testing::internal::fmt(static_cast<double>(tol)) + ")",   \
               fatal)
#define EXPECT_NEAR(a, b, tol) GTS_NEAR_(a, b, tol, false)
#define ASSERT_NEAR(a, b, tol) GTS_NEAR_(a, b, tol, true)

#define GTS_DEQ_(a, b, fatal)                                                                     \
    GTS_CHECK_(::testing::internal::almost_equal(static_cast<double>(a), static_cast<double>(b)), \
               ::testing::internal::cmp_text(#a, "~=", #b, static_cast<double>(a), static_cast<double>(b)), fatal)
#define EXPECT_DOUBLE_EQ(a, b) GTS_DEQ_(a, b, false)
#define ASSERT_DOUBLE_EQ(a, b) GTS_DEQ_(a, b, true)

#define GTS_THROW_(stmt, ex, fatal)                                                               \
    GTS_CHECK_(([&]() -> bool {                                                                   \
                   try {                                                                          \
                       stmt;                                                                      \
                   } catch (const ex&) {                                                          \
                       return true;                                                               \
                   } catch (...) {                                                                \
                       return false;                                                              \
                   }                                                                              \
                   return false;                                                                  \
               }()),                                                                              \
               std::string("Expected: ") + #stmt + " throws " + #ex, fatal)
#define EXPECT_THROW(stmt, ex) GTS_THROW_(stmt, ex, false)
#define ASSERT_THROW(stmt, ex) GTS_THROW_(stmt, ex, true)
#define EXPECT_NO_THROW(stmt)                                                                     \
    GTS_CHECK_(([&]() -> bool { try { stmt; } catch (...) { return false; } return true; }()),   \
               std::string("Expected no throw: ") + #stmt, false)

#define FAIL() GTS_CHECK_(false, std::string("Failed"), true)
#define ADD_FAILURE() GTS_CHECK_(false, std::string("Failed"), false)
#define SUCCEED() static_cast<void>(0)

#define RUN_ALL_TESTS() ::testing::RunAllTests(nullptr)
