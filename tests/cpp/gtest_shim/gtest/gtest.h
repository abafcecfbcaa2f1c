// Minimal GoogleTest-compatible shim (this repo's own code): GTest is not installed in
// this image, and it lets the reference's unit-test sources be compiled, unmodified and
// in place, against the drop-in headers (tests/cpp/build_reftests.sh). Supports the
// assertion subset those sources use; failures print file:line and the streamed message.
#pragma once

#include <cmath>
#include <cstring>
#include <type_traits>
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace gshim {

struct Case {
    const char* suite;
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
inline bool& skipped() {
    static bool s = false;
    return s;
}

struct Registrar {
    Registrar(const char* s, const char* n, std::function<void()> f) { registry().push_back({s, n, std::move(f)}); }
};

// Collects a streamed message; reports on destruction when the check failed.
class Reporter {
public:
    Reporter(bool ok, const char* file, int line, std::string what) : ok_(ok), file_(file), line_(line), what_(std::move(what)) {}
    ~Reporter() {
        if (!ok_) {
            ++failures();
            std::printf("  %s:%d: Failure: %s %s\n", file_, line_, what_.c_str(), msg_.str().c_str());
        }
    }
    template <typename T>
    Reporter& operator<<(const T& v) {
        msg_ << v;
        return *this;
    }
    bool ok() const { return ok_; }

private:
    bool ok_;
    const char* file_;
    int line_;
    std::string what_;
    std::ostringstream msg_;
};

struct Skip {
    template <typename T>
    Skip& operator<<(const T&) {
        return *this;
    }
};

// `return Fatal() = Reporter(...) << msg;` -- the gtest idiom that lets ASSERT_* and
// GTEST_SKIP() take a streamed message and still return from a void test body.
struct Fatal {
    void operator=(const Reporter&) const {}
    void operator=(const Skip&) const {}
};

// float/double equality within 4 ULPs, like GoogleTest's *_FLOAT_EQ / *_DOUBLE_EQ
template <typename F>
bool almost_equal(F a, F b) {
    if (a == b) return true;
    if (std::isnan(a) || std::isnan(b)) return false;
    using I = std::conditional_t<sizeof(F) == 4, long long, long long>;
    auto ord = [](F x) -> I {
        if constexpr (sizeof(F) == 4) {
            int i;
            std::memcpy(&i, &x, 4);
            return i < 0 ? static_cast<I>(static_cast<int>(0x80000000u) - i) : static_cast<I>(i);
        } else {
            long long i;
            std::memcpy(&i, &x, 8);
            return i < 0 ? static_cast<I>(static_cast<long long>(0x8000000000000000ull) - i) : i;
        }
    };
    const I d = ord(a) - ord(b);
    return (d < 0 ? -d : d) <= 4;
}

}  // namespace gshim

#include <cstring>
#include <type_traits>

#define GSHIM_CAT2(a, b) a##b
#define GSHIM_CAT(a, b) GSHIM_CAT2(a, b)

#define TEST(suite, name)                                                                                   \
    static void GSHIM_CAT(gshim_test_, GSHIM_CAT(suite, GSHIM_CAT(_, name)))();                             \
    static ::gshim::Registrar GSHIM_CAT(gshim_reg_, GSHIM_CAT(suite, GSHIM_CAT(_, name)))(                   \
        #suite, #name, GSHIM_CAT(gshim_test_, GSHIM_CAT(suite, GSHIM_CAT(_, name))));                        \
    static void GSHIM_CAT(gshim_test_, GSHIM_CAT(suite, GSHIM_CAT(_, name)))()

#define GSHIM_CHECK(cond, what) ::gshim::Reporter((cond), __FILE__, __LINE__, (what))
// ASSERT_*: report, then return from the test body when the check failed
#define GSHIM_ASSERT(cond, what) \
    if (cond) {                  \
    } else                       \
        return ::gshim::Fatal() = ::gshim::Reporter(false, __FILE__, __LINE__, (what))

#define EXPECT_TRUE(c) GSHIM_CHECK(static_cast<bool>(c), "EXPECT_TRUE(" #c ")")
#define EXPECT_FALSE(c) GSHIM_CHECK(!static_cast<bool>(c), "EXPECT_FALSE(" #c ")")
#define EXPECT_EQ(a, b) GSHIM_CHECK((a) == (b), "EXPECT_EQ(" #a ", " #b ")")
#define EXPECT_NE(a, b) GSHIM_CHECK((a) != (b), "EXPECT_NE(" #a ", " #b ")")
#define EXPECT_LT(a, b) GSHIM_CHECK((a) < (b), "EXPECT_LT(" #a ", " #b ")")
#define EXPECT_LE(a, b) GSHIM_CHECK((a) <= (b), "EXPECT_LE(" #a ", " #b ")")
#define EXPECT_GT(a, b) GSHIM_CHECK((a) > (b), "EXPECT_GT(" #a ", " #b ")")
#define EXPECT_GE(a, b) GSHIM_CHECK((a) >= (b), "EXPECT_GE(" #a ", " #b ")")
#define EXPECT_NEAR(a, b, tol) \
    GSHIM_CHECK(std::fabs(static_cast<double>(a) - static_cast<double>(b)) <= (tol), "EXPECT_NEAR(" #a ", " #b ")")
#define EXPECT_FLOAT_EQ(a, b) \
    GSHIM_CHECK(::gshim::almost_equal<float>(static_cast<float>(a), static_cast<float>(b)), "EXPECT_FLOAT_EQ(" #a ", " #b ")")
#define EXPECT_DOUBLE_EQ(a, b)                                                                  \
    GSHIM_CHECK(::gshim::almost_equal<double>(static_cast<double>(a), static_cast<double>(b)), \
                "EXPECT_DOUBLE_EQ(" #a ", " #b ")")
#define EXPECT_THROW(stmt, ex)                                                    \
    GSHIM_CHECK(([&] {                                                            \
                    try {                                                         \
                        stmt;                                                     \
                    } catch (const ex&) {                                         \
                        return true;                                              \
                    } catch (...) {                                               \
                        return false;                                             \
                    }                                                             \
                    return false;                                                 \
                })(),                                                             \
                "EXPECT_THROW(" #stmt ", " #ex ")")
#define EXPECT_NO_THROW(stmt)                                                     \
    GSHIM_CHECK(([&] {                                                            \
                    try {                                                         \
                        stmt;                                                     \
                    } catch (...) {                                               \
                        return false;                                             \
                    }                                                             \
                    return true;                                                  \
                })(),                                                             \
                "EXPECT_NO_THROW(" #stmt ")")

#define ASSERT_TRUE(c) GSHIM_ASSERT(static_cast<bool>(c), "ASSERT_TRUE(" #c ")")
#define ASSERT_FALSE(c) GSHIM_ASSERT(!static_cast<bool>(c), "ASSERT_FALSE(" #c ")")
#define ASSERT_EQ(a, b) GSHIM_ASSERT((a) == (b), "ASSERT_EQ(" #a ", " #b ")")
#define ASSERT_GE(a, b) GSHIM_ASSERT((a) >= (b), "ASSERT_GE(" #a ", " #b ")")
#define ASSERT_LE(a, b) GSHIM_ASSERT((a) <= (b), "ASSERT_LE(" #a ", " #b ")")

#define FAIL() return ::gshim::Fatal() = ::gshim::Reporter(false, __FILE__, __LINE__, "FAIL()")
#define ADD_FAILURE() GSHIM_CHECK(false, "ADD_FAILURE()")
#define ASSERT_NE(a, b) GSHIM_ASSERT((a) != (b), "ASSERT_NE(" #a ", " #b ")")
#define ASSERT_LT(a, b) GSHIM_ASSERT((a) < (b), "ASSERT_LT(" #a ", " #b ")")
#define ASSERT_GT(a, b) GSHIM_ASSERT((a) > (b), "ASSERT_GT(" #a ", " #b ")")
#define GTEST_SKIP() return ::gshim::Fatal() = (::gshim::skipped() = true, ::gshim::Skip())

int main(int, char**) {
    int failed_tests = 0, skipped_tests = 0;
    for (const auto& c : ::gshim::registry()) {
        const int before = ::gshim::failures();
        ::gshim::skipped() = false;
        std::printf("[ RUN      ] %s.%s\n", c.suite, c.name);
        try {
            c.fn();
        } catch (const std::exception& e) {
            ++::gshim::failures();
            std::printf("  uncaught exception: %s\n", e.what());
        }
        const bool ok = ::gshim::failures() == before;
        if (!ok) ++failed_tests;
        if (::gshim::skipped()) ++skipped_tests;
        std::printf("[ %s ] %s.%s\n", !ok ? " FAILED " : (::gshim::skipped() ? " SKIPPED" : "      OK"), c.suite,
                    c.name);
    }
    std::printf("[==========] %zu tests, %d failed, %d skipped\n", ::gshim::registry().size(), failed_tests,
                skipped_tests);
    return failed_tests == 0 ? 0 : 1;
}
