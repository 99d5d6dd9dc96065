// minitest.hpp -- a tiny self-written test runner (GoogleTest is not in the
// image). TEST(suite, name) registers a case; EXPECT_* record failures and
// continue, ASSERT_* abort the case. main() runs everything (or the cases
// whose "suite.name" contains argv[1]) and returns the failure count.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace minitest {

struct Case {
    std::string name;
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
struct Registrar {
    Registrar(const char* suite, const char* name, std::function<void()> fn) {
        registry().push_back({std::string(suite) + "." + name, std::move(fn)});
    }
};
struct AssertAbort {};

inline void fail(const char* file, int line, const std::string& what) {
    ++failures();
    std::fprintf(stderr, "  FAIL %s:%d: %s\n", file, line, what.c_str());
}

inline int run_all(int argc, char** argv) {
    const std::string filter = argc > 1 ? argv[1] : "";
    int ran = 0, failed_cases = 0;
    for (const Case& c : registry()) {
        if (!filter.empty() && c.name.find(filter) == std::string::npos) continue;
        const int before = failures();
        try {
            c.fn();
        } catch (const AssertAbort&) {
        } catch (const std::exception& e) {
            fail(__FILE__, __LINE__, std::string("uncaught exception: ") + e.what());
        }
        ++ran;
        const bool ok = failures() == before;
        if (!ok) ++failed_cases;
        std::printf("[%s] %s\n", ok ? "  OK  " : " FAIL ", c.name.c_str());
    }
    std::printf("%d cases, %d failed\n", ran, failed_cases);
    return failed_cases;
}

}  // namespace minitest

#define MT_CAT2(a, b) a##b
#define MT_CAT(a, b) MT_CAT2(a, b)
#define TEST(suite, name)                                                                       \
    static void MT_CAT(test_, MT_CAT(suite, MT_CAT(_, name)))();                                \
    static minitest::Registrar MT_CAT(reg_, MT_CAT(suite, MT_CAT(_, name)))(                    \
        #suite, #name, MT_CAT(test_, MT_CAT(suite, MT_CAT(_, name))));                          \
    static void MT_CAT(test_, MT_CAT(suite, MT_CAT(_, name)))()

#define EXPECT_TRUE(c) \
    do { if (!(c)) minitest::fail(__FILE__, __LINE__, "EXPECT_TRUE(" #c ")"); } while (0)
#define EXPECT_FALSE(c) EXPECT_TRUE(!(c))
#define ASSERT_TRUE(c) \
    do { if (!(c)) { minitest::fail(__FILE__, __LINE__, "ASSERT_TRUE(" #c ")"); throw minitest::AssertAbort{}; } } while (0)
#define EXPECT_EQ(a, b) \
    do { if (!((a) == (b))) minitest::fail(__FILE__, __LINE__, "EXPECT_EQ(" #a ", " #b ")"); } while (0)
#define ASSERT_EQ(a, b) \
    do { if (!((a) == (b))) { minitest::fail(__FILE__, __LINE__, "ASSERT_EQ(" #a ", " #b ")"); throw minitest::AssertAbort{}; } } while (0)
#define EXPECT_LT(a, b) \
    do { if (!((a) < (b))) minitest::fail(__FILE__, __LINE__, "EXPECT_LT(" #a ", " #b ") with " + std::to_string(a) + " vs " + std::to_string(b)); } while (0)
#define EXPECT_LE(a, b) \
    do { if (!((a) <= (b))) minitest::fail(__FILE__, __LINE__, "EXPECT_LE(" #a ", " #b ") with " + std::to_string(a) + " vs " + std::to_string(b)); } while (0)
#define EXPECT_GT(a, b) EXPECT_LT(b, a)
#define EXPECT_GE(a, b) EXPECT_LE(b, a)
#define EXPECT_NEAR(a, b, tol) \
    do { const double _x = (a), _y = (b); if (!(std::abs(_x - _y) <= (tol))) minitest::fail(__FILE__, __LINE__, "EXPECT_NEAR(" #a ", " #b ") diff " + std::to_string(std::abs(_x - _y))); } while (0)
#define EXPECT_THROW(stmt, type)                                                              \
    do {                                                                                      \
        bool _caught = false;                                                                 \
        try { stmt; } catch (const type&) { _caught = true; } catch (...) {}                  \
        if (!_caught) minitest::fail(__FILE__, __LINE__, "EXPECT_THROW(" #stmt ", " #type ")"); \
    } while (0)
#define EXPECT_NO_THROW(stmt)                                                                  \
    do { try { stmt; } catch (...) { minitest::fail(__FILE__, __LINE__, "EXPECT_NO_THROW(" #stmt ")"); } } while (0)
