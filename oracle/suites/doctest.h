// TEST INFRASTRUCTURE ONLY -- a minimal stand-in for doctest (absent from the
// reference tree), just enough to compile the reference's own unit
// suites (proj/tests/test_*.cpp) unchanged against this repository's headers
// and library: TEST_CASE, CHECK, CHECK_FALSE, CHECK_THROWS_AS, REQUIRE, FAIL.
// Exit status = number of failed test cases.
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest_shim {

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
inline int& failures_in_case() {
    static int f = 0;
    return f;
}
struct Register {
    Register(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};
struct Abort {};  // thrown by a failed REQUIRE / FAIL to leave the test case

inline void fail(const char* file, int line, const std::string& what, bool fatal) {
    std::printf("  %s:%d: FAILED: %s\n", file, line, what.c_str());
    ++failures_in_case();
    if (fatal) throw Abort{};
}

inline int run_all() {
    int failed = 0, checked = 0;
    for (const Case& c : registry()) {
        failures_in_case() = 0;
        try {
            c.fn();
        } catch (const Abort&) {
        } catch (const std::exception& e) {
            fail(c.file, c.line, std::string("unexpected exception: ") + e.what(), false);
        } catch (...) {
            fail(c.file, c.line, "unexpected non-standard exception", false);
        }
        ++checked;
        if (failures_in_case()) {
            ++failed;
            std::printf("[FAIL] %s\n", c.name);
        } else {
            std::printf("[ ok ] %s\n", c.name);
        }
    }
    std::printf("test cases: %d | %d passed | %d failed\n", checked, checked - failed, failed);
    return failed;
}

}  // namespace doctest_shim

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_CASE(fn, name)                                                       \
    static void fn();                                                                     \
    static doctest_shim::Register DOCTEST_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(doctest_shim_case_, __COUNTER__), name)

#define DOCTEST_SHIM_CHECK(expr, fatal)                                                    \
    do {                                                                                   \
        bool doctest_shim_ok_ = false;                                                     \
        try {                                                                              \
            doctest_shim_ok_ = static_cast<bool>(expr);                                    \
        } catch (const std::exception& e) {                                                \
            doctest_shim::fail(__FILE__, __LINE__, std::string(#expr) + " threw " + e.what(), fatal); \
            break;                                                                         \
        }                                                                                  \
        if (!doctest_shim_ok_) doctest_shim::fail(__FILE__, __LINE__, #expr, fatal);       \
    } while (0)
#define CHECK(...) DOCTEST_SHIM_CHECK((__VA_ARGS__), false)
#define CHECK_FALSE(...) DOCTEST_SHIM_CHECK(!(__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_SHIM_CHECK((__VA_ARGS__), true)
#define CHECK_THROWS_AS(expr, type)                                                           \
    do {                                                                                      \
        bool doctest_shim_thrown_ = false;                                                    \
        try {                                                                                 \
            static_cast<void>(expr);                                                          \
        } catch (const type&) {                                                               \
            doctest_shim_thrown_ = true;                                                      \
        } catch (...) {                                                                       \
        }                                                                                     \
        if (!doctest_shim_thrown_) doctest_shim::fail(__FILE__, __LINE__, #expr " does not throw " #type, false); \
    } while (0)
#define FAIL(msg) doctest_shim::fail(__FILE__, __LINE__, std::string(msg), true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest_shim::run_all(); }
#endif
