// Minimal doctest-compatible test harness: the subset of doctest's macros the
// reference's unit suites use (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// FAIL, DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN), so /root/reference/proj/tests/*.cpp
// compile UNCHANGED against include/ + libdfakit_b200.so (doctest itself is a
// third-party header the reference does not vendor).
//
// Semantics follow doctest: CHECK records a failure and continues (an
// exception thrown by the expression is a failure too); REQUIRE and FAIL
// record a failure and end the current test case; CHECK_THROWS_AS passes only
// if the expression throws the named type.  The main() prints one line per
// failed assertion and a doctest-style summary, and exits non-zero on failure.
#pragma once

#include <cstdio>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

namespace mini_doctest {

struct Case {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, void (*fn)(), const char* file, int line) {
        registry().push_back({name, fn, file, line});
    }
};

struct AbortCase {};

struct State {
    const char* current = "";
    long assertions = 0;
    long failed_assertions = 0;
    bool case_failed = false;
};

inline State& state() {
    static State s;
    return s;
}

inline void report(const char* file, int line, const char* macro, const char* expr, const std::string& extra) {
    State& s = state();
    ++s.failed_assertions;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) in test case \"%s\"%s%s\n", file, line, macro, expr, s.current,
                 extra.empty() ? "" : " -- ", extra.c_str());
}

template <typename M>
std::string to_text(const M& m) {
    std::ostringstream os;
    os << m;
    return os.str();
}

}  // namespace mini_doctest

#define MINI_DOCTEST_CAT2(a, b) a##b
#define MINI_DOCTEST_CAT(a, b) MINI_DOCTEST_CAT2(a, b)
#define MINI_DOCTEST_CASE(fn, reg, name)                                                        \
    static void fn();                                                                          \
    static ::mini_doctest::Registrar reg(name, &fn, __FILE__, __LINE__);                       \
    static void fn()
#define TEST_CASE(name) \
    MINI_DOCTEST_CASE(MINI_DOCTEST_CAT(mini_doctest_case_, __COUNTER__), MINI_DOCTEST_CAT(mini_doctest_reg_, __LINE__), name)

#define MINI_DOCTEST_ASSERT(macro, fatal, ...)                                                           \
    do {                                                                                                \
        ++::mini_doctest::state().assertions;                                                           \
        bool mini_doctest_ok = false;                                                                   \
        std::string mini_doctest_extra;                                                                 \
        try {                                                                                           \
            mini_doctest_ok = static_cast<bool>(__VA_ARGS__);                                           \
        } catch (const ::mini_doctest::AbortCase&) {                                                    \
            throw;                                                                                      \
        } catch (const std::exception& e) {                                                             \
            mini_doctest_extra = std::string("threw: ") + e.what();                                     \
        } catch (...) {                                                                                 \
            mini_doctest_extra = "threw an unknown exception";                                          \
        }                                                                                               \
        if (!mini_doctest_ok) {                                                                         \
            ::mini_doctest::report(__FILE__, __LINE__, macro, #__VA_ARGS__, mini_doctest_extra);         \
            if (fatal) throw ::mini_doctest::AbortCase{};                                               \
        }                                                                                               \
    } while (0)

#define CHECK(...) MINI_DOCTEST_ASSERT("CHECK", false, __VA_ARGS__)
#define REQUIRE(...) MINI_DOCTEST_ASSERT("REQUIRE", true, __VA_ARGS__)

#define CHECK_THROWS_AS(expr, ...)                                                                     \
    do {                                                                                              \
        ++::mini_doctest::state().assertions;                                                         \
        bool mini_doctest_ok = false;                                                                 \
        std::string mini_doctest_extra = "did not throw";                                             \
        try {                                                                                         \
            static_cast<void>(expr);                                                                  \
        } catch (const __VA_ARGS__&) {                                                                \
            mini_doctest_ok = true;                                                                   \
        } catch (const std::exception& e) {                                                           \
            mini_doctest_extra = std::string("threw another type: ") + e.what();                      \
        } catch (...) {                                                                               \
            mini_doctest_extra = "threw another type";                                                \
        }                                                                                             \
        if (!mini_doctest_ok)                                                                         \
            ::mini_doctest::report(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__,     \
                                   mini_doctest_extra);                                               \
    } while (0)

#define FAIL(msg)                                                                                     \
    do {                                                                                              \
        ::mini_doctest::report(__FILE__, __LINE__, "FAIL", "", ::mini_doctest::to_text(msg));         \
        throw ::mini_doctest::AbortCase{};                                                            \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    const char* only = nullptr;  // optional: run only test cases whose name contains argv[1]
    if (argc > 1) only = argv[1];
    long cases = 0, failed = 0, skipped = 0;
    for (const auto& c : ::mini_doctest::registry()) {
        if (only && !std::strstr(c.name, only)) {
            ++skipped;
            continue;
        }
        ::mini_doctest::State& s = ::mini_doctest::state();
        s.current = c.name;
        s.case_failed = false;
        ++cases;
        try {
            c.fn();
        } catch (const ::mini_doctest::AbortCase&) {
        } catch (const std::exception& e) {
            ++s.assertions;  // doctest counts an escaped exception as a failed assertion
            ::mini_doctest::report(c.file, c.line, "TEST_CASE", c.name, std::string("unexpected exception: ") + e.what());
        } catch (...) {
            ++s.assertions;
            ::mini_doctest::report(c.file, c.line, "TEST_CASE", c.name, "unexpected exception");
        }
        failed += s.case_failed;
    }
    const ::mini_doctest::State& s = ::mini_doctest::state();
    std::printf("[doctest] test cases: %ld | %ld passed | %ld failed | %ld skipped\n", cases, cases - failed, failed,
                skipped);
    std::printf("[doctest] assertions: %ld | %ld passed | %ld failed |\n", s.assertions,
                s.assertions - s.failed_assertions, s.failed_assertions);
    std::printf("[doctest] Status: %s!\n", failed ? "FAILURE" : "SUCCESS");
    return failed ? 1 : 0;
}
#endif
