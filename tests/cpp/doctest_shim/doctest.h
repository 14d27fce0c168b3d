// doctest.h -- a minimal, self-written harness with the subset of the doctest
// interface that the reference's unit tests use (TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, CAPTURE, FAIL,
// doctest::Approx, DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN).  The reference
// vendors the real doctest under proj/vendor/, which is absent from the
// reference tree; this shim lets tests/cpp/Makefile compile the
// reference's test sources UNCHANGED against the B200 drop-in headers.
// Test infrastructure only.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double value) : value_(value) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& rhs) {
        const double scale = std::max(std::fabs(lhs), std::fabs(rhs.value_));
        return std::fabs(lhs - rhs.value_) <= rhs.eps_ * (1.0 + scale);
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

private:
    double value_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
};

namespace detail {

struct Case {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};

inline std::vector<Case>& cases() {
    static std::vector<Case> all;
    return all;
}

struct Registrar {
    Registrar(const char* name, void (*fn)(), const char* file, int line) {
        cases().push_back({name, fn, file, line});
    }
};

struct Stats {
    long asserts = 0, failed_asserts = 0;
    bool case_failed = false;
    const char* case_name = "";
    std::vector<std::string> context;
};

inline Stats& stats() {
    static Stats s;
    return s;
}

struct AbortCase {};  // REQUIRE / FAIL end the current test case

inline void record(bool ok, const char* file, int line, const char* what, const std::string& note) {
    Stats& s = stats();
    ++s.asserts;
    if (ok) return;
    ++s.failed_asserts;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: ERROR in TEST_CASE(\"%s\"): %s%s%s\n", file, line, s.case_name, what,
                 note.empty() ? "" : " -- ", note.c_str());
    for (const std::string& c : s.context) std::fprintf(stderr, "    with %s\n", c.c_str());
}

template <typename T, typename = void>
struct streamable : std::false_type {};
template <typename T>
struct streamable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};

template <typename T>
std::string show(const T& v) {
    if constexpr (streamable<T>::value) {
        std::ostringstream o;
        o << v;
        return o.str();
    } else {
        return "{?}";
    }
}

class Capture {
public:
    template <typename T>
    Capture(const char* name, const T& v) {
        stats().context.push_back(std::string(name) + " := " + show(v));
    }
    ~Capture() { stats().context.pop_back(); }
};

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC(name, fn)                                                                    \
    static void fn();                                                                           \
    static const doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC(name, DOCTEST_CAT(doctest_case_, __COUNTER__))

#define DOCTEST_EVAL(expr, want, abort)                                                         \
    do {                                                                                        \
        bool doctest_ok_ = false;                                                               \
        std::string doctest_note_;                                                              \
        try {                                                                                   \
            doctest_ok_ = static_cast<bool>(expr) == (want);                                    \
        } catch (const std::exception& e) {                                                     \
            doctest_note_ = std::string("threw: ") + e.what();                                  \
        } catch (...) {                                                                         \
            doctest_note_ = "threw an unknown exception";                                       \
        }                                                                                       \
        doctest::detail::record(doctest_ok_, __FILE__, __LINE__, #expr, doctest_note_);         \
        if (!doctest_ok_ && (abort)) throw doctest::detail::AbortCase{};                        \
    } while (0)

#define CHECK(...) DOCTEST_EVAL((__VA_ARGS__), true, false)
#define CHECK_FALSE(...) DOCTEST_EVAL((__VA_ARGS__), false, false)
#define REQUIRE(...) DOCTEST_EVAL((__VA_ARGS__), true, true)

#define CHECK_THROWS_AS(expr, type)                                                             \
    do {                                                                                        \
        bool doctest_ok_ = false;                                                               \
        std::string doctest_note_ = "no exception";                                             \
        try {                                                                                   \
            static_cast<void>(expr);                                                            \
        } catch (const type&) {                                                                 \
            doctest_ok_ = true;                                                                 \
        } catch (const std::exception& e) {                                                     \
            doctest_note_ = std::string("wrong exception: ") + e.what();                        \
        } catch (...) {                                                                         \
            doctest_note_ = "wrong exception type";                                             \
        }                                                                                       \
        doctest::detail::record(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #type ")", \
                                doctest_ok_ ? std::string() : doctest_note_);                   \
    } while (0)

#define CHECK_NOTHROW(expr)                                                                     \
    do {                                                                                        \
        bool doctest_ok_ = true;                                                                \
        std::string doctest_note_;                                                              \
        try {                                                                                   \
            static_cast<void>(expr);                                                            \
        } catch (const std::exception& e) {                                                     \
            doctest_ok_ = false;                                                                \
            doctest_note_ = e.what();                                                           \
        } catch (...) {                                                                         \
            doctest_ok_ = false;                                                                \
        }                                                                                       \
        doctest::detail::record(doctest_ok_, __FILE__, __LINE__, "CHECK_NOTHROW(" #expr ")",    \
                                doctest_note_);                                                 \
    } while (0)

#define CAPTURE(x) const doctest::detail::Capture DOCTEST_CAT(doctest_capture_, __COUNTER__)(#x, x)

#define FAIL(msg)                                                                               \
    do {                                                                                        \
        doctest::detail::record(false, __FILE__, __LINE__, "FAIL", doctest::detail::show(msg)); \
        throw doctest::detail::AbortCase{};                                                     \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    using namespace doctest::detail;
    int failed_cases = 0;
    for (const Case& c : cases()) {
        Stats& s = stats();
        s.case_failed = false;
        s.case_name = c.name;
        s.context.clear();
        try {
            c.fn();
        } catch (const AbortCase&) {
        } catch (const std::exception& e) {
            record(false, c.file, c.line, "unexpected exception", e.what());
        } catch (...) {
            record(false, c.file, c.line, "unexpected exception", "unknown");
        }
        failed_cases += s.case_failed ? 1 : 0;
    }
    const Stats& s = stats();
    std::printf("[doctest] test cases: %zu | %zu passed | %d failed\n", cases().size(),
                cases().size() - size_t(failed_cases), failed_cases);
    std::printf("[doctest] assertions: %ld | %ld passed | %ld failed\n", s.asserts,
                s.asserts - s.failed_asserts, s.failed_asserts);
    std::printf("[doctest] Status: %s\n", failed_cases ? "FAILURE!" : "SUCCESS!");
    return failed_cases ? 1 : 0;
}
#endif
