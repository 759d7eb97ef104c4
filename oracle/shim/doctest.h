// Minimal doctest stand-in — TEST INFRASTRUCTURE ONLY.
//
// The reference vendors doctest under proj/vendor/ (proj/CMakeLists.txt:5),
// which is git-ignored and absent from the mount (proj/.gitignore:2).  This
// header implements the subset the reference's unit tests use (TEST_CASE,
// CHECK, CHECK_FALSE, REQUIRE, FAIL, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// doctest::Approx, doctest::Contains) so the unmodified test sources compile
// into oracle/_ref/unit_tests.  Approx follows doctest's definition:
//   |a - b| < eps * (scale + max(|a|, |b|)),  eps = 100 * FLT_EPSILON, scale = 1.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
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
inline const char*& current_test() {
    static const char* t = "";
    return t;
}

struct Registrar {
    Registrar(const char* name, void (*fn)(), const char* file, int line) {
        registry().push_back({name, fn, file, line});
    }
};

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    ++checks();
    if (ok) return;
    ++failures();
    std::printf("%s:%d: FAILED in \"%s\": %s\n", file, line, current_test(), expr);
    if (require) throw RequireFailed{};
}

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) <
               rhs.eps_ * (rhs.scale_ + std::fmax(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return operator==(rhs, lhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !operator==(lhs, rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !operator==(rhs, lhs); }

private:
    double value_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
    double scale_ = 1.0;
};

struct Contains {
    std::string s;
    explicit Contains(const char* x) : s(x) {}
    explicit Contains(std::string x) : s(std::move(x)) {}
    bool check(const std::string& what) const { return what.find(s) != std::string::npos; }
};

inline int run_all() {
    int failed_cases = 0;
    for (const auto& tc : registry()) {
        current_test() = tc.name;
        int before = failures();
        try {
            tc.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++failures();
            std::printf("%s:%d: EXCEPTION in \"%s\": %s\n", tc.file, tc.line, tc.name, e.what());
        }
        if (failures() != before) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
                registry().size() - failed_cases, failed_cases);
    std::printf("[doctest-shim] assertions: %d | %d passed | %d failed\n", checks(),
                checks() - failures(), failures());
    std::printf("[doctest-shim] Status: %s\n", failed_cases ? "FAILURE!" : "SUCCESS!");
    return failed_cases ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                        \
    static void fn();                                                                \
    static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);  \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(msg) doctest::report(false, "FAIL", __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                   \
    do {                                                                             \
        bool ok_ = false;                                                            \
        try {                                                                        \
            (void)(expr);                                                            \
        } catch (const __VA_ARGS__&) {                                               \
            ok_ = true;                                                              \
        } catch (...) {                                                              \
        }                                                                            \
        doctest::report(ok_, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                     \
    do {                                                                             \
        bool ok_ = false;                                                            \
        try {                                                                        \
            (void)(expr);                                                            \
        } catch (const __VA_ARGS__& e_) {                                            \
            ok_ = (matcher).check(e_.what());                                        \
        } catch (...) {                                                              \
        }                                                                            \
        doctest::report(ok_, "throws-with " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
