// Minimal doctest-compatible shim -- TEST INFRASTRUCTURE ONLY.
//
// The reference vendors doctest under proj/vendor/ (git-ignored and absent,
// /root/reference/proj/.gitignore:2). This header implements just the subset
// its hot-path tests use (TEST_CASE, CHECK*, REQUIRE*, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, INFO, FAIL, doctest::Approx, doctest::Contains) so
// proj/tests/test_distattention.cpp and acceptance_test.cpp compile unchanged,
// both against the reference (oracle/_ref) and against the B200 drop-in
// adapter (build/dropin). Run with `-tc=<name>` (or `-tc=<prefix>*`) to select cases.
#pragma once
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    Approx& scale(double s) { scl = s; return *this; }
    double value;
    double eps = 1.1920928955078125e-07 * 100;  // float epsilon x 100, as doctest
    double scl = 1.0;
    bool match(double lhs) const {
        return std::fabs(lhs - value) < eps * (scl + std::max(std::fabs(lhs), std::fabs(value)));
    }
};
inline bool operator==(double l, const Approx& r) { return r.match(l); }
inline bool operator==(const Approx& l, double r) { return l.match(r); }
inline bool operator!=(double l, const Approx& r) { return !r.match(l); }
inline bool operator!=(const Approx& l, double r) { return !l.match(r); }
inline bool operator<=(double l, const Approx& r) { return l < r.value || r.match(l); }
inline bool operator>=(double l, const Approx& r) { return l > r.value || r.match(l); }
inline bool operator<(double l, const Approx& r) { return l < r.value && !r.match(l); }
inline bool operator>(double l, const Approx& r) { return l > r.value && !r.match(l); }

struct Contains {
    explicit Contains(const char* s) : str(s) {}
    std::string str;
    bool check(const std::string& what) const { return what.find(str) != std::string::npos; }
};

namespace detail {
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
struct Registrar {
    Registrar(const char* name, void (*fn)(), const char* file, int line) {
        registry().push_back({name, fn, file, line});
    }
};
struct RequireFailed {};
inline long& asserts() { static long n = 0; return n; }
inline long& failed_asserts() { static long n = 0; return n; }
inline bool& case_failed() { static bool b = false; return b; }
inline std::vector<std::string>& info_stack() { static std::vector<std::string> s; return s; }
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   bool fatal) {
    ++asserts();
    if (ok) return;
    ++failed_asserts();
    case_failed() = true;
    if (failed_asserts() <= 50) {
        std::printf("%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, expr);
        for (auto& s : info_stack()) std::printf("  logged: %s\n", s.c_str());
    }
    if (fatal) throw RequireFailed{};
}
struct InfoScope {
    template <class T>
    explicit InfoScope(const T& v) {
        std::ostringstream os;
        os << v;
        info_stack().push_back(os.str());
    }
    ~InfoScope() { info_stack().pop_back(); }
};
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                   \
    static void fn();                                                               \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, fn, __FILE__,   \
                                                              __LINE__);            \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define DOCTEST_ASSERT_(kind, cond, fatal) \
    ::doctest::detail::report(static_cast<bool>(cond), kind, #cond, __FILE__, __LINE__, fatal)
#define CHECK(...) DOCTEST_ASSERT_("CHECK", (__VA_ARGS__), false)
#define CHECK_FALSE(...) DOCTEST_ASSERT_("CHECK_FALSE", !(__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_ASSERT_("REQUIRE", (__VA_ARGS__), true)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_("REQUIRE_FALSE", !(__VA_ARGS__), true)
#define CHECK_NOTHROW(...)                                                             \
    do {                                                                               \
        bool ok_ = true;                                                               \
        try { (void)(__VA_ARGS__); } catch (...) { ok_ = false; }                      \
        ::doctest::detail::report(ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__, \
                                  false);                                              \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                     \
    do {                                                                               \
        bool ok_ = false;                                                              \
        try { (void)(expr); } catch (const __VA_ARGS__&) { ok_ = true; } catch (...) {} \
        ::doctest::detail::report(ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                          \
    do {                                                                               \
        bool ok_ = false;                                                              \
        try { (void)(expr); } catch (const __VA_ARGS__& e_) {                          \
            ok_ = ::doctest::Contains(with).check(e_.what());                          \
        } catch (...) {}                                                               \
        ::doctest::detail::report(ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__, \
                                  false);                                              \
    } while (0)
#define INFO(...) \
    ::doctest::detail::InfoScope DOCTEST_CAT(doctest_info_, __COUNTER__)(__VA_ARGS__)
#define FAIL(...) ::doctest::detail::report(false, "FAIL", #__VA_ARGS__, __FILE__, __LINE__, true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    std::vector<std::string> include, exclude;
    for (int i = 1; i < argc; ++i) {
        if (!std::strncmp(argv[i], "-tc=", 4)) include.push_back(argv[i] + 4);
        if (!std::strncmp(argv[i], "-tce=", 5)) exclude.push_back(argv[i] + 5);
    }
    int ran = 0, failed = 0;
    for (auto& tc : ::doctest::detail::registry()) {
        std::string name = tc.name;
        // exact name, or prefix match when the filter ends in '*'
        auto match = [&](const std::string& f) {
            if (!f.empty() && f.back() == '*') return name.compare(0, f.size() - 1, f, 0, f.size() - 1) == 0;
            return name == f;
        };
        bool sel = include.empty();
        for (auto& s : include) sel = sel || match(s);
        for (auto& s : exclude) sel = sel && !match(s);
        if (!sel) continue;
        ++ran;
        ::doctest::detail::case_failed() = false;
        try {
            tc.fn();
        } catch (const ::doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            std::printf("%s:%d: ERROR: test case THREW exception: %s\n", tc.file, tc.line, e.what());
            ::doctest::detail::case_failed() = true;
        }
        if (::doctest::detail::case_failed()) {
            ++failed;
            std::printf("[doctest] FAILED: %s\n", tc.name);
        }
        std::fflush(stdout);
    }
    std::printf("[doctest] test cases: %d | %d passed | %d failed\n", ran, ran - failed, failed);
    std::printf("[doctest] assertions: %ld | %ld passed | %ld failed\n",
                ::doctest::detail::asserts(),
                ::doctest::detail::asserts() - ::doctest::detail::failed_asserts(),
                ::doctest::detail::failed_asserts());
    std::printf("[doctest] Status: %s!\n", failed ? "FAILURE" : "SUCCESS");
    return failed ? 1 : 0;
}
#endif
