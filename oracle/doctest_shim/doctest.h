// Minimal doctest-compatible test harness (test infrastructure, not product).
// The reference's tests include <doctest.h>, which is not vendored in
// /root/reference (proj/.gitignore:2).  This header implements the subset those
// tests use -- TEST_CASE, SUBCASE, CHECK*, REQUIRE, INFO, doctest::Approx,
// doctest::Contains -- so the reference's own test files can be compiled
// unmodified against both the reference library and libp2bw.so.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <set>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    Approx& scale(double s) { scale_ = s; return *this; }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) <
               a.eps_ * (a.scale_ + std::fmax(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

private:
    double value_;
    double eps_ = 1.1920928955078125e-07 * 100;
    double scale_ = 1.0;
};

struct Contains {
    std::string needle;
    explicit Contains(const char* s) : needle(s) {}
    bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
};

namespace shim {

struct RequireFailed {};

struct Registry {
    struct Case { const char* name; const char* file; int line; void (*fn)(); };
    std::vector<Case> cases;
    int checks = 0, failures = 0;
    // subcase bookkeeping for the running test case
    std::set<std::pair<std::string, int>> done;
    bool entered = false, discovered_new = false;
    static Registry& get() { static Registry r; return r; }
};

inline int add_case(const char* name, const char* file, int line, void (*fn)()) {
    Registry::get().cases.push_back({name, file, line, fn});
    return 0;
}

inline void report(bool ok, const char* file, int line, const std::string& what) {
    auto& r = Registry::get();
    ++r.checks;
    if (!ok) {
        ++r.failures;
        std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, what.c_str());
    }
}

struct Subcase {
    bool active = false;
    std::pair<std::string, int> id;
    Subcase(const char* file, int line) : id(file, line) {
        auto& r = Registry::get();
        if (r.entered || r.done.count(id)) {
            if (!r.done.count(id)) r.discovered_new = true;
            return;
        }
        r.entered = true;
        active = true;
    }
    ~Subcase() {
        if (active) Registry::get().done.insert(id);
    }
    explicit operator bool() const { return active; }
};

inline bool matches(const Contains& c, const std::string& what) { return c.matches(what); }
inline bool matches(const char* s, const std::string& what) { return what == s; }
inline bool matches(const std::string& s, const std::string& what) { return what == s; }

template <class... Args>
std::string concat(Args&&... args) {
    std::ostringstream os;
    (os << ... << args);
    return os.str();
}

inline int run_all() {
    auto& r = Registry::get();
    int failed_cases = 0;
    for (const auto& c : r.cases) {
        r.done.clear();
        const int before = r.failures;
        for (int pass = 0; pass < 1000; ++pass) {
            r.entered = false;
            r.discovered_new = false;
            try {
                c.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                report(false, c.file, c.line, std::string("unexpected exception: ") + e.what());
            }
            if (!r.discovered_new) break;
        }
        if (r.failures != before) {
            ++failed_cases;
            std::fprintf(stderr, "[doctest-shim] FAILED test case: %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | failed: %d | assertions: %d | failed: %d\n",
                r.cases.size(), failed_cases, r.checks, r.failures);
    return r.failures == 0 ? 0 : 1;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQUE(base) DOCTEST_CAT(base, __LINE__)

#define TEST_CASE(name)                                                                      \
    static void DOCTEST_UNIQUE(doctest_fn_)();                                                \
    static const int DOCTEST_UNIQUE(doctest_reg_) =                                          \
        doctest::shim::add_case(name, __FILE__, __LINE__, &DOCTEST_UNIQUE(doctest_fn_));     \
    static void DOCTEST_UNIQUE(doctest_fn_)()

#define SUBCASE(name) if (const doctest::shim::Subcase DOCTEST_UNIQUE(doctest_sc_){__FILE__, __LINE__})

#define INFO(...) ((void)0)
#define CAPTURE(...) ((void)0)
#define MESSAGE(...) ((void)0)

#define CHECK(...) doctest::shim::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_MESSAGE(cond, ...) \
    doctest::shim::report(static_cast<bool>(cond), __FILE__, __LINE__, doctest::shim::concat(__VA_ARGS__))
#define REQUIRE(...)                                                                   \
    do {                                                                               \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                       \
        doctest::shim::report(doctest_ok_, __FILE__, __LINE__, #__VA_ARGS__);          \
        if (!doctest_ok_) throw doctest::shim::RequireFailed{};                        \
    } while (0)
#define FAIL(...)                                                                       \
    do {                                                                                \
        doctest::shim::report(false, __FILE__, __LINE__, doctest::shim::concat(__VA_ARGS__)); \
        throw doctest::shim::RequireFailed{};                                           \
    } while (0)

#define CHECK_THROWS_AS(expr, type)                                                     \
    do {                                                                                \
        bool doctest_ok_ = false;                                                       \
        try { (void)(expr); } catch (const type&) { doctest_ok_ = true; } catch (...) {} \
        doctest::shim::report(doctest_ok_, __FILE__, __LINE__, "throws " #type ": " #expr); \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, type)                                       \
    do {                                                                                \
        bool doctest_ok_ = false;                                                       \
        try { (void)(expr); } catch (const type& e) {                                   \
            doctest_ok_ = doctest::shim::matches(matcher, e.what());                    \
        } catch (...) {}                                                                \
        doctest::shim::report(doctest_ok_, __FILE__, __LINE__, "throws-with " #expr);   \
    } while (0)

#define CHECK_NOTHROW(expr)                                                             \
    do {                                                                                \
        bool doctest_ok_ = true;                                                        \
        try { (void)(expr); } catch (...) { doctest_ok_ = false; }                      \
        doctest::shim::report(doctest_ok_, __FILE__, __LINE__, "nothrow " #expr);       \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::shim::run_all(); }
#endif
