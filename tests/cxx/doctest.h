// Minimal doctest-compatible harness (doctest itself is not in the image) so the
// reference's own unit suites compile unchanged.  Supports the subset they use:
// TEST_CASE, REQUIRE, REQUIRE_FALSE, CHECK, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// INFO, doctest::Approx (doctest's epsilon * (scale + max(|a|,|b|)) rule).
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {
struct Failure : std::exception {
    std::string what_;
    explicit Failure(std::string w) : what_(std::move(w)) {}
    const char* what() const noexcept override { return what_.c_str(); }
};
struct Case {
    const char* name;
    std::function<void()> fn;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, std::function<void()> fn) { registry().push_back({name, std::move(fn)}); }
};
class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v_) < b.eps_ * (b.scale_ + std::fmax(std::fabs(a), std::fabs(b.v_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }

private:
    double v_, eps_ = 1.1920929e-07f * 100, scale_ = 1.0;
};
inline std::string Contains(const std::string& s) { return s; }
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                          \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                            \
    static doctest::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(name, DOCTEST_CAT(doctest_fn_, __LINE__)); \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define DOCTEST_FAIL(msg)                                                                        \
    do {                                                                                         \
        std::ostringstream os_;                                                                  \
        os_ << __FILE__ << ":" << __LINE__ << ": " << msg;                                       \
        throw doctest::Failure(os_.str());                                                       \
    } while (0)
#define REQUIRE(...)                                                                             \
    do {                                                                                         \
        if (!(__VA_ARGS__)) DOCTEST_FAIL("REQUIRE(" #__VA_ARGS__ ")");                          \
    } while (0)
#define CHECK(...) REQUIRE(__VA_ARGS__)
#define REQUIRE_FALSE(...)                                                                       \
    do {                                                                                         \
        if ((__VA_ARGS__)) DOCTEST_FAIL("REQUIRE_FALSE(" #__VA_ARGS__ ")");                     \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                              \
    do {                                                                                         \
        bool ok_ = false;                                                                        \
        try {                                                                                    \
            (void)(expr);                                                                        \
        } catch (const type&) {                                                                  \
            ok_ = true;                                                                          \
        } catch (...) {                                                                          \
        }                                                                                        \
        if (!ok_) DOCTEST_FAIL("CHECK_THROWS_AS(" #expr ", " #type ")");                         \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, needle, type)                                                 \
    do {                                                                                         \
        bool ok_ = false;                                                                        \
        try {                                                                                    \
            (void)(expr);                                                                        \
        } catch (const type& e_) {                                                               \
            ok_ = std::string(e_.what()).find(needle) != std::string::npos;                     \
        } catch (...) {                                                                          \
        }                                                                                        \
        if (!ok_) DOCTEST_FAIL("CHECK_THROWS_WITH_AS(" #expr ")");                               \
    } while (0)
#define INFO(...) (void)0
