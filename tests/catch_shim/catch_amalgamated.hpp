// Minimal Catch2-v3-compatible test shim (Catch2 is not installed in this
// image). Implements exactly the surface the reference planner's test suites
// use: TEST_CASE, SECTION (flat, one leaf per run, like Catch), CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH, FAIL, CAPTURE,
// Catch::Approx (epsilon / margin) and Catch::Matchers::ContainsSubstring.
// Used to compile the reference's own tests unmodified against both the
// reference library (oracle/_ref) and ours (tests/test_reference_suites.py).
#pragma once

// The real amalgamated header pulls in much of the standard library; the
// reference tests rely on that transitively.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <iostream>
#include <map>
#include <memory>
#include <optional>
#include <string_view>
#include <tuple>
#include <utility>
#include <limits>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace catch_shim {

struct TestCase {
    std::string name, tags;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(void (*fn)(), const char* name, const char* tags) {
        registry().push_back({name, tags, fn});
    }
};

struct RunState {
    std::set<std::string> done_sections;
    bool entered_new = false;
    std::size_t assertions = 0;
    std::size_t failures = 0;
    std::string current;
};

inline RunState& state() {
    static RunState s;
    return s;
}

struct RequireAbort {};

inline void report(bool ok, const char* what, const char* file, int line) {
    auto& s = state();
    ++s.assertions;
    if (!ok) {
        ++s.failures;
        std::fprintf(stderr, "%s:%d: FAILED in '%s': %s\n", file, line, s.current.c_str(), what);
    }
}

// Enter a section iff no section was entered during this run and this one has
// not completed yet.
inline bool enter_section(const char* name) {
    auto& s = state();
    if (s.entered_new || s.done_sections.count(name)) return false;
    s.done_sections.insert(name);
    s.entered_new = true;
    return true;
}

}  // namespace catch_shim

namespace Catch {

class Approx {
public:
    explicit Approx(double v)
        : value_(v), epsilon_(std::numeric_limits<float>::epsilon() * 100.0), margin_(0.0) {}
    Approx& epsilon(double e) {
        epsilon_ = e;
        return *this;
    }
    Approx& margin(double m) {
        margin_ = m;
        return *this;
    }
    bool matches(double other) const {
        const double d = std::fabs(other - value_);
        if (d <= margin_) return true;
        const double scale = std::isinf(value_) ? 0.0 : std::fabs(value_);
        return d <= epsilon_ * (1.0 + scale) || other == value_;
    }
    friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
    friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }

private:
    double value_, epsilon_, margin_;
};

namespace Matchers {
struct ContainsSubstring {
    std::string needle;
    explicit ContainsSubstring(std::string n) : needle(std::move(n)) {}
    bool match(const std::string& s) const { return s.find(needle) != std::string::npos; }
};
}  // namespace Matchers

}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)

#define CATCH_SHIM_TEST_CASE(fn, name, tags)                          \
    static void fn();                                                 \
    static ::catch_shim::Registrar CATCH_SHIM_CAT(fn, _reg)(fn, name, tags); \
    static void fn()

#define TEST_CASE(name, tags) CATCH_SHIM_TEST_CASE(CATCH_SHIM_CAT(catch_shim_tc_, __COUNTER__), name, tags)

#define SECTION(name) if (::catch_shim::enter_section(name))

#define CHECK(...) ::catch_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::catch_shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                   \
    do {                                                                               \
        const bool catch_shim_ok = static_cast<bool>(__VA_ARGS__);                     \
        ::catch_shim::report(catch_shim_ok, #__VA_ARGS__, __FILE__, __LINE__);         \
        if (!catch_shim_ok) throw ::catch_shim::RequireAbort{};                        \
    } while (0)

#define CHECK_THROWS_AS(expr, type)                                                    \
    do {                                                                               \
        bool catch_shim_ok = false;                                                    \
        try {                                                                          \
            static_cast<void>(expr);                                                   \
        } catch (const type&) {                                                        \
            catch_shim_ok = true;                                                      \
        } catch (...) {                                                                \
        }                                                                              \
        ::catch_shim::report(catch_shim_ok, #expr " throws " #type, __FILE__, __LINE__); \
    } while (0)

#define CHECK_THROWS_WITH(expr, matcher)                                               \
    do {                                                                               \
        bool catch_shim_ok = false;                                                    \
        try {                                                                          \
            static_cast<void>(expr);                                                   \
        } catch (const std::exception& e) {                                           \
            catch_shim_ok = (matcher).match(e.what());                                 \
        } catch (...) {                                                                \
        }                                                                              \
        ::catch_shim::report(catch_shim_ok, #expr " throws with " #matcher, __FILE__, __LINE__); \
    } while (0)

#define FAIL(msg)                                                                      \
    do {                                                                               \
        ::catch_shim::report(false, msg, __FILE__, __LINE__);                          \
        throw ::catch_shim::RequireAbort{};                                            \
    } while (0)

#define CAPTURE(...) static_cast<void>(0)
