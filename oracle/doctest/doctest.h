// oracle/doctest/doctest.h -- TEST INFRASTRUCTURE ONLY.
//
// The reference's unit tests (proj/tests/test_*.cpp) are written against the
// doctest single-header framework, which its CMake expects under proj/vendor/
// (proj/CMakeLists.txt:5) and which is not present in /root/reference or in
// this image.  This header is a small from-scratch implementation of the part
// of doctest's documented macro API those files use, so they compile
// UNMODIFIED -- once against the reference itself (oracle/_ref) and once
// against the B200 drop-in library (libspecsense_b200.so):
//
//   TEST_CASE, SUBCASE (re-run-per-leaf semantics), CHECK, CHECK_FALSE,
//   REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS + doctest::Contains,
//   CHECK_NOTHROW, doctest::Approx (+ .epsilon), DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
//
// Approx follows doctest's documented rule: |a - b| < eps * (scale + max(|a|, |b|)),
// default eps = 100 * FLT_EPSILON, scale 1.  No expression decomposition: a failed
// check prints its source text, file and line.  main() accepts substring filters
// (-tc=<substr>, repeatable) and exits nonzero when any check failed.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <set>
#include <string>
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
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double x) const {
        return std::fabs(x - value_) < eps_ * (scale_ + std::fmax(std::fabs(x), std::fabs(value_)));
    }
    template <typename T>
    friend bool operator==(const T& lhs, const Approx& rhs) {
        return rhs.matches(static_cast<double>(lhs));
    }
    template <typename T>
    friend bool operator==(const Approx& lhs, const T& rhs) {
        return lhs.matches(static_cast<double>(rhs));
    }
    template <typename T>
    friend bool operator!=(const T& lhs, const Approx& rhs) {
        return !rhs.matches(static_cast<double>(lhs));
    }
    template <typename T>
    friend bool operator!=(const Approx& lhs, const T& rhs) {
        return !lhs.matches(static_cast<double>(rhs));
    }

  private:
    double value_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
    double scale_ = 1.0;
};

struct Contains {
    std::string needle;
    explicit Contains(const char* s) : needle(s) {}
    bool matches(const char* what) const { return std::strstr(what, needle.c_str()) != nullptr; }
};

namespace detail {

using TestFn = void (*)();

struct TestCase {
    TestFn fn;
    const char* name;
    const char* file;
    int line;
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(TestFn fn, const char* name, const char* file, int line) {
        registry().push_back({fn, name, file, line});
    }
};

struct RequireAbort {};  // thrown by a failed REQUIRE; ends the current run of the test case

struct Frame {
    std::string path;
    bool entered_child = false;
    bool pending = false;
};

struct State {
    const TestCase* tc = nullptr;
    std::vector<Frame> stack;
    std::set<std::string> done;
    long long checks = 0;
    long long failed_checks = 0;
    bool case_failed = false;
};

inline State& state() {
    static State s;
    return s;
}

inline void report_failure(const char* file, int line, const char* kind, const char* expr, const char* extra = nullptr) {
    State& s = state();
    ++s.failed_checks;
    s.case_failed = true;
    std::string where;
    for (std::size_t i = 1; i < s.stack.size(); ++i) where += " / " + s.stack[i].path.substr(s.stack[i].path.rfind('\x1f') + 1);
    std::printf("%s:%d: FAILED %s( %s )%s%s  [test case \"%s\"%s]\n", file, line, kind, expr, extra ? " -- " : "",
                extra ? extra : "", s.tc ? s.tc->name : "?", where.c_str());
    std::fflush(stdout);
}

inline void check(bool ok, const char* file, int line, const char* kind, const char* expr, bool require) {
    ++state().checks;
    if (ok) return;
    report_failure(file, line, kind, expr);
    if (require) throw RequireAbort{};
}

// SUBCASE: the enclosing test case is re-run until every leaf subcase has been
// entered exactly once; each run enters at most one not-yet-finished subcase per
// nesting level (the first one met), as doctest documents.
class Subcase {
  public:
    Subcase(const char* name, const char* file, int line) {
        State& s = state();
        Frame& parent = s.stack.back();
        path_ = parent.path + "\x1e" + file + ":" + std::to_string(line) + "\x1f" + name;
        if (s.done.count(path_)) return;
        if (parent.entered_child) {
            parent.pending = true;
            return;
        }
        parent.entered_child = true;
        s.stack.push_back(Frame{path_});
        entered_ = true;
    }
    ~Subcase() {
        if (!entered_) return;
        State& s = state();
        const Frame f = s.stack.back();
        s.stack.pop_back();
        if (f.pending)
            s.stack.back().pending = true;
        else
            s.done.insert(path_);
    }
    Subcase(const Subcase&) = delete;
    Subcase& operator=(const Subcase&) = delete;
    explicit operator bool() const { return entered_; }

  private:
    std::string path_;
    bool entered_ = false;
};

inline bool selected(const TestCase& tc, const std::vector<std::string>& filters) {
    if (filters.empty()) return true;
    for (const auto& f : filters)
        if (std::strstr(tc.name, f.c_str())) return true;
    return false;
}

inline int run_all(int argc, char** argv) {
    std::vector<std::string> filters;
    for (int i = 1; i < argc; ++i) {
        const char* a = argv[i];
        if (std::strncmp(a, "-tc=", 4) == 0) filters.emplace_back(a + 4);
        if (std::strncmp(a, "--test-case=", 12) == 0) filters.emplace_back(a + 12);
    }
    State& s = state();
    int n_run = 0, n_failed = 0;
    for (const TestCase& tc : registry()) {
        if (!selected(tc, filters)) continue;
        ++n_run;
        s.tc = &tc;
        s.done.clear();
        s.case_failed = false;
        for (int run = 0; run < 100000; ++run) {
            s.stack.assign(1, Frame{std::string(tc.name)});
            const std::size_t done_before = s.done.size();
            bool aborted = true;
            try {
                tc.fn();
                aborted = false;
            } catch (const RequireAbort&) {
            } catch (const std::exception& e) {
                report_failure(tc.file, tc.line, "TEST_CASE", tc.name, (std::string("unexpected exception: ") + e.what()).c_str());
            } catch (...) {
                report_failure(tc.file, tc.line, "TEST_CASE", tc.name, "unexpected non-std exception");
            }
            // an aborted run may have left later sibling subcases undiscovered
            if (aborted && s.done.size() > done_before) continue;
            if (!s.stack.front().pending) break;
        }
        if (s.case_failed) ++n_failed;
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | checks: %lld | %lld failed\n", n_run,
                n_run - n_failed, n_failed, s.checks, s.failed_checks);
    return n_failed == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define DOCTEST_TEST_CASE_IMPL(fn, reg, name)                                                  \
    static void fn();                                                                          \
    static const ::doctest::detail::Registrar reg(&fn, name, __FILE__, __LINE__);              \
    static void fn()
#define DOCTEST_TEST_CASE_2(id, name) \
    DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_tc_fn_, id), DOCTEST_CAT(doctest_tc_reg_, id), name)
#define TEST_CASE(name) DOCTEST_TEST_CASE_2(__COUNTER__, name)

#define SUBCASE(name)                                                                               \
    if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name, __FILE__, __LINE__}; \
        DOCTEST_CAT(doctest_sc_, __LINE__))

#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK", #__VA_ARGS__, false)
#define CHECK_FALSE(...) \
    ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK_FALSE", #__VA_ARGS__, false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "REQUIRE", #__VA_ARGS__, true)

#define CHECK_THROWS_AS(expr, ...)                                                                  \
    do {                                                                                            \
        bool doctest_ok_ = false;                                                                   \
        try {                                                                                       \
            static_cast<void>(expr);                                                                \
        } catch (const __VA_ARGS__&) {                                                              \
            doctest_ok_ = true;                                                                     \
        } catch (...) {                                                                             \
        }                                                                                           \
        ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, false); \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                       \
    do {                                                                                            \
        bool doctest_ok_ = false;                                                                   \
        try {                                                                                       \
            static_cast<void>(expr);                                                                \
        } catch (const __VA_ARGS__& e) {                                                            \
            doctest_ok_ = (with).matches(e.what());                                                 \
        } catch (...) {                                                                             \
        }                                                                                           \
        ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS", #expr ", " #__VA_ARGS__, false); \
    } while (0)

#define CHECK_NOTHROW(...)                                                                          \
    do {                                                                                            \
        bool doctest_ok_ = true;                                                                    \
        try {                                                                                       \
            static_cast<void>(__VA_ARGS__);                                                         \
        } catch (...) {                                                                             \
            doctest_ok_ = false;                                                                    \
        }                                                                                           \
        ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "CHECK_NOTHROW", #__VA_ARGS__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv); }
#endif
