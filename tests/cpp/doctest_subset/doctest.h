// A small, from-scratch subset of the doctest unit-test API -- just what the
// reference's unit suites (/root/reference/proj/tests/test_*.cpp) use, so
// that they compile UNMODIFIED against the B200 drop-in (include/lamfast +
// liblamfast.so).  Not doctest: no third-party code is reproduced here; only
// the macro names and the documented semantics are followed:
//
//   TEST_SUITE(name) { ... }     groups test cases (the name is ignored)
//   TEST_CASE(name) { ... }      registers a test case
//   SUBCASE(name) { ... }        the test case is re-run once per leaf
//                                subcase; each run enters one new path
//   CHECK / REQUIRE (_FALSE)     assertions; REQUIRE aborts the test case
//   CHECK_THROWS, CHECK_THROWS_AS, CHECK_NOTHROW
//   CAPTURE(x)                   prints "x := value" with a failure
//   doctest::Approx(v).epsilon(e).scale(s)
//       |a - v| < e * (s + max(|a|, |v|)), default e = 100 * FLT_EPSILON,
//       s = 1 (doctest's published Approx semantics)
//
// Define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN in exactly one translation unit
// before including this header to get main().  Command line: `-tc=<substr>`
// runs only test cases whose name contains <substr>; `-ltc` lists them.
#ifndef LAMFAST_DOCTEST_SUBSET_H
#define LAMFAST_DOCTEST_SUBSET_H

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double value)
        : value_(value), epsilon_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0),
          scale_(1.0) {}
    Approx& epsilon(double e) {
        epsilon_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double lhs) const {
        return std::fabs(lhs - value_) < epsilon_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
    }
    double value() const { return value_; }

    friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
    friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || rhs.matches(lhs); }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || rhs.matches(lhs); }
    friend bool operator<(double lhs, const Approx& rhs) { return lhs < rhs.value_ && !rhs.matches(lhs); }
    friend bool operator>(double lhs, const Approx& rhs) { return lhs > rhs.value_ && !rhs.matches(lhs); }

private:
    double value_, epsilon_, scale_;
};

namespace detail {

// ---- value printing for failure messages --------------------------------
template <typename T, typename = void>
struct Printable : std::false_type {};
template <typename T>
struct Printable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};

template <typename T>
std::string show(const T& v) {
    if constexpr (std::is_same_v<T, Approx>) {
        std::ostringstream os;
        os.precision(17);
        os << "Approx( " << v.value() << " )";
        return os.str();
    } else if constexpr (std::is_same_v<T, bool>) {
        return v ? "true" : "false";
    } else if constexpr (std::is_arithmetic_v<T>) {
        std::ostringstream os;
        os.precision(17);
        os << v;
        return os.str();
    } else if constexpr (std::is_convertible_v<const T&, std::string>) {
        return "\"" + std::string(v) + "\"";
    } else if constexpr (Printable<T>::value) {
        std::ostringstream os;
        os.precision(17);
        os << v;
        std::string s = os.str();
        return s.size() > 200 ? s.substr(0, 200) + "..." : s;
    } else {
        return "{?}";
    }
}

// ---- run state ------------------------------------------------------------
struct Counters {
    long assertions = 0, failed_assertions = 0;
};

struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct RequireAbort {}; // thrown by a failed REQUIRE: ends the current run of the test case

struct State {
    Counters c;
    const TestCase* current = nullptr;
    bool current_failed = false;
    std::vector<std::string> captures;
    // subcase traversal (see Subcase)
    std::vector<std::string> path;                // names of the subcases entered, outermost first
    std::set<std::vector<std::string>> done;      // fully explored subcase paths
    bool root_child_entered = false;
    bool root_pending = false;
    struct Frame {
        bool child_entered = false;
        bool child_pending = false;
    };
    std::vector<Frame> frames;
};

inline State& state() {
    static State s;
    return s;
}

inline void report_failure(const char* kind, const char* expr, const char* file, int line,
                           const std::string& detail) {
    State& s = state();
    ++s.c.failed_assertions;
    s.current_failed = true;
    std::printf("%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, expr);
    if (!detail.empty())
        std::printf("  values: %s\n", detail.c_str());
    if (s.current)
        std::printf("  in test case: %s\n", s.current->name);
    for (const auto& p : s.path)
        std::printf("  in subcase: %s\n", p.c_str());
    for (const auto& cap : s.captures)
        std::printf("  logged: %s\n", cap.c_str());
}

// ---- expression decomposition: CHECK(a == b) prints both sides ---------------
struct Result {
    bool ok;
    std::string text;
};

template <typename L>
struct Lhs {
    const L& lhs;
    explicit Lhs(const L& l) : lhs(l) {}
#define LAMFAST_DOCTEST_BINOP(op)                                                   \
    template <typename R>                                                           \
    Result operator op(const R& rhs) const {                                        \
        const bool ok = static_cast<bool>(lhs op rhs);                              \
        return {ok, show(lhs) + " " #op " " + show(rhs)};                           \
    }
    LAMFAST_DOCTEST_BINOP(==)
    LAMFAST_DOCTEST_BINOP(!=)
    LAMFAST_DOCTEST_BINOP(<)
    LAMFAST_DOCTEST_BINOP(<=)
    LAMFAST_DOCTEST_BINOP(>)
    LAMFAST_DOCTEST_BINOP(>=)
#undef LAMFAST_DOCTEST_BINOP
    operator Result() const { return {static_cast<bool>(lhs), show(lhs)}; }
};

struct Decomposer {
    template <typename L>
    Lhs<L> operator<<(const L& l) const {
        return Lhs<L>(l);
    }
};

inline Result to_result(const Result& r) { return r; }
template <typename L>
Result to_result(const Lhs<L>& l) {
    return static_cast<Result>(l);
}

inline void assertion(const Result& r, bool expect, bool require, const char* kind, const char* expr,
                      const char* file, int line) {
    State& s = state();
    ++s.c.assertions;
    if (r.ok != expect) {
        report_failure(kind, expr, file, line, r.text);
        if (require)
            throw RequireAbort{};
    }
}

inline void unexpected_exception(const char* kind, const char* expr, const char* file, int line,
                                 const std::string& what, bool require) {
    State& s = state();
    ++s.c.assertions;
    report_failure(kind, expr, file, line, "threw an exception: " + what);
    if (require)
        throw RequireAbort{};
}

inline std::string exception_text(std::exception_ptr p) {
    try {
        std::rethrow_exception(p);
    } catch (const std::exception& e) {
        return e.what();
    } catch (const RequireAbort&) {
        throw;
    } catch (...) {
        return "unknown exception";
    }
}

// ---- registration ------------------------------------------------------------
struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

// ---- SUBCASE ----------------------------------------------------------------
// A test case is run repeatedly.  In one run, inside any scope at most one
// child subcase is entered: the first whose path is not yet fully explored.
// Any other unexplored child seen in that run marks its parent "pending", so
// the test case runs again; a subcase whose run saw no pending descendant is
// marked explored.  The run loop ends when the root has nothing pending.
struct Subcase {
    bool entered = false;
    Subcase(const char* name) {
        State& s = state();
        std::vector<std::string> key = s.path;
        key.push_back(name);
        bool& sibling_entered = s.frames.empty() ? s.root_child_entered : s.frames.back().child_entered;
        if (s.done.count(key))
            return;
        if (sibling_entered) {
            (s.frames.empty() ? s.root_pending : s.frames.back().child_pending) = true;
            return;
        }
        sibling_entered = true;
        entered = true;
        s.path.push_back(name);
        s.frames.push_back({});
    }
    ~Subcase() {
        if (!entered)
            return;
        State& s = state();
        const bool pending = s.frames.back().child_pending;
        s.frames.pop_back();
        if (!pending)
            s.done.insert(s.path);
        else
            (s.frames.empty() ? s.root_pending : s.frames.back().child_pending) = true;
        s.path.pop_back();
    }
    explicit operator bool() const { return entered; }
};

struct Capture {
    Capture(const char* name, const std::string& value) { state().captures.push_back(std::string(name) + " := " + value); }
    ~Capture() { state().captures.pop_back(); }
};

inline int run(int argc, char** argv) {
    std::string filter;
    bool list = false;
    for (int i = 1; i < argc; ++i) {
        if (std::strncmp(argv[i], "-tc=", 4) == 0)
            filter = argv[i] + 4;
        else if (std::strcmp(argv[i], "-ltc") == 0)
            list = true;
    }
    State& s = state();
    long cases = 0, failed_cases = 0, skipped = 0;
    for (const TestCase& tc : registry()) {
        if (!filter.empty() && std::string(tc.name).find(filter) == std::string::npos) {
            ++skipped;
            continue;
        }
        if (list) {
            std::printf("%s\n", tc.name);
            continue;
        }
        ++cases;
        s.current = &tc;
        s.current_failed = false;
        s.done.clear();
        int runs = 0;
        do {
            s.path.clear();
            s.frames.clear();
            s.captures.clear();
            s.root_child_entered = false;
            s.root_pending = false;
            try {
                tc.fn();
            } catch (const RequireAbort&) {
            } catch (const std::exception& e) {
                ++s.c.failed_assertions;
                s.current_failed = true;
                std::printf("%s:%d: ERROR: test case THREW exception: %s\n  in test case: %s\n", tc.file, tc.line,
                            e.what(), tc.name);
            } catch (...) {
                ++s.c.failed_assertions;
                s.current_failed = true;
                std::printf("%s:%d: ERROR: test case THREW an unknown exception\n  in test case: %s\n", tc.file,
                            tc.line, tc.name);
            }
            if (++runs > 100000)
                break;
        } while (s.root_pending);
        if (s.current_failed)
            ++failed_cases;
    }
    if (list)
        return 0;
    std::printf("[doctest-subset] test cases: %ld | %ld passed | %ld failed | %ld skipped\n", cases,
                cases - failed_cases, failed_cases, skipped);
    std::printf("[doctest-subset] assertions: %ld | %ld passed | %ld failed |\n", s.c.assertions,
                s.c.assertions - s.c.failed_assertions, s.c.failed_assertions);
    std::printf("[doctest-subset] Status: %s!\n", failed_cases ? "FAILURE" : "SUCCESS");
    return failed_cases ? 1 : 0;
}

} // namespace detail
} // namespace doctest

#define LAMFAST_DOCTEST_CAT_(a, b) a##b
#define LAMFAST_DOCTEST_CAT(a, b) LAMFAST_DOCTEST_CAT_(a, b)
#define LAMFAST_DOCTEST_UNIQUE(prefix) LAMFAST_DOCTEST_CAT(prefix, __COUNTER__)

#define LAMFAST_DOCTEST_TEST_CASE_IMPL(fn, name)                                                    \
    static void fn();                                                                             \
    static ::doctest::detail::Registrar LAMFAST_DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
    static void fn()
#define TEST_CASE(name) LAMFAST_DOCTEST_TEST_CASE_IMPL(LAMFAST_DOCTEST_UNIQUE(lamfast_doctest_case_), name)

#define TEST_SUITE(name) namespace LAMFAST_DOCTEST_UNIQUE(lamfast_doctest_suite_)

#define SUBCASE(name) if (const ::doctest::detail::Subcase LAMFAST_DOCTEST_UNIQUE(lamfast_doctest_sub_){name})

#define CAPTURE(x) ::doctest::detail::Capture LAMFAST_DOCTEST_UNIQUE(lamfast_doctest_cap_)(#x, ::doctest::detail::show(x))

#define LAMFAST_DOCTEST_ASSERT(kind, expect, require, ...)                                                     \
    do {                                                                                                    \
        try {                                                                                               \
            ::doctest::detail::assertion(                                                                   \
                ::doctest::detail::to_result(::doctest::detail::Decomposer() << __VA_ARGS__), expect, require, \
                kind, #__VA_ARGS__, __FILE__, __LINE__);                                                    \
        } catch (const ::doctest::detail::RequireAbort&) {                                                  \
            throw;                                                                                          \
        } catch (...) {                                                                                     \
            ::doctest::detail::unexpected_exception(                                                        \
                kind, #__VA_ARGS__, __FILE__, __LINE__,                                                     \
                ::doctest::detail::exception_text(std::current_exception()), require);                      \
        }                                                                                                   \
    } while (false)

#define CHECK(...) LAMFAST_DOCTEST_ASSERT("CHECK", true, false, __VA_ARGS__)
#define REQUIRE(...) LAMFAST_DOCTEST_ASSERT("REQUIRE", true, true, __VA_ARGS__)
#define CHECK_FALSE(...) LAMFAST_DOCTEST_ASSERT("CHECK_FALSE", false, false, __VA_ARGS__)
#define REQUIRE_FALSE(...) LAMFAST_DOCTEST_ASSERT("REQUIRE_FALSE", false, true, __VA_ARGS__)

#define LAMFAST_DOCTEST_THROWS(kind, expr, catch_clause)                                                        \
    do {                                                                                                     \
        ++::doctest::detail::state().c.assertions;                                                           \
        bool lamfast_threw_ = false;                                                                         \
        try {                                                                                                \
            expr;                                                                                            \
        } catch_clause catch (...) {                                                                         \
            ::doctest::detail::report_failure(kind, #expr, __FILE__, __LINE__,                                \
                                              "threw a different exception: " +                             \
                                                  ::doctest::detail::exception_text(std::current_exception())); \
            lamfast_threw_ = true;                                                                           \
        }                                                                                                    \
        if (!lamfast_threw_)                                                                                 \
            ::doctest::detail::report_failure(kind, #expr, __FILE__, __LINE__, "did not throw");             \
    } while (false)

#define CHECK_THROWS_AS(expr, ...) \
    LAMFAST_DOCTEST_THROWS("CHECK_THROWS_AS", expr, catch (const __VA_ARGS__&) { lamfast_threw_ = true; })
#define CHECK_THROWS(expr)                                                                             \
    do {                                                                                               \
        ++::doctest::detail::state().c.assertions;                                                     \
        bool lamfast_threw_ = false;                                                                   \
        try {                                                                                          \
            expr;                                                                                      \
        } catch (...) {                                                                                \
            lamfast_threw_ = true;                                                                     \
        }                                                                                              \
        if (!lamfast_threw_)                                                                           \
            ::doctest::detail::report_failure("CHECK_THROWS", #expr, __FILE__, __LINE__, "did not throw"); \
    } while (false)
#define CHECK_NOTHROW(expr)                                                                            \
    do {                                                                                               \
        ++::doctest::detail::state().c.assertions;                                                     \
        try {                                                                                          \
            expr;                                                                                      \
        } catch (...) {                                                                                \
            ::doctest::detail::report_failure("CHECK_NOTHROW", #expr, __FILE__, __LINE__,              \
                                              ::doctest::detail::exception_text(std::current_exception())); \
        }                                                                                              \
    } while (false)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif

#endif // LAMFAST_DOCTEST_SUBSET_H
