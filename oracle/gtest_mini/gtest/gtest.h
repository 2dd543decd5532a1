// gtest_mini — TEST INFRASTRUCTURE ONLY. A minimal GoogleTest-compatible header (GTest is not
// installed in this image) covering exactly the subset the reference's suites use:
// TEST, FAIL, ADD_FAILURE, EXPECT_/ASSERT_ {EQ, NE, LT, LE, GT, GE, TRUE, FALSE, NEAR, THROW, NO_THROW} with
// `<< message` streaming, and a main() with --gtest_filter (':'-separated globs, '-' negatives).
// Lets oracle/Makefile compile the reference's own test files (proj/tests/*.cpp) unmodified
// against (a) the reference library and (b) the B200 drop-in shim.
#pragma once
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include <unistd.h>  // real GTest headers pull this in; the suites use ::getpid

namespace gtest_mini {

struct TestCase {
  std::string suite, name;
  void (*fn)();
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline int& current_failures() {
  static int f = 0;
  return f;
}
struct Registrar {
  Registrar(const char* suite, const char* name, void (*fn)()) { registry().push_back({suite, name, fn}); }
};

template <typename T, typename = void>
struct printable : std::false_type {};
template <typename T>
struct printable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};
template <typename T>
std::string show(const T& v) {
  if constexpr (std::is_enum_v<T>) {
    return std::to_string(static_cast<long long>(v));
  } else if constexpr (printable<T>::value) {
    std::ostringstream os;
    os.precision(17);
    os << v;
    return os.str();
  } else {
    return "<unprintable>";
  }
}

struct Message {
  std::ostringstream os;
  template <typename T>
  Message& operator<<(const T& v) {
    os << v;
    return *this;
  }
};

struct Failure {
  const char* file;
  int line;
  std::string text;
  Failure(const char* f, int l, std::string t) : file(f), line(l), text(std::move(t)) {}
  void operator=(const Message& m) const {
    ++current_failures();
    std::string extra = m.os.str();
    std::fprintf(stderr, "%s:%d: Failure\n%s%s%s\n", file, line, text.c_str(), extra.empty() ? "" : "\n",
                 extra.c_str());
  }
};

template <typename A, typename B, typename Op>
std::pair<bool, std::string> cmp(const A& a, const B& b, Op op, const char* ea, const char* eb, const char* sym) {
  if (op(a, b)) return {true, std::string()};
  return {false, std::string("Expected: (") + ea + ") " + sym + " (" + eb + "), actual: " + show(a) + " vs " +
                     show(b)};
}

inline bool glob(const char* p, const char* s) {
  if (*p == 0) return *s == 0;
  if (*p == '*') return glob(p + 1, s) || (*s && glob(p, s + 1));
  if (*p == '?') return *s && glob(p + 1, s + 1);
  return *p == *s && glob(p + 1, s + 1);
}
inline bool any_glob(const std::string& pats, const std::string& name) {
  size_t i = 0;
  while (i <= pats.size()) {
    size_t j = pats.find(':', i);
    if (j == std::string::npos) j = pats.size();
    if (j > i && glob(pats.substr(i, j - i).c_str(), name.c_str())) return true;
    i = j + 1;
  }
  return false;
}

inline int run_all(int argc, char** argv) {
  std::string pos = "*", neg;
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "--gtest_filter=", 15) == 0) {
      std::string f = argv[i] + 15;
      const size_t dash = f.find('-');
      pos = dash == std::string::npos ? f : f.substr(0, dash);
      neg = dash == std::string::npos ? "" : f.substr(dash + 1);
      if (pos.empty()) pos = "*";
    }
  int ran = 0, failed = 0;
  std::vector<std::string> failed_names;
  for (const auto& t : registry()) {
    const std::string full = t.suite + "." + t.name;
    if (!any_glob(pos, full) || (!neg.empty() && any_glob(neg, full))) continue;
    ++ran;
    current_failures() = 0;
    std::printf("[ RUN      ] %s\n", full.c_str());
    std::fflush(stdout);
    try {
      t.fn();
    } catch (const std::exception& e) {
      ++current_failures();
      std::fprintf(stderr, "uncaught exception: %s\n", e.what());
    } catch (...) {
      ++current_failures();
      std::fprintf(stderr, "uncaught non-std exception\n");
    }
    if (current_failures()) {
      ++failed;
      failed_names.push_back(full);
      std::printf("[  FAILED  ] %s\n", full.c_str());
    } else {
      std::printf("[       OK ] %s\n", full.c_str());
    }
    std::fflush(stdout);
  }
  std::printf("[==========] %d tests ran.\n[  PASSED  ] %d tests.\n", ran, ran - failed);
  for (const auto& n : failed_names) std::printf("[  FAILED  ] %s\n", n.c_str());
  return failed ? 1 : 0;
}

}  // namespace gtest_mini

#define GTM_BLOCKER_ \
  switch (0)         \
  case 0:            \
  default:

#define TEST(suite, name)                                                                        \
  static void gtm_##suite##_##name();                                                            \
  static ::gtest_mini::Registrar gtm_reg_##suite##_##name(#suite, #name, &gtm_##suite##_##name); \
  static void gtm_##suite##_##name()

#define GTM_NONFATAL_(ok, text) \
  GTM_BLOCKER_ if (ok) {} else ::gtest_mini::Failure(__FILE__, __LINE__, text) = ::gtest_mini::Message()
#define GTM_FATAL_(ok, text) \
  GTM_BLOCKER_ if (ok) {} else return ::gtest_mini::Failure(__FILE__, __LINE__, text) = ::gtest_mini::Message()

#define GTM_CMP_(a, b, op, sym, KIND)                                                              \
  if (const auto gtm_r = ::gtest_mini::cmp((a), (b), [](const auto& x, const auto& y) { return x op y; }, \
                                           #a, #b, sym);                                           \
      true)                                                                                        \
  KIND(gtm_r.first, gtm_r.second)

#define EXPECT_EQ(a, b) GTM_CMP_(a, b, ==, "==", GTM_NONFATAL_)
#define EXPECT_NE(a, b) GTM_CMP_(a, b, !=, "!=", GTM_NONFATAL_)
#define EXPECT_LT(a, b) GTM_CMP_(a, b, <, "<", GTM_NONFATAL_)
#define EXPECT_LE(a, b) GTM_CMP_(a, b, <=, "<=", GTM_NONFATAL_)
#define EXPECT_GT(a, b) GTM_CMP_(a, b, >, ">", GTM_NONFATAL_)
#define EXPECT_GE(a, b) GTM_CMP_(a, b, >=, ">=", GTM_NONFATAL_)
#define ASSERT_EQ(a, b) GTM_CMP_(a, b, ==, "==", GTM_FATAL_)
#define ASSERT_NE(a, b) GTM_CMP_(a, b, !=, "!=", GTM_FATAL_)
#define ASSERT_LT(a, b) GTM_CMP_(a, b, <, "<", GTM_FATAL_)
#define ASSERT_LE(a, b) GTM_CMP_(a, b, <=, "<=", GTM_FATAL_)
#define ASSERT_GT(a, b) GTM_CMP_(a, b, >, ">", GTM_FATAL_)
#define ASSERT_GE(a, b) GTM_CMP_(a, b, >=, ">=", GTM_FATAL_)
#define EXPECT_TRUE(c) GTM_NONFATAL_(static_cast<bool>(c), "Expected true: " #c)
#define EXPECT_FALSE(c) GTM_NONFATAL_(!static_cast<bool>(c), "Expected false: " #c)
#define ASSERT_TRUE(c) GTM_FATAL_(static_cast<bool>(c), "Expected true: " #c)
#define ASSERT_FALSE(c) GTM_FATAL_(!static_cast<bool>(c), "Expected false: " #c)
#define EXPECT_NEAR(a, b, tol)                                                                    \
  GTM_NONFATAL_(std::abs(static_cast<double>(a) - static_cast<double>(b)) <= static_cast<double>(tol), \
                std::string("Expected |" #a " - " #b "| <= " #tol ", actual ") +                   \
                    ::gtest_mini::show(static_cast<double>(a)) + " vs " +                          \
                    ::gtest_mini::show(static_cast<double>(b)))

#define GTM_THROW_(stmt, exc, KIND)                                                   \
  if (const int gtm_t = [&]() -> int {                                                \
        try {                                                                         \
          stmt;                                                                       \
        } catch (const exc&) {                                                        \
          return 0;                                                                   \
        } catch (...) {                                                               \
          return 2;                                                                   \
        }                                                                             \
        return 1;                                                                     \
      }();                                                                            \
      true)                                                                           \
  KIND(gtm_t == 0, gtm_t == 1 ? "Expected " #stmt " to throw " #exc ", it threw nothing" \
                              : "Expected " #stmt " to throw " #exc ", it threw another type")
#define EXPECT_THROW(stmt, exc) GTM_THROW_(stmt, exc, GTM_NONFATAL_)
#define ASSERT_THROW(stmt, exc) GTM_THROW_(stmt, exc, GTM_FATAL_)
#define EXPECT_NO_THROW(stmt)                          \
  if (const bool gtm_ok = [&]() -> bool {              \
        try {                                          \
          stmt;                                        \
        } catch (...) {                                \
          return false;                                \
        }                                              \
        return true;                                   \
      }();                                             \
      true)                                            \
  GTM_NONFATAL_(gtm_ok, "Expected " #stmt " not to throw")
#define FAIL() GTM_FATAL_(false, "Failed")
#define ADD_FAILURE() GTM_NONFATAL_(false, "Failed")
#define SUCCEED() GTM_NONFATAL_(true, "")
