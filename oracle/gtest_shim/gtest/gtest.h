// Minimal GoogleTest-compatible subset — TEST INFRASTRUCTURE ONLY.
// GTest is absent from this image; this lets the reference's own test
// sources (proj/tests/*.cpp) compile unmodified into oracle/_ref/ so they can
// validate the Eigen shim. Supports TEST, EXPECT/ASSERT_{EQ,NE,LT,LE,GT,GE,
// TRUE,FALSE,NEAR,DOUBLE_EQ,THROW}, FAIL() and streamed messages.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace testing {

struct TestCase {
  const char* suite;
  const char* name;
  std::function<void()> fn;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline bool& current_failed() {
  static bool f = false;
  return f;
}
inline int& total_failures() {
  static int f = 0;
  return f;
}

struct Registrar {
  Registrar(const char* s, const char* n, std::function<void()> f) { registry().push_back({s, n, std::move(f)}); }
};

// Collects the streamed message and reports on destruction.
class Reporter {
 public:
  Reporter(const char* file, int line, std::string what) : file_(file), line_(line), what_(std::move(what)) {}
  ~Reporter() {
    std::fprintf(stderr, "%s:%d: Failure\n%s%s%s\n", file_, line_, what_.c_str(),
                 msg_.str().empty() ? "" : "\n  ", msg_.str().c_str());
    current_failed() = true;
  }
  template <class T>
  Reporter& operator<<(const T& v) {
    msg_ << v;
    return *this;
  }

 private:
  const char* file_;
  int line_;
  std::string what_;
  std::ostringstream msg_;
};

// Swallows messages when the assertion passed.
struct Sink {
  template <class T>
  Sink& operator<<(const T&) {
    return *this;
  }
};

template <class T>
std::string repr(const T& v) {
  if constexpr (requires(std::ostream& o, const T& x) { o << x; }) {
    std::ostringstream o;
    o.precision(17);
    o << v;
    return o.str();
  } else {
    return "<value>";
  }
}

inline bool almost_equal_ulps(double a, double b) {
  if (std::isnan(a) || std::isnan(b)) return false;
  if (a == b) return true;
  auto biased = [](double x) {
    std::uint64_t u;
    std::memcpy(&u, &x, sizeof u);
    const std::uint64_t sign = std::uint64_t{1} << 63;
    return (u & sign) ? ~u + 1 : sign | u;
  };
  const std::uint64_t ua = biased(a), ub = biased(b);
  return (ua >= ub ? ua - ub : ub - ua) <= 4;
}

struct AssertionAbort {};

}  // namespace testing

#define GTEST_CAT_(a, b) a##b
#define GTEST_CAT(a, b) GTEST_CAT_(a, b)

#define TEST(suite, name)                                                                  \
  static void GTEST_CAT(gtest_fn_##suite##_, name)();                                      \
  static ::testing::Registrar GTEST_CAT(gtest_reg_##suite##_, name)(#suite, #name,         \
                                                                   &GTEST_CAT(gtest_fn_##suite##_, name)); \
  static void GTEST_CAT(gtest_fn_##suite##_, name)()

// The check itself: on failure, a Reporter collects the streamed message.
#define GTEST_CHECK_(cond, text, fatal)                                                        \
  if (cond)                                                                                    \
    ;                                                                                          \
  else                                                                                         \
    for (bool gtest_once_ = true; gtest_once_; gtest_once_ = false,                            \
              (fatal ? throw ::testing::AssertionAbort{} : (void)0))                         \
  ::testing::Reporter(__FILE__, __LINE__, text)

#define GTEST_BINARY_(a, b, op, fatal)                                                         \
  GTEST_CHECK_(((a)op(b)),                                                                     \
               std::string("Expected: (" #a ") " #op " (" #b "), actual: ") +                 \
                   ::testing::repr(a) + " vs " + ::testing::repr(b),                         \
               fatal)

#define EXPECT_EQ(a, b) GTEST_BINARY_(a, b, ==, false)
#define EXPECT_NE(a, b) GTEST_BINARY_(a, b, !=, false)
#define EXPECT_LT(a, b) GTEST_BINARY_(a, b, <, false)
#define EXPECT_LE(a, b) GTEST_BINARY_(a, b, <=, false)
#define EXPECT_GT(a, b) GTEST_BINARY_(a, b, >, false)
#define EXPECT_GE(a, b) GTEST_BINARY_(a, b, >=, false)
#define ASSERT_EQ(a, b) GTEST_BINARY_(a, b, ==, true)
#define ASSERT_NE(a, b) GTEST_BINARY_(a, b, !=, true)
#define ASSERT_LT(a, b) GTEST_BINARY_(a, b, <, true)
#define ASSERT_LE(a, b) GTEST_BINARY_(a, b, <=, true)
#define ASSERT_GT(a, b) GTEST_BINARY_(a, b, >, true)
#define ASSERT_GE(a, b) GTEST_BINARY_(a, b, >=, true)
#define EXPECT_TRUE(c) GTEST_CHECK_(static_cast<bool>(c), "Expected true: " #c, false)
#define EXPECT_FALSE(c) GTEST_CHECK_(!static_cast<bool>(c), "Expected false: " #c, false)
#define ASSERT_TRUE(c) GTEST_CHECK_(static_cast<bool>(c), "Expected true: " #c, true)
#define ASSERT_FALSE(c) GTEST_CHECK_(!static_cast<bool>(c), "Expected false: " #c, true)
#define EXPECT_NEAR(a, b, tol)                                                                  \
  GTEST_CHECK_(std::abs((a) - (b)) <= (tol),                                                  \
               std::string("Expected |" #a " - " #b "| <= " #tol ", actual: ") +              \
                   ::testing::repr(a) + " vs " + ::testing::repr(b),                         \
               false)
#define EXPECT_DOUBLE_EQ(a, b)                                                                  \
  GTEST_CHECK_(::testing::almost_equal_ulps((a), (b)),                                       \
               std::string("Expected double equality of " #a " and " #b ": ") +               \
                   ::testing::repr(a) + " vs " + ::testing::repr(b),                         \
               false)
#define EXPECT_THROW(stmt, exc)                                                                 \
  do {                                                                                          \
    bool gtest_caught_ = false;                                                                 \
    try {                                                                                       \
      stmt;                                                                                     \
    } catch (const exc&) {                                                                      \
      gtest_caught_ = true;                                                                     \
    } catch (...) {                                                                             \
    }                                                                                           \
    if (!gtest_caught_) ::testing::Reporter(__FILE__, __LINE__, "Expected " #stmt " to throw " #exc); \
  } while (0)
#define FAIL() GTEST_CHECK_(false, "Failed", true)
#define ADD_FAILURE() GTEST_CHECK_(false, "Failed", false)
#define SUCCEED() ::testing::Sink()

inline int gtest_shim_run_all(int argc, char** argv) {
  const char* filter = nullptr;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "--gtest_filter=", 15) == 0) filter = argv[i] + 15;
  }
  int passed = 0, failed = 0;
  std::vector<std::string> failed_names;
  for (const auto& tc : ::testing::registry()) {
    const std::string full = std::string(tc.suite) + "." + tc.name;
    if (filter && full.find(filter) == std::string::npos) continue;
    ::testing::current_failed() = false;
    std::printf("[ RUN      ] %s\n", full.c_str());
    std::fflush(stdout);
    try {
      tc.fn();
    } catch (const ::testing::AssertionAbort&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "uncaught exception: %s\n", e.what());
      ::testing::current_failed() = true;
    }
    if (::testing::current_failed()) {
      ++failed;
      failed_names.push_back(full);
      std::printf("[  FAILED  ] %s\n", full.c_str());
    } else {
      ++passed;
      std::printf("[       OK ] %s\n", full.c_str());
    }
    std::fflush(stdout);
  }
  std::printf("[==========] %d tests ran. [  PASSED  ] %d. [  FAILED  ] %d.\n", passed + failed, passed, failed);
  for (const auto& n : failed_names) std::printf("[  FAILED  ] %s\n", n.c_str());
  return failed == 0 ? 0 : 1;
}

#ifndef GTEST_SHIM_NO_MAIN
int main(int argc, char** argv) { return gtest_shim_run_all(argc, argv); }
#endif
