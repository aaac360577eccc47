// Minimal GoogleTest-compatible harness -- TEST INFRASTRUCTURE ONLY.
//
// GoogleTest is not installed in this image, so this header supplies the
// subset of its API that the reference's own unit tests use
// (/root/reference/proj/tests/*.cpp: TEST, TEST_F, EXPECT_*/ASSERT_*,
// GTEST_SKIP, ::testing::Test::HasFailure).  It lets oracle/Makefile compile
// those test files unchanged against the shimmed reference headers, which is
// how the shim SparseSolver (oracle/shim/tpfem/solve.hpp) is pinned to the
// reference's own known-answer tests.  main() is provided when
// GTEST_SHIM_MAIN is defined (the Makefile defines it).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace testing {

namespace internal {

struct Registry {
  struct Entry {
    std::string suite, name;
    std::function<void()> run;
  };
  std::vector<Entry> tests;
  bool current_failed = false;
  bool current_skipped = false;
  static Registry& get() {
    static Registry r;
    return r;
  }
};

struct FatalFailure {};
struct SkipTest {};

// Collects the streamed user message and reports on destruction.
class Reporter {
 public:
  Reporter(bool failed, const char* file, int line, std::string what, bool fatal)
      : failed_(failed), file_(file), line_(line), what_(std::move(what)), fatal_(fatal) {}
  template <class T>
  Reporter& operator<<(const T& v) {
    if (failed_) msg_ << v;
    return *this;
  }
  ~Reporter() noexcept(false) {
    if (!failed_) return;
    Registry::get().current_failed = true;
    std::cerr << file_ << ":" << line_ << ": Failure\n  " << what_;
    const std::string m = msg_.str();
    if (!m.empty()) std::cerr << "\n  " << m;
    std::cerr << "\n";
    if (fatal_ && !std::uncaught_exceptions()) throw FatalFailure{};
  }

 private:
  bool failed_;
  const char* file_;
  int line_;
  std::string what_;
  bool fatal_;
  std::ostringstream msg_;
};

template <class A, class B>
std::string describe(const char* op, const char* ea, const char* eb, const A& a, const B& b) {
  std::ostringstream s;
  s.precision(17);
  s << "Expected: (" << ea << ") " << op << " (" << eb << "), actual: ";
  if constexpr (requires(std::ostream& o) { o << a; o << b; }) {
    s << a << " vs " << b;
  } else {
    s << "<unprintable>";
  }
  return s.str();
}

inline bool double_eq(double a, double b) {
  if (a == b) return true;
  if (std::isnan(a) || std::isnan(b)) return false;
  // 4 ULPs, like gtest's AlmostEquals.
  const double diff = std::fabs(a - b);
  const double scale = std::fmax(std::fabs(a), std::fabs(b));
  return diff <= 4.0 * 2.220446049250313e-16 * scale;
}

}  // namespace internal

class Test {
 public:
  virtual ~Test() = default;
  virtual void SetUp() {}
  virtual void TearDown() {}
  virtual void TestBody() = 0;
  static bool HasFailure() { return internal::Registry::get().current_failed; }
};

inline int RunAllTests() {
  auto& reg = internal::Registry::get();
  int failed = 0, skipped = 0;
  for (auto& t : reg.tests) {
    reg.current_failed = false;
    reg.current_skipped = false;
    std::cout << "[ RUN      ] " << t.suite << "." << t.name << std::endl;
    try {
      t.run();
    } catch (const internal::FatalFailure&) {
    } catch (const internal::SkipTest&) {
      reg.current_skipped = true;
    } catch (const std::exception& e) {
      reg.current_failed = true;
      std::cerr << "  uncaught exception: " << e.what() << "\n";
    }
    if (reg.current_failed) {
      ++failed;
      std::cout << "[  FAILED  ] " << t.suite << "." << t.name << std::endl;
    } else if (reg.current_skipped) {
      ++skipped;
      std::cout << "[  SKIPPED ] " << t.suite << "." << t.name << std::endl;
    } else {
      std::cout << "[       OK ] " << t.suite << "." << t.name << std::endl;
    }
  }
  std::cout << "[==========] " << reg.tests.size() << " tests, " << failed << " failed, "
            << skipped << " skipped" << std::endl;
  return failed == 0 ? 0 : 1;
}

}  // namespace testing

#define GTS_CONCAT_(a, b) a##b
#define GTS_CONCAT(a, b) GTS_CONCAT_(a, b)

#define GTS_DEFINE_TEST_(suite, name, base)                                              \
  class GTS_CONCAT(suite, GTS_CONCAT(_, GTS_CONCAT(name, _Test))) : public base {         \
   public:                                                                               \
    void TestBody() override;                                                            \
  };                                                                                     \
  static const bool GTS_CONCAT(gts_reg_, GTS_CONCAT(suite, GTS_CONCAT(_, name))) = [] {   \
    ::testing::internal::Registry::get().tests.push_back(                                \
        {#suite, #name, [] {                                                             \
           GTS_CONCAT(suite, GTS_CONCAT(_, GTS_CONCAT(name, _Test))) t;                   \
           t.SetUp();                                                                    \
           try {                                                                         \
             t.TestBody();                                                               \
           } catch (...) {                                                               \
             t.TearDown();                                                               \
             throw;                                                                      \
           }                                                                             \
           t.TearDown();                                                                 \
         }});                                                                            \
    return true;                                                                         \
  }();                                                                                   \
  void GTS_CONCAT(suite, GTS_CONCAT(_, GTS_CONCAT(name, _Test)))::TestBody()

namespace testing::internal {
class PlainTest : public ::testing::Test {};
}  // namespace testing::internal

#define TEST(suite, name) GTS_DEFINE_TEST_(suite, name, ::testing::internal::PlainTest)
#define TEST_F(fixture, name) GTS_DEFINE_TEST_(fixture, name, fixture)

#define GTS_CMP_(fatal, op, a, b)                                                          \
  for (bool gts_once = true; gts_once; gts_once = false)                                   \
    for (const auto& gts_a = (a); gts_once; gts_once = false)                              \
      for (const auto& gts_b = (b); gts_once; gts_once = false)                            \
  ::testing::internal::Reporter(!(gts_a op gts_b), __FILE__, __LINE__,                      \
                                ::testing::internal::describe(#op, #a, #b, gts_a, gts_b),   \
                                fatal)

#define EXPECT_EQ(a, b) GTS_CMP_(false, ==, a, b)
#define EXPECT_NE(a, b) GTS_CMP_(false, !=, a, b)
#define EXPECT_LT(a, b) GTS_CMP_(false, <, a, b)
#define EXPECT_LE(a, b) GTS_CMP_(false, <=, a, b)
#define EXPECT_GT(a, b) GTS_CMP_(false, >, a, b)
#define EXPECT_GE(a, b) GTS_CMP_(false, >=, a, b)
#define ASSERT_EQ(a, b) GTS_CMP_(true, ==, a, b)
#define ASSERT_NE(a, b) GTS_CMP_(true, !=, a, b)
#define ASSERT_LT(a, b) GTS_CMP_(true, <, a, b)
#define ASSERT_LE(a, b) GTS_CMP_(true, <=, a, b)
#define ASSERT_GT(a, b) GTS_CMP_(true, >, a, b)
#define ASSERT_GE(a, b) GTS_CMP_(true, >=, a, b)

#define GTS_BOOL_(fatal, cond, want)                                                      \
  ::testing::internal::Reporter(static_cast<bool>(cond) != (want), __FILE__, __LINE__,     \
                                std::string("Value of: ") + #cond + " expected " #want,    \
                                fatal)
#define EXPECT_TRUE(c) GTS_BOOL_(false, c, true)
#define EXPECT_FALSE(c) GTS_BOOL_(false, c, false)
#define ASSERT_TRUE(c) GTS_BOOL_(true, c, true)
#define ASSERT_FALSE(c) GTS_BOOL_(true, c, false)

#define GTS_DEQ_(fatal, a, b)                                                               \
  for (bool gts_once = true; gts_once; gts_once = false)                                    \
    for (const double gts_a = (a), gts_b = (b); gts_once; gts_once = false)                 \
  ::testing::internal::Reporter(!::testing::internal::double_eq(gts_a, gts_b), __FILE__,     \
                                __LINE__,                                                   \
                                ::testing::internal::describe("~=", #a, #b, gts_a, gts_b),  \
                                fatal)
#define EXPECT_DOUBLE_EQ(a, b) GTS_DEQ_(false, a, b)
#define ASSERT_DOUBLE_EQ(a, b) GTS_DEQ_(true, a, b)

#define GTS_NEAR_(fatal, a, b, tol)                                                        \
  for (bool gts_once = true; gts_once; gts_once = false)                                   \
    for (const double gts_a = (a), gts_b = (b), gts_t = (tol); gts_once; gts_once = false) \
  ::testing::internal::Reporter(!(std::fabs(gts_a - gts_b) <= gts_t), __FILE__, __LINE__,   \
                                ::testing::internal::describe("near", #a, #b, gts_a, gts_b) + \
                                    " tol " + std::to_string(gts_t),                        \
                                fatal)
#define EXPECT_NEAR(a, b, tol) GTS_NEAR_(false, a, b, tol)
#define ASSERT_NEAR(a, b, tol) GTS_NEAR_(true, a, b, tol)

#define GTS_THROW_(fatal, stmt, exc)                                                       \
  for (bool gts_once = true; gts_once; gts_once = false)                                   \
    for (int gts_state = [&]() -> int {                                                    \
           try {                                                                           \
             stmt;                                                                         \
           } catch (const exc&) {                                                          \
             return 0;                                                                     \
           } catch (...) {                                                                 \
             return 2;                                                                     \
           }                                                                               \
           return 1;                                                                       \
         }();                                                                              \
         gts_once; gts_once = false)                                                       \
  ::testing::internal::Reporter(gts_state != 0, __FILE__, __LINE__,                         \
                                std::string("Expected: ") + #stmt + " throws " #exc,       \
                                fatal)
#define EXPECT_THROW(stmt, exc) GTS_THROW_(false, stmt, exc)
#define ASSERT_THROW(stmt, exc) GTS_THROW_(true, stmt, exc)

#define GTS_NOTHROW_(fatal, stmt)                                                          \
  for (bool gts_once = true; gts_once; gts_once = false)                                   \
    for (bool gts_threw = [&]() -> bool {                                                  \
           try {                                                                           \
             stmt;                                                                         \
           } catch (...) {                                                                 \
             return true;                                                                  \
           }                                                                               \
           return false;                                                                   \
         }();                                                                              \
         gts_once; gts_once = false)                                                       \
  ::testing::internal::Reporter(gts_threw, __FILE__, __LINE__,                              \
                                std::string("Expected: ") + #stmt + " does not throw",     \
                                fatal)
#define EXPECT_NO_THROW(stmt) GTS_NOTHROW_(false, stmt)
#define ASSERT_NO_THROW(stmt) GTS_NOTHROW_(true, stmt)

#define GTEST_SKIP() \
  for (;;) throw ::testing::internal::SkipTest{}; \
  std::cout

#ifdef GTEST_SHIM_MAIN
int main() { return ::testing::RunAllTests(); }
#endif
