// A minimal GoogleTest-compatible shim (GTest is not installed in this
// image).  Enough of the API for the reference's unit suites to compile
// unchanged against the drop-in headers: TEST, EXPECT_/ASSERT_ comparisons,
// NEAR / DOUBLE_EQ, THROW / NO_THROW, streamed messages, TempDir.
// Test infrastructure only.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace testing {

class Message {
 public:
  template <class T>
  Message& operator<<(const T& v) {
    ss_ << v;
    return *this;
  }
  std::string str() const { return ss_.str(); }

 private:
  std::ostringstream ss_;
};

class AssertionResult {
 public:
  AssertionResult(bool ok, std::string msg = "") : ok_(ok), msg_(std::move(msg)) {}
  explicit operator bool() const { return ok_; }
  const std::string& message() const { return msg_; }

 private:
  bool ok_;
  std::string msg_;
};

inline AssertionResult AssertionSuccess() { return AssertionResult(true); }
inline AssertionResult AssertionFailure(const std::string& m) { return AssertionResult(false, m); }

inline std::string TempDir() {
  const char* t = std::getenv("TEST_TMPDIR");
  std::string d = t ? t : "/tmp";
  if (d.empty() || d.back() != '/') d += '/';
  return d;
}

namespace internal {

struct State {
  int failures = 0;  // in the running test
};
inline State& state() {
  static State s;
  return s;
}

template <class T, class = void>
struct streamable : std::false_type {};
template <class T>
struct streamable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};

template <class T>
std::string show(const T& v);

template <class T, class = void>
struct iterable : std::false_type {};
template <class T>
struct iterable<T, std::void_t<decltype(std::declval<const T&>().begin())>> : std::true_type {};

template <class T>
std::string show(const T& v) {
  std::ostringstream o;
  if constexpr (std::is_floating_point_v<T>) {
    o.precision(17);
    o << v;
  } else if constexpr (streamable<T>::value) {
    o << v;
  } else if constexpr (iterable<T>::value) {
    o << "{";
    bool first = true;
    for (const auto& e : v) {
      o << (first ? "" : ", ") << show(e);
      first = false;
    }
    o << "}";
  } else {
    o << "<value>";
  }
  return o.str();
}

template <class A, class B, class Op>
AssertionResult compare(const char* ea, const char* eb, const A& a, const B& b, Op op, const char* opname) {
  if (op(a, b)) return AssertionSuccess();
  return AssertionFailure(std::string("Expected: (") + ea + ") " + opname + " (" + eb + "), actual: " +
                          show(a) + " vs " + show(b));
}

inline AssertionResult near(const char* ea, const char* eb, const char* et, double a, double b, double tol) {
  const double d = std::fabs(a - b);
  if (d <= tol) return AssertionSuccess();
  return AssertionFailure(std::string("The difference between ") + ea + " and " + eb + " is " + show(d) +
                          ", which exceeds " + et + ", where " + ea + " = " + show(a) + ", " + eb +
                          " = " + show(b) + ", " + et + " = " + show(tol));
}

// GoogleTest's DOUBLE_EQ: within 4 ULPs (NaN never equal).
inline AssertionResult double_eq(const char* ea, const char* eb, double a, double b) {
  auto biased = [](double x) {
    uint64_t u;
    std::memcpy(&u, &x, 8);
    const uint64_t sign = 1ull << 63;
    return (u & sign) ? ~u + 1 : u | sign;
  };
  bool ok = !(std::isnan(a) || std::isnan(b));
  if (ok) {
    const uint64_t x = biased(a), y = biased(b);
    ok = (x >= y ? x - y : y - x) <= 4;
  }
  if (ok) return AssertionSuccess();
  return AssertionFailure(std::string("Expected equality of these values:\n  ") + ea + "\n    " + show(a) +
                          "\n  " + eb + "\n    " + show(b));
}

struct AssertHelper {
  const char* file;
  int line;
  std::string msg;
  AssertHelper(const char* f, int l, std::string m) : file(f), line(l), msg(std::move(m)) {}
  void operator=(const Message& m) const {
    state().failures += 1;
    std::cout << file << ":" << line << ": Failure\n" << msg;
    const std::string extra = m.str();
    if (!extra.empty()) std::cout << "\n" << extra;
    std::cout << std::endl;
  }
};

struct TestInfo {
  std::string suite, name;
  void (*body)();
};
inline std::vector<TestInfo>& registry() {
  static std::vector<TestInfo> r;
  return r;
}
struct Registrar {
  Registrar(const char* s, const char* n, void (*f)()) { registry().push_back({s, n, f}); }
};

}  // namespace internal

inline void InitGoogleTest(int*, char**) {}
inline void InitGoogleTest() {}

}  // namespace testing

inline int RUN_ALL_TESTS() {
  using namespace testing::internal;
  int failed = 0, run = 0;
  std::vector<std::string> bad;
  for (const TestInfo& t : registry()) {
    const std::string id = t.suite + "." + t.name;
    std::cout << "[ RUN      ] " << id << std::endl;
    state().failures = 0;
    try {
      t.body();
    } catch (const std::exception& e) {
      std::cout << "unexpected exception: " << e.what() << std::endl;
      state().failures += 1;
    } catch (...) {
      std::cout << "unexpected non-std exception" << std::endl;
      state().failures += 1;
    }
    ++run;
    if (state().failures) {
      ++failed;
      bad.push_back(id);
      std::cout << "[  FAILED  ] " << id << std::endl;
    } else {
      std::cout << "[       OK ] " << id << std::endl;
    }
  }
  std::cout << "[==========] " << run << " tests ran." << std::endl;
  std::cout << "[  PASSED  ] " << (run - failed) << " tests." << std::endl;
  if (failed) {
    std::cout << "[  FAILED  ] " << failed << " tests, listed below:" << std::endl;
    for (const auto& b : bad) std::cout << "[  FAILED  ] " << b << std::endl;
  }
  return failed ? 1 : 0;
}

#define GTEST_SHIM_CHECK_(res, on_fail)                        \
  if (const ::testing::AssertionResult gtest_ar_ = (res)) \
    ;                                                          \
  else                                                         \
    on_fail ::testing::internal::AssertHelper(__FILE__, __LINE__, gtest_ar_.message()) = ::testing::Message()

#define GTEST_SHIM_NONFATAL_
#define GTEST_SHIM_FATAL_ return

#define GTEST_SHIM_CMP_(a, b, op, name, kind)                                                             \
  GTEST_SHIM_CHECK_(::testing::internal::compare(#a, #b, (a), (b),                                        \
                                                 [](const auto& x, const auto& y) { return x op y; }, name), \
                    kind)

#define EXPECT_EQ(a, b) GTEST_SHIM_CMP_(a, b, ==, "==", GTEST_SHIM_NONFATAL_)
#define EXPECT_NE(a, b) GTEST_SHIM_CMP_(a, b, !=, "!=", GTEST_SHIM_NONFATAL_)
#define EXPECT_LT(a, b) GTEST_SHIM_CMP_(a, b, <, "<", GTEST_SHIM_NONFATAL_)
#define EXPECT_LE(a, b) GTEST_SHIM_CMP_(a, b, <=, "<=", GTEST_SHIM_NONFATAL_)
#define EXPECT_GT(a, b) GTEST_SHIM_CMP_(a, b, >, ">", GTEST_SHIM_NONFATAL_)
#define EXPECT_GE(a, b) GTEST_SHIM_CMP_(a, b, >=, ">=", GTEST_SHIM_NONFATAL_)
#define ASSERT_EQ(a, b) GTEST_SHIM_CMP_(a, b, ==, "==", GTEST_SHIM_FATAL_)
#define ASSERT_NE(a, b) GTEST_SHIM_CMP_(a, b, !=, "!=", GTEST_SHIM_FATAL_)
#define ASSERT_LT(a, b) GTEST_SHIM_CMP_(a, b, <, "<", GTEST_SHIM_FATAL_)
#define ASSERT_LE(a, b) GTEST_SHIM_CMP_(a, b, <=, "<=", GTEST_SHIM_FATAL_)
#define ASSERT_GT(a, b) GTEST_SHIM_CMP_(a, b, >, ">", GTEST_SHIM_FATAL_)
#define ASSERT_GE(a, b) GTEST_SHIM_CMP_(a, b, >=, ">=", GTEST_SHIM_FATAL_)

#define GTEST_SHIM_BOOL_(c, want, kind)                                                                   \
  GTEST_SHIM_CHECK_(((bool)(c)) == (want) ? ::testing::AssertionSuccess()                                 \
                                          : ::testing::AssertionFailure(std::string("Value of: ") + #c + \
                                                                        "\n  Expected: " #want),          \
                    kind)
#define EXPECT_TRUE(c) GTEST_SHIM_BOOL_(c, true, GTEST_SHIM_NONFATAL_)
#define EXPECT_FALSE(c) GTEST_SHIM_BOOL_(c, false, GTEST_SHIM_NONFATAL_)
#define ASSERT_TRUE(c) GTEST_SHIM_BOOL_(c, true, GTEST_SHIM_FATAL_)
#define ASSERT_FALSE(c) GTEST_SHIM_BOOL_(c, false, GTEST_SHIM_FATAL_)

#define EXPECT_NEAR(a, b, t) \
  GTEST_SHIM_CHECK_(::testing::internal::near(#a, #b, #t, (a), (b), (t)), GTEST_SHIM_NONFATAL_)
#define ASSERT_NEAR(a, b, t) \
  GTEST_SHIM_CHECK_(::testing::internal::near(#a, #b, #t, (a), (b), (t)), GTEST_SHIM_FATAL_)
#define EXPECT_DOUBLE_EQ(a, b) \
  GTEST_SHIM_CHECK_(::testing::internal::double_eq(#a, #b, (a), (b)), GTEST_SHIM_NONFATAL_)
#define ASSERT_DOUBLE_EQ(a, b) \
  GTEST_SHIM_CHECK_(::testing::internal::double_eq(#a, #b, (a), (b)), GTEST_SHIM_FATAL_)

#define GTEST_SHIM_THROW_(stmt, exc, kind)                                                        \
  GTEST_SHIM_CHECK_(([&]() -> ::testing::AssertionResult {                                        \
                      try {                                                                       \
                        stmt;                                                                     \
                      } catch (const exc&) {                                                      \
                        return ::testing::AssertionSuccess();                                     \
                      } catch (const std::exception& e_) {                                        \
                        return ::testing::AssertionFailure(std::string("Expected: " #stmt         \
                                                                       " throws " #exc            \
                                                                       ".\n  Actual: it throws ") + \
                                                           e_.what());                            \
                      } catch (...) {                                                             \
                        return ::testing::AssertionFailure("Expected: " #stmt " throws " #exc     \
                                                           ".\n  Actual: a different type.");     \
                      }                                                                           \
                      return ::testing::AssertionFailure("Expected: " #stmt " throws " #exc       \
                                                         ".\n  Actual: it throws nothing.");      \
                    }()),                                                                         \
                    kind)
#define EXPECT_THROW(stmt, exc) GTEST_SHIM_THROW_(stmt, exc, GTEST_SHIM_NONFATAL_)
#define ASSERT_THROW(stmt, exc) GTEST_SHIM_THROW_(stmt, exc, GTEST_SHIM_FATAL_)
#define EXPECT_ANY_THROW(stmt) GTEST_SHIM_THROW_(stmt, std::exception, GTEST_SHIM_NONFATAL_)

#define GTEST_SHIM_NO_THROW_(stmt, kind)                                                        \
  GTEST_SHIM_CHECK_(([&]() -> ::testing::AssertionResult {                                      \
                      try {                                                                     \
                        stmt;                                                                   \
                      } catch (const std::exception& e_) {                                      \
                        return ::testing::AssertionFailure(                                     \
                            std::string("Expected: " #stmt " doesn't throw.\n  Actual: ") +     \
                            e_.what());                                                         \
                      } catch (...) {                                                           \
                        return ::testing::AssertionFailure("Expected: " #stmt " doesn't throw."); \
                      }                                                                         \
                      return ::testing::AssertionSuccess();                                     \
                    }()),                                                                       \
                    kind)
#define EXPECT_NO_THROW(stmt) GTEST_SHIM_NO_THROW_(stmt, GTEST_SHIM_NONFATAL_)
#define ASSERT_NO_THROW(stmt) GTEST_SHIM_NO_THROW_(stmt, GTEST_SHIM_FATAL_)

#define TEST(suite, name)                                                                  \
  static void suite##_##name##_gtest_body();                                               \
  static ::testing::internal::Registrar suite##_##name##_gtest_reg(#suite, #name,         \
                                                                   &suite##_##name##_gtest_body); \
  static void suite##_##name##_gtest_body()
