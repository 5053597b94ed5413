// Minimal GoogleTest-compatible shim (GTest is not installed in this image).
// Supports what the reference's proj/tests sources use: TEST, EXPECT_* /
// ASSERT_* (EQ NE LT LE GT GE TRUE FALSE NEAR DOUBLE_EQ THROW) with `<<`
// messages, TEST_F fixtures (SetUp/TearDown) and RecordProperty.  main() lives in gtest_main.cpp.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace gtshim {

struct TestCase {
  const char* suite;
  const char* name;
  std::function<void()> fn;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}

struct Registrar {
  Registrar(const char* s, const char* n, std::function<void()> f) {
    registry().push_back({s, n, std::move(f)});
  }
};

// Collects an optional `<< message` and reports on destruction.
class Failure {
 public:
  Failure(const char* file, int line, const std::string& what) {
    os_ << file << ":" << line << ": Failure: " << what;
  }
  Failure(const Failure&) = delete;
  ~Failure() {
    std::cerr << os_.str() << std::endl;
    ++failures();
  }
  template <typename T>
  Failure& operator<<(const T& v) {
    os_ << " " << v;
    return *this;
  }

 private:
  std::ostringstream os_;
};
struct Voidify {
  void operator=(const Failure&) {}
};

template <typename A, typename B>
std::string vals(const A& a, const B& b) {
  std::ostringstream os;
  os << " (" << a << " vs " << b << ")";
  return os.str();
}
template <typename A, typename B>
std::string vals_np(const A&, const B&) {
  return "";
}

inline bool almost_equal(double a, double b) {  // 4 ULPs, as gtest
  if (std::isnan(a) || std::isnan(b)) return false;
  if (a == b) return true;
  int64_t ia, ib;
  std::memcpy(&ia, &a, 8);
  std::memcpy(&ib, &b, 8);
  if ((ia < 0) != (ib < 0)) return false;
  const int64_t d = ia > ib ? ia - ib : ib - ia;
  return d <= 4;
}

}  // namespace gtshim

inline void RecordProperty(const std::string& k, const std::string& v) {
  std::cerr << "  [property] " << k << " = " << v << std::endl;
}

namespace testing {
// Fixture base (TEST_F): SetUp before and TearDown after each test body.
class Test {
 public:
  virtual ~Test() = default;
  virtual void SetUp() {}
  virtual void TearDown() {}
};
}  // namespace testing

#define GTSHIM_CAT(a, b) a##b
#define TEST_F(fixture, name)                                                          \
  struct GTSHIM_CAT(fixture##_, name) : public fixture {                               \
    void Body();                                                                       \
    void Run() {                                                                       \
      this->SetUp();                                                                   \
      Body();                                                                          \
      this->TearDown();                                                                \
    }                                                                                  \
  };                                                                                   \
  static ::gtshim::Registrar GTSHIM_CAT(gtshim_reg_##fixture##_, name)(                \
      #fixture, #name, [] {                                                            \
        GTSHIM_CAT(fixture##_, name) t;                                                \
        t.Run();                                                                       \
      });                                                                              \
  void GTSHIM_CAT(fixture##_, name)::Body()
#define TEST(suite, name)                                                              \
  static void GTSHIM_CAT(gtshim_##suite##_, name)();                                   \
  static ::gtshim::Registrar GTSHIM_CAT(gtshim_reg_##suite##_, name)(                  \
      #suite, #name, &GTSHIM_CAT(gtshim_##suite##_, name));                            \
  static void GTSHIM_CAT(gtshim_##suite##_, name)()

#define GTSHIM_CHECK(cond, text, fatal) \
  if (cond)                             \
    ;                                   \
  else                                  \
    fatal ::gtshim::Voidify() = ::gtshim::Failure(__FILE__, __LINE__, text)

#define GTSHIM_RET return
#define GTSHIM_NORET

#define GTSHIM_CMP(a, b, op, fatal) \
  GTSHIM_CHECK(((a)op(b)), std::string(#a " " #op " " #b), fatal)

#define EXPECT_EQ(a, b) GTSHIM_CMP(a, b, ==, GTSHIM_NORET)
#define EXPECT_NE(a, b) GTSHIM_CMP(a, b, !=, GTSHIM_NORET)
#define EXPECT_LT(a, b) GTSHIM_CMP(a, b, <, GTSHIM_NORET)
#define EXPECT_LE(a, b) GTSHIM_CMP(a, b, <=, GTSHIM_NORET)
#define EXPECT_GT(a, b) GTSHIM_CMP(a, b, >, GTSHIM_NORET)
#define EXPECT_GE(a, b) GTSHIM_CMP(a, b, >=, GTSHIM_NORET)
#define ASSERT_EQ(a, b) GTSHIM_CMP(a, b, ==, GTSHIM_RET)
#define ASSERT_NE(a, b) GTSHIM_CMP(a, b, !=, GTSHIM_RET)
#define ASSERT_LT(a, b) GTSHIM_CMP(a, b, <, GTSHIM_RET)
#define ASSERT_LE(a, b) GTSHIM_CMP(a, b, <=, GTSHIM_RET)
#define ASSERT_GT(a, b) GTSHIM_CMP(a, b, >, GTSHIM_RET)
#define ASSERT_GE(a, b) GTSHIM_CMP(a, b, >=, GTSHIM_RET)
#define EXPECT_TRUE(c) GTSHIM_CHECK(static_cast<bool>(c), std::string(#c), GTSHIM_NORET)
#define EXPECT_FALSE(c) GTSHIM_CHECK(!static_cast<bool>(c), std::string("!" #c), GTSHIM_NORET)
#define ASSERT_TRUE(c) GTSHIM_CHECK(static_cast<bool>(c), std::string(#c), GTSHIM_RET)
#define ASSERT_FALSE(c) GTSHIM_CHECK(!static_cast<bool>(c), std::string("!" #c), GTSHIM_RET)
#define EXPECT_NEAR(a, b, tol) \
  GTSHIM_CHECK(std::fabs((a) - (b)) <= (tol), std::string("|" #a " - " #b "| <= " #tol), GTSHIM_NORET)
#define EXPECT_DOUBLE_EQ(a, b) \
  GTSHIM_CHECK(::gtshim::almost_equal((a), (b)), std::string(#a " ~= " #b), GTSHIM_NORET)
#define EXPECT_THROW(stmt, exc)                                                  \
  do {                                                                           \
    bool gtshim_ok = false;                                                      \
    try {                                                                        \
      stmt;                                                                      \
    } catch (const exc&) {                                                       \
      gtshim_ok = true;                                                          \
    } catch (...) {                                                              \
    }                                                                            \
    if (!gtshim_ok) ::gtshim::Failure(__FILE__, __LINE__, "expected " #exc);     \
  } while (0)
