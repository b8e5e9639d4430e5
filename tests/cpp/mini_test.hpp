// mini_test.hpp — a few doctest-style macros so the C++ tests read like the
// reference's proj/tests (doctest is not available in this image).
#pragma once
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace mini {
struct Case {
  const char* name;
  std::function<void()> fn;
};
inline std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
inline int& failures() {
  static int f = 0;
  return f;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { cases().push_back({n, std::move(f)}); }
};
inline int run_all() {
  for (auto& c : cases()) {
    const int before = failures();
    try {
      c.fn();
    } catch (const std::exception& e) {
      std::printf("  exception: %s\n", e.what());
      ++failures();
    }
    std::printf("[%s] %s\n", failures() == before ? "ok" : "FAIL", c.name);
  }
  std::printf("%zu cases, %d failures\n", cases().size(), failures());
  return failures() ? 1 : 0;
}
}  // namespace mini

#define MINI_CAT2(a, b) a##b
#define MINI_CAT(a, b) MINI_CAT2(a, b)
#define TEST_CASE(name)                                             \
  static void MINI_CAT(case_, __LINE__)();                          \
  static mini::Reg MINI_CAT(reg_, __LINE__)(name, MINI_CAT(case_, __LINE__)); \
  static void MINI_CAT(case_, __LINE__)()
#define CHECK(x)                                                          \
  do {                                                                    \
    if (!(x)) {                                                           \
      std::printf("  %s:%d CHECK(%s) failed\n", __FILE__, __LINE__, #x); \
      ++mini::failures();                                                 \
    }                                                                     \
  } while (0)
#define REQUIRE(x)                                                            \
  do {                                                                        \
    if (!(x)) {                                                               \
      std::printf("  %s:%d REQUIRE(%s) failed\n", __FILE__, __LINE__, #x);    \
      ++mini::failures();                                                     \
      return;                                                                 \
    }                                                                         \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                           \
  do {                                                                     \
    bool thrown_ = false;                                                  \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (const T&) {                                                   \
      thrown_ = true;                                                      \
    }                                                                      \
    if (!thrown_) {                                                        \
      std::printf("  %s:%d %s did not throw %s\n", __FILE__, __LINE__, #expr, #T); \
      ++mini::failures();                                                  \
    }                                                                      \
  } while (0)
#define MINI_MAIN() \
  int main() { return mini::run_all(); }
