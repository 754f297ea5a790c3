// Minimal test harness (doctest is not available in this image): CHECK and
// REQUIRE record failures with file:line; main() runs every registered case.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace th {

struct Case {
  const char* name;
  std::function<void()> fn;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
struct RequireFailed {};

// doctest::Approx(x).epsilon(e): |a - b| < e (1 + max(|a|, |b|))
inline bool approx(double a, double b, double eps) {
  return std::fabs(a - b) < eps * (1.0 + std::fmax(std::fabs(a), std::fabs(b)));
}

}  // namespace th

#define TH_CAT2(a, b) a##b
#define TH_CAT(a, b) TH_CAT2(a, b)
#define TEST_CASE(name)                                            \
  static void TH_CAT(th_case_, __LINE__)();                        \
  static th::Reg TH_CAT(th_reg_, __LINE__)(name, TH_CAT(th_case_, __LINE__)); \
  static void TH_CAT(th_case_, __LINE__)()
#define CHECK(cond)                                                                      \
  do {                                                                                   \
    if (!(cond)) {                                                                       \
      std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);              \
      ++th::failures();                                                                  \
    }                                                                                    \
  } while (0)
#define REQUIRE(cond)                                                                    \
  do {                                                                                   \
    if (!(cond)) {                                                                       \
      std::printf("  REQUIRE failed %s:%d: %s\n", __FILE__, __LINE__, #cond);            \
      ++th::failures();                                                                  \
      throw th::RequireFailed{};                                                         \
    }                                                                                    \
  } while (0)
#define CHECK_THROWS(expr)                                                               \
  do {                                                                                   \
    bool th_thrown = false;                                                              \
    try {                                                                                \
      (void)(expr);                                                                      \
    } catch (...) {                                                                      \
      th_thrown = true;                                                                  \
    }                                                                                    \
    if (!th_thrown) {                                                                    \
      std::printf("  CHECK_THROWS failed %s:%d: %s\n", __FILE__, __LINE__, #expr);       \
      ++th::failures();                                                                  \
    }                                                                                    \
  } while (0)

#define TH_MAIN                                                                          \
  int main(int argc, char** argv) {                                                      \
    int run = 0;                                                                         \
    for (auto& c : th::registry()) {                                                     \
      if (argc > 1 && std::string(c.name).find(argv[1]) == std::string::npos) continue;  \
      const int before = th::failures();                                                 \
      try {                                                                              \
        c.fn();                                                                          \
      } catch (const th::RequireFailed&) {                                               \
      } catch (const std::exception& e) {                                                \
        std::printf("  exception: %s\n", e.what());                                      \
        ++th::failures();                                                                \
      }                                                                                  \
      std::printf("[%s] %s\n", th::failures() == before ? "PASS" : "FAIL", c.name);     \
      ++run;                                                                             \
    }                                                                                    \
    std::printf("%d cases, %d failed checks\n", run, th::failures());                    \
    return th::failures() == 0 ? 0 : 1;                                                  \
  }
