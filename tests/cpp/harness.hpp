// Minimal test harness for the C++ contract tests (doctest is not vendored).
#pragma once

#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

namespace th {

struct Case {
  const char* name;
  const char* group;  // "cpu" or "gpu"
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
  Reg(const char* n, const char* g, std::function<void()> f) { registry().push_back({n, g, std::move(f)}); }
};

struct Fatal {};

}  // namespace th

#define TH_CAT2(a, b) a##b
#define TH_CAT(a, b) TH_CAT2(a, b)
#define TEST(group, name)                                                 \
  static void TH_CAT(th_fn_, __LINE__)();                                 \
  static th::Reg TH_CAT(th_reg_, __LINE__)(name, group, TH_CAT(th_fn_, __LINE__)); \
  static void TH_CAT(th_fn_, __LINE__)()

#define CHECK(cond)                                                                  \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      std::printf("    CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
      ++th::failures();                                                              \
    }                                                                                \
  } while (0)

#define REQUIRE(cond)                                                                \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      std::printf("    REQUIRE failed %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
      ++th::failures();                                                              \
      throw th::Fatal{};                                                             \
    }                                                                                \
  } while (0)

#define CHECK_THROWS_AS(expr, T)                                                     \
  do {                                                                               \
    bool th_caught = false;                                                          \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const T&) {                                                             \
      th_caught = true;                                                              \
    } catch (...) {                                                                  \
    }                                                                                \
    if (!th_caught) {                                                                \
      std::printf("    CHECK_THROWS_AS failed %s:%d: %s\n", __FILE__, __LINE__, #expr); \
      ++th::failures();                                                              \
    }                                                                                \
  } while (0)

inline int th_main(int argc, char** argv) {
  const std::string group = argc > 1 ? argv[1] : "all";
  const std::string filter = argc > 2 ? argv[2] : "";
  int ran = 0, failed_cases = 0;
  for (auto& c : th::registry()) {
    if (group != "all" && group != c.group) continue;
    if (!filter.empty() && std::string(c.name).find(filter) == std::string::npos) continue;
    const int before = th::failures();
    std::printf("[ RUN  ] %s\n", c.name);
    std::fflush(stdout);
    try {
      c.fn();
    } catch (const th::Fatal&) {
    } catch (const std::exception& e) {
      std::printf("    uncaught exception: %s\n", e.what());
      ++th::failures();
    }
    const bool ok = th::failures() == before;
    std::printf("[ %s ] %s\n", ok ? " OK " : "FAIL", c.name);
    std::fflush(stdout);
    ++ran;
    if (!ok) ++failed_cases;
  }
  std::printf("%d cases, %d failed\n", ran, failed_cases);
  return failed_cases ? 1 : 0;
}
