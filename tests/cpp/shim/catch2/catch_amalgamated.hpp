// Minimal stand-in for Catch2 v3 (absent from this image; the reference's
// unit tests expect it under /usr/local/include, proj/tests/CMakeLists.txt:1-2).
// Test infrastructure only: TEST_CASE registration, CHECK / CHECK_FALSE /
// REQUIRE / CHECK_THROWS_AS / FAIL and a main() that runs every case and
// reports "N cases, M checks, F failed".
#pragma once
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace shim {
struct Case {
  const char* name;
  std::function<void()> fn;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Stats {
  long checks = 0, failures = 0;
  const char* current = "";
};
inline Stats& stats() {
  static Stats s;
  return s;
}
struct Abort {};
struct Reg {
  Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
inline void record(bool ok, const char* expr, const char* file, int line) {
  ++stats().checks;
  if (!ok) {
    ++stats().failures;
    std::printf("FAILED: %s\n  %s:%d: %s\n", stats().current, file, line, expr);
  }
}
}  // namespace shim

#define SHIM_CAT2(a, b) a##b
#define SHIM_CAT(a, b) SHIM_CAT2(a, b)
#define TEST_CASE(name, ...)                                                        \
  static void SHIM_CAT(shim_case_, __LINE__)();                                     \
  static shim::Reg SHIM_CAT(shim_reg_, __LINE__)(name, &SHIM_CAT(shim_case_, __LINE__)); \
  static void SHIM_CAT(shim_case_, __LINE__)()
#define CHECK(...) shim::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  shim::record(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                  \
  do {                                                                                \
    const bool shim_ok_ = static_cast<bool>(__VA_ARGS__);                             \
    shim::record(shim_ok_, #__VA_ARGS__, __FILE__, __LINE__);                         \
    if (!shim_ok_) throw shim::Abort{};                                               \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                   \
  do {                                                                                \
    bool shim_thrown_ = false;                                                        \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (const type&) {                                                           \
      shim_thrown_ = true;                                                            \
    } catch (...) {                                                                   \
    }                                                                                 \
    shim::record(shim_thrown_, "throws " #type ": " #expr, __FILE__, __LINE__);       \
  } while (0)
#define FAIL(msg)                                                                     \
  do {                                                                                \
    shim::record(false, msg, __FILE__, __LINE__);                                     \
    throw shim::Abort{};                                                              \
  } while (0)

int main() {
  long cases = 0;
  for (auto& c : shim::registry()) {
    shim::stats().current = c.name;
    ++cases;
    try {
      c.fn();
    } catch (const shim::Abort&) {
    } catch (const std::exception& e) {
      ++shim::stats().failures;
      std::printf("FAILED: %s\n  unexpected exception: %s\n", c.name, e.what());
    }
  }
  std::printf("%ld cases, %ld checks, %ld failed\n", cases, shim::stats().checks,
              shim::stats().failures);
  return shim::stats().failures == 0 ? 0 : 1;
}
