// f2s.cuh (the device float formatter) against std::to_chars(float): every
// float with argument "all" (2^32, threaded), else the special values, every
// exponent's extremes and a few million random bit patterns.
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#define __host__
#define __device__
#define __forceinline__ inline
#include "../../paper_2203_09087_b200/csrc/f2s.cuh"

static bool check(uint32_t u) {
  float f;
  std::memcpy(&f, &u, 4);
  char a[64], b[64];
  const auto r = std::to_chars(a, a + 64, f);
  const int na = (int)(r.ptr - a);
  const int nb = eccb::f2s::format(u, b);
  const int nlen = eccb::f2s::format(u, nullptr);
  if (na != nb || nlen != nb || std::memcmp(a, b, na) != 0) {
    std::printf("mismatch %08x: std '%.*s' ours '%.*s'\n", u, na, a, nb, b);
    return false;
  }
  return true;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "all") {
    const unsigned nt = std::max(1u, std::thread::hardware_concurrency());
    std::vector<std::thread> ts;
    std::vector<int> bad(nt, 0);
    for (unsigned t = 0; t < nt; ++t)
      ts.emplace_back([&, t] {
        for (uint64_t u = t; u < (1ull << 32); u += nt)
          if (!check((uint32_t)u) && ++bad[t] > 5) return;
      });
    for (auto& t : ts) t.join();
    int nbad = 0;
    for (int b : bad) nbad += b;
    std::printf("f2s all 2^32 floats: %s\n", nbad ? "FAIL" : "ok");
    return nbad ? 1 : 0;
  }
  long n = 0;
  bool ok = true;
  const uint32_t specials[] = {0u, 0x80000000u, 0x7F800000u, 0xFF800000u, 0x7FC00000u, 1u, 0x7F7FFFFFu,
                               0x00800000u, 0x007FFFFFu, 0x3F800000u, 0x38D1B717u, 0x4B000000u};
  for (uint32_t u : specials) ok &= check(u), ++n;
  for (uint32_t e = 0; e < 255; ++e)
    for (uint32_t m : {0u, 1u, 2u, 0x7FFFFEu, 0x7FFFFFu, 0x400000u, 0x3FFFFFu})
      for (uint32_t s : {0u, 1u}) ok &= check((s << 31) | (e << 23) | m), ++n;
  std::mt19937 rng(5);
  for (int i = 0; i < 4000000 && ok; ++i) ok &= check((uint32_t)rng()), ++n;
  // decimal-looking values (short digit strings) -- the cases where shortest matters
  for (int d = 1; d < 200000 && ok; ++d)
    for (float sc : {1e-7f, 1e-3f, 0.01f, 1.0f, 10.0f, 1e5f}) {
      const float f = (float)d * sc;
      uint32_t u;
      std::memcpy(&u, &f, 4);
      ok &= check(u);
      ++n;
    }
  std::printf("f2s %s (%ld values)\n", ok ? "ok" : "FAIL", n);
  return ok ? 0 : 1;
}
