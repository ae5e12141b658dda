// CPU check of the bit-sliced carry-save sum used by k_u8_3d.cu
// (bits::sum_code): random masks, every lane-bit compared with a scalar sum.
// Built and run by tests/test_native_cpu.py.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>

#define __host__
#define __device__
#define __forceinline__ inline
#include "../../paper_2203_09087_b200/csrc/bits.cuh"
#include "../../paper_2203_09087_b200/csrc/hist16.cuh"

int main() {
  std::mt19937 rng(7);
  for (int it = 0; it < 20000; ++it) {
    uint32_t w1[17], w2[9], out[4];
    const int bias = it % 5;  // vary densities
    for (auto& x : w1) x = bias == 0 ? rng() : (bias == 1 ? rng() & rng() : (bias == 2 ? rng() | rng() : (bias == 3 ? 0xFFFFFFFFu : 0u)));
    for (auto& x : w2) x = bias == 4 ? rng() : (bias == 3 ? rng() | rng() : rng() & rng());
    eccb::bits::sum_code(w1, w2, out);
    for (int p = 0; p < 32; ++p) {
      int s = 0;
      for (auto x : w1) s += (x >> p) & 1;
      for (auto x : w2) s += 2 * ((x >> p) & 1);
      int got = 0;
      for (int k = 0; k < 4; ++k) got |= ((out[k] >> p) & 1) << k;
      if (got != (s & 15)) {
        std::printf("mismatch it=%d p=%d want %d got %d\n", it, p, s & 15, got);
        return 1;
      }
    }
  }
  std::printf("sum_code ok\n");
  return 0;
}
// (appended) transpose_codes == transpose8 on {p0..p3, 0, 0, 0, 0}
int test_transpose_codes() {
  std::mt19937 rng(11);
  for (int it = 0; it < 20000; ++it) {
    uint32_t p[4] = {(uint32_t)rng(), (uint32_t)rng(), (uint32_t)rng(), (uint32_t)rng()};
    uint32_t a[8] = {p[0], p[1], p[2], p[3], 0, 0, 0, 0}, b[8];
    eccb::bits::transpose8(a);
    eccb::bits::transpose_codes(p[0], p[1], p[2], p[3], b);
    for (int r = 0; r < 8; ++r)
      if (a[r] != b[r]) { std::printf("transpose_codes mismatch\n"); return 1; }
    // and the meaning: byte b of w[r] = code of lane-bit 8b + r
    for (int q = 0; q < 32; ++q) {
      int want = 0;
      for (int k = 0; k < 4; ++k) want |= ((p[k] >> q) & 1) << k;
      if ((int)((b[q & 7] >> (8 * (q >> 3))) & 0xFF) != want) { std::printf("code layout mismatch\n"); return 1; }
    }
  }
  std::printf("transpose_codes ok\n");
  return 0;
}
static int run_extra = [] { if (test_transpose_codes()) std::exit(1); return 0; }();  // a failure fails the binary
// (appended) sum_blocks9: every one of the 3^9 per-block (h, l) patterns
int test_sum_blocks9() {
  int pat = 0;
  uint32_t h[9] = {}, l[9] = {};
  int total = 1;
  for (int b = 0; b < 9; ++b) total *= 3;
  for (int base = 0; base < total; base += 32) {
    for (int b = 0; b < 9; ++b) h[b] = l[b] = 0;
    for (int p = 0; p < 32 && base + p < total; ++p) {
      int t = base + p;
      for (int b = 0; b < 9; ++b, t /= 3) {
        const int q = t % 3;
        if (q == 2) h[b] |= 1u << p;
        if (q == 1) l[b] |= 1u << p;
      }
    }
    uint32_t out[4];
    eccb::bits::sum_blocks9(h, l, out);
    for (int p = 0; p < 32 && base + p < total; ++p, ++pat) {
      int s = 0;
      for (int b = 0; b < 9; ++b) s += 2 * ((h[b] >> p) & 1) + ((l[b] >> p) & 1);
      int got = 0;
      for (int k = 0; k < 4; ++k) got |= ((out[k] >> p) & 1) << k;
      if (got != (s & 15)) { std::printf("sum_blocks9 mismatch\n"); return 1; }
    }
  }
  std::printf("sum_blocks9 ok (%d patterns)\n", pat);
  return 0;
}
static int run_extra9 = [] { if (test_sum_blocks9()) std::exit(1); return 0; }();  // a failure fails the binary

// hist16.cuh's packed encoding: every pair of half sums |v| < 32768 decodes
// exactly from the word  BIAS + v_lo + (v_hi << 16)  (plain 32-bit adds, the
// low half borrowing from the high one), and the one-mask band flag fires for
// every half outside the band widened by one count (the borrow's lag).
static int test_hist16() {
  using namespace eccb::hist16;
  std::mt19937 rng(11);
  const int edges[] = {-32767, -28672, -4098, -4097, -4096, -4095, -1, 0, 1, 4094, 4095, 4096, 4097, 28671, 32767};
  long n = 0;
  for (int vlo = -32767; vlo <= 32767; ++vlo) {
    for (int k = 0; k < 15 + 8; ++k) {
      const int vhi = k < 15 ? edges[k] : (int)(rng() % 65535) - 32767;
      const uint32_t w = BIAS + (uint32_t)vlo + ((uint32_t)vhi << 16);
      const int t = (int)(w - BIAS);  // k_batch16's pass-1 sum of both halves
      if (t - 65535 * ((t + 32768) >> 16) != vlo + vhi) {
        std::printf("hist16 pair sum mismatch %d %d\n", vlo, vhi);
        return 1;
      }
      if (lo_value(w) != vlo || hi_value(w) != vhi || half_value(w, 0) != vlo || half_value(w, 1) != vhi) {
        std::printf("hist16 decode mismatch %d %d\n", vlo, vhi);
        return 1;
      }
      const bool flo = (w & FLAG & 0xFFFFu) != 0, fhi = (w & FLAG & 0xFFFF0000u) != 0;
      const bool olo = vlo < -BAND || vlo >= BAND;
      if (flo != olo) { std::printf("hist16 low flag %d\n", vlo); return 1; }
      if ((vhi < -BAND - 1 || vhi > BAND) && !fhi) { std::printf("hist16 high flag missed %d %d\n", vlo, vhi); return 1; }
      if (vlo >= -BAND && (vhi < -BAND || vhi >= BAND) != fhi) { std::printf("hist16 high flag %d %d\n", vlo, vhi); return 1; }
      ++n;
    }
  }
  std::printf("hist16 encoding ok (%ld words)\n", n);
  return 0;
}
static int run_hist16 = [] { if (test_hist16()) std::exit(1); return 0; }();  // a failure fails the binary

// Column layout of the bit-sliced 3D kernels (bits.cuh cols): every width
// is covered exactly, interior columns own <= 30, the two edge columns <= 31
// (one column: <= 32), and no smaller column count could hold the width.
static int test_cols() {
  for (int W = 1; W <= 20000; ++W) {
    const int G = eccb::cols::groups(W);
    if (eccb::cols::start(0, G, W) != 0 || eccb::cols::start(G, G, W) != W) {
      std::printf("cols ends W=%d\n", W);
      return 1;
    }
    for (int k = 0; k < G; ++k) {
      const int n = eccb::cols::start(k + 1, G, W) - eccb::cols::start(k, G, W);
      const int cap = G == 1 ? 32 : (k == 0 || k == G - 1) ? 31 : 30;
      if (n < 1 || n > cap) {
        std::printf("cols W=%d G=%d k=%d owns %d\n", W, G, k, n);
        return 1;
      }
    }
    const int cap_less = G - 1 == 1 ? 32 : 30 * (G - 1) + 2;
    if (G > 1 && W <= cap_less) {
      std::printf("cols W=%d: %d columns not minimal\n", W, G);
      return 1;
    }
  }
  std::printf("cols layout ok\n");
  return 0;
}
static int run_cols = [] { if (test_cols()) std::exit(1); return 0; }();
