// bits.cuh -- bit-sliced helpers for the sm_100a stencil kernels.
//
// A "plane set" holds one 32-voxel run along axis 2 in bit-sliced form:
// P[k] bit p = bit k of voxel (z0 + p).  Comparisons of two runs then cost
// one LOP3 per bit plane (a carry chain over 32 voxel pairs at once) instead
// of one compare per voxel, which is what makes the u8 stencil fit the ALU
// budget of an HBM-speed sweep ("K1: bit-sliced tournament").
#pragma once
#include <cstdint>


namespace eccb {
namespace bits {

// One LOP3 with a compile-time truth table (operands a, b, c carry the
// canonical tables 0xF0, 0xCC, 0xAA).  Written as inline PTX because ptxas
// otherwise splits several of the 3-input functions below into 2-3 ops.
template <int LUT>
__host__ __device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
#ifdef __CUDA_ARCH__
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
  return d;
#else
  uint32_t d = 0;
  for (int i = 0; i < 32; ++i) {
    const int k = (((a >> i) & 1) << 2) | (((b >> i) & 1) << 1) | ((c >> i) & 1);
    d |= (uint32_t)((LUT >> k) & 1) << i;
  }
  return d;
#endif
}

// [a > b] for 32 lanes of NB-bit unsigned numbers: carry-out of a + ~b,
// one LOP3 per bit (0xB2 = (a & ~b) | ((a | ~b) & c)).
template <int NB>
__host__ __device__ __forceinline__ uint32_t gt(const uint32_t (&a)[NB], const uint32_t (&b)[NB]) {
  uint32_t c = a[0] & ~b[0];
#pragma unroll
  for (int i = 1; i < NB; ++i) c = lop3<0xB2>(a[i], b[i], c);
  return c;
}

// out = g ? b : a   (the minimum when g = [a > b])
template <int NB>
__host__ __device__ __forceinline__ void sel(uint32_t (&out)[NB], uint32_t g, const uint32_t (&a)[NB],
                                    const uint32_t (&b)[NB]) {
#pragma unroll
  for (int i = 0; i < NB; ++i) out[i] = lop3<0xE2>(b[i], g, a[i]);
}

// (a & m) | (b & ~m) as ONE lop3 (ptxas splits the C++ form into two LOP3s
// plus a shift when m is an immediate).
__host__ __device__ __forceinline__ uint32_t bsel(uint32_t a, uint32_t m, uint32_t b) {
#ifdef __CUDA_ARCH__
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xE2;" : "=r"(d) : "r"(a), "r"(m), "r"(b));
  return d;
#else
  return (a & m) | (b & ~m);
#endif
}

// x >> k computed on the FMA pipe (IMAD.HI: the high word of x * 2^(32-k))
// instead of the integer ALU pipe, which is the stencil kernel's bottleneck.
__host__ __device__ __forceinline__ uint32_t shr_fma(uint32_t x, int k) {
#ifdef __CUDA_ARCH__
  return __umulhi(x, 1u << (32 - k));
#else
  return x >> k;
#endif
}

// (x >> 1) + a and (x << 1) + a as ONE FMA-pipe instruction each (IMAD.HI /
// IMAD with an addend): the shift plus a bit that lands where the shift
// left a zero (a < 2^31, resp. a in {0, 1}).
__host__ __device__ __forceinline__ uint32_t shr1_add(uint32_t x, uint32_t a) {
#ifdef __CUDA_ARCH__
  uint32_t d;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(0x80000000u), "r"(a));
  return d;
#else
  return (x >> 1) + a;
#endif
}
__host__ __device__ __forceinline__ uint32_t shl1_add(uint32_t x, uint32_t a) {
#ifdef __CUDA_ARCH__
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(2u), "r"(a));
  return d;
#else
  return (x << 1) + a;
#endif
}

// (x >> p) & 1 for a compile-time p on the FMA pipe: IMAD.SHL moves bit p
// to bit 31, IMAD.HI by 2 brings it down alone.
__host__ __device__ __forceinline__ uint32_t bit_fma(uint32_t x, int p) {
#ifdef __CUDA_ARCH__
  return __umulhi(x << (31 - p), 2u);
#else
  return (x >> p) & 1u;
#endif
}

// Merge-style delta swap between w[i] and w[i+s] on bit distance `sh` with
// mask m (bits that stay in w[i]): one shift + one lop3 per output word
// (the left shift becomes IMAD.SHL, the right one IMAD.HI: both FMA pipe).
__host__ __device__ __forceinline__ void dswap(uint32_t& lo, uint32_t& hi, int sh, uint32_t m) {
  const uint32_t a = lo, b = hi;
  lo = bsel(a, m, b << sh);
  hi = bsel(shr_fma(a, sh), m, b);
}

// 8x8 bit-matrix transpose applied to the four bytes of 8 words in
// parallel: bit (8b + k) of w[r]  <->  bit (8b + r) of w[k].  An involution.
__host__ __device__ __forceinline__ void transpose8(uint32_t (&w)[8]) {
#pragma unroll
  for (int r = 0; r < 4; ++r) dswap(w[r], w[r + 4], 4, 0x0F0F0F0Fu);
#pragma unroll
  for (int r = 0; r < 8; r += 4) {
    dswap(w[r], w[r + 2], 2, 0x33333333u);
    dswap(w[r + 1], w[r + 3], 2, 0x33333333u);
  }
#pragma unroll
  for (int r = 0; r < 8; r += 2) dswap(w[r], w[r + 1], 1, 0x55555555u);
}

// prmt.b32 in its default mode: selector nibbles with bit 3 set replicate
// the sign bit of the selected byte (__byte_perm ignores that bit).
__host__ __device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
#ifdef __CUDA_ARCH__
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
#else
  const uint64_t v = ((uint64_t)b << 32) | a;
  uint32_t r = 0;
  for (int i = 0; i < 4; ++i) {
    const uint32_t n = (sel >> (4 * i)) & 15;
    uint32_t byte = (uint32_t)((v >> (8 * (n & 7))) & 0xFF);
    if (n & 8) byte = (byte & 0x80) ? 0xFF : 0x00;
    r |= byte << (8 * i);
  }
  return r;
#endif
}

// Full adder on bit-sliced operands.
__host__ __device__ __forceinline__ void fa(uint32_t a, uint32_t b, uint32_t c, uint32_t& s, uint32_t& cy) {
  s = a ^ b ^ c;
  cy = (a & b) | (c & (a ^ b));
}

// 4x4 byte transposes of (a0,a2,a4,a6) and (a1,a3,a5,a7): returns w[r] with
// byte b = byte (r % 4) of a[2b + r / 4], i.e. for 32 contiguous bytes in
// a[0..7], byte b of w[r] is source byte 8b + r.  After transpose8 this puts
// source byte p at bit p of every plane.
__host__ __device__ __forceinline__ void byte_interleave(const uint32_t (&a)[8], uint32_t (&w)[8]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t x0 = a[h], x1 = a[h + 2], x2 = a[h + 4], x3 = a[h + 6];
    const uint32_t t0 = prmt(x0, x1, 0x5140);  // x0.0 x1.0 x0.1 x1.1
    const uint32_t t1 = prmt(x0, x1, 0x7362);  // x0.2 x1.2 x0.3 x1.3
    const uint32_t t2 = prmt(x2, x3, 0x5140);
    const uint32_t t3 = prmt(x2, x3, 0x7362);
    w[4 * h + 0] = prmt(t0, t2, 0x5410);  // x0.0 x1.0 x2.0 x3.0
    w[4 * h + 1] = prmt(t0, t2, 0x7632);  // x0.1 x1.1 x2.1 x3.1
    w[4 * h + 2] = prmt(t1, t3, 0x5410);
    w[4 * h + 3] = prmt(t1, t3, 0x7632);
  }
}


// transpose8 of {p0, p1, p2, p3, 0, 0, 0, 0} (four code planes -> bytes):
// the butterfly stages commute, so the two within-nibble stages run on the
// four live words first and the nibble split last (28 ops instead of 44).
// Result: byte b of w[r] = (p3 p2 p1 p0 bits of lane-bit 8b + r).
__host__ __device__ __forceinline__ void transpose_codes(uint32_t p0, uint32_t p1, uint32_t p2,
                                                         uint32_t p3, uint32_t (&w)[8]) {
  w[0] = p0; w[1] = p1; w[2] = p2; w[3] = p3;
  dswap(w[0], w[2], 2, 0x33333333u);
  dswap(w[1], w[3], 2, 0x33333333u);
  dswap(w[0], w[1], 1, 0x55555555u);
  dswap(w[2], w[3], 1, 0x55555555u);
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    w[r + 4] = (w[r] >> 4) & 0x0F0F0F0Fu;
    w[r] &= 0x0F0F0F0Fu;
  }
}

}  // namespace bits
}  // namespace eccb

namespace eccb {
namespace bits {

// Bit-sliced S mod 16 for S = sum(w1[0..16]) + 2 * sum(w2[0..8]) (a
// carry-save tree of 19 full adders).  out[k] bit p = bit k of S at lane-bit
// p.  __host__ so tests/test_bits.cpp can check it exhaustively on the CPU.
__host__ __device__ __forceinline__ void fa3(uint32_t a, uint32_t b, uint32_t c, uint32_t& s,
                                             uint32_t& cy) {
  s = a ^ b ^ c;
  cy = (a & b) | (c & (a ^ b));
}

__host__ __device__ __forceinline__ void csa17(const uint32_t (&a)[17], uint32_t& bit,
                                               uint32_t (&carry)[8]) {
  uint32_t s[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) fa3(a[3 * i], a[3 * i + 1], a[3 * i + 2], s[i], carry[i]);
  uint32_t t0, t1;
  fa3(s[0], s[1], s[2], t0, carry[5]);
  fa3(s[3], s[4], a[15], t1, carry[6]);
  fa3(t0, t1, a[16], bit, carry[7]);
}

__host__ __device__ __forceinline__ void sum_code(const uint32_t (&w1)[17], const uint32_t (&w2)[9],
                                                  uint32_t (&out)[4]) {
  uint32_t c2[8];
  csa17(w1, out[0], c2);
  uint32_t b[17];
#pragma unroll
  for (int i = 0; i < 9; ++i) b[i] = w2[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) b[9 + i] = c2[i];
  uint32_t c4[8];
  csa17(b, out[1], c4);
  uint32_t s0, s1, s2, k0, k1, k2;
  fa3(c4[0], c4[1], c4[2], s0, k0);
  fa3(c4[3], c4[4], c4[5], s1, k1);
  fa3(s0, s1, c4[6], s2, k2);
  out[2] = s2 ^ c4[7];
  const uint32_t k3 = s2 & c4[7];
  out[3] = k0 ^ k1 ^ k2 ^ k3;
}

// Bit-sliced S mod 16 for S = sum_b (2 h[b] + l[b]) over the nine in-plane
// blocks of a voxel (h[b] & l[b] == 0, so each block adds 0, 1 or 2): the
// per-block form of the tournament sum, change + 9 = sum_b q_b with
// q_b = 1 + s_b I_b (X_b - Xp_b) (k_u8_3d.cu).  12 full adders, one half
// adder and one 3-input XOR; out[k] bit p = bit k of S at lane-bit p.
__host__ __device__ __forceinline__ void sum_blocks9(const uint32_t (&h)[9], const uint32_t (&l)[9],
                                                     uint32_t (&out)[4]) {
  // weight 1: the nine l's
  uint32_t a0, c0, a1, c1, a2, c2, c3;
  fa3(l[0], l[1], l[2], a0, c0);
  fa3(l[3], l[4], l[5], a1, c1);
  fa3(l[6], l[7], l[8], a2, c2);
  fa3(a0, a1, a2, out[0], c3);
  // weight 2: the nine h's and four carries
  uint32_t b0, d0, b1, d1, b2, d2, b3, d3, e0, f0, f1;
  fa3(h[0], h[1], h[2], b0, d0);
  fa3(h[3], h[4], h[5], b1, d1);
  fa3(h[6], h[7], h[8], b2, d2);
  fa3(c0, c1, c2, b3, d3);
  fa3(b0, b1, b2, e0, f0);
  fa3(e0, b3, c3, out[1], f1);
  // weight 4: six carries
  uint32_t g0, k0, g1, k1;
  fa3(d0, d1, d2, g0, k0);
  fa3(d3, f0, f1, g1, k1);
  out[2] = g0 ^ g1;
  // weight 8 (mod 16): three carries
  out[3] = k0 ^ k1 ^ (g0 & g1);
}

}  // namespace bits
namespace cols {
// Column groups of the bit-sliced 3D kernels (k_u8_3d.cu, k_u16_3d.cu)
// along an in-plane axis of width W.  A column's window is 32
// rows (lanes) / bits; an interior column owns 30 of them (one halo on each
// side), but the image's first and last columns own 31: the collar beyond
// the image edge is VIRTUAL (no lane / bit holds it, its comparisons are
// substituted in sweep_step), so 512 = 31 + 15 x 30 + 31 takes 17 columns
// instead of 18 (-11 % plane steps at 512^2 per plane).
__host__ __device__ __forceinline__ int groups(int W) {
  return W <= 32 ? 1 : 2 + (W - 62 + 29) / 30 * (W > 62);
}
// First owned index of group k (k = G: W).  W = q G + r; the r groups one
// voxel larger are taken in the order 0, G-1, 1, 2, ... (only the two edge
// groups may own 31).
__host__ __device__ __forceinline__ int start(int k, int G, int W) {
  if (k <= 0) return 0;
  if (k >= G) return W;
  const int q = W / G, r = W - q * G;
  const int m = k - 1 < r - 2 ? k - 1 : r - 2;  // interior groups before k with an extra voxel
  return k * q + (r > 0) + (m > 0 ? m : 0);
}

}  // namespace cols

}  // namespace eccb
