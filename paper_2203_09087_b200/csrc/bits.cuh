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

// [a > b] for 32 lanes of NB-bit unsigned numbers: carry-out of a + ~b.
template <int NB>
__device__ __forceinline__ uint32_t gt(const uint32_t (&a)[NB], const uint32_t (&b)[NB]) {
  uint32_t c = a[0] & ~b[0];
#pragma unroll
  for (int i = 1; i < NB; ++i) c = (a[i] & ~b[i]) | ((a[i] | ~b[i]) & c);
  return c;
}

// out = g ? b : a   (the minimum when g = [a > b])
template <int NB>
__device__ __forceinline__ void sel(uint32_t (&out)[NB], uint32_t g, const uint32_t (&a)[NB],
                                    const uint32_t (&b)[NB]) {
#pragma unroll
  for (int i = 0; i < NB; ++i) out[i] = (g & b[i]) | (~g & a[i]);
}

// Merge-style delta swap between w[i] and w[i+s] on bit distance `sh` with
// mask m (bits that stay in w[i]).
__device__ __forceinline__ void dswap(uint32_t& lo, uint32_t& hi, int sh, uint32_t m) {
  const uint32_t a = lo, b = hi;
  lo = (a & m) | ((b << sh) & ~m);
  hi = ((a >> sh) & m) | (b & ~m);
}

// 8x8 bit-matrix transpose applied to the four bytes of 8 words in
// parallel: bit (8b + k) of w[r]  <->  bit (8b + r) of w[k].  An involution.
__device__ __forceinline__ void transpose8(uint32_t (&w)[8]) {
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
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// Full adder on bit-sliced operands.
__device__ __forceinline__ void fa(uint32_t a, uint32_t b, uint32_t c, uint32_t& s, uint32_t& cy) {
  s = a ^ b ^ c;
  cy = (a & b) | (c & (a ^ b));
}

// 4x4 byte transposes of (a0,a2,a4,a6) and (a1,a3,a5,a7): returns w[r] with
// byte b = byte (r % 4) of a[2b + r / 4], i.e. for 32 contiguous bytes in
// a[0..7], byte b of w[r] is source byte 8b + r.  After transpose8 this puts
// source byte p at bit p of every plane.
__device__ __forceinline__ void byte_interleave(const uint32_t (&a)[8], uint32_t (&w)[8]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t x0 = a[h], x1 = a[h + 2], x2 = a[h + 4], x3 = a[h + 6];
    const uint32_t t0 = __byte_perm(x0, x1, 0x5140);  // x0.0 x1.0 x0.1 x1.1
    const uint32_t t1 = __byte_perm(x0, x1, 0x7362);  // x0.2 x1.2 x0.3 x1.3
    const uint32_t t2 = __byte_perm(x2, x3, 0x5140);
    const uint32_t t3 = __byte_perm(x2, x3, 0x7362);
    w[4 * h + 0] = __byte_perm(t0, t2, 0x5410);  // x0.0 x1.0 x2.0 x3.0
    w[4 * h + 1] = __byte_perm(t0, t2, 0x7632);  // x0.1 x1.1 x2.1 x3.1
    w[4 * h + 2] = __byte_perm(t1, t3, 0x5410);
    w[4 * h + 3] = __byte_perm(t1, t3, 0x7632);
  }
}

}  // namespace bits
}  // namespace eccb
