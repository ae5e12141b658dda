// tourney.cuh -- scalar-key tournament stencil shared by the generic kernels
// (k_generic.cu: any shape / dtype / slab, the sorted-f32 changes, the
// per-face masks behind the C++ introduced()) and the batched 2D kernel
// (k_batch.cu).  The bit-sliced kernels (k_u8_3d.cu, k_u16_3d.cu, ...) use
// the same algebra on 32 voxels at a time; this is its one-voxel-per-thread
// form for order-preserving uint32 keys (ecc_common.cuh KeyTraits).
//
// Semantics (kernel.hpp:21-74).  A voxel introduces the face between it and
// the voxels of a block (2, 4 or 8 voxels around a face / edge / vertex) iff
// it is the block's minimum, ties going to the voxel that comes first in
// row-major order.  Every block is decided by a tournament over its axes
// from the least significant (axis 2) to the most significant (axis 0): at
// each stage the two halves being compared are separated along a more
// significant axis than anything inside them, so the whole earlier half
// precedes the whole later half and "the later half wins" is simply
// key(later) < key(earlier), with no per-voxel tie test.  Collar positions
// carry the dtype's sentinel key and take part like any voxel (a +inf voxel
// ties with the +inf collar exactly as in the reference).
//
// Per voxel v the blocks split by their extent along the sweep axis (axis 0):
// the in-plane blocks b containing v (v itself, its pairs, its quads) and
// each of them extended to the previous or the next plane.  With I_b = "v
// wins b inside its plane" and X_b(i) = "plane i+1's copy of b beats plane
// i's" (minimum against minimum):
//     v wins b extended to i+1  <=>  I_b & !X_b(i)
//     v wins b extended to i-1  <=>  I_b &  X_b(i-1)
// and the extended block has the opposite Euler sign, so
//     change(v) = sum_b  s_b * I_b * (X_b(i) - X_b(i-1)),
// s_b = (-1)^d for v itself and alternating with block size.
#pragma once
#include <cstdint>

namespace eccb {
namespace tour {

// In-plane blocks of a 3D voxel v = (j, k) (axis 1, axis 2):
//   0 v   1 Z(k-1)   2 Z(k)   3 Y(j-1)   4 Y(j)
//   5 Q(j-1,k-1)   6 Q(j-1,k)   7 Q(j,k-1)   8 Q(j,k)
// Z = pair along axis 2 anchored at k, Y = pair along axis 1, Q = 2 x 2.
constexpr int NB3 = 9;
constexpr uint32_t POS3 = 0x1Eu;   // the four pairs: sign +1 (v and quads: -1)
// 2D (axis 0 = sweep, axis 1 = in-row):  0 v   1 B(j-1)   2 B(j)
constexpr int NB2 = 3;
constexpr uint32_t POS2 = 0x1u;    // v: sign +1 (pairs: -1)

template <int NB>
struct Plane {
  uint32_t M[NB];  // block minima (keys)
  uint32_t I;      // bit b: v wins block b inside the plane
};

// X mask: bit b = [next.M[b] < cur.M[b]] (the later plane's block wins).
template <int NB>
__device__ __forceinline__ uint32_t xmask(const Plane<NB>& nxt, const Plane<NB>& cur) {
  uint32_t x = 0;
#pragma unroll
  for (int b = 0; b < NB; ++b) x |= (uint32_t)(nxt.M[b] < cur.M[b]) << b;
  return x;
}

// change = sum_b s_b I_b (X_b - Xp_b): the +1 terms are blocks whose sign
// is +1 and X - Xp = +1, or sign -1 and X - Xp = -1; the -1 terms the rest.
template <uint32_t POS>
__device__ __forceinline__ int change_of(uint32_t I, uint32_t X, uint32_t Xp) {
  const uint32_t up = I & X & ~Xp, dn = I & ~X & Xp;
  return __popc((up & POS) | (dn & ~POS)) - __popc((up & ~POS) | (dn & POS));
}

// Face bit f = (o0+1)*9 + (o1+1)*3 + (o2+1) of the FaceOffset o a voxel
// introduces (kernel.hpp:32-53); f = 13 (no offset) is never set.
__device__ __forceinline__ uint32_t faces3(uint32_t I, uint32_t X, uint32_t Xp) {
  // (o1, o2) of in-plane block b
  constexpr int o1[NB3] = {0, 0, 0, -1, 1, -1, -1, 1, 1};
  constexpr int o2[NB3] = {0, -1, 1, 0, 0, -1, 1, -1, 1};
  uint32_t f = 0;
#pragma unroll
  for (int b = 0; b < NB3; ++b) {
    const int c = (o1[b] + 1) * 3 + (o2[b] + 1);
    const uint32_t ib = (I >> b) & 1u;
    if (b) f |= ib << (9 + c);                      // o0 = 0
    f |= (ib & ~(X >> b)) << (18 + c);              // o0 = +1
    f |= (ib & (Xp >> b)) << c;                     // o0 = -1
  }
  return f;
}

__device__ __forceinline__ uint32_t faces2(uint32_t I, uint32_t X, uint32_t Xp) {
  constexpr int o1[NB2] = {0, -1, 1};
  uint32_t f = 0;
#pragma unroll
  for (int b = 0; b < NB2; ++b) {
    const int c = (o1[b] + 1) * 3 + 1;
    const uint32_t ib = (I >> b) & 1u;
    if (b) f |= ib << (9 + c);
    f |= (ib & ~(X >> b)) << (18 + c);
    f |= (ib & (Xp >> b)) << c;
  }
  return f;
}

// In-row blocks of a 2D pixel from its own key c and its row neighbours
// l (j-1) and r (j+1): B(j-1) = {j-1, j} is won by j iff c < l (j-1 comes
// first), B(j) = {j, j+1} iff not r < c.
__device__ __forceinline__ Plane<NB2> row2(uint32_t l, uint32_t c, uint32_t r) {
  Plane<NB2> p;
  p.M[0] = c;
  p.M[1] = min(l, c);
  p.M[2] = min(c, r);
  p.I = 1u | ((uint32_t)(c < l) << 1) | ((uint32_t)!(r < c) << 2);
  return p;
}

}  // namespace tour
}  // namespace eccb
