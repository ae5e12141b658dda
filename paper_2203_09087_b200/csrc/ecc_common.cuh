// ecc_common.cuh -- device-side vocabulary shared by the ECC kernels.
//
// Keys.  Every comparison of the reference stencil is done on a uint32 key
// that preserves the order of the extended value domain
// (value_traits<T>::extended, common.hpp:49-66):
//   u8  -> value,        collar sentinel 256     (common.hpp:54-59)
//   u16 -> value,        collar sentinel 65536   (the f32 path's +inf)
//   f32 -> order key (value_index.hpp:95-99; -0 folds onto +0), collar
//          sentinel = key(+inf), so a +inf voxel ties with the collar exactly
//          as in the reference.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace eccb {

template <class T>
struct KeyTraits;

template <>
struct KeyTraits<uint8_t> {
  static constexpr uint32_t kSentinel = 256u;
  __device__ __forceinline__ static uint32_t key(uint8_t v) { return v; }
};

template <>
struct KeyTraits<uint16_t> {
  static constexpr uint32_t kSentinel = 65536u;
  __device__ __forceinline__ static uint32_t key(uint16_t v) { return v; }
};

__host__ __device__ __forceinline__ uint32_t float_order_key_bits(uint32_t u) {
  if (u == 0x80000000u) u = 0;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

template <>
struct KeyTraits<float> {
  static constexpr uint32_t kSentinel = 0xFF800000u;  // key(+inf)
  __device__ __forceinline__ static uint32_t key(float v) {
    return float_order_key_bits(__float_as_uint(v));
  }
};

// Error flags raised by kernels (read back by the host after a launch).
enum : uint32_t {
  kFlagBinmap = 1u,  // value outside the affine bin grid
  kFlagNaN = 2u,
};

// ---------------------------------------------------------------------------
// Per-voxel change, 3D (kernel.hpp:99-137).  w[a][b][c] is the neighbour at
// offset (a-1, b-1, c-1) along (axis0, axis1, axis2).  Offsets whose first
// nonzero component is negative are earlier in row-major order
// (kernel.hpp:21-27) and compare strictly.
__device__ __forceinline__ int change3(const uint32_t (&w)[3][3][3]) {
  const uint32_t c = w[1][1][1];
  const unsigned xm = c < w[0][1][1], xp = c <= w[2][1][1];
  const unsigned ym = c < w[1][0][1], yp = c <= w[1][2][1];
  const unsigned zm = c < w[1][1][0], zp = c <= w[1][1][2];
  const unsigned exy_mm = xm & ym & (unsigned)(c < w[0][0][1]);
  const unsigned exy_mp = xm & yp & (unsigned)(c < w[0][2][1]);
  const unsigned exy_pm = xp & ym & (unsigned)(c <= w[2][0][1]);
  const unsigned exy_pp = xp & yp & (unsigned)(c <= w[2][2][1]);
  const unsigned exz_mm = xm & zm & (unsigned)(c < w[0][1][0]);
  const unsigned exz_mp = xm & zp & (unsigned)(c < w[0][1][2]);
  const unsigned exz_pm = xp & zm & (unsigned)(c <= w[2][1][0]);
  const unsigned exz_pp = xp & zp & (unsigned)(c <= w[2][1][2]);
  const unsigned eyz_mm = ym & zm & (unsigned)(c < w[1][0][0]);
  const unsigned eyz_mp = ym & zp & (unsigned)(c < w[1][0][2]);
  const unsigned eyz_pm = yp & zm & (unsigned)(c <= w[1][2][0]);
  const unsigned eyz_pp = yp & zp & (unsigned)(c <= w[1][2][2]);
  unsigned v = 0;
  v += exy_mm & exz_mm & eyz_mm & (unsigned)(c < w[0][0][0]);
  v += exy_mm & exz_mp & eyz_mp & (unsigned)(c < w[0][0][2]);
  v += exy_mp & exz_mm & eyz_pm & (unsigned)(c < w[0][2][0]);
  v += exy_mp & exz_mp & eyz_pp & (unsigned)(c < w[0][2][2]);
  v += exy_pm & exz_pm & eyz_mm & (unsigned)(c <= w[2][0][0]);
  v += exy_pm & exz_pp & eyz_mp & (unsigned)(c <= w[2][0][2]);
  v += exy_pp & exz_pm & eyz_pm & (unsigned)(c <= w[2][2][0]);
  v += exy_pp & exz_pp & eyz_pp & (unsigned)(c <= w[2][2][2]);
  const unsigned sq = xm + xp + ym + yp + zm + zp;
  const unsigned ed = exy_mm + exy_mp + exy_pm + exy_pp + exz_mm + exz_mp +
                      exz_pm + exz_pp + eyz_mm + eyz_mp + eyz_pm + eyz_pp;
  return -1 + (int)sq - (int)ed + (int)v;
}

// Per-voxel change, 2D over axes 0 and 1 (kernel.hpp:81-94).  w[a][b] is the
// neighbour at offset (a-1, b-1).
__device__ __forceinline__ int change2(const uint32_t (&w)[3][3]) {
  const uint32_t c = w[1][1];
  const unsigned am = c < w[0][1], ap = c <= w[2][1];
  const unsigned bm = c < w[1][0], bp = c <= w[1][2];
  unsigned v = 0;
  v += am & bm & (unsigned)(c < w[0][0]);
  v += am & bp & (unsigned)(c < w[0][2]);
  v += ap & bm & (unsigned)(c <= w[2][0]);
  v += ap & bp & (unsigned)(c <= w[2][2]);
  return 1 + (int)v - (int)(am + ap + bm + bp);
}

// Affine f32 bin map: bin = (v - lo) * inv_step must be an exact integer in
// [0, nbins) whose inverse lo + bin * step reproduces v (== compares -0 and
// +0 equal, so -0 lands on +0's bin as in value_index.hpp:97).  The inverse
// is evaluated in double, identically on host and device.
struct AffineMap {
  float lo, step;
  double inv_step;
  uint32_t nbins;
  float pow2_scale;  // 1/step when lo == 0 and step is a power of two, else 0
  // "keyed" map of the dense sorted-f32 path: bin = order key - key_lo
  // (value_index.hpp:95-99 order, every distinct value its own bin)
  int keyed = 0;
  uint32_t key_lo = 0;
};

__host__ __device__ __forceinline__ float affine_value(const AffineMap& m,
                                                      uint32_t bin) {
#ifdef __CUDA_ARCH__
  return __double2float_rn(__dadd_rn((double)m.lo, __dmul_rn((double)bin, (double)m.step)));
#else
  volatile double prod = (double)bin * (double)m.step;
  volatile double sum = (double)m.lo + prod;
  return (float)sum;
#endif
}

__device__ __forceinline__ uint32_t affine_bin(const AffineMap& m, float v,
                                               uint32_t* flags) {
  if (m.pow2_scale != 0.0f) {
    // lo = 0, step = 2^-k: v * 2^k is exact, and v is on the grid iff that
    // product is an integer (2^23 magic rounding); same accepted set and
    // bins as the double-precision check below (BASELINE config 4's grid).
    const float t = v * m.pow2_scale;
    if (t >= 0.0f && t < (float)m.nbins) {
      const float mg = t + 8388608.0f;
      if (mg - 8388608.0f == t) return __float_as_uint(mg) - 0x4B000000u;
    }
    atomicOr(flags, v != v ? kFlagNaN : kFlagBinmap);
    return 0;
  }
  const double t = __dmul_rn(__dadd_rn((double)v, -(double)m.lo), m.inv_step);
  const double r = rint(t);
  uint32_t bin = 0;
  bool ok = (r >= 0.0) && (r < (double)m.nbins);
  if (ok) {
    bin = (uint32_t)r;
    ok = affine_value(m, bin) == v;
  }
  if (!ok) {
    atomicOr(flags, v != v ? kFlagNaN : kFlagBinmap);
    bin = 0;
  }
  return bin;
}

// Slab description shared by the kernels (see ecc_accumulate_slab).
struct Slab {
  const void* base;  // device pointer to image plane `plane0`
  int64_t plane0, nplanes;
  int64_t w0, w1, w2;
  int64_t own0, own1;
  int64_t pitch = 0;  // elements between consecutive rows in memory (0 = w2)
  int64_t ppitch = 0; // elements between consecutive planes (0 = w1 * row_pitch())
  __host__ __device__ int64_t row_pitch() const { return pitch ? pitch : w2; }
  __host__ __device__ int64_t plane_pitch() const { return ppitch ? ppitch : w1 * row_pitch(); }
};

}  // namespace eccb
