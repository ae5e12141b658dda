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

// Key images (the device copy of a PaddedChunk, ecc_chunk_*): the values are
// already order-preserving keys; the sentinel beyond the image is above them.
template <>
struct KeyTraits<uint32_t> {
  static constexpr uint32_t kSentinel = 0xFFFFFFFFu;
  __device__ __forceinline__ static uint32_t key(uint32_t v) { return v; }
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
  // value-index map (ValueIndex<float>::bin_of, value_index.hpp:40-45): bin =
  // position of the value's order key in this ascending device table, which
  // must hold it exactly (else ECC_EBINMAP)
  const uint32_t* table = nullptr;
  uint32_t table_n = 0;
  // key images without a table: bin = (key - key_lo) & key_mask
  uint32_t key_mask = 0xFFFFFFFFu;
  // the generic kernels' histogram as packed words (HistSink, <= 2^28 voxels)
  int packed = 0;
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
  // owned box along axes 1 and 2 (generic kernels only; -1 = the full axis):
  // a PaddedChunk's collar is part of the device image but owns no voxels
  int64_t oj0 = 0, oj1 = -1, ok0 = 0, ok1 = -1;
  __host__ __device__ int64_t own_j1() const { return oj1 < 0 ? w1 : oj1; }
  __host__ __device__ int64_t own_k1() const { return ok1 < 0 ? w2 : ok1; }
  __host__ __device__ int64_t row_pitch() const { return pitch ? pitch : w2; }
  __host__ __device__ int64_t plane_pitch() const { return ppitch ? ppitch : w1 * row_pitch(); }
};

}  // namespace eccb
