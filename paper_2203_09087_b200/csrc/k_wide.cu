// k_wide.cu -- K1+K2 for 3D images with large bin counts (u16 -> 65536 bins,
// affine-quantised f32 -> up to 65536 bins; BASELINE config 4).
//
// Replaces, for those inputs, the reference's change_row_3d + radix
// argsort + reduce-by-key path (kernel.hpp:143-188, value_index.hpp:159-197):
// the value -> bin map is applied once per voxel (the centre) and the
// stencil compares the raw values (u16 as integers, f32 as floats with the
// +inf collar sentinel -- the reference's own extended-float comparison,
// so -0 == +0 and a +inf voxel ties the collar exactly as in
// common.hpp:61-66).
//
// Mapping: one CTA per SM (persistent), 32 x 16 threads over an (axis-2,
// axis-1) tile; every thread sweeps a segment of axis-0 planes keeping the
// 3 x 3 x 3 window in registers, so each value is loaded once per plane step
// and the two column neighbours hit L1.
//
// Histogram: 65536 signed 16-bit halves packed two per word in shared
// memory (128 KB) plus an occupancy bitmap (8 KB).  A half that leaves
// [-16384, 16383] is spilled exactly to the global int64 histogram by the
// thread whose atomic crossed the bound (atomicAdd returns the old word), so
// no half can ever wrap.  The CTA flushes its halves once at the end; the
// occupancy half of the global histogram receives the number of CTAs in
// which the value occurs (> 0 iff it occurs, which is all K3 reads).
#include <algorithm>
#include <cstdint>

#include "ecc_common.cuh"
#include "internal.h"

namespace eccb {
namespace wide {

constexpr int BX = 32, BY = 16;  // threads along axis 2 / axis 1

template <class K>
struct Sent;
template <>
struct Sent<uint32_t> {
  __device__ static uint32_t v(uint32_t s) { return s; }
};
template <>
struct Sent<float> {
  __device__ static float v(uint32_t) { return __int_as_float(0x7f800000); }
};

// change_3d (kernel.hpp:99-137) on any ordered key type
template <class K>
__device__ __forceinline__ int change3k(const K (&w)[3][3][3]) {
  const K c = w[1][1][1];
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
  const unsigned ed = exy_mm + exy_mp + exy_pm + exy_pp + exz_mm + exz_mp + exz_pm + exz_pp +
                      eyz_mm + eyz_mp + eyz_pm + eyz_pp;
  return -1 + (int)sq - (int)ed + (int)v;
}

__device__ __forceinline__ int sext16(uint32_t v) { return (int)(int16_t)(v & 0xFFFFu); }

// words[bin/2] holds bins 2q (low half) and 2q+1 (high half) as one integer
// lo + 65536 * hi; halves stay within [-16384, 16383] (each change moves a
// half by at most 7) because the crossing thread spills.
__device__ __forceinline__ void packed_add(uint32_t* words, uint32_t bin, int ch,
                                           int64_t* gsum) {
  const uint32_t q = bin >> 1;
  const bool hi = bin & 1;
  const uint32_t add = hi ? ((uint32_t)ch << 16) : (uint32_t)ch;
  const uint32_t old = atomicAdd(&words[q], add);
  const uint32_t nw = old + add;
  const int lo_old = sext16(old), lo_new = sext16(nw);
  const int before = hi ? (int)((int32_t)(old - (uint32_t)lo_old) >> 16) : lo_old;
  const int after = hi ? (int)((int32_t)(nw - (uint32_t)lo_new) >> 16) : lo_new;
  const bool in_before = before >= -16384 && before <= 16383;
  const bool in_after = after >= -16384 && after <= 16383;
  if (in_before && !in_after) {
    atomicAdd(&words[q], hi ? (uint32_t)(-after) << 16 : (uint32_t)(-after));
    atomicAdd(reinterpret_cast<unsigned long long*>(&gsum[bin]),
              static_cast<unsigned long long>(static_cast<long long>(after)));
  }
}

template <class T>
struct KeyOf;  // value type -> comparison key type
template <>
struct KeyOf<uint16_t> {
  using K = uint32_t;
  static constexpr uint32_t kSent = 65536u;
  __device__ static K key(uint16_t v) { return v; }
};
template <>
struct KeyOf<float> {
  using K = float;
  static constexpr uint32_t kSent = 0;
  __device__ static K key(float v) { return v; }
};

template <class T, bool AFFINE>
__global__ void __launch_bounds__(BX * BY, 1)
    k_wide3(Slab s, int seglen, int nseg, int tz, int ty, AffineMap am, int64_t* ghist,
            uint32_t nbins, uint32_t* flags) {
  using KO = KeyOf<T>;
  using K = typename KO::K;
  extern __shared__ uint32_t sm[];
  const uint32_t nwords = (nbins + 1) / 2;
  uint32_t* words = sm;
  uint32_t* pres = sm + nwords;
  const int tid = threadIdx.y * BX + threadIdx.x;
  for (uint32_t i = tid; i < nwords + (nbins + 31) / 32; i += BX * BY) sm[i] = 0;
  __syncthreads();

  const K SENT = Sent<K>::v(KO::kSent);
  const T* base = static_cast<const T*>(s.base);
  const int64_t W0 = s.w0, W1 = s.w1, W2 = s.w2;
  const int64_t plane = W1 * W2;
  const long long items = (long long)nseg * ty * tz;
  for (long long it = blockIdx.x; it < items; it += gridDim.x) {
    const int seg = (int)(it / ((long long)ty * tz));
    const int rest = (int)(it - (long long)seg * ty * tz);
    const int yt = rest / tz, zt = rest - yt * tz;
    const int64_t j = (int64_t)yt * BY + threadIdx.y;
    const int64_t k = (int64_t)zt * BX + threadIdx.x;
    const int64_t i0 = s.own0 + (int64_t)seg * seglen;
    const int64_t i1 = min(i0 + seglen, s.own1);
    if (j >= W1 || k >= W2 || i0 >= i1) continue;
    // column validity of the 3 x 3 neighbourhood (fixed over the sweep)
    bool cv[3][3];
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        cv[b][c] = (j - 1 + b >= 0) && (j - 1 + b < W1) && (k - 1 + c >= 0) && (k - 1 + c < W2);
    const bool interior = j >= 1 && j + 1 < W1 && k >= 1 && k + 1 < W2;
    // the 9 values of one plane around (j, k): row pointers advance by one
    // plane per step; loads for plane i + 2 are issued before the stencil
    // of plane i runs (one plane of prefetch hides the L1/L2 latency)
    const T* p0 = base + (j * W2 + k) + (i0 - 1 - s.plane0) * plane;
    auto fetch = [&](const T* p, int64_t i, T (&raw)[3][3]) {
      const bool in = i >= 0 && i < W0;
#pragma unroll
      for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (in && (interior || cv[b][c])) raw[b][c] = __ldg(p + (b - 1) * W2 + (c - 1));
    };
    auto keys = [&](int64_t i, const T (&raw)[3][3], K (&dst)[3][3]) {
      const bool in = i >= 0 && i < W0;
#pragma unroll
      for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          dst[b][c] = (in && (interior || cv[b][c])) ? KO::key(raw[b][c]) : SENT;
    };
    K w[3][3][3];
    T r0[3][3], r1[3][3];
    fetch(p0, i0 - 1, r0);
    fetch(p0 + plane, i0, r1);
    keys(i0 - 1, r0, w[0]);
    keys(i0, r1, w[1]);
    fetch(p0 + 2 * plane, i0 + 1, r0);  // plane i0 + 1
    const T* pc = p0 + plane;            // centre voxel of plane i
    for (int64_t i = i0; i < i1; ++i) {
      keys(i + 1, r0, w[2]);
      if (i + 1 < i1) fetch(pc + 2 * plane, i + 2, r0);  // prefetch plane i + 2
      const int ch = change3k<K>(w);
      const T v = w[1][1][1] == SENT ? T(0) : static_cast<T>(w[1][1][1]);
      uint32_t bin;
      if constexpr (AFFINE)
        bin = affine_bin(am, static_cast<float>(v), flags);
      else
        bin = static_cast<uint32_t>(v);
      atomicOr(&pres[bin >> 5], 1u << (bin & 31));
      if (ch != 0) packed_add(words, bin, ch, ghist);
#pragma unroll
      for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          w[0][b][c] = w[1][b][c];
          w[1][b][c] = w[2][b][c];
        }
      pc += plane;
    }
  }
  __syncthreads();
  for (uint32_t b = tid; b < nbins; b += BX * BY) {
    const uint32_t word = words[b >> 1];
    const int lo = sext16(word);
    const int sum = (b & 1) ? (int)((int32_t)(word - (uint32_t)lo) >> 16) : lo;
    if (sum != 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(&ghist[b]),
                static_cast<unsigned long long>(static_cast<long long>(sum)));
    if ((pres[b >> 5] >> (b & 31)) & 1u)
      atomicAdd(reinterpret_cast<unsigned long long*>(&ghist[nbins + b]), 1ull);
  }
}

template <class T, bool AFFINE>
cudaError_t launch_t(const Slab& s, const AffineMap& am, int64_t* ghist, uint32_t nbins,
                     uint32_t* flags, int sms, cudaStream_t st) {
  const size_t smem = ((nbins + 1) / 2 + (nbins + 31) / 32) * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_wide3<T, AFFINE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)((32768 + 2048) * 4));
    attr = true;
  }
  const int ty = (int)((s.w1 + BY - 1) / BY), tz = (int)((s.w2 + BX - 1) / BX);
  const long long tiles = (long long)ty * tz;
  const int64_t owned = s.own1 - s.own0;
  // ~8 work items per SM, segments of >= 16 planes
  long long nseg = (8LL * sms + tiles - 1) / tiles;
  nseg = std::max<long long>(1, std::min<long long>(nseg, (owned + 15) / 16));
  const int seglen = (int)((owned + nseg - 1) / nseg);
  nseg = (owned + seglen - 1) / seglen;
  const long long items = nseg * tiles;
  const unsigned grid = (unsigned)std::min<long long>(items, sms);
  k_wide3<T, AFFINE><<<grid, dim3(BX, BY), smem, st>>>(s, seglen, (int)nseg, tz, ty, am, ghist,
                                                       nbins, flags);
  return cudaGetLastError();
}

}  // namespace wide

bool wide_supported(const Slab& s, int dtype, bool affine, uint32_t nbins) {
  return s.w2 > 1 && nbins <= 65536 && nbins > 8192 &&
         ((dtype == 1 && !affine) || (dtype == 2 && affine)) &&
         s.w1 * s.w2 < (1ll << 40);
}

cudaError_t launch_wide(const Slab& s, int dtype, bool affine, const AffineMap& am, int64_t* ghist,
                        uint32_t nbins, uint32_t* flags, int sms, cudaStream_t st) {
  if (dtype == 1) return wide::launch_t<uint16_t, false>(s, am, ghist, nbins, flags, sms, st);
  return wide::launch_t<float, true>(s, am, ghist, nbins, flags, sms, st);
}

}  // namespace eccb
