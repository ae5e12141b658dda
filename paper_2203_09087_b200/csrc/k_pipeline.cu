// k_pipeline.cu -- the GPU-resident pipeline of the reference's in-memory
// benchmark: uniform noise and separable Gaussian
// smoothing on the device, bit-identical to the reference generator.
//
//   uniform_noise   datagen.hpp:57-62  (counter_uniform, datagen.hpp:30-32)
//   gaussian_smooth datagen.hpp:108-122 (convolve_axis, datagen.hpp:80-105)
//
// Exactness.  counter_uniform is integer work ((H >> 40) * 2^-24 is exact in
// binary32).  convolve_axis accumulates, in tap order k = -half..half, the
// double products kernel[k] * value into a double starting at 0 and rounds
// the sum to float; the reference is ISO C++ built for x86-64 (SSE2 doubles,
// no FMA contraction), so with the same weights (computed on the host with
// the same libm, capi.cu) and explicitly rounded __dmul_rn / __dadd_rn steps
// the device produces the same floats.  Edge clamping as in the reference.
//
// Layout.  Per smoothed axis the volume is (outer, L, inner).  Inputs are
// staged once per CTA as doubles in shared memory, edge-clamped (the float
// -> double conversion is exact and now happens once per input instead of
// once per tap), then every thread runs several outputs: per tap one
// conflict-free LDS.64, a DMUL and a DADD (no FMA: the reference rounds the
// product).  inner == 1: row tiles of 1024 outputs; inner > 1: tiles of 32
// coalesced inner positions x 64 outputs along the axis.
#include <cstdint>
#include <type_traits>

#include "ecc_common.cuh"
#include "internal.h"

namespace eccb {
namespace pipe {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void k_uniform(float* __restrict__ d, uint64_t n, uint64_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    d[i] = (float)(splitmix64(seed + i * 0x9E3779B97F4A7C15ull) >> 40) * 0x1p-24f;
}

constexpr int MAXW = 255;  // kernel taps (shared-memory tiles hold width - 1 halo lines)

// The volume seen as (outer, L, inner) around the smoothed axis (inner =
// product of the later extents, the axis stride).  Inputs are staged once
// as doubles in shared memory (edge-clamped), so a tap is one LDS.64, a
// DMUL and a DADD; each thread produces several outputs.

// inner == 1 (the contiguous axis): a CTA smooths 256 J consecutive outputs
// of one line (J = 1, 2 or 4 by line length); thread t owns outputs
// t + 256 j (conflict-free reads).
constexpr int ROW_T = 256;

template <int J>
__global__ void __launch_bounds__(ROW_T)
    k_smooth_rows(const float* __restrict__ in, float* __restrict__ out, uint32_t L,
                  uint32_t tiles, const double* __restrict__ w, int width) {
  constexpr int ROW_J = J, ROW_OUT = ROW_T * J;
  extern __shared__ double sh[];
  double* ws = sh;                  // [width]
  double* xs = sh + width;          // [J * ROW_T + width - 1]
  const int half = width / 2;
  const uint64_t line = blockIdx.x / tiles;
  const int64_t p0 = (int64_t)(blockIdx.x - line * tiles) * ROW_OUT;
  const float* src = in + line * L;
  for (int k = threadIdx.x; k < width; k += ROW_T) ws[k] = w[k];
  // staging: eight loads in flight per thread before any conversion
  const int ne = J * ROW_T + width - 1;
  for (int e0 = 0; e0 < ne; e0 += 8 * ROW_T) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * ROW_T + threadIdx.x;
      int64_t q = p0 - half + e;
      q = q < 0 ? 0 : (q > (int64_t)L - 1 ? (int64_t)L - 1 : q);
      v[u] = e < ne ? __ldg(src + q) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * ROW_T + threadIdx.x;
      if (e < ne) xs[e] = (double)v[u];
    }
  }
  __syncthreads();
  double acc[ROW_J];
#pragma unroll
  for (int j = 0; j < ROW_J; ++j) acc[j] = 0.0;
  for (int k = 0; k < width; ++k) {
    const double wk = ws[k];
#pragma unroll
    for (int j = 0; j < ROW_J; ++j)
      acc[j] = __dadd_rn(acc[j], __dmul_rn(wk, xs[threadIdx.x + ROW_T * j + k]));
  }
  float* dst = out + line * L;
#pragma unroll
  for (int j = 0; j < ROW_J; ++j) {
    const int64_t p = p0 + threadIdx.x + ROW_T * j;
    if (p < (int64_t)L) dst[p] = __double2float_rn(acc[j]);
  }
}

// The contiguous axis, pipelined: a CTA runs UPB consecutive (line, tile)
// units and issues the next unit's loads before computing the current one,
// so the load latency hides behind the taps (widths up to 64).
constexpr int UPB = 8;

// mm != nullptr (the last pass of a smoothing whose result is ECC'ed next):
// also reduce the outputs' order-key range into mm[0] (min) / mm[1] (max)
// and raise kFlagNaN in *flags -- the key-range pass of the sorted-f32 ECC,
// fused (the values are in registers here anyway).
template <int J>
__global__ void __launch_bounds__(ROW_T)
    k_smooth_rows_p(const float* __restrict__ in, float* __restrict__ out, uint32_t L,
                    uint32_t tiles, uint64_t units, const double* __restrict__ w, int width,
                    uint32_t* __restrict__ mm, uint32_t* __restrict__ flags) {
  uint32_t klo = 0xFFFFFFFFu, khi = 0;
  bool nan = false;
  constexpr int ROW_OUT = ROW_T * J, NV = (ROW_OUT + 63 + ROW_T - 1) / ROW_T;
  extern __shared__ double sh[];
  double* ws = sh;          // [width]
  double* xs = sh + width;  // [ROW_OUT + width - 1]
  const int half = width / 2;
  const int ne = ROW_OUT + width - 1;
  for (int k = threadIdx.x; k < width; k += ROW_T) ws[k] = w[k];
  const uint64_t u0 = (uint64_t)blockIdx.x * UPB;
  const uint64_t u1 = u0 + UPB < units ? u0 + UPB : units;
  float v[NV];
  auto load = [&](uint64_t u) {
    const uint64_t line = u / tiles;
    const int64_t p0 = (int64_t)(u - line * tiles) * ROW_OUT;
    const float* src = in + line * L;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int e = i * ROW_T + threadIdx.x;
      int64_t q = p0 - half + e;
      q = q < 0 ? 0 : (q > (int64_t)L - 1 ? (int64_t)L - 1 : q);
      v[i] = e < ne ? __ldg(src + q) : 0.0f;
    }
  };
  if (u0 < u1) load(u0);
  for (uint64_t u = u0; u < u1; ++u) {
    __syncthreads();  // the previous unit's taps are done with xs
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int e = i * ROW_T + threadIdx.x;
      if (e < ne) xs[e] = (double)v[i];
    }
    __syncthreads();
    if (u + 1 < u1) load(u + 1);  // in flight during the taps below
    double acc[J];
#pragma unroll
    for (int j = 0; j < J; ++j) acc[j] = 0.0;
    for (int k = 0; k < width; ++k) {
      const double wk = ws[k];
#pragma unroll
      for (int j = 0; j < J; ++j)
        acc[j] = __dadd_rn(acc[j], __dmul_rn(wk, xs[threadIdx.x + ROW_T * j + k]));
    }
    const uint64_t line = u / tiles;
    const int64_t p0 = (int64_t)(u - line * tiles) * ROW_OUT;
    float* dst = out + line * L;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int64_t p = p0 + threadIdx.x + ROW_T * j;
      if (p < (int64_t)L) {
        const float f = __double2float_rn(acc[j]);
        dst[p] = f;
        if (mm) {
          const uint32_t kk = float_order_key_bits(__float_as_uint(f));
          klo = min(klo, kk);
          khi = max(khi, kk);
          nan |= f != f;
        }
      }
    }
  }
  if (mm) {
    klo = __reduce_min_sync(0xFFFFFFFFu, klo);
    khi = __reduce_max_sync(0xFFFFFFFFu, khi);
    if ((threadIdx.x & 31) == 0) {
      atomicMin(mm, klo);
      atomicMax(mm + 1, khi);
    }
    if (nan) atomicOr(flags, kFlagNaN);
  }
}

// inner > 1: a CTA smooths COL_W inner positions x COL_OUT outputs along the
// axis; thread (c, g) owns column c, outputs g + COL_G j.
constexpr int COL_W = 32, COL_G = 8, COL_J = 8, COL_OUT = COL_G * COL_J;

// Register-blocked taps for a compile-time width W: the thread's COL_J
// consecutive outputs share one window of COL_J + W - 1 inputs held in
// registers, so a tap costs a DMUL + DADD and no shared-memory load.  The
// accumulation order per output (taps k = 0 .. W-1) is the reference's.
template <int W, int STRIDE>
__device__ __forceinline__ void taps_blocked(const double* xs, const double* ws, int first, int c,
                                            double (&acc)[COL_J]) {
  double x[COL_J + W - 1], wr[W];
#pragma unroll
  for (int m = 0; m < COL_J + W - 1; ++m) x[m] = xs[(first + m) * STRIDE + c];
#pragma unroll
  for (int k = 0; k < W; ++k) wr[k] = ws[k];
#pragma unroll
  for (int k = 0; k < W; ++k)
#pragma unroll
    for (int j = 0; j < COL_J; ++j) acc[j] = __dadd_rn(acc[j], __dmul_rn(wr[k], x[j + k]));
}

template <int W>
__global__ void __launch_bounds__(COL_W * COL_G)
    k_smooth_cols(const float* __restrict__ in, float* __restrict__ out, uint32_t L,
                  uint64_t inner, uint32_t ctiles, const double* __restrict__ w, int width) {
  extern __shared__ double sh[];
  double* ws = sh;                  // [width]
  double* xs = sh + width;          // [(COL_OUT + width - 1) * COL_W]
  const int half = width / 2;
  const uint64_t outer = blockIdx.x / ctiles;
  const uint64_t c0 = (uint64_t)(blockIdx.x - outer * ctiles) * COL_W;
  const int64_t p0 = (int64_t)blockIdx.y * COL_OUT;
  const float* src = in + outer * L * inner;
  const int c = threadIdx.x & (COL_W - 1), g = threadIdx.x / COL_W;
  const bool col_in = c0 + c < inner;
  for (int k = threadIdx.x; k < width; k += COL_W * COL_G) ws[k] = w[k];
  // staging: the whole tile's loads in flight per thread (one latency per
  // tile) before any conversion; compile-time widths know the count
  const int nr = COL_OUT + width - 1;
  constexpr int NL = W > 0 ? (COL_OUT + W - 1 + COL_G - 1) / COL_G : 8;
  for (int r0 = g; r0 < nr; r0 += NL * COL_G) {
    float v[NL];
#pragma unroll
    for (int u = 0; u < NL; ++u) {
      const int r = r0 + u * COL_G;
      int64_t q = p0 - half + r;
      q = q < 0 ? 0 : (q > (int64_t)L - 1 ? (int64_t)L - 1 : q);
      v[u] = (col_in && r < nr) ? __ldg(src + (uint64_t)q * inner + c0 + c) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < NL; ++u) {
      const int r = r0 + u * COL_G;
      if (r < nr) xs[r * COL_W + c] = (double)v[u];
    }
  }
  __syncthreads();
  double acc[COL_J];
#pragma unroll
  for (int j = 0; j < COL_J; ++j) acc[j] = 0.0;
  if constexpr (W > 0) {
    taps_blocked<W, COL_W>(xs, ws, g * COL_J, c, acc);  // outputs g COL_J + j
  } else {
    for (int k = 0; k < width; ++k) {                    // outputs g + COL_G j
      const double wk = ws[k];
#pragma unroll
      for (int j = 0; j < COL_J; ++j)
        acc[j] = __dadd_rn(acc[j], __dmul_rn(wk, xs[(g + COL_G * j + k) * COL_W + c]));
    }
  }
  if (!col_in) return;
  float* dst = out + outer * L * inner + c0 + c;
#pragma unroll
  for (int j = 0; j < COL_J; ++j) {
    const int64_t p = p0 + (W > 0 ? g * COL_J + j : g + COL_G * j);
    if (p < (int64_t)L) dst[(uint64_t)p * inner] = __double2float_rn(acc[j]);
  }
}

// Strided axes with a compile-time width, pipelined: a CTA runs PT
// consecutive position tiles of one column tile and issues the next tile's
// loads before the current tile's register-blocked taps.
constexpr int PT = 4;

template <int W>
__global__ void __launch_bounds__(COL_W * COL_G)
    k_smooth_cols_p(const float* __restrict__ in, float* __restrict__ out, uint32_t L,
                    uint64_t inner, uint32_t ctiles, uint32_t ptiles,
                    const double* __restrict__ w) {
  constexpr int NR = COL_OUT + W - 1, NL = (NR + COL_G - 1) / COL_G;
  __shared__ double ws[W];
  __shared__ double xs[NR * COL_W];
  const int half = W / 2;
  const uint64_t outer = blockIdx.x / ctiles;
  const uint64_t c0 = (uint64_t)(blockIdx.x - outer * ctiles) * COL_W;
  const float* src = in + outer * L * inner;
  const int c = threadIdx.x & (COL_W - 1), g = threadIdx.x / COL_W;
  const bool col_in = c0 + c < inner;
  for (int k = threadIdx.x; k < W; k += COL_W * COL_G) ws[k] = w[k];
  const uint32_t t0 = blockIdx.y * PT, t1 = min(t0 + PT, ptiles);
  float v[NL];
  auto load = [&](uint32_t t) {
    const int64_t p0 = (int64_t)t * COL_OUT;
#pragma unroll
    for (int u = 0; u < NL; ++u) {
      const int r = g + u * COL_G;
      int64_t q = p0 - half + r;
      q = q < 0 ? 0 : (q > (int64_t)L - 1 ? (int64_t)L - 1 : q);
      v[u] = (col_in && r < NR) ? __ldg(src + (uint64_t)q * inner + c0 + c) : 0.0f;
    }
  };
  if (t0 < t1) load(t0);
  for (uint32_t t = t0; t < t1; ++t) {
    __syncthreads();  // the previous tile's taps are done with xs
#pragma unroll
    for (int u = 0; u < NL; ++u) {
      const int r = g + u * COL_G;
      if (r < NR) xs[r * COL_W + c] = (double)v[u];
    }
    __syncthreads();
    if (t + 1 < t1) load(t + 1);  // in flight during the taps
    double acc[COL_J];
#pragma unroll
    for (int j = 0; j < COL_J; ++j) acc[j] = 0.0;
    taps_blocked<W, COL_W>(xs, ws, g * COL_J, c, acc);
    if (col_in) {
      float* dst = out + outer * L * inner + c0 + c;
      const int64_t p0 = (int64_t)t * COL_OUT;
#pragma unroll
      for (int j = 0; j < COL_J; ++j) {
        const int64_t p = p0 + g * COL_J + j;
        if (p < (int64_t)L) dst[(uint64_t)p * inner] = __double2float_rn(acc[j]);
      }
    }
  }
}

}  // namespace pipe

cudaError_t launch_uniform_noise(float* d, uint64_t n, uint64_t seed, int sms, cudaStream_t st) {
  pipe::k_uniform<<<sms * 16, 256, 0, st>>>(d, n, seed);
  return cudaGetLastError();
}

int gaussian_max_width() { return pipe::MAXW; }

cudaError_t launch_convolve_axis(const float* in, float* out, uint64_t w0, uint64_t w1,
                                 uint64_t w2, int axis, const double* d_weights, int width,
                                 cudaStream_t st, uint32_t* mm, uint32_t* flags, bool* ranged) {
  if (ranged) *ranged = false;
  using namespace pipe;
  const uint64_t ext[3] = {w0, w1, w2};
  const uint64_t L = ext[axis];
  uint64_t outer = 1, inner = 1;
  for (int a = 0; a < axis; ++a) outer *= ext[a];
  for (int a = axis + 1; a < 3; ++a) inner *= ext[a];
  if (L > 0x7FFFFFFFull) return cudaErrorInvalidValue;
  // compile-time widths get the register-blocked kernels
  auto blocked = [&](auto wc) -> bool {
    constexpr int W = decltype(wc)::value;
    if (width != W) return false;
    if (inner == 1) {
      // the contiguous axis keeps the plain row tiles: a transposed-tile
      // register-blocked variant measured slower (826 vs 794 us at 512^3)
      return false;
    } else {
      const uint64_t ctiles = (inner + COL_W - 1) / COL_W;
      const uint64_t ptiles = (L + COL_OUT - 1) / COL_OUT;
      if (outer * ctiles > 0x7FFFFFFFull || ptiles > 65535) return false;
      if (((COL_OUT + W - 1) * COL_W + W) * 8 <= 48 * 1024) {  // static shared memory
        k_smooth_cols_p<W><<<dim3((unsigned)(outer * ctiles), (unsigned)((ptiles + PT - 1) / PT)),
                             COL_W * COL_G, 0, st>>>(in, out, (uint32_t)L, inner, (uint32_t)ctiles,
                                                     (uint32_t)ptiles, d_weights);
        return true;
      }
      const size_t smem = (size_t)(width + (COL_OUT + width - 1) * COL_W) * 8;
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_smooth_cols<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_smooth_cols<W><<<dim3((unsigned)(outer * ctiles), (unsigned)ptiles), COL_W * COL_G, smem,
                         st>>>(in, out, (uint32_t)L, inner, (uint32_t)ctiles, d_weights, width);
    }
    return true;
  };
  using std::integral_constant;
  if (blocked(integral_constant<int, 5>{}) || blocked(integral_constant<int, 7>{}) ||
      blocked(integral_constant<int, 9>{}) || blocked(integral_constant<int, 13>{}) ||
      blocked(integral_constant<int, 25>{}))
    return cudaGetLastError();
  if (inner == 1) {
    const int J = L <= 256 ? 1 : (L <= 512 ? 2 : 4);
    const uint64_t tiles = (L + (uint64_t)ROW_T * J - 1) / ((uint64_t)ROW_T * J);
    if (outer * tiles > 0x7FFFFFFFull) return cudaErrorInvalidValue;
    const size_t smem = (size_t)(width + ROW_T * J + width - 1) * 8;
    const uint64_t units = outer * tiles;
    if (width <= 64 && (units + UPB - 1) / UPB <= 0x7FFFFFFFull) {
      const unsigned grid = (unsigned)((units + UPB - 1) / UPB);
      auto go = [&](auto kern) {
        if (smem > 48 * 1024)
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, ROW_T, smem, st>>>(in, out, (uint32_t)L, (uint32_t)tiles, units, d_weights,
                                        width, mm, flags);
      };
      if (ranged) *ranged = mm != nullptr;
      if (J == 1)
        go(k_smooth_rows_p<1>);
      else if (J == 2)
        go(k_smooth_rows_p<2>);
      else
        go(k_smooth_rows_p<4>);
      return cudaGetLastError();
    }
    const unsigned grid = (unsigned)(outer * tiles);
    auto go = [&](auto kern) {
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<grid, ROW_T, smem, st>>>(in, out, (uint32_t)L, (uint32_t)tiles, d_weights, width);
    };
    if (J == 1)
      go(k_smooth_rows<1>);
    else if (J == 2)
      go(k_smooth_rows<2>);
    else
      go(k_smooth_rows<4>);
  } else {
    const uint64_t ctiles = (inner + COL_W - 1) / COL_W;
    const uint64_t ptiles = (L + COL_OUT - 1) / COL_OUT;
    if (outer * ctiles > 0x7FFFFFFFull || ptiles > 65535) return cudaErrorInvalidValue;
    const size_t smem = (size_t)(width + (COL_OUT + width - 1) * COL_W) * 8;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(k_smooth_cols<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_smooth_cols<0><<<dim3((unsigned)(outer * ctiles), (unsigned)ptiles), COL_W * COL_G, smem, st>>>(
        in, out, (uint32_t)L, inner, (uint32_t)ctiles, d_weights, width);
  }
  return cudaGetLastError();
}

}  // namespace eccb
