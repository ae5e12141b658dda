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
// Layout.  One thread per output voxel, a CTA row per image row (no 64-bit
// index division); the taps of the contiguous axis hit L1, those of axes
// 0 / 1 are coalesced rows that stay in L2 while a plane band is swept (13
// planes x w1 x w2 x 4 B for the bench's width 13).  Double arithmetic: a
// DMUL and a DADD per tap (no FMA: the reference rounds the product).
#include <cstdint>

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

constexpr int MAXW = 1023;  // kernel taps held in shared memory

// One CTA row per image row (axes 0, 1 flattened: blockIdx.x), threads
// along axis 2 (blockIdx.y tiles): no 64-bit division per voxel.
__global__ void k_convolve_axis(const float* __restrict__ in, float* __restrict__ out,
                                uint32_t w1, uint32_t w2, uint32_t axis_w, int axis,
                                const double* __restrict__ w, int width) {
  __shared__ double ws[MAXW];
  for (int k = threadIdx.x; k < width; k += blockDim.x) ws[k] = w[k];
  __syncthreads();
  const uint32_t c = blockIdx.y * blockDim.x + threadIdx.x;
  if (c >= w2) return;
  const uint32_t r = blockIdx.x;
  const uint32_t i0 = r / w1, i1 = r - i0 * w1;
  const uint64_t i = (uint64_t)r * w2 + c;
  const int64_t pos = axis == 0 ? i0 : (axis == 1 ? i1 : c);
  const uint64_t s = axis == 0 ? (uint64_t)w1 * w2 : (axis == 1 ? w2 : 1);
  const float* base = in + (i - (uint64_t)pos * s);
  const int half = width / 2;
  double acc = 0.0;
  if (pos >= half && pos + half < (int64_t)axis_w) {
    // interior (every voxel but the 2 x half nearest the ends): a running
    // pointer, no clamping, no 64-bit index multiply per tap
    const float* q = base + (uint64_t)(pos - half) * s;
#pragma unroll 4
    for (int k = 0; k < width; ++k, q += s)
      acc = __dadd_rn(acc, __dmul_rn(ws[k], (double)__ldg(q)));
  } else {
    for (int k = -half; k <= half; ++k) {
      int64_t qq = pos + k;
      qq = qq < 0 ? 0 : (qq > (int64_t)axis_w - 1 ? (int64_t)axis_w - 1 : qq);
      acc = __dadd_rn(acc, __dmul_rn(ws[k + half], (double)__ldg(base + (uint64_t)qq * s)));
    }
  }
  out[i] = __double2float_rn(acc);
}

}  // namespace pipe

cudaError_t launch_uniform_noise(float* d, uint64_t n, uint64_t seed, int sms, cudaStream_t st) {
  pipe::k_uniform<<<sms * 16, 256, 0, st>>>(d, n, seed);
  return cudaGetLastError();
}

int gaussian_max_width() { return pipe::MAXW; }

cudaError_t launch_convolve_axis(const float* in, float* out, uint64_t w0, uint64_t w1,
                                 uint64_t w2, int axis, const double* d_weights, int width,
                                 cudaStream_t st) {
  const uint64_t rows = w0 * w1;
  const uint64_t ext = axis == 0 ? w0 : (axis == 1 ? w1 : w2);
  if (rows > 0x7FFFFFFFull || (w2 + 255) / 256 > 65535 || ext > 0xFFFFFFFFull)
    return cudaErrorInvalidValue;
  const dim3 grid((unsigned)rows, (unsigned)((w2 + 255) / 256));
  pipe::k_convolve_axis<<<grid, 256, 0, st>>>(in, out, (uint32_t)w1, (uint32_t)w2, (uint32_t)ext,
                                               axis, d_weights, width);
  return cudaGetLastError();
}

}  // namespace eccb
