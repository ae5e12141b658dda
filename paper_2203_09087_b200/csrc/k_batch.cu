// k_batch.cu -- batched 2D ECC (the reference has no
// in-memory batched entry point; BASELINE config 3 needs one).
//
// One CTA per image.  The histogram of per-pixel changes (change_2d,
// kernel.hpp:81-94) is built in the output row itself and then prefix-summed
// in place, so each image's curve is produced without leaving the CTA:
//   * <= 8192 bins (u8): shared-memory bins, one flush per CTA;
//   * 65536 bins (u16): packed 16-bit bin pairs in shared memory (128 KB)
//     plus an 8 KB presence bitmap, with exact overflow spill to the global
//     row (see PackedBins below).
#include <cub/cub.cuh>

#include "ecc_common.cuh"
#include "internal.h"

namespace eccb {

namespace {

template <class T>
__device__ __forceinline__ uint32_t key_at(const T* img, int h, int w, int i,
                                           int j) {
  if (i < 0 || i >= h || j < 0 || j >= w) return KeyTraits<T>::kSentinel;
  return KeyTraits<T>::key(__ldg(img + (size_t)i * w + j));
}

// Shared-memory bins for 65536 values in 128 KB: word q holds bins 2q (low
// half) and 2q+1 (high half) as one integer V = S_lo + 65536 * S_hi, which
// an atomicAdd of `change` or `change << 16` updates exactly.  The halves
// decode unambiguously while each |S| < 32768.  Every change moves a half
// by at most 3 (2D range [-3, 1]); the thread whose update
// carries a half out of [-16384, 16383] subtracts exactly what it observed
// and spills it to the global row, so halves never get near the limit.
__device__ __forceinline__ int sext16(uint32_t v) { return (int)(int16_t)(v & 0xFFFF); }

__device__ __forceinline__ void packed_add(uint32_t* words, uint32_t bin, int ch,
                                           int32_t* grow) {
  const uint32_t q = bin >> 1;
  const bool hi = bin & 1;
  const uint32_t add = hi ? ((uint32_t)ch << 16) : (uint32_t)ch;
  const uint32_t old = atomicAdd(&words[q], add);
  const uint32_t nw = old + add;
  // decode the touched half before and after
  const int lo_old = sext16(old), lo_new = sext16(nw);
  int before, after;
  if (hi) {
    before = (int)((int32_t)(old - (uint32_t)lo_old) >> 16);
    after = (int)((int32_t)(nw - (uint32_t)lo_new) >> 16);
  } else {
    before = lo_old;
    after = lo_new;
  }
  const bool in_before = before >= -16384 && before <= 16383;
  const bool in_after = after >= -16384 && after <= 16383;
  if (in_before && !in_after) {
    atomicAdd(&words[q], hi ? (uint32_t)(-after) << 16 : (uint32_t)(-after));
    atomicAdd(&grow[bin], after);
  }
}

}  // namespace

template <class T, bool PACKED>
__global__ void __launch_bounds__(1024) k_batch2d(const T* __restrict__ data, int h,
                                                  int w, uint32_t nbins,
                                                  int32_t* __restrict__ chi,
                                                  uint32_t* __restrict__ presence) {
  extern __shared__ uint32_t sm[];
  const size_t img_id = blockIdx.x;
  const T* img = data + img_id * (size_t)h * w;
  int32_t* row = chi + img_id * (size_t)nbins;
  uint32_t* pres_row = presence + img_id * (size_t)(nbins / 32);
  const uint32_t nwords = PACKED ? nbins / 2 : nbins;
  uint32_t* bins = sm;
  uint32_t* pres = sm + nwords;
  for (uint32_t q = threadIdx.x; q < nwords + nbins / 32; q += blockDim.x) sm[q] = 0;
  for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) row[b] = 0;
  __syncthreads();
  // pixels in row-major order, a 3x3 key window per pixel
  const int n = h * w;
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    const int i = p / w, j = p - i * w;
    uint32_t win[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) win[a][b] = key_at<T>(img, h, w, i - 1 + a, j - 1 + b);
    const int ch = change2(win);
    const uint32_t v = win[1][1];
    atomicOr(&pres[v >> 5], 1u << (v & 31));
    if (ch != 0) {
      if constexpr (PACKED)
        packed_add(bins, v, ch, row);
      else
        atomicAdd(&bins[v], (uint32_t)ch);
    }
  }
  __syncthreads();
  // fold shared bins into the row (spills already there), then scan in place
  const uint32_t per = (nbins + blockDim.x - 1) / blockDim.x;
  const uint32_t b0 = min(nbins, threadIdx.x * per), b1 = min(nbins, b0 + per);
  int32_t local = 0;
  for (uint32_t b = b0; b < b1; ++b) {
    int s;
    if constexpr (PACKED) {
      const uint32_t word = bins[b >> 1];
      const int lo = sext16(word);
      s = (b & 1) ? (int)((int32_t)(word - (uint32_t)lo) >> 16) : lo;
    } else {
      s = (int)bins[b];
    }
    local += s + row[b];
  }
  using Scan = cub::BlockScan<int32_t, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  int32_t ex;
  Scan(tmp).ExclusiveSum(local, ex);
  for (uint32_t b = b0; b < b1; ++b) {
    int s;
    if constexpr (PACKED) {
      const uint32_t word = bins[b >> 1];
      const int lo = sext16(word);
      s = (b & 1) ? (int)((int32_t)(word - (uint32_t)lo) >> 16) : lo;
    } else {
      s = (int)bins[b];
    }
    ex += s + row[b];
    row[b] = ex;
  }
  for (uint32_t q = threadIdx.x; q < nbins / 32; q += blockDim.x) pres_row[q] = pres[q];
}

cudaError_t launch_batch2d(const void* data, int dtype, uint64_t count, int h, int w,
                           int32_t* chi, uint32_t* presence, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  if (dtype == 0) {
    const uint32_t nbins = 256;
    const size_t smem = (nbins + nbins / 32) * 4;
    k_batch2d<uint8_t, false><<<(unsigned)count, 1024, smem, st>>>(
        (const uint8_t*)data, h, w, nbins, chi, presence);
  } else if (dtype == 1) {
    const uint32_t nbins = 65536;
    const size_t smem = (nbins / 2 + nbins / 32) * 4;
    cudaFuncSetAttribute(k_batch2d<uint16_t, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_batch2d<uint16_t, true><<<(unsigned)count, 1024, smem, st>>>(
        (const uint16_t*)data, h, w, nbins, chi, presence);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace eccb
