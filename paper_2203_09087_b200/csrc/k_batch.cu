// k_batch.cu -- batched 2D ECC (the reference has no
// in-memory batched entry point; BASELINE config 3 needs one).
//
// One CTA per image (1024 threads).  Thread t owns column j = t % w of a
// band of rows and slides a window of three rows of (j-1, j, j+1) keys down
// it (one new row per step, prefetched one step ahead), carrying each row's
// in-row block minima and deciding the pixel's blocks by the tournament of
// tourney.cuh (the 2D stencil of kernel.hpp:81-94).  The per-image histogram lives in shared
// memory:
//   * <= 8192 bins (u8): int32 change sums + occupancy bits;
//   * 65536 bins (u16 images wider than the bit-sliced k_batch16.cu takes):
//     the packed biased 16-bit halves of hist16.cuh (128 KB) with exact
//     compare-and-swap spills to a per-SM global scratch row (one CTA per
//     SM, so rows are private), marking the bin in a "spilled" bitmap so the
//     epilogue reads back and re-zeroes exactly those scratch entries.
// The epilogue prefix-sums the bins in place (block scan over per-thread
// runs) and writes the dense chi row and the occupancy bitmap -- one pass,
// no zero-fill of the output.
#include <cub/cub.cuh>

#include "ecc_common.cuh"
#include "hist16.cuh"
#include "internal.h"
#include "tourney.cuh"

namespace eccb {

namespace {

constexpr int NT = 1024;
static_assert(hist16::no_wrap(NT, 1, 3), "2D changes reach -3: the packed halves could wrap");

__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

}  // namespace

template <class T, bool PACKED>
__global__ void __launch_bounds__(NT, 1)
    k_batch2d(const T* __restrict__ data, int h, int w, uint32_t nbins, int32_t* __restrict__ chi,
              uint32_t* __restrict__ presence, int32_t* __restrict__ spill_scratch) {
  extern __shared__ uint32_t sm[];
  const uint32_t nwords = PACKED ? nbins / 2 : nbins;
  uint32_t* bins = sm;
  uint32_t* pres = sm + nwords;
  uint32_t* spilled = pres + nbins / 32;  // PACKED only
  const uint32_t nsm = nwords + nbins / 32 + (PACKED ? nbins / 32 : 0);
  for (uint32_t q = threadIdx.x; q < nsm; q += NT)
    sm[q] = (PACKED && q < nwords) ? hist16::BIAS : 0u;  // packed halves start at the bias
  __syncthreads();
  const uint32_t hbase = static_cast<uint32_t>(__cvta_generic_to_shared(bins));
  const T* img = data + (size_t)blockIdx.x * h * w;
  int32_t* row = chi + (size_t)blockIdx.x * nbins;
  uint32_t* pres_row = presence + (size_t)blockIdx.x * (nbins / 32);
  int32_t* scratch = PACKED ? spill_scratch + (size_t)smid() * nbins : nullptr;
  constexpr uint32_t SENT = KeyTraits<T>::kSentinel;

  // thread -> (column, band of rows)
  const int bands = max(1, NT / w);
  const int cols_per_pass = NT / bands;  // >= w when bands > 1
  for (int j0 = 0; j0 < w; j0 += cols_per_pass) {
    const int j = j0 + (int)threadIdx.x % cols_per_pass;
    const int band = (int)threadIdx.x / cols_per_pass;
    if (j >= w || band >= bands) continue;
    const int rows = (h + bands - 1) / bands;
    const int i0 = band * rows, i1 = min(h, i0 + rows);
    if (i0 >= i1) continue;
    const bool lv = j >= 1, rv = j + 1 < w;
    // one running pointer per thread; rows outside the image read the
    // sentinel (the loop bounds keep the pointer inside for i in [0, h))
    const T* p = img + (ptrdiff_t)(i0 - 1) * w + j;
    auto fetch = [&](int i, const T* q, uint32_t (&r)[3]) {
      if (i < 0 || i >= h) {
        r[0] = r[1] = r[2] = SENT;
        return;
      }
      r[0] = lv ? (uint32_t)__ldg(q - 1) : SENT;
      r[1] = (uint32_t)__ldg(q);
      r[2] = rv ? (uint32_t)__ldg(q + 1) : SENT;
    };
    uint32_t r0[3], r1[3], nxt[3];
    fetch(i0 - 1, p, r0);
    fetch(i0, p + w, r1);
    fetch(i0 + 1, p + 2 * w, nxt);
    p += 3 * w;  // row i0 + 2
    tour::Plane<tour::NB2> prev = tour::row2(r0[0], r0[1], r0[2]);
    tour::Plane<tour::NB2> cur = tour::row2(r1[0], r1[1], r1[2]);
    uint32_t Xp = tour::xmask(cur, prev);
    for (int i = i0; i < i1; ++i, p += w) {
      const tour::Plane<tour::NB2> next = tour::row2(nxt[0], nxt[1], nxt[2]);
      fetch(i + 2, p, nxt);  // prefetch
      const uint32_t X = tour::xmask(next, cur);
      const int ch = tour::change_of<tour::POS2>(cur.I, X, Xp);
      const uint32_t v = cur.M[0];
      // occupancy: a plain load first; the atomic only the first time
      if (!((pres[v >> 5] >> (v & 31)) & 1u)) atomicOr(&pres[v >> 5], 1u << (v & 31));
      if (ch != 0) {
        if constexpr (PACKED) {
          // the packed table of hist16.cuh: exact out-of-band moves to the
          // per-SM scratch row
          hist16::Upd u;
          hist16::issue(hbase, v, (uint32_t)ch, u);  // 32-bit two's complement
          auto spill = [&](uint32_t key, int val) {
            atomicAdd(&scratch[key], val);
            atomicOr(&spilled[key >> 5], 1u << (key & 31));
          };
          hist16::fix(hbase, u, spill);
        } else {
          atomicAdd(&bins[v], (uint32_t)ch);
        }
      }
      Xp = X;
      cur = next;
    }
  }
  __syncthreads();
  // epilogue: thread t owns bins [t * per, (t + 1) * per)
  const uint32_t per = (nbins + NT - 1) / NT;
  const uint32_t b0 = min(nbins, threadIdx.x * per), b1 = min(nbins, b0 + per);
  auto bin_sum = [&](uint32_t b) -> int {
    if constexpr (PACKED) {
      int s = hist16::half_value(bins[b >> 1], b & 1u);
      if ((spilled[b >> 5] >> (b & 31)) & 1u) s += scratch[b];
      return s;
    } else {
      return (int)bins[b];
    }
  };
  int32_t local = 0;
  for (uint32_t b = b0; b < b1; ++b) local += bin_sum(b);
  using Scan = cub::BlockScan<int32_t, NT>;
  __shared__ typename Scan::TempStorage tmp;
  int32_t ex;
  Scan(tmp).ExclusiveSum(local, ex);
  for (uint32_t b = b0; b < b1; ++b) {
    ex += bin_sum(b);
    row[b] = ex;
  }
  if constexpr (PACKED) {
    __syncthreads();  // all reads of the scratch row are done
    for (uint32_t b = b0; b < b1; ++b)
      if ((spilled[b >> 5] >> (b & 31)) & 1u) scratch[b] = 0;
  }
  for (uint32_t q = threadIdx.x; q < nbins / 32; q += NT) pres_row[q] = pres[q];
}

bool batch16_supported(int h, int w);
cudaError_t launch_batch_u8(const uint8_t* data, uint64_t count, int h, int w, int32_t* chi,
                            uint32_t* presence, cudaStream_t st);
cudaError_t launch_batch16(const uint16_t* data, uint64_t count, int h, int w, int32_t* chi,
                           uint32_t* presence, int32_t* spill_scratch, cudaStream_t st);

cudaError_t launch_batch2d(const void* data, int dtype, uint64_t count, int h, int w,
                           int32_t* chi, uint32_t* presence, int32_t* spill_scratch,
                           cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  if (dtype == 0) {
    // rows of a multiple of 16 bytes: the bit-sliced kernel (k_u8_2d.cu)
    const cudaError_t e = launch_batch_u8(static_cast<const uint8_t*>(data), count, h, w, chi,
                                          presence, st);
    if (e != cudaErrorNotSupported) return e;
    const uint32_t nbins = 256;
    const size_t smem = (nbins + nbins / 32) * 4;
    k_batch2d<uint8_t, false><<<(unsigned)count, NT, smem, st>>>(
        (const uint8_t*)data, h, w, nbins, chi, presence, nullptr);
  } else if (dtype == 1 && batch16_supported(h, w)) {
    return launch_batch16(static_cast<const uint16_t*>(data), count, h, w, chi, presence,
                          spill_scratch, st);
  } else if (dtype == 1) {
    const uint32_t nbins = 65536;
    const size_t smem = (nbins / 2 + 2 * nbins / 32) * 4;
    cudaFuncSetAttribute(k_batch2d<uint16_t, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_batch2d<uint16_t, true><<<(unsigned)count, NT, smem, st>>>(
        (const uint16_t*)data, h, w, nbins, chi, presence, spill_scratch);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace eccb
