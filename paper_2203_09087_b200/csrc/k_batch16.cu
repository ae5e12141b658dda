// k_batch16.cu -- batched 2D ECC for u16 images (BASELINE config 3), bit
// sliced.  One CTA per image; the image's 65536-bin histogram lives in
// shared memory (packed biased 16-bit halves with exact spills, as in
// k_u16_3d.cu) and the epilogue writes the dense chi row + occupancy bitmap.
//
// Mapping.  A lane owns a 32-pixel chunk of a row (bit p = pixel 32c + p
// along axis 1) and sweeps a band of rows (axis 0); the L lanes of a band
// hold the row's consecutive chunks, so a pixel's axis-1 neighbour across a
// chunk boundary arrives by a warp shuffle (funnel shift) -- no halo bits.
// Per row the lane bit-transposes its 32 keys into 16 planes, then, with the
// tie rule of change_2d (kernel.hpp:81-94; ties go to the earlier pixel):
//   pairs along axis 1: gz = [c(p) > c(p+1)], pair minimum mz;
//   pairs along axis 0: gx = [P(p) > N(p)] between consecutive rows;
//   2 x 2 quads: gq = [mz of row X-1 > mz of row X];
// and a pixel of row X-1 changes chi by 1 + #quads won - #pairs won
// (range [-3, 1]).  The 8 win bits go through a small
// carry-save adder; the result minus 3 is the change in 4-bit two's
// complement, transposed back to signed bytes for the histogram.
#include <type_traits>

#include "bits.cuh"
#include "hist16.cuh"
#include "ecc_common.cuh"
#include "internal.h"

namespace eccb {
namespace b16 {

#ifndef ECC_B16_NW
#define ECC_B16_NW 16
#endif
constexpr int NW = ECC_B16_NW;  // warps per CTA
constexpr int NT = NW * 32;
constexpr int HWORDS = 32768, PWORDS = 2048;
constexpr uint32_t FULL = 0xFFFFFFFFu;
#ifndef ECC_HGRP
#define ECC_HGRP 16  // (8 in round 1; 16 measured 1.71 vs 1.72 ms once the band test got cheaper)
#endif
constexpr int HGRP = ECC_HGRP;  // pixels per atomic group (divides 32)
#ifndef ECC_B16_ASYNC
#define ECC_B16_ASYNC 1
#endif
static_assert(hist16::no_wrap(NT, HGRP, 3), "2D changes reach -3: the packed halves could wrap");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// 32 keys (two per word, natural order) -> 16 bit planes
__device__ __forceinline__ void planes16(const uint32_t (&W)[16], uint32_t (&C)[16]) {
  uint32_t lo[8], hi[8], t[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    lo[j] = bits::prmt(W[2 * j], W[2 * j + 1], 0x6420);
    hi[j] = bits::prmt(W[2 * j], W[2 * j + 1], 0x7531);
  }
  bits::byte_interleave(lo, t);
  bits::transpose8(t);
#pragma unroll
  for (int i = 0; i < 8; ++i) C[i] = t[i];
  bits::byte_interleave(hi, t);
  bits::transpose8(t);
#pragma unroll
  for (int i = 0; i < 8; ++i) C[8 + i] = t[i];
}

struct Row {
  uint32_t C[16], mz[16];
  uint32_t gz;
  uint32_t W[16];
};

__global__ void __launch_bounds__(NT, 1)
    k_batch16(const uint16_t* __restrict__ data, int h, int w, int L, int32_t* __restrict__ chi,
              uint32_t* __restrict__ presence, int32_t* __restrict__ spill_scratch) {
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* hw = sm;                    // packed halves
  uint32_t* pres = hw + HWORDS;         // occupancy bits
  uint32_t* spilled = pres + PWORDS;    // bins with a spilled partial in `scratch`
  {  // 16-byte stores (the table is 128 KB: 16 per thread)
    const uint4 bias = make_uint4(hist16::BIAS, hist16::BIAS, hist16::BIAS, hist16::BIAS);
    for (int i = threadIdx.x; i < HWORDS / 4; i += NT) reinterpret_cast<uint4*>(hw)[i] = bias;
    for (int i = threadIdx.x; i < 2 * PWORDS / 4; i += NT)
      reinterpret_cast<uint4*>(pres)[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  const uint16_t* img = data + (size_t)blockIdx.x * h * w;
  int32_t* scratch = spill_scratch + (size_t)smid() * 65536;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nchunks = (w + 31) / 32;
  const int bpw = 32 / L;                       // bands per warp
  const int nbands = NW * bpw;
  const int band = warp * bpw + lane / L, c = lane % L;
  // every band runs the same number of row steps (warp-wide shuffles stay
  // converged); rows past the image are collar and emit nothing
  const int rows = (h + nbands - 1) / nbands;
  const int R0 = band * rows;
  // pixels of this chunk outside [0, w) (all of them for dummy lanes)
  const int lo = 32 * c;
  uint32_t zout = FULL;
  if (c < nchunks) zout = (w - lo >= 32) ? 0u : (FULL << (w - lo));
  const uint32_t vm = ~zout;
  const bool first = c == 0, last = c == nchunks - 1;
  const bool vec = (w & 7) == 0;
  const uint32_t hbase = smem_u32(hw), pbase = smem_u32(pres);

#if ECC_B16_ASYNC
  // the next row is staged in shared memory by cp.async (no registers held
  // for it across the step): two slots per thread, slot = row parity
  uint32_t* stage = spilled + PWORDS;  // [2][NT][16] words
  auto issue_row = [&](int i) {
    uint32_t* dst = stage + ((i & 1) * NT + threadIdx.x) * 16;
    if (i < 0 || i >= h || c >= nchunks) {
#pragma unroll
      for (int q = 0; q < 4; ++q) reinterpret_cast<uint4*>(dst)[q] = make_uint4(FULL, FULL, FULL, FULL);
    } else {
      const uint16_t* p = img + (size_t)i * w + lo;
      if (vec && w - lo >= 32) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + 4 * q)),
                       "l"(p + 8 * q)
                       : "memory");
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t a = (lo + 2 * j < w) ? __ldg(p + 2 * j) : 0xFFFFu;
          const uint32_t b = (lo + 2 * j + 1 < w) ? __ldg(p + 2 * j + 1) : 0xFFFFu;
          dst[j] = a | (b << 16);
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto take_row = [&](int i, uint32_t (&W)[16]) {
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // row i landed, row i + 1 in flight
    const uint4* src = reinterpret_cast<const uint4*>(stage + ((i & 1) * NT + threadIdx.x) * 16);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 v = src[q];
      W[4 * q] = v.x; W[4 * q + 1] = v.y; W[4 * q + 2] = v.z; W[4 * q + 3] = v.w;
    }
  };
  Row A, B;
  uint32_t xgx = 0, xgq = 0, xgq1 = 0;  // previous row pair's results
  issue_row(R0 - 1);
  // steps: rows R0-1 .. R0+rows arrive; at the arrival of row X the changes
  // of row X-1 are emitted (X-1 in [R0, R0 + rows) and inside the image)
  auto step = [&](int X, Row& P, Row& N, auto kind) {
    constexpr int K = decltype(kind)::value;  // 0 first, 1 no emission, 2 emit
    issue_row(X + 1);  // prefetch (collar past the band's last row + 1 is harmless)
    take_row(X, N.W);
#else
  auto load_row = [&](int i, uint32_t (&W)[16]) {
    if (i < 0 || i >= h || c >= nchunks) {
#pragma unroll
      for (int j = 0; j < 16; ++j) W[j] = FULL;
      return;
    }
    const uint16_t* p = img + (size_t)i * w + lo;
    if (vec && w - lo >= 32) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(p) + q);
        W[4 * q] = v.x; W[4 * q + 1] = v.y; W[4 * q + 2] = v.z; W[4 * q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t a = (lo + 2 * j < w) ? __ldg(p + 2 * j) : 0xFFFFu;
        const uint32_t b = (lo + 2 * j + 1 < w) ? __ldg(p + 2 * j + 1) : 0xFFFFu;
        W[j] = a | (b << 16);
      }
    }
  };

  Row A, B;
  uint32_t xgx = 0, xgq = 0, xgq1 = 0;  // previous row pair's results
  uint32_t nxt[16];
  load_row(R0 - 1, nxt);
  // steps: rows R0-1 .. R0+rows arrive; at the arrival of row X the changes
  // of row X-1 are emitted (X-1 in [R0, R0 + rows) and inside the image)
  auto step = [&](int X, Row& P, Row& N, auto kind) {
    constexpr int K = decltype(kind)::value;  // 0 first, 1 no emission, 2 emit
#pragma unroll
    for (int j = 0; j < 16; ++j) N.W[j] = nxt[j];
    load_row(X + 1, nxt);  // prefetch (collar past the band's last row + 1 is harmless)
#endif
    planes16(N.W, N.C);
    const bool xout = X < 0 || X >= h;
    const uint32_t om = xout ? FULL : zout;
#pragma unroll
    for (int i = 0; i < 16; ++i) N.C[i] |= om;
    {
      uint32_t t[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        uint32_t nb = __shfl_down_sync(FULL, N.C[i], 1, L);
        if (last) nb = FULL;  // right collar (later side: loses every tie)
        t[i] = __funnelshift_r(N.C[i], nb, 1);
      }
      N.gz = bits::gt<16>(N.C, t);
      bits::sel<16>(N.mz, N.gz, N.C, t);
    }
    if constexpr (K >= 1) {
      uint32_t gx = bits::gt<16>(P.C, N.C);
      uint32_t gq = bits::gt<16>(P.mz, N.mz);
      if (X - 1 < 0) gx = gq = FULL;  // row -1 never wins
      // quad anchored one pixel to the left: from the previous chunk, or for
      // the first chunk the quad over the left collar, whose minima are the
      // pixels at 0 -- its comparison is gx bit 0
      uint32_t qprev = __shfl_up_sync(FULL, gq, 1, L);
      if (first) qprev = gx << 31;
      const uint32_t gq1 = __funnelshift_l(qprev, gq, 1);
      if constexpr (K == 2) {
        uint32_t zprev = __shfl_up_sync(FULL, P.gz, 1, L);
        if (first) zprev = FULL;  // the left collar never wins
        const uint32_t Z0 = ~P.gz;
        const uint32_t Z1 = __funnelshift_l(zprev, P.gz, 1);
        // S = 4 quads won + 4 negated pairs won = change + 3
        const uint32_t t0 = Z0 & ~gq, t1 = Z0 & xgq, t2 = Z1 & ~gq1, t3 = Z1 & xgq1;
        const uint32_t t4 = ~Z0, t5 = ~Z1, t6 = gx, t7 = ~xgx;
        uint32_t s0, c0, s1, c1, s2, c2;
        bits::fa3(t0, t1, t2, s0, c0);
        bits::fa3(t3, t4, t5, s1, c1);
        bits::fa3(t6, t7, s0, s2, c2);
        const uint32_t b0 = s1 ^ s2, k0 = s1 & s2;             // weight 1
        uint32_t b1, k1;
        bits::fa3(c0, c1, c2, b1, k1);                         // weight 2
        const uint32_t b1x = b1 ^ k0, k1x = b1 & k0;
        const uint32_t b2 = k1 ^ k1x;                          // weight 4 (S <= 4)
        // d = S - 3 (mod 16), 4-bit two's complement, masked to owned pixels
        // S - 3 = S + 13: add 1101b
        const uint32_t d0 = ~b0;                               // b0 + 1
        const uint32_t cy1 = b0;
        const uint32_t d1 = b1x ^ cy1;                         // + 0
        const uint32_t cy2 = b1x & cy1;
        const uint32_t d2 = ~(b2 ^ cy2);                       // + 1
        const uint32_t cy3 = b2 | cy2;
        const uint32_t d3 = ~cy3;                              // + 1 (no carry out needed)
        const uint32_t vmr = (X - 1 < h) ? vm : 0u;
        uint32_t V[8] = {d0 & vmr, d1 & vmr, d2 & vmr, d3 & vmr, d3 & vmr, d3 & vmr, d3 & vmr, d3 & vmr};
        bits::transpose8(V);
        // histogram: groups of HGRP pixels (atomic latencies overlap), one vote
        // per group for the rare out-of-band fix
        auto spill = [&](uint32_t key, int after) {
          atomicAdd(&scratch[key], after);
          atomicOr(&spilled[key >> 5], 1u << (key & 31));
        };
        // every pixel of the chunk owned (the common case: whole rows inside
        // the image) -> the occupancy bit needs no per-pixel ownership test
        auto pixels = [&](auto all_owned) {
#pragma unroll
          for (int g4 = 0; g4 < 32; g4 += HGRP) {
            hist16::Upd u[HGRP];
#pragma unroll
            for (int j = 0; j < HGRP; ++j) {
              const int p = g4 + j, r = p & 7, b = p >> 3;
              const uint32_t chu =
                  bits::prmt(V[r], 0u, b | ((8 | b) << 4) | ((8 | b) << 8) | ((8 | b) << 12));
              // (the key and the shifted change built with IMADs instead of
              // PRMT / SHF measured slower, 1.78 / 1.81 ms vs 1.73: the FMA
              // pipe and issue slots, not the ALU, bound this loop now)
              const uint32_t key = bits::prmt(P.W[p >> 1], 0u, (p & 1) ? 0x4432 : 0x4410);
              hist16::mark(pbase, key, decltype(all_owned)::value ? 1u : bits::bit_fma(vmr, p));
              hist16::issue(hbase, key, chu, u[j]);
            }
            uint32_t any = 0;
#pragma unroll
            for (int j = 0; j < HGRP; ++j) any |= hist16::crossed(u[j]);
            if (__any_sync(FULL, any != 0)) {
#pragma unroll
              for (int j = 0; j < HGRP; ++j) hist16::fix(hbase, u[j], spill);
            }
          }
        };
        if (__all_sync(FULL, vmr == FULL))
          pixels(std::true_type{});
        else
          pixels(std::false_type{});
      }
      xgx = gx;
      xgq = gq;
      xgq1 = gq1;
    }
  };
  step(R0 - 1, B, A, std::integral_constant<int, 0>{});
  step(R0, A, B, std::integral_constant<int, 1>{});
  int X = R0 + 1;
  for (; X + 1 <= R0 + rows; X += 2) {
    step(X, B, A, std::integral_constant<int, 2>{});
    step(X + 1, A, B, std::integral_constant<int, 2>{});
  }
  if (X <= R0 + rows) step(X, B, A, std::integral_constant<int, 2>{});
  __syncthreads();
  // epilogue, conflict-free: warp w owns a contiguous run of 256-bin chunks
  // (16 for 16 warps); lane l holds 8 consecutive bins of a chunk (one
  // 16-byte shared load, the chunk's spill bits one broadcast word).  Pass 1
  // sums the warp's bins, pass 2 scans chunk by chunk and writes chi
  // coalesced (two 16-byte stores per lane).
  const uint32_t c0 = (uint32_t)warp * 256u / NW, c1 = (uint32_t)(warp + 1) * 256u / NW;
  int32_t* row = chi + (size_t)blockIdx.x * 65536;
  auto sums8 = [&](uint32_t b, int (&x)[8]) {  // b % 8 == 0
    const uint4 w4 = *reinterpret_cast<const uint4*>(hw + (b >> 1));
    x[0] = hist16::lo_value(w4.x);
    x[1] = hist16::hi_value(w4.x);
    x[2] = hist16::lo_value(w4.y);
    x[3] = hist16::hi_value(w4.y);
    x[4] = hist16::lo_value(w4.z);
    x[5] = hist16::hi_value(w4.z);
    x[6] = hist16::lo_value(w4.w);
    x[7] = hist16::hi_value(w4.w);
    const uint32_t sp = (spilled[b >> 5] >> (b & 31)) & 0xFFu;
    if (sp) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if ((sp >> k) & 1u) x[k] += scratch[b + k];
    }
  };
  __shared__ int32_t wsum[NW];
  const uint32_t wb = 8u * lane;
  int32_t part = 0;
  for (uint32_t i = c0 * 256u; i < c1 * 256u; i += 256) {
    // lo + hi of a word without unpacking: t = w - BIAS = hi * 65536 + lo
    // exactly, hi = (t + 32768) >> 16 (arithmetic), so lo + hi = t - 65535 hi
    // (tests/cpp/test_bits.cpp checks the identity; 1.635 vs 1.644 ms for C3)
    const uint32_t b = wb + i;
    const uint4 w4 = *reinterpret_cast<const uint4*>(hw + (b >> 1));
    const uint32_t ws[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = (int)(ws[q] - hist16::BIAS);
      part += t - 65535 * ((t + 32768) >> 16);
    }
    const uint32_t sp = (spilled[b >> 5] >> (b & 31)) & 0xFFu;
    if (sp) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if ((sp >> k) & 1u) part += scratch[b + k];
    }
  }
  part = __reduce_add_sync(FULL, part);
  if (lane == 0) wsum[warp] = part;
  __syncthreads();
  int32_t carry = 0;
  for (int j = 0; j < warp; ++j) carry += wsum[j];
  for (uint32_t i = c0 * 256u; i < c1 * 256u; i += 256) {
    int x[8];
    sums8(wb + i, x);
#pragma unroll
    for (int k = 1; k < 8; ++k) x[k] += x[k - 1];
    int t = x[7];  // inclusive scan of the lane totals
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, t, o);
      if (lane >= o) t += y;
    }
    const int base = carry + t - x[7];
    int4* dst = reinterpret_cast<int4*>(row + wb + i);
    dst[0] = make_int4(base + x[0], base + x[1], base + x[2], base + x[3]);
    dst[1] = make_int4(base + x[4], base + x[5], base + x[6], base + x[7]);
    carry += __shfl_sync(FULL, t, 31);
  }
  __syncthreads();  // every read of the scratch row is done
  for (int q = threadIdx.x; q < PWORDS; q += NT) {
    uint32_t m = spilled[q];
    while (m) {
      const int bit = __ffs(m) - 1;
      m &= m - 1;
      scratch[q * 32 + bit] = 0;
    }
  }
  uint32_t* pres_row = presence + (size_t)blockIdx.x * PWORDS;
  for (int q = threadIdx.x; q < PWORDS; q += NT) pres_row[q] = pres[q];
}

}  // namespace b16

bool batch16_supported(int h, int w) { return w >= 1 && w <= 1024 && h >= 1; }

cudaError_t launch_batch16(const uint16_t* data, uint64_t count, int h, int w, int32_t* chi,
                           uint32_t* presence, int32_t* spill_scratch, cudaStream_t st) {
  using namespace b16;
  if (count == 0) return cudaSuccess;
  int L = 1;
  while (L < (w + 31) / 32) L <<= 1;
  const size_t smem = (size_t)(HWORDS + 2 * PWORDS + (ECC_B16_ASYNC ? 2 * NT * 16 : 0)) * 4;
  smem_optin<k_batch16>((int)smem);
  k_batch16<<<(unsigned)count, NT, smem, st>>>(data, h, w, L, chi, presence, spill_scratch);
  return cudaGetLastError();
}

}  // namespace eccb
