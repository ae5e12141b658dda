// k_u16_2d.cu -- K1+K2 for single 2D images with 16-bit keys (u16 images,
// affine-quantised f32 images after k_affine_keys) on sm_100a.
//
// Replaces, for those images, the reference hot loop
//   accumulate_chunk / build_index_counts over change_2d
//   (kernel.hpp:81-94, 229-239; value_index.hpp:159-197)
// and produces the same per-bin change sums and occupancy bit-exactly.
//
// The mapping is k_u8_2d.cu's (a warp holds 32 consecutive 32-pixel chunks
// of a row, lanes 0 / 31 halo, and sweeps a band of rows; units are (band,
// strip) pairs, band-major), the stencil is k_batch16.cu's 16-plane form,
// and the histogram is the packed 65536-bin shared-memory table of
// hist16.cuh (one CTA per SM): out-of-band spills go straight to the global
// int64 histogram, occupancy is a shared bitmap, and each CTA flushes its
// table once at the end (sums to ghist[b], one count per CTA to
// ghist[nbins + b] for occupied bins).
#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "bits.cuh"
#include "ecc_common.cuh"
#include "hist16.cuh"
#include "internal.h"

namespace eccb {
namespace u162d {

#ifndef ECC_U162D_NW
#define ECC_U162D_NW 16
#endif
constexpr int NW = ECC_U162D_NW;  // warps per CTA (one CTA per SM: the table fills shared memory)
constexpr int NT = NW * 32;
constexpr int HWORDS = 32768, PWORDS = 2048;
constexpr int SMEM_BYTES = (HWORDS + PWORDS) * 4;
constexpr int STRIP = 30;
constexpr uint32_t FULL = 0xFFFFFFFFu;
#ifndef ECC_HGRP
#define ECC_HGRP 8
#endif
constexpr int HGRP = ECC_HGRP;  // pixels per atomic group (divides 32)
static_assert(hist16::no_wrap(NT, HGRP, 3), "2D changes reach -3: the packed halves could wrap");

struct Geom {
  const uint16_t* base;  // row plane0 of the slab
  long long pitch;       // elements between rows (multiple of 8)
  int W0, W1, plane0, nheld, own0, P, nchunks, nstrips, band, nunits;
  uint32_t nbins;
};

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

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__global__ void __launch_bounds__(NT, 1)
    k_u16_2d(const Geom g, int64_t* __restrict__ ghist) {
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* hw = sm;              // packed biased halves
  uint32_t* pres = hw + HWORDS;   // occupancy bits
  for (int i = threadIdx.x; i < HWORDS; i += NT) hw[i] = hist16::BIAS;
  for (int i = threadIdx.x; i < PWORDS; i += NT) pres[i] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwt = gridDim.x * NW;
  const uint32_t hbase = smem_u32(hw), pbase = smem_u32(pres);
  auto spill = [&](uint32_t key, int after) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&ghist[key]),
              static_cast<unsigned long long>(static_cast<long long>(after)));
  };

  // units dealt round-robin over the CTAs: a small image spreads over every
  // SM (a few warps each) instead of filling a few SMs' 16 warps
  for (int u = warp * gridDim.x + blockIdx.x; u < g.nunits; u += nwt) {
    const int bi = u / g.nstrips, strip = u - bi * g.nstrips;
    const int R0 = g.own0 + bi * g.band;
    const int rows = min(g.band, g.own0 + g.P - R0);
    const int c = strip * STRIP - 1 + lane;
    const int lo = 32 * c;
    const bool chunk_in = c >= 0 && c < g.nchunks;
    uint32_t zout = FULL;
    if (chunk_in) zout = (g.W1 - lo >= 32) ? 0u : (FULL << (g.W1 - lo));
    const uint32_t vm = (lane >= 1 && lane <= STRIP) ? ~zout : 0u;
    const bool first = c == 0;
    const int nq = chunk_in ? min(4, (g.W1 - lo + 7) / 8) : 0;  // 16-byte groups holding pixels

    auto load_row = [&](int i, uint32_t (&W)[16]) {
      // rows outside the image are collar; rows outside the held range are
      // only the prefetch past a band's halo row (never used)
      if (i < 0 || i >= g.W0 || i < g.plane0 || i >= g.plane0 + g.nheld || !chunk_in) {
#pragma unroll
        for (int j = 0; j < 16; ++j) W[j] = FULL;
        return;
      }
      const uint16_t* p = g.base + (long long)(i - g.plane0) * g.pitch + lo;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q < nq) {
          const uint4 v = ldg_stream(p + 8 * q);
          W[4 * q] = v.x; W[4 * q + 1] = v.y; W[4 * q + 2] = v.z; W[4 * q + 3] = v.w;
        } else {
          W[4 * q] = W[4 * q + 1] = W[4 * q + 2] = W[4 * q + 3] = FULL;
        }
      }
    };

    Row A, B;
    uint32_t xgx = 0, xgq = 0, xgq1 = 0;
    uint32_t nxt[16];
    load_row(R0 - 1, nxt);
    auto step = [&](int X, Row& P, Row& N, auto kind) {
      constexpr int K = decltype(kind)::value;  // 0 first, 1 no emission, 2 emit
#pragma unroll
      for (int j = 0; j < 16; ++j) N.W[j] = nxt[j];
      load_row(X + 1, nxt);
      planes16(N.W, N.C);
      const uint32_t om = (X < 0 || X >= g.W0) ? FULL : zout;
#pragma unroll
      for (int i = 0; i < 16; ++i) N.C[i] |= om;
      {
        uint32_t t[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          t[i] = __funnelshift_r(N.C[i], __shfl_down_sync(FULL, N.C[i], 1), 1);
        N.gz = bits::gt<16>(N.C, t);
        bits::sel<16>(N.mz, N.gz, N.C, t);
      }
      if constexpr (K >= 1) {
        uint32_t gx = bits::gt<16>(P.C, N.C);
        uint32_t gq = bits::gt<16>(P.mz, N.mz);
        if (X - 1 < 0) gx = gq = FULL;  // row -1 never wins
        uint32_t qprev = __shfl_up_sync(FULL, gq, 1);
        if (first) qprev = gx << 31;    // the quad over the left collar
        const uint32_t gq1 = __funnelshift_l(qprev, gq, 1);
        if constexpr (K == 2) {
          uint32_t zprev = __shfl_up_sync(FULL, P.gz, 1);
          if (first) zprev = FULL;      // column -1 never wins
          const uint32_t vmr = (X - 1 < g.W0) ? vm : 0u;
          const uint32_t Z0 = ~P.gz;
          const uint32_t Z1 = __funnelshift_l(zprev, P.gz, 1);
          // S = 4 quads won + 4 negated pairs won = change + 3 (k_batch16.cu)
          const uint32_t t0 = Z0 & ~gq, t1 = Z0 & xgq, t2 = Z1 & ~gq1, t3 = Z1 & xgq1;
          const uint32_t t4 = ~Z0, t5 = ~Z1, t6 = gx, t7 = ~xgx;
          uint32_t s0, c0, s1, c1, s2, c2;
          bits::fa3(t0, t1, t2, s0, c0);
          bits::fa3(t3, t4, t5, s1, c1);
          bits::fa3(t6, t7, s0, s2, c2);
          const uint32_t b0 = s1 ^ s2, k0 = s1 & s2;
          uint32_t b1, k1;
          bits::fa3(c0, c1, c2, b1, k1);
          const uint32_t b1x = b1 ^ k0, k1x = b1 & k0;
          const uint32_t b2 = k1 ^ k1x;
          // d = S - 3 (mod 16) in 4-bit two's complement, 0 where not emitted
          const uint32_t d0 = ~b0;
          const uint32_t d1 = b1x ^ b0;
          const uint32_t cy2 = b1x & b0;
          const uint32_t d2 = ~(b2 ^ cy2);
          const uint32_t d3 = ~(b2 | cy2);
          uint32_t V[8] = {d0 & vmr, d1 & vmr, d2 & vmr, d3 & vmr,
                           d3 & vmr, d3 & vmr, d3 & vmr, d3 & vmr};
          bits::transpose8(V);
#pragma unroll
          for (int g4 = 0; g4 < 32; g4 += HGRP) {
            hist16::Upd up[HGRP];
#pragma unroll
            for (int j = 0; j < HGRP; ++j) {
              const int p = g4 + j, r = p & 7, b = p >> 3;
              const uint32_t chu =
                  bits::prmt(V[r], 0u, b | ((8 | b) << 4) | ((8 | b) << 8) | ((8 | b) << 12));
              const uint32_t key = bits::prmt(P.W[p >> 1], 0u, (p & 1) ? 0x4432 : 0x4410);
              hist16::mark(pbase, key, bits::bit_fma(vmr, p));  // (vmr >> p) & 1 on the FMA pipe
              hist16::issue(hbase, key, chu, up[j]);
            }
            uint32_t any = 0;
#pragma unroll
            for (int j = 0; j < HGRP; ++j) any |= hist16::crossed(up[j]);
            if (__any_sync(FULL, any != 0)) {
#pragma unroll
              for (int j = 0; j < HGRP; ++j) hist16::fix(hbase, up[j], spill);
            }
          }
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
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < g.nbins; b += NT) {
    const int sum = hist16::half_value(hw[b >> 1], b & 1u);
    if (sum != 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(&ghist[b]),
                static_cast<unsigned long long>(static_cast<long long>(sum)));
    if ((pres[b >> 5] >> (b & 31)) & 1u)
      atomicAdd(reinterpret_cast<unsigned long long*>(&ghist[g.nbins + b]), 1ull);
  }
}

}  // namespace u162d

bool u16_2d_supported(const Slab& s) {
  return s.w2 == 1 && s.w1 >= 1 && s.plane_pitch() % 8 == 0 &&
         (reinterpret_cast<uintptr_t>(s.base) % 16) == 0 && s.w0 < (1ll << 31) &&
         s.w1 < (1ll << 31) - 64;
}

cudaError_t launch_u16_2d(const Slab& s, uint32_t nbins, int64_t* ghist, int sms,
                          cudaStream_t st) {
  using namespace u162d;
  Geom g;
  g.base = static_cast<const uint16_t*>(s.base);
  g.pitch = s.plane_pitch();
  g.W0 = (int)s.w0;
  g.W1 = (int)s.w1;
  g.plane0 = (int)s.plane0;
  g.nheld = (int)s.nplanes;
  g.own0 = (int)s.own0;
  g.P = (int)(s.own1 - s.own0);
  g.nchunks = (g.W1 + 31) / 32;
  g.nstrips = (g.nchunks + STRIP - 1) / STRIP;
  g.nbins = nbins;
  if (g.P <= 0) return cudaErrorInvalidValue;
  const long long cap_warps = (long long)sms * NW;
  // bands of >= 32 rows (2 halo rows each), ~4 units per resident warp when
  // the image is large, else one wave of shorter bands (>= MINBAND rows: a
  // small image is latency-bound, so more, shorter bands finish sooner)
#ifndef ECC_U162D_MINBAND
#define ECC_U162D_MINBAND 2
#endif
  const long long nb = std::max<long long>(1, (4 * cap_warps) / g.nstrips);
  long long band = std::max<long long>(32, (g.P + nb - 1) / nb);
  if ((g.P + band - 1) / band * g.nstrips < cap_warps)
    band = std::max<long long>(ECC_U162D_MINBAND, ((long long)g.P * g.nstrips + cap_warps - 1) / cap_warps);
  band = std::max<long long>(1, std::min<long long>(band, g.P));
  g.band = (int)band;
  const long long units = (g.P + band - 1) / band * g.nstrips;
  if (units > (1ll << 30)) return cudaErrorInvalidValue;
  g.nunits = (int)units;
  smem_optin<k_u16_2d>(SMEM_BYTES);
  const long long grid = std::min<long long>(units, sms);
  k_u16_2d<<<(unsigned)grid, NT, SMEM_BYTES, st>>>(g, ghist);
  return cudaGetLastError();
}

}  // namespace eccb
