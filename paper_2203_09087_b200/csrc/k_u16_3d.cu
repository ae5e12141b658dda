// k_u16_3d.cu -- K1+K2 for 3D volumes with 16-bit keys on sm_100a: the
// bit-sliced tournament of k_u8_3d.cu widened to 16 bit planes, with a
// 65536-bin shared-memory histogram.  Serves u16 volumes directly and
// affine-quantised f32 volumes (BASELINE config 4) after a one-pass
// f32 -> bin-index conversion (the affine map is monotone, so comparing bin
// indices is comparing values -- value_index.hpp:159-197 relies on the same
// order-only dependence, test_kernel.cpp:175-200).
//
// Differences from the u8 kernel (see k_u8_3d.cu for the stencil algebra):
//  * TMA boxes of 40 u16 x 32 rows; a lane funnel-shifts its 32-key window
//    out of five LDS.128 and splits it into low / high bytes, each
//    bit-transposed into 8 planes (planes 0-7 and 8-15).
//  * Only the value planes and the three in-plane "upper side wins" words of
//    the previous plane are carried (19 registers); its block minima are
//    recomputed at the x comparison instead of stored, which keeps the
//    16-plane state inside the register budget of 12 warps per SM.
//  * The per-block carry-save sum (bits::sum_blocks9, as k_u8_3d.cu) gives
//    change + 9; adding 7 mod 16 makes its 4 planes the change in 4-bit two's
//    complement, and replicating the sign plane makes the code transpose
//    produce signed bytes that one PRMT sign-extends.
//  * Histogram: 65536 signed 16-bit halves packed two per word in shared
//    memory, stored as v + 0x1000 (hist16.cuh): an update that leaves its
//    half outside [-4096, 4095] moves the half's current value to the global
//    int64 histogram with a compare-and-swap, so the half is reset to exactly
//    0; the group size keeps the worst-case drift before the first reset
//    below the wrap (hist16.cuh's bound, asserted below).  Occupancy is a
//    65536-bit map.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "bits.cuh"
#include "hist16.cuh"
#include "ecc_common.cuh"
#include "internal.h"

namespace eccb {
namespace u163d {

constexpr int NW = 12;     // warps per CTA (one CTA per SM: the histogram fills shared memory)
constexpr int NS = 2;      // TMA ring stages per warp
constexpr int BOXE = 40;   // box elements along axis 2 (window of 32 + alignment)
constexpr int BOXY = 32;
constexpr int STAGE = BOXE * 2 * BOXY;  // bytes
constexpr int HWORDS = 32768;           // 65536 packed halves
constexpr int PWORDS = 2048;            // 65536 occupancy bits
constexpr int RING_BYTES = NW * NS * STAGE;
constexpr int BAR_BYTES = NW * NS * 8;
constexpr int SMEM_BYTES = RING_BYTES + BAR_BYTES + (HWORDS + PWORDS + 1) * 4;  // + set-bit count
constexpr uint32_t FULL = 0xFFFFFFFFu;
#ifndef ECC_AFF_U
#define ECC_AFF_U 8
#endif
#ifndef ECC_U16_GRP
#define ECC_U16_GRP 10
#endif
constexpr int GRP = ECC_U16_GRP;  // voxels per atomic group (divides 30)
static_assert(30 % GRP == 0, "a group size divides the 30 owned bits");
static_assert(hist16::no_wrap(NW * 32, GRP, 7), "3D changes reach -7: the packed halves could wrap");

struct Geom {
  int W0, W1, W2, plane0, own0, P, Gy, Gz, ncols, seglen, nunits;
  int vc;  // virtual-collar column layout (k_u16_3d<true>)
  uint32_t nbins;
  int rr;  // units < resident warps: dealt round-robin over the CTAs (every SM busy)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  const uint32_t a = smem_u32(bar);
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// Columns as in k_u8_3d.cu: the first / last column along each in-plane
// axis owns 31 rows / bits with a virtual collar (bits.cuh cols).
struct Cursor {
  int u, k, len, x0, ys, ye, zs, ze, yb, zb;  // owned [ys, ye) x [zs, ze); window origin (yb, zb)
  __device__ __forceinline__ void set(const Geom& g) {
    const int seg = u / g.ncols, col = u - seg * g.ncols;
    x0 = g.own0 + seg * g.seglen;
    len = min(g.seglen, g.P - seg * g.seglen);
    const int gy = col / g.Gz, gz = col - gy * g.Gz;
    if (g.vc) {
      ys = cols::start(gy, g.Gy, g.W1);
      ye = cols::start(gy + 1, g.Gy, g.W1);
      zs = cols::start(gz, g.Gz, g.W2);
      ze = cols::start(gz + 1, g.Gz, g.W2);
      yb = ys > 0 ? ys - 1 : 0;
      zb = zs > 0 ? zs - 1 : 0;
    } else {  // every column owns <= 30; the image-edge collar sits in lane 0 / bit 0
      ys = (int)((long long)gy * g.W1 / g.Gy);
      ye = (int)((long long)(gy + 1) * g.W1 / g.Gy);
      zs = (int)((long long)gz * g.W2 / g.Gz);
      ze = (int)((long long)(gz + 1) * g.W2 / g.Gz);
      yb = ys - 1;
      zb = zs - 1;
    }
  }
  __device__ __forceinline__ void start(const Geom& g, int u0) {
    u = u0;
    k = 0;
    if (u < g.nunits) set(g);
  }
  __device__ __forceinline__ bool valid(const Geom& g) const { return u < g.nunits; }
  __device__ __forceinline__ void next(const Geom& g, int nwt) {
    if (++k == len + 2) {
      u += nwt;
      k = 0;
      if (u < g.nunits) set(g);
    }
  }
};

struct Row {
  uint32_t C[16];        // value planes
  uint32_t gz, gy, gyz;  // "upper side wins" of the z / y pairs, yz blocks
  uint32_t W[16];        // the row's 32 keys (two per word, natural order)
};

struct XCarry {
  uint32_t gxa, gxz, gxz1, gxy, gxyu, g8, g81, g8u, g8u1;
};

struct RunGeom {
  int y, o;
  uint32_t zout, vm;
  uint32_t vlo, zf, zl;  // virtual-collar substitutions (k_u8_3d.cu RunGeom)
  bool yout, zlo, edge, b0, b31;
  __device__ __forceinline__ void set(const Geom& g, const Cursor& c, int lane) {
    y = c.yb + lane;
    const int z0 = c.zb;
    o = z0 & 7;  // element offset of the window in the 16-byte aligned box row
    yout = (y < 0) | (y >= g.W1);
    zlo = z0 < 0;  // the layout without virtual collars: bit 0 is the z = -1 collar
    const int hi = g.W2 - z0;
    zout = (hi < 32 ? ~((1u << hi) - 1u) : 0u) | (zlo ? 1u : 0u);
    const int lo_b = c.zs - z0, hi_b = c.ze - z0;  // owned bits [lo_b, hi_b)
    const uint32_t own = (hi_b >= 32 ? FULL : ((1u << hi_b) - 1u)) & (FULL << lo_b);
    vm = (lane >= c.ys - c.yb && lane < c.ye - c.yb) ? own : 0u;
    vlo = (lane == 0 && c.ys == 0) ? FULL : 0u;
    zf = c.zs == 0 ? 1u : 0u;
    zl = z0 + 32 >= g.W2 ? 0x80000000u : 0u;
    b0 = lo_b == 0;
    b31 = hi_b >= 32;
    edge = __any_sync(FULL, yout | (zout != 0));
  }
};

// (x >> 1) + a, a < 2^31 (the z + 1 neighbours; a = the virtual collar bit)
__device__ __forceinline__ uint32_t shr1_add(uint32_t x, uint32_t a) {
  uint32_t d;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(0x80000000u), "r"(a));
  return d;
}

// minima of the previous row's blocks, recomputed from its planes
__device__ __forceinline__ void row_minima(const Row& P, uint32_t zl, uint32_t (&mz)[16],
                                           uint32_t (&my)[16], uint32_t (&myz)[16]) {
  uint32_t t[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) t[i] = shr1_add(P.C[i], zl);
  bits::sel<16>(mz, P.gz, P.C, t);
#pragma unroll
  for (int i = 0; i < 16; ++i) t[i] = __shfl_down_sync(FULL, P.C[i], 1);
  bits::sel<16>(my, P.gy, P.C, t);
#pragma unroll
  for (int i = 0; i < 16; ++i) t[i] = __shfl_down_sync(FULL, mz[i], 1);
  bits::sel<16>(myz, P.gyz, mz, t);
}

template <bool VC, int KIND, class Issue>
__device__ __forceinline__ void sweep_step(const Geom& g, const int X, const RunGeom& rg, int& step,
                                           uint8_t (*myring)[STAGE], uint64_t* myfull,
                                           uint32_t* hwords, uint32_t* pres, int64_t* ghist,
                                           const Cursor& pc, int lane, Row& P, Row& N, XCarry& xc,
                                           Issue& issue) {
  const int slot = step & (NS - 1);
  const uint32_t phase = (uint32_t)((step / NS) & 1);
  mbar_wait(&myfull[slot], phase);
  {
    const uint4* rowp = reinterpret_cast<const uint4*>(myring[slot] + lane * BOXE * 2);
    uint32_t Wd[20];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const uint4 q = rowp[i];
      Wd[4 * i] = q.x; Wd[4 * i + 1] = q.y; Wd[4 * i + 2] = q.z; Wd[4 * i + 3] = q.w;
    }
    const int sh = 16 * (rg.o & 1);
#define ECC_WINDOW16(Q)                                                                    \
  _Pragma("unroll") for (int j = 0; j < 16; ++j) N.W[j] =                                 \
      __funnelshift_r(Wd[(Q) + j], Wd[(Q) + j + 1], sh)
    switch (rg.o >> 1) {
      case 0: ECC_WINDOW16(0); break;
      case 1: ECC_WINDOW16(1); break;
      case 2: ECC_WINDOW16(2); break;
      default: ECC_WINDOW16(3); break;
    }
#undef ECC_WINDOW16
  }
  __syncwarp();
  if (pc.valid(g)) {
    if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    issue(slot);
  }
  uint32_t (&C)[16] = N.C;
  {
    uint32_t lo[8], hi[8], t[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      lo[j] = bits::prmt(N.W[2 * j], N.W[2 * j + 1], 0x6420);
      hi[j] = bits::prmt(N.W[2 * j], N.W[2 * j + 1], 0x7531);
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
  const bool xout = (KIND == 0 ? X < 0 : false) | (X >= g.W0);
  if (rg.edge | xout) {  // collar voxels hold 0xFFFF; see k_u8_3d.cu
    const uint32_t om = (rg.yout | xout) ? FULL : rg.zout;
#pragma unroll
    for (int i = 0; i < 16; ++i) C[i] |= om;
  }
  uint32_t Nmz[16], Nmy[16], Nmyz[16];
  {
    uint32_t t[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i] = shr1_add(C[i], VC ? rg.zl : 0u);
    uint32_t gz = bits::gt<16>(C, t);
    if (!VC && rg.zlo) gz |= 1u;  // z = -1 never wins as the lower side
    bits::sel<16>(Nmz, gz, C, t);
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i] = __shfl_down_sync(FULL, C[i], 1);
    uint32_t gy = bits::gt<16>(C, t);
    if (!VC && rg.y < 0) gy = FULL;  // y = -1 never wins
    bits::sel<16>(Nmy, gy, C, t);
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i] = __shfl_down_sync(FULL, Nmz[i], 1);
    uint32_t gyz = bits::gt<16>(Nmz, t);
    if (!VC && rg.y < 0) gyz = FULL;
    bits::sel<16>(Nmyz, gyz, Nmz, t);
    N.gz = gz;
    N.gy = gy;
    N.gyz = gyz;
  }
  if constexpr (KIND >= 1) {
    uint32_t gxa, gxz, gxy, g8;
    {
      uint32_t Pmz[16], Pmy[16], Pmyz[16];
      row_minima(P, VC ? rg.zl : 0u, Pmz, Pmy, Pmyz);
      gxa = bits::gt<16>(P.C, N.C);
      gxz = bits::gt<16>(Pmz, Nmz);
      gxy = bits::gt<16>(Pmy, Nmy);
      g8 = bits::gt<16>(Pmyz, Nmyz);
    }
    if (KIND == 1 && X - 1 < 0) gxa = gxz = gxy = g8 = FULL;
    // across a virtual collar (k_u8_3d.cu): first columns' bit 0 / lane 0
    const uint32_t zf = VC ? rg.zf : 0u, vlo = VC ? rg.vlo : 0u;
    const uint32_t gxz1 = (gxz << 1) | (gxa & zf), g81 = (g8 << 1) | (gxy & zf);
    const uint32_t gxyu = VC ? bits::bsel(gxa, vlo, __shfl_up_sync(FULL, gxy, 1)) : __shfl_up_sync(FULL, gxy, 1);
    const uint32_t g8u = VC ? bits::bsel(gxz, vlo, __shfl_up_sync(FULL, g8, 1)) : __shfl_up_sync(FULL, g8, 1);
    const uint32_t g8u1 = (g8u << 1) | (gxyu & zf);
    if constexpr (KIND == 2) {
      const uint32_t gyu = __shfl_up_sync(FULL, P.gy, 1) | vlo;
      const uint32_t gyzu = __shfl_up_sync(FULL, P.gyz, 1) | vlo;
      // the nine in-plane blocks of each voxel (k_u8_3d.cu): I_b wins b in
      // the plane, X_b / Xp_b the axis-0 comparisons of b, q_b = 2 h_b + l_b
      const uint32_t Z0 = ~P.gz, Z1 = (P.gz << 1) | zf;
      const uint32_t I[9] = {FULL, Z1, Z0, gyu, ~P.gy, ((P.gz & gyzu) << 1) | (gyu & zf),
                             Z0 & gyzu, ((P.gz & ~P.gyz) << 1) | (~P.gy & zf), Z0 & ~P.gyz};
      const uint32_t Xn[9] = {gxa, gxz1, gxz, gxyu, gxy, g8u1, g8u, g81, g8};
      const uint32_t Xp[9] = {xc.gxa, xc.gxz1, xc.gxz, xc.gxyu, xc.gxy,
                              xc.g8u1, xc.g8u, xc.g81, xc.g8};
      uint32_t h[9], l[9];
#pragma unroll
      for (int b = 0; b < 9; ++b) {
        l[b] = bits::lop3<0x9F>(I[b], Xn[b], Xp[b]);  // ~(I & (X ^ Xp))
        h[b] = (b >= 1 && b <= 4) ? bits::lop3<0x40>(I[b], Xn[b], Xp[b])   // I & X & ~Xp
                                  : bits::lop3<0x20>(I[b], Xn[b], Xp[b]);  // I & ~X & Xp
      }
      // S = change + 9; change = S + 7 mod 16 in 4-bit two's complement
      uint32_t s[4];
      bits::sum_blocks9(h, l, s);
      const uint32_t vm = rg.vm;
      const uint32_t c2 = s[1] | s[0], c3 = s[2] | c2;
      const uint32_t d0 = ~s[0] & vm, d1 = ~(s[1] ^ s[0]) & vm, d2 = ~(s[2] ^ c2) & vm,
                     d3 = (s[3] ^ c3) & vm;  // non-emitted voxels: change 0
      uint32_t V[8] = {d0, d1, d2, d3, d3, d3, d3, d3};
      bits::transpose8(V);  // byte b of V[r] = int8 change of voxel 8b + r
      const uint32_t hbase = smem_u32(hwords), pbase = smem_u32(pres);
      // branch-free per voxel: predicated shared-memory ops (no divergence
      // bookkeeping), the rare out-of-band fix behind a warp vote.  Once
      // every bin's occupancy bit is set (random 16-bit data fills the map
      // early) the occupancy code is skipped for the whole step.
      auto spill = [&](uint32_t key, int after) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&ghist[key]),
                  static_cast<unsigned long long>(static_cast<long long>(after)));
      };
      // one group of NJ voxels p = p0 + j * ps: atomic latencies overlap, one
      // vote per group for the rare out-of-band fix (hist16.cuh)
      auto group = [&](auto with_presence, auto nj_c, const int p0, const int ps) {
        constexpr int NJ = decltype(nj_c)::value;
        {
          hist16::Upd u[NJ];
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            const int p = p0 + j * ps, r = p & 7, b = p >> 3;
            const uint32_t chu =
                bits::prmt(V[r], 0u, b | ((8 | b) << 4) | ((8 | b) << 8) | ((8 | b) << 12));
            const uint32_t key = bits::prmt(P.W[p >> 1], 0u, (p & 1) ? 0x4432 : 0x4410);
            if constexpr (decltype(with_presence)::value) {
              const uint32_t pa = pbase + ((key >> 3) & ~3u);
              const uint32_t bit = 1u << (key & 31);
              uint32_t pw;
              asm volatile("ld.shared.u32 %0, [%1];" : "=r"(pw) : "r"(pa) : "memory");
              const uint32_t need = ((vm >> p) & 1u) & (uint32_t)((pw & bit) == 0);
              uint32_t prev;
              asm volatile(
                  "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\tmov.u32 %0, %3;\n\t"
                  "@q atom.shared.or.b32 %0, [%2], %3;\n\t}"
                  : "=r"(prev)
                  : "r"(need), "r"(pa), "r"(bit)
                  : "memory");
              // count newly set bits so the map's saturation can be detected
              const uint32_t fresh = need & (uint32_t)((prev & bit) == 0);
              asm volatile(
                  "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q red.shared.add.u32 [%1], 1;\n\t}" ::"r"(fresh),
                  "r"(pbase + PWORDS * 4)
                  : "memory");
            }
            hist16::issue(hbase, key, chu, u[j]);
          }
          uint32_t any = 0;
#pragma unroll
          for (int j = 0; j < NJ; ++j) any |= hist16::crossed(u[j]);
          if (__any_sync(FULL, any != 0)) {
#pragma unroll
            for (int j = 0; j < NJ; ++j) hist16::fix(hbase, u[j], spill);
          }
        }
      };
      auto voxels = [&](auto wp) {
#pragma unroll
        for (int g5 = 1; g5 <= 30; g5 += GRP) group(wp, std::integral_constant<int, GRP>{}, g5, 1);
        // bits 0 / 31 are owned only in a first / last column (warp-uniform)
        if constexpr (VC)
          if (rg.b0 | rg.b31) group(wp, std::integral_constant<int, 2>{}, 0, 31);
      };
      uint32_t nset;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(nset) : "r"(pbase + PWORDS * 4) : "memory");
      if (nset >= g.nbins)
        voxels(std::false_type{});
      else
        voxels(std::true_type{});
    }
    xc.gxa = gxa; xc.gxz = gxz; xc.gxz1 = gxz1; xc.gxy = gxy; xc.gxyu = gxyu;
    xc.g8 = g8; xc.g81 = g81; xc.g8u = g8u; xc.g8u1 = g8u1;
  }
  ++step;
}

template <bool VC>
__global__ void __launch_bounds__(NW * 32, 1)
    k_u16_3d(const __grid_constant__ CUtensorMap map, Geom g, int64_t* __restrict__ ghist) {
  extern __shared__ __align__(128) uint8_t dsm[];
  auto ring = reinterpret_cast<uint8_t(*)[NS][STAGE]>(dsm);
  auto full = reinterpret_cast<uint64_t(*)[NS]>(dsm + RING_BYTES);
  uint32_t* hwords = reinterpret_cast<uint32_t*>(dsm + RING_BYTES + BAR_BYTES);
  uint32_t* pres = hwords + HWORDS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t(*myring)[STAGE] = ring[warp];
  uint64_t* myfull = full[warp];
  for (int i = threadIdx.x; i < HWORDS; i += NW * 32) hwords[i] = hist16::BIAS;
  for (int i = threadIdx.x; i <= PWORDS; i += NW * 32) pres[i] = 0;  // bitmap + count
  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&myfull[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nwt = gridDim.x * NW;
  const int gw = g.rr ? warp * (int)gridDim.x + (int)blockIdx.x : (int)blockIdx.x * NW + warp;
  Cursor pc;
  pc.start(g, gw);
  auto issue = [&](int slot) {
    if (lane == 0) {
      const int X = pc.x0 - 1 + pc.k;
      mbar_expect_tx(&myfull[slot], STAGE);
      tma_load3(myring[slot], &map, (pc.zb >> 3) << 3, pc.yb, X - g.plane0,
                &myfull[slot]);
    }
    pc.next(g, nwt);
  };
  for (int s = 0; s < NS && pc.valid(g); ++s) issue(s);
  Row A, B;
  XCarry xc;
  RunGeom rg;
  int step = 0;
  for (int u = gw; u < g.nunits; u += nwt) {
    Cursor cc;
    cc.start(g, u);
    rg.set(g, cc, lane);
    const int x0 = cc.x0, len = cc.len;
    sweep_step<VC, 0>(g, x0 - 1, rg, step, myring, myfull, hwords, pres, ghist, pc, lane, B, A, xc, issue);
    sweep_step<VC, 1>(g, x0, rg, step, myring, myfull, hwords, pres, ghist, pc, lane, A, B, xc, issue);
    int X = x0 + 1;
    for (; X + 1 <= x0 + len; X += 2) {
      sweep_step<VC, 2>(g, X, rg, step, myring, myfull, hwords, pres, ghist, pc, lane, B, A, xc, issue);
      sweep_step<VC, 2>(g, X + 1, rg, step, myring, myfull, hwords, pres, ghist, pc, lane, A, B, xc,
                    issue);
    }
    if (X <= x0 + len)
      sweep_step<VC, 2>(g, X, rg, step, myring, myfull, hwords, pres, ghist, pc, lane, B, A, xc, issue);
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < g.nbins; b += NW * 32) {
    const uint32_t word = hwords[b >> 1];
    const int sum = hist16::half_value(word, b & 1u);
    if (sum != 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(&ghist[b]),
                static_cast<unsigned long long>(static_cast<long long>(sum)));
    if ((pres[b >> 5] >> (b & 31)) & 1u)
      atomicAdd(reinterpret_cast<unsigned long long*>(&ghist[g.nbins + b]), 1ull);
  }
}

// f32 slab -> affine bin indices (u16), same exactness check as the other
// f32 paths (ecc_common.cuh:affine_bin): off-grid values raise kFlagBinmap,
// NaN raises kFlagNaN.
__global__ void k_affine_keys(const float* __restrict__ v, uint64_t rows, uint32_t w2,
                              uint32_t pitch, AffineMap am, uint16_t* __restrict__ keys,
                              uint32_t* flags) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  if (pitch == w2 && (w2 & 3) == 0) {
    // contiguous rows: a flat grid-stride over float4 groups, ECC_AFF_U (8)
    // loads in flight per thread (measured 1.08 ms at 8, 1.14 at 4, 1.30 at 2
    // for C4's 4.3 GB read + 2.1 GB written: 90 % of HBM)
    const uint64_t n4 = rows * w2 / 4;
    const float4* src = reinterpret_cast<const float4*>(v);
    uint2* dst = reinterpret_cast<uint2*>(keys);
    constexpr int U = ECC_AFF_U;
    uint64_t i = tid;
    for (; i + (U - 1) * nthreads < n4; i += U * nthreads) {
      float4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) x[u] = __ldcs(src + i + u * nthreads);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t k0 = affine_bin(am, x[u].x, flags), k1 = affine_bin(am, x[u].y, flags);
        const uint32_t k2 = affine_bin(am, x[u].z, flags), k3 = affine_bin(am, x[u].w, flags);
        dst[i + u * nthreads] = make_uint2(k0 | (k1 << 16), k2 | (k3 << 16));
      }
    }
    for (; i < n4; i += nthreads) {
      const float4 x = __ldcs(src + i);
      const uint32_t k0 = affine_bin(am, x.x, flags), k1 = affine_bin(am, x.y, flags);
      const uint32_t k2 = affine_bin(am, x.z, flags), k3 = affine_bin(am, x.w, flags);
      dst[i] = make_uint2(k0 | (k1 << 16), k2 | (k3 << 16));
    }
    return;
  }
  // padded key rows: one warp per row at a time, coalesced reads of w2
  // floats, writes of w2 keys
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = tid >> 5;
  const uint64_t nwarps = nthreads >> 5;
  const bool vec = (w2 & 3) == 0 && (pitch & 3) == 0;
  for (uint64_t r = warp; r < rows; r += nwarps) {
    const float* src = v + r * w2;
    uint16_t* dst = keys + r * pitch;
    if (vec) {
      for (uint32_t c = 4 * lane; c < w2; c += 128) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(src + c));
        const uint32_t k0 = affine_bin(am, x.x, flags), k1 = affine_bin(am, x.y, flags);
        const uint32_t k2 = affine_bin(am, x.z, flags), k3 = affine_bin(am, x.w, flags);
        *reinterpret_cast<uint2*>(dst + c) = make_uint2(k0 | (k1 << 16), k2 | (k3 << 16));
      }
    } else {
      for (uint32_t c = lane; c < w2; c += 32) dst[c] = (uint16_t)affine_bin(am, __ldg(src + c), flags);
    }
  }
}

}  // namespace u163d

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode16() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}
}  // namespace

// Number of axis-0 segments: minimises the modelled time of the persistent
// grid, max units per warp x (segment length + 2 halo planes).
long long best_segments(long long ncols, long long P, long long cap_warps) {
  long long best = 1;
  double best_cost = 1e300;
  for (long long n = 1; n <= std::max<long long>(1, P / 4); ++n) {  // segments >= 4 planes
    const long long len = (P + n - 1) / n;
    const long long units = ((P + len - 1) / len) * ncols;
    const long long per_warp = (units + cap_warps - 1) / cap_warps;
    const double cost = (double)per_warp * (double)(len + 2);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = (P + len - 1) / len;
    }
  }
  return best;
}

bool u16_3d_supported(const Slab& s) {
  return s.w2 > 1 && (s.row_pitch() * 2) % 16 == 0 &&
         (reinterpret_cast<uintptr_t>(s.base) % 16) == 0 && s.w1 <= (1 << 30) &&
         s.w2 <= (1 << 30) && s.w0 <= (1 << 30);
}

cudaError_t launch_affine_keys(const float* v, uint64_t rows, uint32_t w2, uint32_t pitch,
                               const AffineMap& am, uint16_t* keys, uint32_t* flags, int sms,
                               cudaStream_t st) {
  u163d::k_affine_keys<<<sms * 8, 256, 0, st>>>(v, rows, w2, pitch, am, keys, flags);
  return cudaGetLastError();
}

cudaError_t launch_u16_3d(const Slab& s, uint32_t nbins, int64_t* ghist, int sms,
                          cudaStream_t st) {
  using namespace u163d;
  auto enc = encode16();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap map;
  const cuuint64_t dims[3] = {(cuuint64_t)s.w2, (cuuint64_t)s.w1, (cuuint64_t)s.nplanes};
  const cuuint64_t strides[2] = {(cuuint64_t)s.row_pitch() * 2,
                                 (cuuint64_t)(s.w1 * s.row_pitch() * 2)};
  const cuuint32_t box[3] = {BOXE, BOXY, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void*>(s.base), dims, strides, box,
          es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  Geom g;
  g.W0 = (int)s.w0;
  g.W1 = (int)s.w1;
  g.W2 = (int)s.w2;
  g.plane0 = (int)s.plane0;
  g.own0 = (int)s.own0;
  g.P = (int)(s.own1 - s.own0);
  // The virtual-collar layout (first / last columns own 31) only where it
  // saves columns (512: 17 instead of 18 per axis; 1024: 35 either way) --
  // its substitutions cost registers, so C4's 1024^3 keeps the plain layout.
  {
    const int vy = cols::groups(g.W1), vz = cols::groups(g.W2);
    const int py = (g.W1 + 29) / 30, pz = (g.W2 + 29) / 30;
    g.vc = (long long)vy * vz < (long long)py * pz;
    g.Gy = g.vc ? vy : py;
    g.Gz = g.vc ? vz : pz;
  }
  g.ncols = g.Gy * g.Gz;
  g.nbins = nbins;
  smem_optin<k_u16_3d<false>>(SMEM_BYTES);
  smem_optin<k_u16_3d<true>>(SMEM_BYTES);
  const long long cap_warps = (long long)sms * NW;
  const long long nseg = best_segments(g.ncols, g.P, cap_warps);
  g.seglen = (int)((g.P + nseg - 1) / nseg);
  const long long units = nseg * g.ncols;
  if (units > (1ll << 30)) return cudaErrorInvalidValue;
  g.nunits = (int)units;
  // fewer units than resident warps: one unit per warp on as many SMs as
  // possible (a small volume is latency-bound)
  g.rr = units < cap_warps;
  const long long grid = g.rr ? std::min<long long>(units, sms)
                              : std::min<long long>((units + NW - 1) / NW, sms);
  if (g.vc)
    k_u16_3d<true><<<(unsigned)grid, NW * 32, SMEM_BYTES, st>>>(map, g, ghist);
  else
    k_u16_3d<false><<<(unsigned)grid, NW * 32, SMEM_BYTES, st>>>(map, g, ghist);
  return cudaGetLastError();
}

}  // namespace eccb
