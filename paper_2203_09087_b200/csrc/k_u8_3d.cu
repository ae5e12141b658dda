// k_u8_3d.cu -- K1+K2 for 3D u8 volumes on sm_100a: bit-sliced tournament
// stencil + per-CTA (code, value) shared-memory histogram, TMA-fed.
//
// Replaces, for u8 3D images, the reference hot loop
//   run_chunk_kernel_u8 (streaming.hpp:146-174)
//     -> accumulate_dense_u8 (kernel.hpp:268-277)
//     -> for_each_change / change_3d (kernel.hpp:99-137, 193-216)
// and produces the same per-value change sums (plus per-value voxel counts
// for the occurrence list, value_index.hpp:63-71) bit-exactly.
//
// Mapping.  A warp owns a "column": 32 rows along axis 1 (one per lane) x
// 32 voxels along axis 2 (one per bit of a bit plane) and sweeps a segment
// of axis 0.  Lane 0 / 31 and bit 0 / 31 are halo, so an interior column
// yields up to 30 x 30 voxels per plane; the first / last column along an
// axis owns 31 there, its collar lane / bit being virtual (bits.cuh cols,
// the substitutions in sweep_step).  Work units are (segment, column) pairs in
// segment-major order: warps that run at the same time hold neighbouring
// columns at the same axis-0 position, so the halo rows/bytes a column
// shares with its neighbours are read from DRAM once and hit in L2 after.
// Each plane of a column arrives by one TMA box (48 B x 32 rows; the box
// origin along axis 2 must be 16-byte aligned) into a per-warp ring; a lane
// reads its 48-byte row with three LDS.128 and funnel-shifts out its
// 32-byte window, byte-interleaves and bit-transposes it into 8 bit planes.
//
// Stencil (validated by tools/tournament_model.py).  With ties going to
// the earlier voxel (kernel.hpp:21-27), a voxel introduces a face / edge /
// vertex iff it is the minimum of the 2 / 4 / 8 voxels around it, so the
// change is  -1 + #2-blocks won - #4-blocks won + #8-blocks won.  Block
// winners come from a tournament: 7 bit-sliced comparisons (z, y, yz in the
// plane; x, xz, xy, xyz against the next plane) and 3 bit-sliced minimum
// selections per voxel.  Each of the voxel's nine in-plane blocks b (the
// voxel, 4 pairs, 4 yz 4-blocks) contributes s_b I_b (X_b - Xp_b) -- I_b:
// the voxel wins b in its plane; X_b / Xp_b: the next / this plane's copy of
// b wins the axis-0 comparison (tourney.cuh derives it) -- entered as
// q_b = 1 + that in {0, 1, 2} = 2 h_b + l_b with two LOP3s; the 18 bit
// vectors go through a 12-full-adder carry-save tree (bits::sum_blocks9)
// giving code = change + 9 in [2, 14] per voxel.
//
// Histogram (K2).  The 4 code planes are transposed back to bytes and each
// voxel does ONE shared-memory atomic increment at hist[code][value] (one
// PRMT builds the index from the value byte and the code byte); the table
// (16 x 256 x u32 per CTA) is reduced to per-value change sums and counts
// once at the end and flushed with int64 global atomics.  Voxels the lane
// does not own go to code 15, which no real change produces.
//
// Collar.  Voxels outside the image hold 255 in the planes; that is only
// wrong when an outside voxel is the EARLIER side of a comparison (the
// reference's sentinel 256 must lose), and those comparisons are forced to
// "later wins" (z = -1, y = -1, x = -1), see tools/tournament_model.py.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <algorithm>
#include <cstdint>

#include <cub/cub.cuh>

#include "bits.cuh"
#include "ecc_common.cuh"
#include "fin_u8.cuh"
#include "internal.h"

namespace eccb {
namespace u83d {
using u8fin::flush_and_finalize;

#ifndef ECC_U83D_NW
#define ECC_U83D_NW 16
#endif
constexpr int NW = ECC_U83D_NW;  // warps per CTA
#ifndef ECC_U83D_NS
#define ECC_U83D_NS 2
#endif
constexpr int NS = ECC_U83D_NS;  // TMA ring stages per warp (a power of two)
#ifndef ECC_U83D_PB
#define ECC_U83D_PB 2
#endif
constexpr int PB = ECC_U83D_PB;  // planes per TMA box (1 or 2): one wait + one refill per box
constexpr int BOXZ = 48;   // box bytes along axis 2 (window of 32 + alignment)
constexpr int BOXY = 32;   // rows per box (one per lane)
constexpr int PLANE_BYTES = BOXZ * BOXY;
constexpr int STAGE = PLANE_BYTES * PB;
constexpr int NCODE = 16;
#ifndef ECC_U83D_HREP
#define ECC_U83D_HREP 4
#endif
constexpr int HREP = ECC_U83D_HREP;  // histogram replicas (one per 32 / HREP lanes: fewer bank conflicts)
constexpr int HIST_WORDS = NCODE * 256 * HREP;
constexpr int RING_BYTES = NW * NS * STAGE;
constexpr int BAR_BYTES = NW * NS * 8;
constexpr int SMEM_BYTES = RING_BYTES + BAR_BYTES + HIST_WORDS * 4;
#ifndef ECC_U83D_CTAS
#define ECC_U83D_CTAS 1
#endif
constexpr int CTAS_PER_SM = ECC_U83D_CTAS;
constexpr uint32_t FULL = 0xFFFFFFFFu;

struct Geom {
  int W0, W1, W2;  // image dims
  int plane0;      // image plane held at tensor-map coordinate 0
  int own0;        // first owned plane
  int P;           // owned planes
  int Gy, Gz;      // column groups along axes 1 and 2
  int ncols;       // Gy * Gz
  int seglen;      // planes per segment
  int nunits;      // ncols * segments
  int8_t* chg;     // CH mode: per-voxel changes of the owned planes (compute_changes)
  uint32_t four;   // = 4, opaque to ptxas so the histogram address stays an IMAD
  int rr;          // units < resident warps: dealt round-robin over the CTAs (every SM busy)
};

// Fused K3 (optional, fin_u8.cuh): the last CTA to finish turns the global
// histogram into the curve.
using u8fin::Fin;

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

// Position of one warp in its sequence of work units (unit u = gw + i *
// nwt, segment-major) and of the plane step k in [0, len + 2) within it
// (one halo plane on each side along axis 0); the producer moves a box of
// PB planes at a time.
struct Cursor {
  int u, k, len, x0, ys, ye, zs, ze, yb, zb;  // owned [ys, ye) x [zs, ze); window origin (yb, zb)
  __device__ __forceinline__ void set(const Geom& g) {
    const int seg = u / g.ncols, col = u - seg * g.ncols;
    x0 = g.own0 + seg * g.seglen;
    len = min(g.seglen, g.P - seg * g.seglen);
    const int gy = col / g.Gz, gz = col - gy * g.Gz;
    ys = cols::start(gy, g.Gy, g.W1);
    ye = cols::start(gy + 1, g.Gy, g.W1);
    zs = cols::start(gz, g.Gz, g.W2);
    ze = cols::start(gz + 1, g.Gz, g.W2);
    yb = ys > 0 ? ys - 1 : 0;  // the first column starts at the image edge (virtual collar)
    zb = zs > 0 ? zs - 1 : 0;
  }
  __device__ __forceinline__ void start(const Geom& g, int u0) {
    u = u0;
    k = 0;
    if (u < g.nunits) set(g);
  }
  __device__ __forceinline__ bool valid(const Geom& g) const { return u < g.nunits; }
  __device__ __forceinline__ void next(const Geom& g, int nwt) {
    k += PB;
    if (k >= len + 2) {
      u += nwt;
      k = 0;
      if (u < g.nunits) set(g);
    }
  }
};

// Carried state of one row of a column (plane X-1 while plane X arrives).
struct Row {
  uint32_t C[8], mz[8], my[8], myz[8];  // value planes and z / y / yz block minima
  uint32_t gz, gy, gyz;                 // "upper side wins" bits of the z / y pairs, yz blocks
  uint32_t W[8];                        // the row's 32 value bytes (natural order)
};

// x-comparison results between planes X-2 and X-1 ("X-1 wins" bits).
struct XCarry {
  uint32_t gxa, gxz, gxz1, gxy, gxyu, g8, g81, g8u, g8u1;
  __device__ __forceinline__ void clear() { gxa = gxz = gxz1 = gxy = gxyu = g8 = g81 = g8u = g8u1 = 0; }
};

// Per-unit constants of this lane.
struct RunGeom {
  int y;          // this lane's row
  int o;          // byte offset of the window in the 16-byte aligned box row
  uint32_t zout;  // bits whose voxel lies outside [0, W2)
  uint32_t vm;    // bits whose change this lane emits (0 for halo lanes)
  uint32_t vlo;   // FULL on lane 0 of a first column: its y - 1 neighbour is the virtual collar
  uint32_t zf;    // 1 in a first column: bit 0's z - 1 neighbour is the virtual collar
  uint32_t zl;    // bit 31 in a last column: bit 31's z + 1 neighbour is the virtual collar
  bool yout;      // this lane's row lies outside [0, W1)
  bool edge;      // some lane of the column holds collar voxels (warp-uniform)
  bool b0, b31;   // bit 0 / bit 31 owned (first / last columns; warp-uniform)
  __device__ __forceinline__ void set(const Geom& g, const Cursor& c, int lane) {
    y = c.yb + lane;
    const int z0 = c.zb;
    o = z0 & 15;
    yout = y >= g.W1;
    const int hi = g.W2 - z0;   // one past the last in-image bit
    zout = hi < 32 ? ~((1u << hi) - 1u) : 0u;
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

__device__ __forceinline__ int decode_change(uint32_t code) { return (int)code - 9; }

// code = change + 9 in [2, 14]; 15 = not emitted
struct Codes {
  static constexpr int n = NCODE;
  static __device__ __forceinline__ bool live(int c) { return c != 15; }
  static __device__ __forceinline__ int change(int c) { return decode_change((uint32_t)c); }
};

// One plane step of a column: plane X arrives as row N, row P holds plane
// X-1.  KIND 0: the unit's first (halo) plane, tournament only; KIND 1: +
// x comparisons against P (P may be the x = -1 collar); KIND 2: + the
// changes of P (X-1 is an owned plane).
template <bool CH, int KIND, int SUB, bool RELEASE, class Issue>
__device__ __forceinline__ void sweep_step(const Geom& g, const int X, const int zs,
                                           const RunGeom& rg, uint32_t& step,
                                           uint8_t (*myring)[STAGE], uint64_t* myfull,
                                           const uint32_t hist_s, const Cursor& pc, int lane,
                                           Row& P, Row& N, XCarry& xc, Issue& issue) {
  // `step` counts boxes: plane SUB of the box in ring slot step % NS
  const uint32_t slot = step & (NS - 1);
  const uint32_t phase = (step / NS) & 1u;
  if (SUB == 0) mbar_wait(&myfull[slot], phase);
  {
    const uint4* rowp =
        reinterpret_cast<const uint4*>(myring[slot] + SUB * PLANE_BYTES + lane * BOXZ);
    const uint4 q0 = rowp[0], q1 = rowp[1], q2 = rowp[2];
    const uint32_t Wd[12] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w,
                             q2.x, q2.y, q2.z, q2.w};
    // the 32-voxel window starts at byte o (warp-uniform) of the row
    const int sh = 8 * (rg.o & 3);
#define ECC_WINDOW(Q)                                                        \
  _Pragma("unroll") for (int j = 0; j < 8; ++j) N.W[j] = __funnelshift_r(Wd[(Q) + j], Wd[(Q) + j + 1], sh)
    switch (rg.o >> 2) {
      case 0: ECC_WINDOW(0); break;
      case 1: ECC_WINDOW(1); break;
      case 2: ECC_WINDOW(2); break;
      default: ECC_WINDOW(3); break;
    }
#undef ECC_WINDOW
  }
  __syncwarp();
  // after the box's last plane: refill this slot with the box NS ahead.
  // Every lane has consumed its LDS results (the funnel shifts above) before
  // the __syncwarp, so the async-proxy write cannot overtake a generic read.
  if (RELEASE) {
    if (pc.valid(g)) issue(slot);
    ++step;
  }
  uint32_t (&C)[8] = N.C;
  bits::byte_interleave(N.W, C);
  bits::transpose8(C);
  // collar: voxels outside the image hold 255 (TMA filled zeros)
  const bool xout = (KIND == 0 ? X < 0 : false) | (X >= g.W0);
  if (rg.edge | xout) {  // warp-uniform: only columns / planes touching the collar
    const uint32_t om = (rg.yout | xout) ? FULL : rg.zout;
#pragma unroll
    for (int i = 0; i < 8; ++i) C[i] |= om;
  }

  // ---- tournament on the new row (plane X)
  {
    uint32_t Cz[8], Cy[8], mzy[8];
#pragma unroll
    // z + 1 neighbours; in a last column bit 31's is the virtual collar
    // (key 255 in every plane: it never wins as the later side)
    for (int i = 0; i < 8; ++i) Cz[i] = bits::shr1_add(C[i], rg.zl);
    const uint32_t gz = bits::gt<8>(C, Cz);
    bits::sel<8>(N.mz, gz, C, Cz);
#pragma unroll
    for (int i = 0; i < 8; ++i) Cy[i] = __shfl_down_sync(FULL, C[i], 1);
    // (lane 31 of a last column reads itself: "y + 1 never wins", the
    // virtual collar's outcome)
    const uint32_t gy = bits::gt<8>(C, Cy);
    bits::sel<8>(N.my, gy, C, Cy);
#pragma unroll
    for (int i = 0; i < 8; ++i) mzy[i] = __shfl_down_sync(FULL, N.mz[i], 1);
    const uint32_t gyz = bits::gt<8>(N.mz, mzy);
    bits::sel<8>(N.myz, gyz, N.mz, mzy);
    N.gz = gz;
    N.gy = gy;
    N.gyz = gyz;
  }

  if constexpr (KIND >= 1) {
    // ---- x comparisons between planes X-1 (P) and X (N): "X wins" bits
    uint32_t gxa = bits::gt<8>(P.C, N.C);
    uint32_t gxz = bits::gt<8>(P.mz, N.mz);
    uint32_t gxy = bits::gt<8>(P.my, N.my);
    uint32_t g8 = bits::gt<8>(P.myz, N.myz);
    if (KIND == 1 && X - 1 < 0) gxa = gxz = gxy = g8 = FULL;  // x = -1 never wins
    // z - 1 / y - 1 neighbours' outcomes; across a virtual collar (first
    // columns: bit 0, lane 0) a block with the collar has the in-image
    // part's minimum, so its x outcome is that part's
    const uint32_t gxz1 = bits::shl1_add(gxz, gxa & rg.zf), g81 = bits::shl1_add(g8, gxy & rg.zf);
    const uint32_t gxyu = bits::bsel(gxa, rg.vlo, __shfl_up_sync(FULL, gxy, 1));
    const uint32_t g8u = bits::bsel(gxz, rg.vlo, __shfl_up_sync(FULL, g8, 1));
    const uint32_t g8u1 = bits::shl1_add(g8u, gxyu & rg.zf);
    if constexpr (KIND == 2) {
      // ---- changes of row X-1: each voxel gathers its 26 block wins
      // the virtual y = -1 collar never wins: v wins its pair / quads with it
      const uint32_t gyu = __shfl_up_sync(FULL, P.gy, 1) | rg.vlo;
      const uint32_t gyzu = __shfl_up_sync(FULL, P.gyz, 1) | rg.vlo;
      // the nine in-plane blocks b of each voxel and I_b = "wins b inside
      // the plane": 0 the voxel, 1 / 2 its z- / z+ pair, 3 / 4 its y- / y+
      // pair, 5..8 the yz 4-blocks (y-,z-) (y-,z+) (y+,z-) (y+,z+)
      // (bit 0 of a first column: the z - 1 pair with the virtual collar is
      // won by v, and a quad with it reduces to v's y pair)
      const uint32_t Z0 = ~P.gz, Z1 = bits::shl1_add(P.gz, rg.zf);
      const uint32_t I[9] = {FULL,
                             Z1,
                             Z0,
                             gyu,
                             ~P.gy,
                             bits::shl1_add(P.gz & gyzu, gyu & rg.zf),
                             Z0 & gyzu,
                             bits::shl1_add(P.gz & ~P.gyz, ~P.gy & rg.zf),
                             Z0 & ~P.gyz};
      // X_b: the next plane's copy of b beats this plane's; Xp_b the same
      // one step earlier (the previous plane against this one)
      const uint32_t Xn[9] = {gxa, gxz1, gxz, gxyu, gxy, g8u1, g8u, g81, g8};
      const uint32_t Xp[9] = {xc.gxa, xc.gxz1, xc.gxz, xc.gxyu, xc.gxy,
                              xc.g8u1, xc.g8u, xc.g81, xc.g8};
      // q_b = 1 + s_b I_b (X_b - Xp_b) in {0, 1, 2} as 2 h_b + l_b (signs:
      // pairs +1, the voxel and the 4-blocks -1); change + 9 = sum_b q_b
      uint32_t h[9], l[9];
#pragma unroll
      for (int b = 0; b < 9; ++b) {
        l[b] = bits::lop3<0x9F>(I[b], Xn[b], Xp[b]);  // ~(I & (X ^ Xp))
        h[b] = (b >= 1 && b <= 4) ? bits::lop3<0x40>(I[b], Xn[b], Xp[b])   // I & X & ~Xp
                                  : bits::lop3<0x20>(I[b], Xn[b], Xp[b]);  // I & ~X & Xp
      }
      // S = change + 9 in [2, 14]; code = S mod 16; not emitted -> 15
      uint32_t s[4];
      bits::sum_blocks9(h, l, s);
      const uint32_t vm = rg.vm;
      uint32_t V[8];
      bits::transpose_codes(s[0] | ~vm, s[1] | ~vm, s[2] | ~vm, s[3] | ~vm, V);
      if constexpr (CH) {
#pragma unroll
        for (int p = 0; p <= 31; ++p) {
          const int r = p & 7, b = p >> 3;
          const uint32_t idx = bits::prmt(P.W[p >> 2], V[r],
                                          (p & 3) | ((4 + b) << 4) | ((0xC + b) << 8) | ((0xC + b) << 12));
          if ((vm >> p) & 1) {
            const long long row = (long long)(X - 1 - g.own0) * g.W1 + rg.y;
            const long long vox = row * g.W2 + (long long)(zs + p);
            g.chg[vox] = (int8_t)decode_change(idx >> 8);
          }
        }
      } else {
        // one shared-memory increment per voxel at hist[code][value]; the
        // address (hist + 4 * idx) is an IMAD on the FMA pipe rather than an
        // ALU-pipe LEA (the integer ALU pipe is this kernel's bottleneck).
        // (Predicating the halo lanes' atomics off through grouped asm was
        // measured slower: 161 vs 141 us, the grouping serialises the
        // address computation.)
        auto bump = [&](int p) {
          const int r = p & 7, b = p >> 3;
          const uint32_t idx = bits::prmt(P.W[p >> 2], V[r],
                                          (p & 3) | ((4 + b) << 4) | ((0xC + b) << 8) | ((0xC + b) << 12));
          uint32_t addr;
          asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(addr) : "r"(idx), "r"(g.four), "r"(hist_s));
          asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
        };
#pragma unroll
        for (int p = 1; p <= 30; ++p) bump(p);
        // bits 0 / 31 are owned only in a first / last column (warp-uniform)
        if (rg.b0) bump(0);
        if (rg.b31) bump(31);

      }
    }
    xc.gxa = gxa; xc.gxz = gxz; xc.gxz1 = gxz1; xc.gxy = gxy; xc.gxyu = gxyu;
    xc.g8 = g8; xc.g81 = g81; xc.g8u = g8u; xc.g8u1 = g8u1;
  }
}

template <bool CH>
__global__ void __launch_bounds__(NW * 32, CTAS_PER_SM)
    k_u8_3d(const __grid_constant__ CUtensorMap map, Geom g, int64_t* __restrict__ ghist, Fin fin) {
  extern __shared__ __align__(128) uint8_t dsm[];
  auto ring = reinterpret_cast<uint8_t(*)[NS][STAGE]>(dsm);              // [NW][NS][STAGE]
  auto full = reinterpret_cast<uint64_t(*)[NS]>(dsm + RING_BYTES);       // [NW][NS]
  uint32_t* hist = reinterpret_cast<uint32_t*>(dsm + RING_BYTES + BAR_BYTES);  // [NCODE][256]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t(*myring)[STAGE] = ring[warp];
  uint64_t* myfull = full[warp];

  if (!CH)
    for (int i = threadIdx.x; i < HIST_WORDS; i += NW * 32) hist[i] = 0;
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
      const int X = pc.x0 - 1 + pc.k;  // image plane
      mbar_expect_tx(&myfull[slot], STAGE);
      // TMA needs the axis-2 box origin on a 16-byte boundary
      tma_load3(myring[slot], &map, (pc.zb >> 4) << 4, pc.yb, X - g.plane0, &myfull[slot]);
    }
    pc.next(g, nwt);
  };
  for (int s = 0; s < NS && pc.valid(g); ++s) issue(s);

  Row A, B;
  XCarry xc;
  RunGeom rg;
  uint32_t step = 0;
  // this lane's replica of the table: entry e at word e * HREP + replica
  const uint32_t hist_s = smem_u32(hist) + (uint32_t)((lane * HREP) >> 5) * 4u;
  for (int u = gw; u < g.nunits; u += nwt) {
    Cursor cc;
    cc.start(g, u);
    rg.set(g, cc, lane);
    const int x0 = cc.x0, zs = cc.zb, len = cc.len;  // zs: the window's first bit
    // unit planes k = 0 .. len+1 (X = x0-1+k); box b holds planes 2b, 2b+1
    // when PB == 2, one plane per box when PB == 1
    constexpr int S1 = PB == 2 ? 1 : 0;
    constexpr bool R0 = PB == 1;
    sweep_step<CH, 0, 0, R0>(g, x0 - 1, zs, rg, step, myring, myfull, hist_s, pc, lane, B, A, xc, issue);
    sweep_step<CH, 1, S1, true>(g, x0, zs, rg, step, myring, myfull, hist_s, pc, lane, A, B, xc, issue);
    // planes x0+1 .. x0+len: the changes of x0 .. x0+len-1
    int X = x0 + 1;
    for (; X + 1 <= x0 + len; X += 2) {
      sweep_step<CH, 2, 0, R0>(g, X, zs, rg, step, myring, myfull, hist_s, pc, lane, B, A, xc, issue);
      sweep_step<CH, 2, S1, true>(g, X + 1, zs, rg, step, myring, myfull, hist_s, pc, lane, A, B, xc, issue);
    }
    if (X <= x0 + len)  // odd plane count: the last box's second plane is unused
      sweep_step<CH, 2, 0, true>(g, X, zs, rg, step, myring, myfull, hist_s, pc, lane, B, A, xc, issue);
  }
  if constexpr (!CH) flush_and_finalize<NW * 32, Codes, HREP>(hist, ghist, fin);
}

}  // namespace u83d

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// Shape gate for the fast path: 3D, axis-2 rows a multiple of 16 bytes (TMA
// stride rule), 16-byte aligned slab base, and per-CTA voxel counts that fit
// the 32-bit shared counters.
bool u8_3d_supported(const Slab& s) {
  return s.w2 > 1 && s.row_pitch() % 16 == 0 && (reinterpret_cast<uintptr_t>(s.base) % 16) == 0 &&
         s.w1 <= (1 << 30) && s.w2 <= (1 << 30) && s.w0 <= (1 << 30) &&
         (s.own1 - s.own0) * s.w1 * s.w2 < (1ll << 40);
}

cudaError_t launch_u8_3d(const Slab& s, int64_t* ghist, int8_t* chg, int sms, cudaStream_t st,
                         const U83dFinalize* fz) {
  using namespace u83d;
  // the tensor map of the last slab is cached per host thread (encoding it
  // is host work on every call otherwise)
  thread_local struct {
    const void* base = nullptr;
    int64_t w1 = 0, w2 = 0, np = 0, pitch = 0;
    CUtensorMap map;
  } cache;
  if (cache.base != s.base || cache.w1 != s.w1 || cache.w2 != s.w2 || cache.np != s.nplanes ||
      cache.pitch != s.row_pitch()) {
    auto enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    const cuuint64_t dims[3] = {(cuuint64_t)s.w2, (cuuint64_t)s.w1, (cuuint64_t)s.nplanes};
    const cuuint64_t strides[2] = {(cuuint64_t)s.row_pitch(), (cuuint64_t)(s.w1 * s.row_pitch())};
    const cuuint32_t box[3] = {BOXZ, BOXY, PB};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&cache.map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(s.base), dims,
                     strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      cache.base = nullptr;
      return cudaErrorInvalidValue;
    }
    cache.base = s.base;
    cache.w1 = s.w1;
    cache.w2 = s.w2;
    cache.np = s.nplanes;
    cache.pitch = s.row_pitch();
  }
  const CUtensorMap& map = cache.map;
  Geom g;
  g.W0 = (int)s.w0;
  g.W1 = (int)s.w1;
  g.W2 = (int)s.w2;
  g.plane0 = (int)s.plane0;
  g.own0 = (int)s.own0;
  g.P = (int)(s.own1 - s.own0);
  g.Gy = cols::groups(g.W1);
  g.Gz = cols::groups(g.W2);
  g.ncols = g.Gy * g.Gz;
  g.chg = chg;
  g.four = 4 * HREP;
  smem_optin<k_u8_3d<false>>(SMEM_BYTES);
  smem_optin<k_u8_3d<true>>(SMEM_BYTES);
  static int per_sm = -1;  // same on every B200
  if (per_sm < 0) {
    int v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_u8_3d<false>, NW * 32, SMEM_BYTES) !=
            cudaSuccess ||
        v < 1)
      v = 1;
    per_sm = v;
  }
  const long long cap_warps = (long long)sms * per_sm * NW;
  // Segments along axis 0: one wave of (segment, column) units when the
  // columns alone under-fill the GPU, else ~8 units per resident warp.
  long long nseg;
  if (g.ncols <= cap_warps)
    nseg = std::max<long long>(1, cap_warps / g.ncols);
  else
    nseg = (8 * cap_warps + g.ncols - 1) / g.ncols;
#ifndef ECC_U83D_MINSEG
#define ECC_U83D_MINSEG 4
#endif
  nseg = std::min<long long>(nseg, std::max(1, g.P / ECC_U83D_MINSEG));  // segments of >= MINSEG planes
  g.seglen = (int)((g.P + nseg - 1) / nseg);
  nseg = (g.P + g.seglen - 1) / g.seglen;
  const long long units = nseg * g.ncols;
  if (units > (1ll << 30)) return cudaErrorInvalidValue;
  g.nunits = (int)units;
#ifndef ECC_U83D_RR
#define ECC_U83D_RR 1
#endif
  // fewer units than resident warps: one unit per warp on as many SMs as
  // possible (a small volume is latency-bound: a few warps per SM step faster)
  g.rr = ECC_U83D_RR && units < cap_warps;
  const long long grid = g.rr ? std::min<long long>(units, cap_warps / NW)
                              : std::min<long long>((units + NW - 1) / NW, cap_warps / NW);
  Fin fin{};
  if (fz) {
    fin = Fin{fz->ticket, fz->bins, fz->changes, fz->chi, fz->count};
    fin.x = u8fin::Xchg{fz->world, fz->rank, fz->epoch, fz->slots, fz->flags, fz->my_slots,
                        fz->my_flags, fz->err};
  }
  if (chg)
    k_u8_3d<true><<<(unsigned)grid, NW * 32, SMEM_BYTES, st>>>(map, g, ghist, fin);
  else
    k_u8_3d<false><<<(unsigned)grid, NW * 32, SMEM_BYTES, st>>>(map, g, ghist, fin);
  return cudaGetLastError();
}

}  // namespace eccb
