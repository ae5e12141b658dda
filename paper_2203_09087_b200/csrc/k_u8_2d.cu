// k_u8_2d.cu -- K1+K2 for single 2D u8 images (w2 == 1) on sm_100a:
// bit-sliced stencil + per-CTA (code, value) shared-memory histogram, with
// the optional fused K3 of fin_u8.cuh (the whole curve in one launch).
//
// Replaces, for 2D u8 images, the reference hot loop
//   run_chunk_kernel_u8 (streaming.hpp:146-174)
//     -> accumulate_dense_u8 (kernel.hpp:268-277)
//     -> for_each_change / change_2d (kernel.hpp:81-94, 193-216)
// and produces the same per-value change sums and pixel counts bit-exactly.
//
// Mapping.  Rows run along axis 0, pixels of a row along axis 1.  A lane
// owns a 32-pixel chunk of a row (bit p = pixel 32c + p) and a warp holds 32
// consecutive chunks of the same row; lanes 0 and 31 are halo, so a warp
// "strip" is 30 chunks (960 pixels) wide.  Rows of at most 16 chunks are
// packed instead (PACK): L lanes per whole row, 32 / L rows per warp.  A work unit is (band of rows,
// strip), band-major, so warps running together read neighbouring strips of
// the same rows and the halo chunks / rows hit in L2.  The warp sweeps its
// band row by row (one row prefetched ahead, two 16-byte loads per lane).
//
// Stencil (the 2D form of the tournament in k_u8_3d.cu, as in
// k_batch16.cu).  Ties go to the earlier pixel (kernel.hpp:21-27):
//   pairs along axis 1: gz = [c(p) > c(p+1)], pair minimum mz;
//   pairs along axis 0: gx = [P(p) > N(p)] between consecutive rows;
//   2 x 2 quads:        gq = [mz of row X-1 > mz of row X];
// a pixel of row X-1 changes chi by 1 + #quads won - #pairs won, range
// [-3, 1].  S = change + 3 (8 win bits through a small carry-save adder) is
// the code; the three code planes are transposed back to bytes and every
// pixel does ONE shared-memory red at hist[code][value].  Pixels the lane
// does not emit get code 7.
//
// Collar.  Pixels outside the image hold 255; only an outside pixel on the
// EARLIER side of a comparison is wrong (the reference's sentinel 256 must
// lose), and those comparisons are forced: row -1 never wins (gx = gq =
// FULL), column -1 never wins (the first chunk's left pair / quad).
#include <algorithm>
#include <cstdint>

#include "bits.cuh"
#include "ecc_common.cuh"
#include "fin_u8.cuh"
#include "internal.h"

namespace eccb {
namespace u82d {

#ifndef ECC_U82D_NW
#define ECC_U82D_NW 16
#endif
#ifndef ECC_U82D_CTAS
#define ECC_U82D_CTAS 1
#endif
#ifndef ECC_U82D_HREP
#define ECC_U82D_HREP 4
#endif
constexpr int NW = ECC_U82D_NW;  // warps per CTA
constexpr int NT = NW * 32;
constexpr int NCODE = 8;         // S = change + 3 in [0, 4]; 7 = not emitted
constexpr int HREP = ECC_U82D_HREP;  // table replicas, one per 32 / HREP lanes (bank spread)
constexpr int HIST_WORDS = NCODE * 256 * HREP;
constexpr int CTAS_PER_SM = ECC_U82D_CTAS;
constexpr int STRIP = 30;  // owned chunks per warp
constexpr uint32_t FULL = 0xFFFFFFFFu;

struct Geom {
  const uint8_t* base;  // row plane0 of the slab
  long long pitch;      // bytes between rows (multiple of 16)
  int W0, W1;           // image rows, pixels per row
  int plane0;           // image row held at base
  int nheld;            // rows held from plane0 (a streamed slab holds only its halo'd range)
  int own0, P;          // first owned row, owned rows
  int nchunks;          // 32-pixel chunks per row
  int nstrips;          // warps across a row
  int band;             // rows per unit
  int nunits;           // bands * nstrips (strips); ceil(bands / G) (packed rows)
  int L, G;             // packed rows: lanes per row (a power of two >= nchunks), rows per warp
  uint32_t four;        // = 4, opaque to ptxas (IMAD address, not an ALU LEA)
  long long img_stride;  // BATCH: bytes between images (image blockIdx.y)
  int32_t* chi;          // BATCH: dense rows [count][256]
  uint32_t* pres;        // BATCH: occupancy bitmaps [count][8]
};

#ifndef ECC_U82D_MINBAND
#define ECC_U82D_MINBAND 1
#endif
constexpr int MINBAND = ECC_U82D_MINBAND;  // shortest band of rows a warp sweeps

struct Codes {
  static constexpr int n = 5;  // S = change + 3 in [0, 4]
  static __device__ __forceinline__ bool live(int) { return true; }
  static __device__ __forceinline__ int change(int c) { return c - 3; }
};

struct Row {
  uint32_t C[8], mz[8];  // value planes, axis-1 pair minima
  uint32_t gz;           // "right pixel wins" bits of the axis-1 pairs
  uint32_t W[8];         // the chunk's 32 value bytes (natural order)
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

// PACK: rows of at most 16 chunks are packed G = 32 / L to a warp (L lanes
// per row, no halo lanes: the whole row is in the warp), each lane group
// sweeping its own band; otherwise a warp holds a strip of 30 chunks of one
// row between two halo lanes.  CLUSTER: units are dealt round-robin over the
// CTAs (few warps per SM for a small image) and the curve is reduced in the
// cluster (fin_u8.cuh, cluster_finalize).
template <bool CLUSTER, bool PACK, bool BATCH = false>
__global__ void __launch_bounds__(NT, CTAS_PER_SM)
    k_u8_2d(const Geom g, int64_t* __restrict__ ghist, const u8fin::Fin fin) {
  if constexpr (CLUSTER || BATCH) u8fin::cluster_started_arrive();
  // BATCH: image blockIdx.y, one thread-block cluster (gridDim.x CTAs) per image
  const uint8_t* const base = BATCH ? g.base + (size_t)blockIdx.y * g.img_stride : g.base;
  __shared__ __align__(16) uint32_t hist[HIST_WORDS];
  for (int i = threadIdx.x; i < HIST_WORDS; i += NT) hist[i] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwt = gridDim.x * NW;
  const uint32_t hist_s = smem_u32(hist) + (uint32_t)(((threadIdx.x & 31) * HREP) >> 5) * 4u;

  const int W = PACK ? g.L : 32;  // shuffle width: the lanes of one row
  for (int u = CLUSTER ? warp * gridDim.x + blockIdx.x : blockIdx.x * NW + warp; u < g.nunits;
       u += nwt) {
    int R0, rows, c, steps;
    if constexpr (PACK) {
      const int grp = lane / g.L;
      c = lane - grp * g.L;
      R0 = g.own0 + (u * g.G + grp) * g.band;
      rows = max(0, min(g.band, g.own0 + g.P - R0));  // 0: a group past the last band
      steps = g.band;                                 // warp-uniform sweep length
    } else {
      const int bi = u / g.nstrips, strip = u - bi * g.nstrips;
      R0 = g.own0 + bi * g.band;
      rows = min(g.band, g.own0 + g.P - R0);
      c = strip * STRIP - 1 + lane;  // this lane's chunk (may be -1 or >= nchunks)
      steps = rows;
    }
    const int lo = 32 * c;
    uint32_t zout = FULL;  // pixels of the chunk outside [0, W1)
    if (c >= 0 && c < g.nchunks) zout = (g.W1 - lo >= 32) ? 0u : (FULL << (g.W1 - lo));
    const uint32_t vm = PACK ? (c < g.nchunks ? ~zout : 0u) : ((lane >= 1 && lane <= STRIP) ? ~zout : 0u);
    const bool first = c == 0;
    // packed rows: the last lane of a row group has no right neighbour lane
    // (the row's right collar, which never wins as the later side)
    const uint32_t rcol = (PACK && c == g.L - 1) ? 1u : 0u;
    const int Rend = R0 + rows;
    const bool chunk_in = c >= 0 && c < g.nchunks;
    const bool hi_in = lo + 16 < g.W1;  // the chunk's second 16 bytes hold image pixels

    auto load_row = [&](int i, uint32_t (&W)[8]) {
      // rows outside the image are collar; rows outside the held range are
      // only the prefetch past a band's halo row (never used)
      if (i < 0 || i >= g.W0 || i < g.plane0 || i >= g.plane0 + g.nheld || !chunk_in) {
#pragma unroll
        for (int j = 0; j < 8; ++j) W[j] = FULL;
        return;
      }
      const uint8_t* p = base + (long long)(i - g.plane0) * g.pitch + lo;
      const uint4 a = ldg_stream(p);
      W[0] = a.x; W[1] = a.y; W[2] = a.z; W[3] = a.w;
      if (hi_in) {
        const uint4 b = ldg_stream(p + 16);
        W[4] = b.x; W[5] = b.y; W[6] = b.z; W[7] = b.w;
      } else {
        W[4] = W[5] = W[6] = W[7] = FULL;
      }
    };

    Row A, B;
    uint32_t xgx = 0, xgq = 0, xgq1 = 0;  // the previous row pair's results
    uint32_t nxt[8];
    load_row(R0 - 1, nxt);
    // rows R0-1 .. R0+rows arrive; at the arrival of row X the changes of row
    // X-1 are emitted (X-1 in [R0, R0 + rows), inside the image)
    auto step = [&](int X, Row& P, Row& N, auto kind) {
      constexpr int K = decltype(kind)::value;  // 0 first, 1 no emission, 2 emit
#pragma unroll
      for (int j = 0; j < 8; ++j) N.W[j] = nxt[j];
      load_row(X + 1, nxt);  // prefetch
      uint32_t (&C)[8] = N.C;
      bits::byte_interleave(N.W, C);
      bits::transpose8(C);
      const uint32_t om = (X < 0 || X >= g.W0) ? FULL : zout;
#pragma unroll
      for (int i = 0; i < 8; ++i) C[i] |= om;
      {
        uint32_t t[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          t[i] = __funnelshift_r(C[i], __shfl_down_sync(FULL, C[i], 1, W), 1);
          if constexpr (PACK) t[i] |= rcol << 31;
        }
        N.gz = bits::gt<8>(C, t);
        bits::sel<8>(N.mz, N.gz, C, t);
      }
      if constexpr (K >= 1) {
        uint32_t gx = bits::gt<8>(P.C, N.C);
        uint32_t gq = bits::gt<8>(P.mz, N.mz);
        if (X - 1 < 0) gx = gq = FULL;  // row -1 never wins
        // the quad anchored one pixel to the left: from the previous chunk,
        // or for chunk 0 the quad over the left collar, whose minima are the
        // pixels at 0 -- its comparison is gx bit 0
        uint32_t qprev = __shfl_up_sync(FULL, gq, 1, W);
        if (first) qprev = gx << 31;
        const uint32_t gq1 = __funnelshift_l(qprev, gq, 1);
        if constexpr (K == 2) {
          const uint32_t vmr = (X - 1 < g.W0 && X - 1 < Rend) ? vm : 0u;
          uint32_t zprev = __shfl_up_sync(FULL, P.gz, 1, W);
          if (first) zprev = FULL;  // column -1 never wins
          if (vmr) {
            const uint32_t Z0 = ~P.gz;
            const uint32_t Z1 = __funnelshift_l(zprev, P.gz, 1);
            // S = 4 quads won + 4 negated pairs won = change + 3
            const uint32_t t0 = Z0 & ~gq, t1 = Z0 & xgq, t2 = Z1 & ~gq1, t3 = Z1 & xgq1;
            const uint32_t t4 = ~Z0, t5 = ~Z1, t6 = gx, t7 = ~xgx;
            uint32_t s0, c0, s1, c1, s2, c2;
            bits::fa3(t0, t1, t2, s0, c0);
            bits::fa3(t3, t4, t5, s1, c1);
            bits::fa3(t6, t7, s0, s2, c2);
            const uint32_t b0 = s1 ^ s2, k0 = s1 & s2;  // weight 1
            uint32_t b1, k1;
            bits::fa3(c0, c1, c2, b1, k1);              // weight 2
            const uint32_t b1x = b1 ^ k0, k1x = b1 & k0;
            const uint32_t b2 = k1 ^ k1x;               // weight 4 (S <= 4)
            const uint32_t nv = ~vmr;
            uint32_t V[8];
            bits::transpose_codes(b0 | nv, b1x | nv, b2 | nv, 0u, V);
#pragma unroll
            for (int p = 0; p < 32; ++p) {
              const int r = p & 7, b = p >> 3;
              const uint32_t idx = bits::prmt(
                  P.W[p >> 2], V[r], (p & 3) | ((4 + b) << 4) | ((0xC + b) << 8) | ((0xC + b) << 12));
              uint32_t addr;
              asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(addr) : "r"(idx), "r"(g.four), "r"(hist_s));
              asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
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
    int t = 1;  // rows R0 + t arrive; the sweep length is warp-uniform
    for (; t + 1 <= steps; t += 2) {
      step(R0 + t, B, A, std::integral_constant<int, 2>{});
      step(R0 + t + 1, A, B, std::integral_constant<int, 2>{});
    }
    if (t <= steps) step(R0 + t, B, A, std::integral_constant<int, 2>{});
  }
  extern __shared__ __align__(16) int cluster_rows[];
  if constexpr (BATCH) {
    u8fin::batch_finalize<NT, Codes, HREP>(hist, cluster_rows, g.chi + (size_t)blockIdx.y * 256,
                                          g.pres + (size_t)blockIdx.y * 8);
  } else if constexpr (CLUSTER) {
    u8fin::cluster_finalize<NT, Codes, HREP>(hist, cluster_rows, fin);
  } else {
    u8fin::flush_and_finalize<NT, Codes, HREP>(hist, ghist, fin);
  }
}

}  // namespace u82d

bool u8_2d_supported(const Slab& s) {
  return s.w2 == 1 && s.w1 >= 1 && s.plane_pitch() % 16 == 0 &&
         (reinterpret_cast<uintptr_t>(s.base) % 16) == 0 && s.w0 < (1ll << 31) &&
         s.w1 < (1ll << 31) - 64 && (s.own1 - s.own0) * s.w1 < (1ll << 38);  // u32 per-CTA counts
}

cudaError_t launch_u8_2d(const Slab& s, int64_t* ghist, int sms, cudaStream_t st,
                         const U83dFinalize* fz) {
  using namespace u82d;
  Geom g;
  g.base = static_cast<const uint8_t*>(s.base);
  g.pitch = s.plane_pitch();
  g.W0 = (int)s.w0;
  g.W1 = (int)s.w1;
  g.plane0 = (int)s.plane0;
  g.nheld = (int)s.nplanes;
  g.own0 = (int)s.own0;
  g.P = (int)(s.own1 - s.own0);
  g.nchunks = (g.W1 + 31) / 32;
  g.nstrips = (g.nchunks + STRIP - 1) / STRIP;
  g.four = 4 * HREP;
  u8fin::Fin fin{};
  if (fz) {
    fin = u8fin::Fin{fz->ticket, fz->bins, fz->changes, fz->chi, fz->count};
    fin.x = u8fin::Xchg{fz->world, fz->rank, fz->epoch, fz->slots, fz->flags, fz->my_slots,
                        fz->my_flags, fz->err};
  }
  // rows of <= 16 chunks: packed, G = 32 / L rows per warp
#ifndef ECC_U82D_PACK
#define ECC_U82D_PACK 1
#endif
  const bool pack = ECC_U82D_PACK && g.nchunks <= 16;
  g.L = 1;
  while (g.L < g.nchunks) g.L *= 2;
  g.G = pack ? 32 / g.L : 1;
  if (!pack) g.L = 32;
  // band slots one unit covers: strips -> 1 / nstrips of a band, packed -> G bands
  auto units_of = [&](long long band) {
    const long long nbands = (g.P + band - 1) / band;
    return pack ? (nbands + g.G - 1) / g.G : nbands * g.nstrips;
  };
  // Small images with the fused curve on one GPU (C1): all CTAs in one
  // thread-block cluster, units dealt round-robin over the CTAs, the curve
  // reduced over distributed shared memory (fin_u8.cuh, cluster_finalize) --
  // bands of up to 4 rows so the units fit one cluster of the largest size
  // this kernel can be co-scheduled with.
  // the opt-ins are per device; the largest co-schedulable cluster is the
  // same on every B200 (measured once)
  smem_optin<k_u8_2d<true, false>>(u8fin::cluster_rows_bytes);
  smem_optin<k_u8_2d<true, true>>(u8fin::cluster_rows_bytes);
  cluster16_optin<k_u8_2d<true, false>>();
  cluster16_optin<k_u8_2d<true, true>>();
  static int max_cluster = -1;
  if (max_cluster < 0) {
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(u8fin::kMaxCluster);
    q.blockDim = dim3(NT);
    q.dynamicSmemBytes = u8fin::cluster_rows_bytes;
    int cs = 0;
    max_cluster = cudaOccupancyMaxPotentialClusterSize(&cs, k_u8_2d<true, false>, &q) == cudaSuccess
                      ? std::min(cs, u8fin::kMaxCluster)
                      : 0;
    (void)cudaGetLastError();
  }
  if (fz && fz->world <= 1 && max_cluster >= 2 && g.P > 0 && (long long)g.P * g.W1 <= (1ll << 22)) {
    const long long cap_units = (long long)max_cluster * NW;
    long long band = 1;
    while (band <= 4 && units_of(band) > cap_units) ++band;
    if (band <= 4) {
      Geom gc = g;
      gc.band = (int)band;
      gc.nunits = (int)units_of(band);
      const unsigned grid = (unsigned)std::min<long long>(max_cluster, gc.nunits);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(NT);
      cfg.dynamicSmemBytes = u8fin::cluster_rows_bytes;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = grid;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      const cudaError_t e = pack ? cudaLaunchKernelEx(&cfg, k_u8_2d<true, true>, gc, ghist, fin)
                                 : cudaLaunchKernelEx(&cfg, k_u8_2d<true, false>, gc, ghist, fin);
      if (e == cudaSuccess) return cudaSuccess;
      // the cluster could not be placed (e.g. SMs held by other work): the
      // regular launch below computes the same curve
      (void)cudaGetLastError();
    }
  }
  const long long cap_warps = (long long)sms * CTAS_PER_SM * NW;
  // bands of >= 32 rows (2 halo rows per band); ~4 units per resident warp
  // when the image is large enough, else one wave of shorter bands (>= MINBAND:
  // small images are latency-bound, so more, shorter bands finish sooner)
  long long band;
  if (!pack) {
    const long long nb = std::max<long long>(1, (4 * cap_warps) / g.nstrips);
    band = std::max<long long>(32, (g.P + nb - 1) / nb);
    if ((long long)((g.P + band - 1) / band) * g.nstrips < cap_warps)
      band = std::max<long long>(MINBAND, ((long long)g.P * g.nstrips + cap_warps - 1) / cap_warps);
  } else {
    const long long slots = cap_warps * g.G;  // bands in one wave of warps
    band = std::max<long long>(32, (g.P + 4 * slots - 1) / (4 * slots));
    if ((g.P + band - 1) / band < slots) band = std::max<long long>(MINBAND, (g.P + slots - 1) / slots);
  }
  band = std::max<long long>(1, std::min<long long>(band, std::max(1, g.P)));
  g.band = (int)band;
  const long long units = units_of(band);
  if (g.P <= 0 || units > (1ll << 30)) return cudaErrorInvalidValue;
  g.nunits = (int)units;
  const long long grid = std::min<long long>((units + NW - 1) / NW, cap_warps / NW);
  if (pack)
    k_u8_2d<false, true><<<(unsigned)grid, NT, 0, st>>>(g, ghist, fin);
  else
    k_u8_2d<false, false><<<(unsigned)grid, NT, 0, st>>>(g, ghist, fin);
  return cudaGetLastError();
}

// A batch of 2D u8 images (ecc_batch2d): one thread-block cluster of k CTAs
// per image (k > 1 only when the batch is too small to fill the GPU), rows
// packed or in strips as for one image, the dense chi row and occupancy
// bitmap written by the cluster's CTA 0 (fin_u8.cuh, batch_finalize).
// Needs rows of a multiple of 16 bytes (16-byte loads); returns
// cudaErrorNotSupported otherwise (the caller runs k_batch.cu).
cudaError_t launch_batch_u8(const uint8_t* data, uint64_t count, int h, int w, int32_t* chi,
                            uint32_t* presence, cudaStream_t st) {
  using namespace u82d;
  if (w % 16 != 0 || (reinterpret_cast<uintptr_t>(data) % 16) != 0 || (long long)h * w > (1ll << 26))
    return cudaErrorNotSupported;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sms = 148;
    (void)cudaGetLastError();
  }
  smem_optin<k_u8_2d<false, true, true>>(u8fin::cluster_rows_bytes);
  smem_optin<k_u8_2d<false, false, true>>(u8fin::cluster_rows_bytes);
  Geom g{};
  g.base = data;
  g.pitch = w;
  g.W0 = h;
  g.W1 = w;
  g.plane0 = 0;
  g.nheld = h;
  g.own0 = 0;
  g.P = h;
  g.nchunks = (w + 31) / 32;
  g.nstrips = (g.nchunks + STRIP - 1) / STRIP;
  g.four = 4 * HREP;
  g.img_stride = (long long)h * w;
  g.chi = chi;
  g.pres = presence;
  const bool pack = ECC_U82D_PACK && g.nchunks <= 16;
  g.L = 1;
  while (g.L < g.nchunks) g.L *= 2;
  g.G = pack ? 32 / g.L : 1;
  if (!pack) g.L = 32;
  // CTAs per image: enough images per wave to fill the GPU, else up to 8 per image
  const long long k = std::max<long long>(1, std::min<long long>(8, (2 * sms + (long long)count - 1) /
                                                                      (long long)count));
  // bands so the image's units fill its k x NW warps once (>= 8 rows a band)
  const long long warps = k * NW;
  long long band;
  if (pack)
    band = std::max<long long>(std::min<long long>(8, h), (h + warps * g.G - 1) / (warps * g.G));
  else
    band = std::max<long long>(std::min<long long>(8, h), ((long long)h * g.nstrips + warps - 1) / warps);
  g.band = (int)band;
  const long long nbands = (h + band - 1) / band;
  g.nunits = (int)(pack ? (nbands + g.G - 1) / g.G : nbands * g.nstrips);
  const u8fin::Fin fin{};
  // grid.y holds at most 65535 images: larger batches in slices
  for (uint64_t i0 = 0; i0 < count; i0 += 65535) {
    const uint64_t n = std::min<uint64_t>(65535, count - i0);
    Geom gi = g;
    gi.base = data + i0 * (uint64_t)g.img_stride;
    gi.chi = chi + i0 * 256;
    gi.pres = presence + i0 * 8;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)k, (unsigned)n);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = u8fin::cluster_rows_bytes;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)k;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t e =
        pack ? cudaLaunchKernelEx(&cfg, k_u8_2d<false, true, true>, gi, (int64_t*)nullptr, fin)
             : cudaLaunchKernelEx(&cfg, k_u8_2d<false, false, true>, gi, (int64_t*)nullptr, fin);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace eccb
