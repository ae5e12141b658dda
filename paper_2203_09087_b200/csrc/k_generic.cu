// k_generic.cu -- the general-shape stencil kernels (any dims, any slab, any
// value type) and the K3 finalize kernel.
//
// These serve every shape the bit-sliced kernels (k_u8_3d.cu, k_u16_3d.cu,
// k_u8_2d.cu, k_u16_2d.cu) do not take: ragged dims, thin slabs, the general
// (sorted) f32 path, value-index tables, and the per-face masks behind the
// C++ introduced().  They evaluate the scalar tournament of tourney.cuh: one
// thread per axis-1/axis-2 position (3D) or axis-1 position (2D) sweeps a
// segment of axis-0 planes carrying the previous plane's block minima, so a
// plane step costs three key loads (3D), the in-plane tournament on
// warp-shuffled neighbours, nine minimum-vs-minimum comparisons along axis 0
// and two popcounts.  Lanes 0 and 31 of a warp are halo (their keys feed the
// neighbouring lanes' blocks); lanes 1..30 own voxels.
#include <type_traits>

#include <cub/cub.cuh>

#include "ecc_common.cuh"
#include "internal.h"
#include "tourney.cuh"

namespace eccb {

template <class T, bool AFFINE>
__device__ __forceinline__ uint32_t bin_of(T v, const AffineMap& am, uint32_t* flags) {
  if constexpr (std::is_same_v<T, uint32_t>) {  // key image (PaddedChunk on the device)
    if (am.table) {
      uint32_t lo = 0, hi = am.table_n;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (am.table[mid] < v) lo = mid + 1; else hi = mid;
      }
      if (lo < am.table_n && am.table[lo] == v) return lo;
      atomicOr(flags, kFlagBinmap);
      return 0;
    }
    return (v - am.key_lo) & am.key_mask;
  } else if constexpr (AFFINE) {
    if (am.table) {  // ValueIndex::bin_of (value_index.hpp:40-45): exact match in the table
      const uint32_t k = float_order_key_bits(__float_as_uint(static_cast<float>(v)));
      uint32_t lo = 0, hi = am.table_n;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (am.table[mid] < k) lo = mid + 1; else hi = mid;
      }
      if (lo < am.table_n && am.table[lo] == k) return lo;
      atomicOr(flags, v != v ? kFlagNaN : kFlagBinmap);
      return 0;
    }
    if (am.keyed)  // dense sorted-f32 path: the order key relative to the minimum
      return float_order_key_bits(__float_as_uint(static_cast<float>(v))) - am.key_lo;
    return affine_bin(am, static_cast<float>(v), flags);
  } else {
    return static_cast<uint32_t>(v);
  }
}

// Histogram sink: per-CTA shared bins (SMEM) flushed once, straight to the
// global int64 histogram for large bin counts, or (PACKED) one 64-bit
// atomic per voxel adding 2^32 + (change + 8) to bin's word of a packed
// table: the high word counts the voxels, the low word is sum(change + 8),
// exact while a table takes <= 2^28 voxels (13 * 2^28 < 2^32).  Half the
// atomics and half the table (a 2^24-bin table fits the 126 MB L2).
template <bool SMEM, bool PACKED = false>
struct HistSink {
  int32_t* sums;
  uint32_t* counts;
  int64_t* ghist;
  uint32_t nbins;
  __device__ __forceinline__ void add(uint32_t bin, int change) {
    if constexpr (PACKED) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&ghist[bin]),
                (1ull << 32) | (unsigned long long)(uint32_t)(change + 8));
    } else if constexpr (SMEM) {
      atomicAdd(&sums[bin], change);
      atomicAdd(&counts[bin], 1u);
    } else {
      atomicAdd(reinterpret_cast<unsigned long long*>(&ghist[bin]),
                static_cast<unsigned long long>(static_cast<long long>(change)));
      atomicAdd(reinterpret_cast<unsigned long long*>(&ghist[nbins + bin]), 1ull);
    }
  }
};

template <bool SMEM, bool PK>
__device__ __forceinline__ void sink_init(HistSink<SMEM, PK>& h, int64_t* ghist,
                                          uint32_t nbins, int32_t* sh) {
  h.ghist = ghist;
  h.nbins = nbins;
  if constexpr (SMEM) {
    h.sums = sh;
    h.counts = reinterpret_cast<uint32_t*>(sh + nbins);
    const int nt = blockDim.x * blockDim.y;
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    for (uint32_t b = tid; b < 2 * nbins; b += nt) sh[b] = 0;
    __syncthreads();
  }
}

template <bool SMEM, bool PK>
__device__ __forceinline__ void sink_flush(HistSink<SMEM, PK>& h) {
  if constexpr (SMEM) {
    __syncthreads();
    const int nt = blockDim.x * blockDim.y;
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    for (uint32_t b = tid; b < h.nbins; b += nt) {
      const uint32_t c = h.counts[b];
      if (c) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&h.ghist[b]),
                  static_cast<unsigned long long>(static_cast<long long>(h.sums[b])));
        atomicAdd(reinterpret_cast<unsigned long long*>(&h.ghist[h.nbins + b]),
                  static_cast<unsigned long long>(c));
      }
    }
  }
}

// What a generic launch produces.
enum Mode : int {
  kHistSmem = 0,   // per-bin change sums + counts, shared bins flushed per CTA
  kHistGlobal = 1, // same, straight to the global int64 histogram
  kChanges = 2,    // int8 change per owned voxel (compute_changes)
  kFaces = 3,      // uint32 introduced-face mask per owned voxel (tourney.cuh faces3/faces2)
  kHistPacked = 4  // packed 64-bit count / sum words, one atomic per voxel (HistSink)
};

constexpr uint32_t FULLMASK = 0xFFFFFFFFu;
constexpr int LANES_OWNED = 30;  // lanes 1..30 of a warp own voxels

// ---------------------------------------------------------------- 3D
// block (32, BY): lane -> axis 2 (k = 30 * blockIdx.x + lane - 1); each warp
// owns TWO consecutive rows j0, j0 + 1 (j0 = 2 (BY blockIdx.y + threadIdx.y)):
// the rows j0-1 .. j0+2 it loads serve both voxels, and the axis-1 pair and
// 2 x 2 block between them are decided once.  blockIdx.z -> segment of
// `seg` owned planes, swept with the previous plane's minima carried.
struct Plane2v {
  tour::Plane<tour::NB3> v[2];  // the two voxels (rows j0, j0 + 1)
};

template <class T, bool AFFINE, int MODE>
__global__ void __launch_bounds__(256) k_tour3(Slab s, int64_t seg, AffineMap am, int64_t* ghist,
                                               uint32_t nbins, uint32_t* flags, void* out) {
  extern __shared__ int32_t sh[];
  constexpr bool HIST = MODE == kHistSmem || MODE == kHistGlobal || MODE == kHistPacked;
  HistSink<MODE == kHistSmem, MODE == kHistPacked> sink;
  if constexpr (HIST) sink_init(sink, ghist, nbins, sh);
  constexpr uint32_t SENT = KeyTraits<T>::kSentinel;
  const int lane = threadIdx.x;
  const int64_t k = (int64_t)blockIdx.x * LANES_OWNED + lane - 1;
  const int64_t j0 = 2 * ((int64_t)blockIdx.y * blockDim.y + threadIdx.y);
  const int64_t i0 = s.own0 + (int64_t)blockIdx.z * seg;
  const int64_t i1 = min(i0 + seg, s.own1);
  if (j0 < s.w1 && i0 < i1) {  // warp-uniform (a warp is one row pair)
    const bool kin = k >= 0 && k < s.w2;
    const int64_t OW1 = s.own_j1() - s.oj0, OW2 = s.own_k1() - s.ok0;
    const bool kown = kin && lane >= 1 && lane <= LANES_OWNED && k >= s.ok0 && k < s.own_k1();
    const bool own0 = kown && j0 >= s.oj0 && j0 < s.own_j1();
    const bool own1 = kown && j0 + 1 >= s.oj0 && j0 + 1 < s.own_j1();
    // rows j0-1, j0, j0+1, j0+2 present?
    const bool rm = j0 > 0, r1 = j0 + 1 < s.w1, r2 = j0 + 2 < s.w1;
    const int64_t rp = s.row_pitch(), pp = s.plane_pitch();
    const T* ctr = static_cast<const T*>(s.base) + j0 * rp + (kin ? k : 0) - s.plane0 * pp;

    // block minima and in-plane wins of plane i for the two voxels
    auto plane = [&](int64_t i, Plane2v& P, T (&val)[2]) {
      uint32_t am_ = SENT, a0 = SENT, a1 = SENT, a2 = SENT;
      if (kin && i >= 0 && i < s.w0) {
        const T* pc = ctr + i * pp;
        val[0] = __ldg(pc);
        a0 = KeyTraits<T>::key(val[0]);
        if (rm) am_ = KeyTraits<T>::key(__ldg(pc - rp));
        if (r1) {
          val[1] = __ldg(pc + rp);
          a1 = KeyTraits<T>::key(val[1]);
        }
        if (r2) a2 = KeyTraits<T>::key(__ldg(pc + 2 * rp));
      }
      // the same rows at k + 1 (lane + 1)
      const uint32_t bm_ = __shfl_down_sync(FULLMASK, am_, 1);
      const uint32_t b0 = __shfl_down_sync(FULLMASK, a0, 1);
      const uint32_t b1 = __shfl_down_sync(FULLMASK, a1, 1);
      const uint32_t b2 = __shfl_down_sync(FULLMASK, a2, 1);
      // pairs along axis 2 anchored at k (rows j0-1 .. j0+2)
      const uint32_t mzm = min(am_, bm_), mz0 = min(a0, b0), mz1 = min(a1, b1), mz2 = min(a2, b2);
      const bool hz0 = b0 < a0, hz1 = b1 < a1;  // k+1 beats k in rows j0, j0+1
      // pairs along axis 1 anchored at rows j0-1, j0, j0+1: the later row wins?
      const bool hym = a0 < am_, hy0 = a1 < a0, hy1 = a2 < a1;
      // 2 x 2 blocks anchored at rows j0-1, j0, j0+1: the later row's pair wins?
      const bool hqm = mz0 < mzm, hq0 = mz1 < mz0, hq1 = mz2 < mz1;
      const uint32_t mqm = min(mzm, mz0), mq0 = min(mz0, mz1), mq1 = min(mz1, mz2);
      // the blocks anchored at k - 1 come from lane - 1
      const uint32_t Lmz0 = __shfl_up_sync(FULLMASK, mz0, 1);
      const uint32_t Lmz1 = __shfl_up_sync(FULLMASK, mz1, 1);
      const uint32_t Lmqm = __shfl_up_sync(FULLMASK, mqm, 1);
      const uint32_t Lmq0 = __shfl_up_sync(FULLMASK, mq0, 1);
      const uint32_t Lmq1 = __shfl_up_sync(FULLMASK, mq1, 1);
      const uint32_t Lb = __shfl_up_sync(
          FULLMASK, (uint32_t)hz0 | ((uint32_t)hz1 << 1) | ((uint32_t)hqm << 2) |
                        ((uint32_t)hq0 << 3) | ((uint32_t)hq1 << 4), 1);
      const uint32_t Lhz0 = Lb & 1u, Lhz1 = (Lb >> 1) & 1u, Lhqm = (Lb >> 2) & 1u,
                     Lhq0 = (Lb >> 3) & 1u, Lhq1 = (Lb >> 4) & 1u;
      const uint32_t nz0 = !hz0, nz1 = !hz1;
      const uint32_t my_m = min(am_, a0), my_0 = min(a0, a1), my_1 = min(a1, a2);
      tour::Plane<tour::NB3>& v = P.v[0];
      v.M[0] = a0;   v.M[1] = Lmz0; v.M[2] = mz0; v.M[3] = my_m; v.M[4] = my_0;
      v.M[5] = Lmqm; v.M[6] = mqm;  v.M[7] = Lmq0; v.M[8] = mq0;
      v.I = 1u | (Lhz0 << 1) | (nz0 << 2) | ((uint32_t)hym << 3) | ((uint32_t)!hy0 << 4) |
            ((Lhz0 & Lhqm) << 5) | ((nz0 & (uint32_t)hqm) << 6) | ((Lhz0 & (Lhq0 ^ 1u)) << 7) |
            ((nz0 & (uint32_t)!hq0) << 8);
      tour::Plane<tour::NB3>& w = P.v[1];
      w.M[0] = a1;   w.M[1] = Lmz1; w.M[2] = mz1; w.M[3] = my_0; w.M[4] = my_1;
      w.M[5] = Lmq0; w.M[6] = mq0;  w.M[7] = Lmq1; w.M[8] = mq1;
      w.I = 1u | (Lhz1 << 1) | (nz1 << 2) | ((uint32_t)hy0 << 3) | ((uint32_t)!hy1 << 4) |
            ((Lhz1 & Lhq0) << 5) | ((nz1 & (uint32_t)hq0) << 6) | ((Lhz1 & (Lhq1 ^ 1u)) << 7) |
            ((nz1 & (uint32_t)!hq1) << 8);
    };

    auto emit = [&](int64_t i, const Plane2v& C, const uint32_t (&X)[2], const uint32_t (&Xp)[2],
                    const T (&val)[2]) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        if (r == 0 ? own0 : own1) {
          const int64_t vox = ((i - s.own0) * OW1 + (j0 + r - s.oj0)) * OW2 + (k - s.ok0);
          if constexpr (HIST) {
            const uint32_t bin = (AFFINE && am.keyed && !am.table)
                                     ? C.v[r].M[0] - am.key_lo
                                     : bin_of<T, AFFINE>(val[r], am, flags);
            sink.add(bin, tour::change_of<tour::POS3>(C.v[r].I, X[r], Xp[r]));
          } else if constexpr (MODE == kChanges) {
            static_cast<int8_t*>(out)[vox] = (int8_t)tour::change_of<tour::POS3>(C.v[r].I, X[r], Xp[r]);
          } else {
            static_cast<uint32_t*>(out)[vox] = tour::faces3(C.v[r].I, X[r], Xp[r]);
          }
        }
      }
    };
    auto xm = [&](const Plane2v& N, const Plane2v& C, uint32_t (&X)[2]) {
      X[0] = tour::xmask(N.v[0], C.v[0]);
      X[1] = tour::xmask(N.v[1], C.v[1]);
    };

    // two planes per iteration with the roles of A and B swapped: no copies
    Plane2v A, B;
    T va[2] = {T(0), T(0)}, vb[2] = {T(0), T(0)};
    uint32_t X[2], Xp[2];
    plane(i0 - 1, A, va);
    plane(i0, B, vb);
    xm(B, A, Xp);
    for (int64_t i = i0; i < i1; i += 2) {
      plane(i + 1, A, va);  // plane i lives in B
      xm(A, B, X);
      emit(i, B, X, Xp, vb);
      Xp[0] = X[0];
      Xp[1] = X[1];
      if (i + 1 >= i1) break;
      plane(i + 2, B, vb);  // plane i + 1 lives in A
      xm(B, A, X);
      emit(i + 1, A, X, Xp, va);
      Xp[0] = X[0];
      Xp[1] = X[1];
    }
  }
  if constexpr (HIST) sink_flush(sink);
}

// ---------------------------------------------------------------- 2D
// Stencil over axes 0 and 1 (w2 == 1, kernel.hpp:81-94).  Block of 8 warps,
// warp w of block b covers j = 30 * (8 b + w) + lane - 1.
template <class T, bool AFFINE, int MODE>
__global__ void __launch_bounds__(256) k_tour2(Slab s, int64_t seg, AffineMap am, int64_t* ghist,
                                               uint32_t nbins, uint32_t* flags, void* out) {
  extern __shared__ int32_t sh[];
  constexpr bool HIST = MODE == kHistSmem || MODE == kHistGlobal || MODE == kHistPacked;
  HistSink<MODE == kHistSmem, MODE == kHistPacked> sink;
  if constexpr (HIST) sink_init(sink, ghist, nbins, sh);
  constexpr uint32_t SENT = KeyTraits<T>::kSentinel;
  const int lane = threadIdx.x & 31;
  const int64_t j = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * LANES_OWNED +
                    lane - 1;
  const int64_t i0 = s.own0 + (int64_t)blockIdx.z * seg;
  const int64_t i1 = min(i0 + seg, s.own1);
  if (i0 < i1) {
    const bool jin = j >= 0 && j < s.w1;
    const int64_t OW1 = s.own_j1() - s.oj0;
    const bool own = jin && lane >= 1 && lane <= LANES_OWNED && j >= s.oj0 && j < s.own_j1();
    const int64_t pp = s.plane_pitch();
    const T* ctr = static_cast<const T*>(s.base) + (jin ? j : 0) - s.plane0 * pp;
    auto row = [&](int64_t i, tour::Plane<tour::NB2>& P, T& val) {
      uint32_t a = SENT;
      if (jin && i >= 0 && i < s.w0) {
        val = __ldg(ctr + i * pp);
        a = KeyTraits<T>::key(val);
      }
      const uint32_t b = __shfl_down_sync(FULLMASK, a, 1);  // j + 1
      const uint32_t mb = min(a, b);
      const bool hb = b < a;
      const uint32_t Lmb = __shfl_up_sync(FULLMASK, mb, 1);   // pair anchored at j - 1
      const uint32_t Lhb = __shfl_up_sync(FULLMASK, (uint32_t)hb, 1);
      P.M[0] = a;
      P.M[1] = Lmb;
      P.M[2] = mb;
      P.I = 1u | (Lhb << 1) | ((uint32_t)!hb << 2);
    };
    tour::Plane<tour::NB2> cur, nxt;
    T vcur = T(0), vnxt = T(0);
    row(i0 - 1, nxt, vnxt);
    row(i0, cur, vcur);
    uint32_t Xp = tour::xmask(cur, nxt);
    for (int64_t i = i0; i < i1; ++i) {
      row(i + 1, nxt, vnxt);
      const uint32_t X = tour::xmask(nxt, cur);
      if (own) {
        const int64_t vox = (i - s.own0) * OW1 + (j - s.oj0);
        if constexpr (HIST) {
          const uint32_t bin = (AFFINE && am.keyed && !am.table) ? cur.M[0] - am.key_lo
                                                                 : bin_of<T, AFFINE>(vcur, am, flags);
          sink.add(bin, tour::change_of<tour::POS2>(cur.I, X, Xp));
        } else if constexpr (MODE == kChanges) {
          static_cast<int8_t*>(out)[vox] = (int8_t)tour::change_of<tour::POS2>(cur.I, X, Xp);
        } else {
          static_cast<uint32_t*>(out)[vox] = tour::faces2(cur.I, X, Xp);
        }
      }
      Xp = X;
      cur = nxt;
      vcur = vnxt;
    }
  }
  if constexpr (HIST) sink_flush(sink);
}

// ---------------------------------------------------------------- launch
namespace {

constexpr uint32_t kSmemBinLimit = 8192;  // 2 x 8192 x 4 B = 64 KB

template <class T, bool AFFINE, int MODE>
cudaError_t launch_generic_t(const Slab& s, const AffineMap& am, int64_t* ghist,
                             uint32_t nbins, uint32_t* flags, void* out, int sms,
                             cudaStream_t st) {
  const int64_t owned = s.own1 - s.own0;
  const bool d3 = s.w2 > 1;
  dim3 block, grid;
  if (d3) {
    block = dim3(32, 8, 1);
    grid = dim3((unsigned)((s.w2 + LANES_OWNED - 1) / LANES_OWNED), (unsigned)((s.w1 + 15) / 16), 1);
  } else {
    block = dim3(256, 1, 1);
    grid = dim3((unsigned)((s.w1 + 8 * LANES_OWNED - 1) / (8 * LANES_OWNED)), 1, 1);
  }
  const int64_t cols = (int64_t)grid.x * grid.y;
  // enough CTAs for ~8 per SM, but segments of at least 8 planes
  int64_t nseg = (8LL * sms + cols - 1) / cols;
  nseg = std::max<int64_t>(1, std::min<int64_t>(nseg, (owned + 7) / 8));
  nseg = std::min<int64_t>(nseg, 65535);
  const int64_t seg = (owned + nseg - 1) / nseg;
  grid.z = (unsigned)((owned + seg - 1) / seg);
  const size_t smem = MODE == kHistSmem ? 2 * nbins * sizeof(int32_t) : 0;
  auto fn = d3 ? k_tour3<T, AFFINE, MODE> : k_tour2<T, AFFINE, MODE>;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fn<<<grid, block, smem, st>>>(s, seg, am, ghist, nbins, flags, out);
  return cudaGetLastError();
}

template <class T, bool AFFINE>
cudaError_t launch_generic_hist(const Slab& s, const AffineMap& am, int64_t* ghist,
                                uint32_t nbins, uint32_t* flags, int sms,
                                cudaStream_t st) {
  if (am.packed)
    return launch_generic_t<T, AFFINE, kHistPacked>(s, am, ghist, nbins, flags, nullptr, sms, st);
  if (nbins <= kSmemBinLimit)
    return launch_generic_t<T, AFFINE, kHistSmem>(s, am, ghist, nbins, flags, nullptr, sms, st);
  return launch_generic_t<T, AFFINE, kHistGlobal>(s, am, ghist, nbins, flags, nullptr, sms, st);
}

template <int MODE>
cudaError_t launch_generic_out(const Slab& s, int dtype, void* out, int sms, cudaStream_t st) {
  AffineMap am{};
  switch (dtype) {
    case 0:
      return launch_generic_t<uint8_t, false, MODE>(s, am, nullptr, 0, nullptr, out, sms, st);
    case 1:
      return launch_generic_t<uint16_t, false, MODE>(s, am, nullptr, 0, nullptr, out, sms, st);
    case 2:
      return launch_generic_t<float, false, MODE>(s, am, nullptr, 0, nullptr, out, sms, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_generic_accumulate(const Slab& s, int dtype, bool affine,
                                      const AffineMap& am, int64_t* ghist,
                                      uint32_t nbins, uint32_t* flags, int sms,
                                      cudaStream_t st) {
  switch (dtype) {
    case 0:
      return launch_generic_hist<uint8_t, false>(s, am, ghist, nbins, flags, sms, st);
    case 1:
      return launch_generic_hist<uint16_t, false>(s, am, ghist, nbins, flags, sms, st);
    case 2:
      if (!affine) return cudaErrorInvalidValue;
      return launch_generic_hist<float, true>(s, am, ghist, nbins, flags, sms, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_generic_changes(const Slab& s, int dtype, int8_t* out, int sms,
                                   cudaStream_t st) {
  return launch_generic_out<kChanges>(s, dtype, out, sms, st);
}

cudaError_t launch_generic_faces(const Slab& s, int dtype, uint32_t* out, int sms,
                                 cudaStream_t st) {
  return launch_generic_out<kFaces>(s, dtype, out, sms, st);
}

// ---------------------------------------------------------------- padded chunks
// A PaddedChunk's extended storage (chunk.hpp:50-127: u8 -> int16 with the
// sentinel 256, u16 -> int32, f32 -> float with +inf) turned into a key image
// on the device: order-preserving uint32 keys of exactly the stored values,
// collar included, so ties with the collar behave as in the reference.  2D
// chunks keep only the middle column of the padded axis 2.  `interior`
// writes only the owned voxels (rows 1..np-2, collar stripped) densely.
__global__ void k_chunk_keys(const void* __restrict__ padded, int etype, uint64_t np, uint64_t w1p,
                             uint64_t w2p, int is2d, int interior, uint32_t* __restrict__ keys) {
  const uint64_t o0 = interior ? 1 : 0, o1 = interior ? 1 : 0, o2 = (interior || is2d) ? 1 : 0;
  const uint64_t n0 = np - 2 * o0, n1 = w1p - 2 * o1, n2 = is2d ? 1 : w2p - 2 * o2;
  const uint64_t n = n0 * n1 * n2;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = t % n2, r = (t / n2) % n1, p = t / (n1 * n2);
    const uint64_t src = ((p + o0) * w1p + (r + o1)) * w2p + (c + o2);
    uint32_t k;
    if (etype == 0)
      k = (uint32_t)((int32_t)static_cast<const int16_t*>(padded)[src] + 32768);
    else if (etype == 1)
      k = (uint32_t)static_cast<const int32_t*>(padded)[src] ^ 0x80000000u;
    else
      k = float_order_key_bits(__float_as_uint(static_cast<const float*>(padded)[src]));
    keys[t] = k;
  }
}

cudaError_t launch_chunk_keys(const void* padded, int etype, uint64_t np, uint64_t w1p,
                              uint64_t w2p, bool is2d, bool interior, uint32_t* keys, int sms,
                              cudaStream_t st) {
  k_chunk_keys<<<sms * 4, 256, 0, st>>>(padded, etype, np, w1p, w2p, is2d ? 1 : 0,
                                        interior ? 1 : 0, keys);
  return cudaGetLastError();
}

cudaError_t launch_keyimage(const Slab& s, int mode, const AffineMap& am, int64_t* ghist,
                            uint32_t nbins, uint32_t* flags, void* out, int sms, cudaStream_t st) {
  switch (mode) {
    case kChanges:
      return launch_generic_t<uint32_t, true, kChanges>(s, am, nullptr, 0, nullptr, out, sms, st);
    case kFaces:
      return launch_generic_t<uint32_t, true, kFaces>(s, am, nullptr, 0, nullptr, out, sms, st);
    default:
      if (nbins <= kSmemBinLimit)
        return launch_generic_t<uint32_t, true, kHistSmem>(s, am, ghist, nbins, flags, nullptr,
                                                           sms, st);
      return launch_generic_t<uint32_t, true, kHistGlobal>(s, am, ghist, nbins, flags, nullptr,
                                                           sms, st);
  }
}

// Value lists (ValueIndex::build, merge_local): keys of n values of a dtype
// (u8 / u16: the value; f32: the order key, NaN flagged).
__global__ void k_value_keys(const void* __restrict__ v, int dtype, uint64_t n,
                             uint32_t* __restrict__ keys, uint32_t* flags) {
  bool nan = false;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t k;
    if (dtype == 0) {
      k = static_cast<const uint8_t*>(v)[i];
    } else if (dtype == 1) {
      k = static_cast<const uint16_t*>(v)[i];
    } else {
      const float x = static_cast<const float*>(v)[i];
      nan |= x != x;
      k = float_order_key_bits(__float_as_uint(x));
    }
    keys[i] = k;
  }
  if (nan) atomicOr(flags, kFlagNaN);
}

// merge_local's incoming entries: sums[i] = local[bin of value i], bin = the
// value (u8 / u16 keys) or the position i (a float value index).
__global__ void k_gather_local(const uint32_t* __restrict__ keys, int by_value, uint64_t n,
                               const int64_t* __restrict__ local, uint64_t nlocal,
                               int64_t* __restrict__ sums, uint32_t* flags) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = by_value ? keys[i] : i;
    if (b < nlocal) {
      sums[i] = local[b];
    } else {
      sums[i] = 0;
      atomicOr(flags, kFlagBinmap);
    }
  }
}

cudaError_t launch_value_keys(const void* v, int dtype, uint64_t n, uint32_t* keys,
                              uint32_t* flags, int sms, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_value_keys<<<sms * 4, 256, 0, st>>>(v, dtype, n, keys, flags);
  return cudaGetLastError();
}

cudaError_t launch_gather_local(const uint32_t* keys, bool by_value, uint64_t n,
                                const int64_t* local, uint64_t nlocal, int64_t* sums,
                                uint32_t* flags, int sms, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_gather_local<<<sms * 2, 256, 0, st>>>(keys, by_value ? 1 : 0, n, local, nlocal, sums, flags);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- order keys
// Sorted path, pass 1: min / max order key of the owned voxels and the NaN
// check (ValueIndex<float>::build rejects NaN, value_index.hpp:29).
// mm[0] = min (start 0xFFFFFFFF), mm[1] = max (start 0).
__global__ void k_key_range(const float* __restrict__ v, uint64_t n, uint32_t* flags,
                            uint32_t* mm) {
  uint32_t lo = 0xFFFFFFFFu, hi = 0;
  bool nan = false;
  auto take = [&](float x) {
    nan |= x != x;
    const uint32_t k = float_order_key_bits(__float_as_uint(x));
    lo = min(lo, k);
    hi = max(hi, k);
  };
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  const bool vec = (reinterpret_cast<uintptr_t>(v) & 15) == 0;
  const uint64_t n4 = vec ? n / 4 : 0;
  const float4* v4 = reinterpret_cast<const float4*>(v);
  // float4 groups, four loads in flight per thread
  uint64_t i = tid;
  for (; i + 3 * nt < n4; i += 4 * nt) {
    float4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = __ldcs(v4 + i + u * nt);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      take(x[u].x); take(x[u].y); take(x[u].z); take(x[u].w);
    }
  }
  for (; i < n4; i += nt) {
    const float4 x = __ldcs(v4 + i);
    take(x.x); take(x.y); take(x.z); take(x.w);
  }
  for (uint64_t j = 4 * n4 + tid; j < n; j += nt) take(__ldg(v + j));
  if (nan) atomicOr(flags, kFlagNaN);
  lo = __reduce_min_sync(0xFFFFFFFFu, lo);
  hi = __reduce_max_sync(0xFFFFFFFFu, hi);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
  }
}

// Pass 2: order keys (value_index.hpp:95-99) minus the minimum -- still
// order-preserving, and only the low bits of (max - min) vary, so the radix
// sort covers fewer bits (the reference skips trivial passes,
// value_index.hpp:125-131, for the same reason).
__global__ void k_order_keys(const float* __restrict__ v, uint64_t n,
                             uint32_t* __restrict__ keys, const uint32_t* mm) {
  const uint32_t lo = mm[0];
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(keys)) & 15) == 0;
  const uint64_t n4 = vec ? n / 4 : 0;
  auto key = [&](float x) { return float_order_key_bits(__float_as_uint(x)) - lo; };
  const float4* v4 = reinterpret_cast<const float4*>(v);
  uint4* k4 = reinterpret_cast<uint4*>(keys);
  uint64_t i = tid;
  for (; i + 3 * nt < n4; i += 4 * nt) {
    float4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = __ldcs(v4 + i + u * nt);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      k4[i + u * nt] = make_uint4(key(x[u].x), key(x[u].y), key(x[u].z), key(x[u].w));
  }
  for (; i < n4; i += nt) {
    const float4 x = __ldcs(v4 + i);
    k4[i] = make_uint4(key(x.x), key(x.y), key(x.z), key(x.w));
  }
  for (uint64_t j = 4 * n4 + tid; j < n; j += nt) keys[j] = key(__ldg(v + j));
}

__global__ void k_add_key(uint32_t* keys, uint64_t n, const uint32_t* mm) {
  const uint32_t lo = mm[0];
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    keys[i] += lo;
}

cudaError_t launch_key_range(const float* v, uint64_t n, uint32_t* flags, uint32_t* mm, int sms,
                             cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_key_range<<<sms * 8, 256, 0, st>>>(v, n, flags, mm);
  return cudaGetLastError();
}

cudaError_t launch_order_keys(const float* v, uint64_t n, uint32_t* keys, const uint32_t* mm,
                              int sms, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_order_keys<<<sms * 8, 256, 0, st>>>(v, n, keys, mm);
  return cudaGetLastError();
}

cudaError_t launch_add_key(uint32_t* keys, uint64_t n, const uint32_t* mm, int sms,
                           cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_add_key<<<sms * 4, 256, 0, st>>>(keys, n, mm);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- K3
// merge_local (vcec.hpp:35-66) + vcec_to_ecc (curve.hpp:28-35) over a dense
// histogram: occurring bins (count > 0) are compacted in ascending order
// and their change sums prefix-summed.  Bins that never occur have a zero
// change sum, so chi at an occurring bin is the prefix over all bins.  The
// histogram is int64[2][nbins] (sums, counts) or, PACKED, the generic
// kernels' uint64[nbins] words count << 32 | sum(change + 8).
template <bool PACKED>
__device__ __forceinline__ void bin_at(const int64_t* __restrict__ hist, uint32_t nbins, uint32_t b,
                                       long long& sum, long long& cnt) {
  if constexpr (PACKED) {
    const unsigned long long w = (unsigned long long)hist[b];
    cnt = (long long)(w >> 32);
    sum = (long long)(w & 0xFFFFFFFFull) - 8 * cnt;
  } else {
    sum = hist[b];
    cnt = hist[nbins + b];
  }
}

// One CTA of 1024 threads, each owning a contiguous run of bins.
template <bool PACKED>
__global__ void __launch_bounds__(1024) k_finalize(const int64_t* __restrict__ hist,
                                                   uint32_t nbins, uint32_t* bins,
                                                   int64_t* changes, int64_t* chi,
                                                   uint64_t* count) {
  using Scan = cub::BlockScan<longlong2, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  const uint32_t per = (nbins + 1023) / 1024;
  const uint32_t b0 = min(nbins, threadIdx.x * per);
  const uint32_t b1 = min(nbins, b0 + per);
  long long npres = 0, sum = 0;
  for (uint32_t b = b0; b < b1; ++b) {
    long long sm, ct;
    bin_at<PACKED>(hist, nbins, b, sm, ct);
    npres += ct != 0;
    sum += sm;
  }
  longlong2 in = make_longlong2(npres, sum), ex;
  struct Add {
    __device__ longlong2 operator()(const longlong2& a, const longlong2& b) const {
      return make_longlong2(a.x + b.x, a.y + b.y);
    }
  };
  longlong2 total;
  Scan(tmp).ExclusiveScan(in, ex, make_longlong2(0, 0), Add(), total);
  long long pos = ex.x, acc = ex.y;
  for (uint32_t b = b0; b < b1; ++b) {
    long long sm, ct;
    bin_at<PACKED>(hist, nbins, b, sm, ct);
    acc += sm;
    if (ct != 0) {
      bins[pos] = b;
      changes[pos] = sm;
      chi[pos] = acc;
      ++pos;
    }
  }
  if (threadIdx.x == 1023) *count = (uint64_t)total.x;
}

// Large bin counts (65536 for u16 / quantised f32, up to 2^24 for the dense
// sorted-f32 path): three small grids -- per-1024-bin partial (count, sum),
// one scan of the partials, and the block-local scan that writes the
// compacted curve -- instead of one CTA walking all bins.
namespace fin {
constexpr int T = 256, PER = 4, B = T * PER;

struct Add2 {
  __device__ longlong2 operator()(const longlong2& a, const longlong2& b) const {
    return make_longlong2(a.x + b.x, a.y + b.y);
  }
};

template <bool PACKED>
__global__ void __launch_bounds__(T) k_partials(const int64_t* __restrict__ hist, uint32_t nbins,
                                                longlong2* __restrict__ part) {
  using Red = cub::BlockReduce<longlong2, T>;
  __shared__ typename Red::TempStorage tmp;
  const uint32_t b0 = blockIdx.x * B + threadIdx.x * PER;
  longlong2 v = make_longlong2(0, 0);
#pragma unroll
  for (int i = 0; i < PER; ++i)
    if (b0 + i < nbins) {
      long long sm, ct;
      bin_at<PACKED>(hist, nbins, b0 + i, sm, ct);
      v.x += ct != 0;
      v.y += sm;
    }
  const longlong2 t = Red(tmp).Reduce(v, Add2());
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ void __launch_bounds__(1024) k_scan_partials(longlong2* part, uint32_t nblk,
                                                        uint64_t* count) {
  using Scan = cub::BlockScan<longlong2, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  const uint32_t per = (nblk + 1023) / 1024;
  const uint32_t a = min(nblk, threadIdx.x * per), b = min(nblk, a + per);
  longlong2 loc = make_longlong2(0, 0);
  for (uint32_t j = a; j < b; ++j) loc = Add2()(loc, part[j]);
  longlong2 ex, total;
  Scan(tmp).ExclusiveScan(loc, ex, make_longlong2(0, 0), Add2(), total);
  for (uint32_t j = a; j < b; ++j) {
    const longlong2 p = part[j];
    part[j] = ex;
    ex = Add2()(ex, p);
  }
  if (threadIdx.x == 0) *count = (uint64_t)total.x;
}

// SCAN: `part` holds the raw per-block totals (nblk <= T) and every block
// reduces those of the blocks before it itself -- no k_scan_partials launch;
// the last block writes the point count.
template <bool PACKED, bool SCAN = false>
__global__ void __launch_bounds__(T) k_write(const int64_t* __restrict__ hist, uint32_t nbins,
                                             const longlong2* __restrict__ part, uint32_t* bins,
                                             int64_t* changes, int64_t* chi, uint64_t* count = nullptr) {
  using Scan = cub::BlockScan<longlong2, T>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ longlong2 base;
  if constexpr (SCAN) {
    using Red = cub::BlockReduce<longlong2, T>;
    __shared__ typename Red::TempStorage rtmp;
    const longlong2 p = threadIdx.x < blockIdx.x ? part[threadIdx.x] : make_longlong2(0, 0);
    const longlong2 t = Red(rtmp).Reduce(p, Add2());
    if (threadIdx.x == 0) {
      base = t;
      if (blockIdx.x + 1 == gridDim.x) *count = (uint64_t)(t.x + part[blockIdx.x].x);
    }
    __syncthreads();
  } else {
    if (threadIdx.x == 0) base = part[blockIdx.x];
    __syncthreads();
  }
  const uint32_t b0 = blockIdx.x * B + threadIdx.x * PER;
  long long s[PER], n[PER];
  longlong2 v = make_longlong2(0, 0);
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    s[i] = n[i] = 0;
    if (b0 + i < nbins) bin_at<PACKED>(hist, nbins, b0 + i, s[i], n[i]);
    v.x += n[i] != 0;
    v.y += s[i];
  }
  longlong2 ex;
  Scan(tmp).ExclusiveScan(v, ex, make_longlong2(0, 0), Add2());
  long long pos = base.x + ex.x, acc = base.y + ex.y;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    acc += s[i];
    if (n[i] != 0) {
      bins[pos] = b0 + i;
      changes[pos] = s[i];
      chi[pos] = acc;
      ++pos;
    }
  }
}
}  // namespace fin

cudaError_t launch_finalize(const int64_t* hist, uint32_t nbins, uint32_t* bins,
                            int64_t* changes, int64_t* chi, uint64_t* count, void* scratch,
                            cudaStream_t st, bool packed) {
  if (nbins <= 4096 || !scratch) {
    if (packed)
      k_finalize<true><<<1, 1024, 0, st>>>(hist, nbins, bins, changes, chi, count);
    else
      k_finalize<false><<<1, 1024, 0, st>>>(hist, nbins, bins, changes, chi, count);
    return cudaGetLastError();
  }
  const uint32_t nblk = (nbins + fin::B - 1) / fin::B;  // scratch: nblk x 16 bytes
  longlong2* part = static_cast<longlong2*>(scratch);
  if (packed)
    fin::k_partials<true><<<nblk, fin::T, 0, st>>>(hist, nbins, part);
  else
    fin::k_partials<false><<<nblk, fin::T, 0, st>>>(hist, nbins, part);
  if (nblk <= (uint32_t)fin::T) {  // <= 256 K bins: the prefix of the partials in k_write
    if (packed)
      fin::k_write<true, true><<<nblk, fin::T, 0, st>>>(hist, nbins, part, bins, changes, chi, count);
    else
      fin::k_write<false, true><<<nblk, fin::T, 0, st>>>(hist, nbins, part, bins, changes, chi, count);
    return cudaGetLastError();
  }
  fin::k_scan_partials<<<1, 1024, 0, st>>>(part, nblk, count);
  if (packed)
    fin::k_write<true><<<nblk, fin::T, 0, st>>>(hist, nbins, part, bins, changes, chi);
  else
    fin::k_write<false><<<nblk, fin::T, 0, st>>>(hist, nbins, part, bins, changes, chi);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- raw-file fixups
// image.hpp:39-52 on the device: big-endian f32 byte swap in place and the
// smallest linear index of a NaN (atomicMin; ~0 when there is none).
__global__ void k_fixup_f32(uint32_t* d, uint64_t n, uint64_t base, bool swap,
                            unsigned long long* nan_min) {
  unsigned long long first = ~0ull;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t u = d[i];
    if (swap) {
      u = __byte_perm(u, 0, 0x0123);
      d[i] = u;
    }
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu) && first == ~0ull) first = base + i;
  }
  if (first != ~0ull) atomicMin(nan_min, first);
}

cudaError_t launch_fixup(void* d, int dtype, uint64_t n, uint64_t base, bool big_endian,
                         unsigned long long* nan_min, int sms, cudaStream_t st) {
  if (dtype != 2) return cudaSuccess;
  k_fixup_f32<<<sms * 8, 256, 0, st>>>(static_cast<uint32_t*>(d), n, base, big_endian, nan_min);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- inputs
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

template <class T>
__global__ void k_fill(T* d, uint64_t n, uint64_t seed, uint64_t base) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t h = splitmix64(seed + (base + i) * 0x9E3779B97F4A7C15ull);
    if constexpr (sizeof(T) == 1)
      d[i] = (T)(h >> 56);
    else if constexpr (sizeof(T) == 2)
      d[i] = (T)(h >> 48);
    else
      d[i] = (float)(h >> 48) * 0x1p-16f;
  }
}

cudaError_t launch_fill(void* d, int dtype, uint64_t n, uint64_t seed,
                        uint64_t base, int sms, cudaStream_t st) {
  const int grid = sms * 16;
  switch (dtype) {
    case 0: k_fill<uint8_t><<<grid, 256, 0, st>>>((uint8_t*)d, n, seed, base); break;
    case 1: k_fill<uint16_t><<<grid, 256, 0, st>>>((uint16_t*)d, n, seed, base); break;
    case 2: k_fill<float><<<grid, 256, 0, st>>>((float*)d, n, seed, base); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace eccb
