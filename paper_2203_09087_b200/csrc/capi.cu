// capi.cu -- implementation of the C ABI in include/ecc_b200.h.
//
// Host orchestration only: argument validation with the reference's error
// wording, scratch management, the streaming driver (pinned staging, a copy
// stream and a compute stream), and dispatch to the kernels.  All voxel
// work happens in the kernels; there is no host compute path.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cub/cub.cuh>
#include <thrust/iterator/transform_iterator.h>

#include "../../include/ecc_b200.h"
#include "internal.h"

using namespace eccb;

namespace eccb {
cudaError_t launch_batch2d(const void* data, int dtype, uint64_t count, int h, int w,
                           int32_t* chi, uint32_t* presence, int32_t* spill_scratch,
                           cudaStream_t st);
cudaError_t launch_fixup(void* d, int dtype, uint64_t n, uint64_t base, bool big_endian,
                         unsigned long long* nan_min, int sms, cudaStream_t st);
cudaError_t launch_accumulate_fast(const Slab& s, int dtype, bool affine,
                                   const AffineMap& am, int64_t* ghist,
                                   uint32_t nbins, uint32_t* flags, int sms,
                                   cudaStream_t st, bool* handled);
cudaError_t launch_changes_fast(const Slab& s, int dtype, int8_t* out, int sms, cudaStream_t st,
                                bool* handled);
}  // namespace eccb

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CKR(x)                                                               \
  do {                                                                       \
    cudaError_t e_ = (x);                                                    \
    if (e_ != cudaSuccess)                                                   \
      return fail(e_ == cudaErrorMemoryAllocation ? ECC_ENOMEM : ECC_ECUDA,  \
                  std::string("CUDA error in ") + #x + ": " +                \
                      cudaGetErrorString(e_));                               \
  } while (0)

#define CKI(x)                        \
  do {                                \
    int rc_ = (x);                    \
    if (rc_ != ECC_OK) return rc_;    \
  } while (0)

size_t esize(ecc_dtype t) { return t == ECC_U8 ? 1 : (t == ECC_U16 ? 2 : 4); }

std::string dims_str(const ecc_dims& d) {
  return std::to_string(d.w0) + "x" + std::to_string(d.w1) + "x" + std::to_string(d.w2);
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  int ensure(size_t bytes) {
    if (bytes <= cap) return ECC_OK;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(bytes, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(ECC_ENOMEM, "device allocation of " + std::to_string(want) +
                                  " bytes failed: " + cudaGetErrorString(e));
    }
    cap = want;
    return ECC_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct PinBuf {
  void* p = nullptr;
  size_t cap = 0;
  int ensure(size_t bytes) {
    if (bytes <= cap) return ECC_OK;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocDefault);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(ECC_ENOMEM, "pinned allocation of " + std::to_string(bytes) +
                                  " bytes failed: " + cudaGetErrorString(e));
    }
    cap = bytes;
    return ECC_OK;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

}  // namespace

// Host vectors of a result: no value-initialisation on resize (every
// element is then written by a device copy), kept in the context between
// calls so a large result reuses already-touched pages.
template <class T>
struct NoInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = NoInitAlloc<U>;
  };
  NoInitAlloc() = default;
  template <class U>
  NoInitAlloc(const NoInitAlloc<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
};
template <class T>
using HostVec = std::vector<T, NoInitAlloc<T>>;

struct BinResult {
  HostVec<uint32_t> bins;     // identity / affine
  HostVec<uint32_t> keys;     // sorted path (order keys)
  HostVec<int64_t> changes;
  HostVec<int64_t> chi;
};

struct ecc_ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;  // compute
  cudaStream_t copy = nullptr;    // H2D
  uint64_t launches = 0;
  DevBuf input, hist, bins, changes, chi, count, flags;
  DevBuf keys, keys2, ch8, ch8b, sums, tmp;
  DevBuf slab[3];
  PinBuf staging[2];
  PinBuf host_small;
  DevBuf fused;  // ticket + 512 x int64 histogram of the fused u8 launch (kept zero)
  DevBuf pad;       // row-padded copy of a u8 slab for the TMA kernel
  DevBuf finscr;    // K3 partials for large bin counts
  DevBuf res;       // result block (count, flags, curve) read back in one copy
  PinBuf res_host;
  DevBuf keys16;    // 16-bit keys (u16 padded / f32 bin indices) for the 16-bit kernels
  DevBuf akeys, asums, sums2;  // sorted f32 path: per-slab runs and their merge
  DevBuf sm_tmp[2], sm_w;     // gaussian_smooth: axis temporaries and the taps
  DevBuf nanidx;    // per-chunk first NaN index of the file path
  DevBuf bscratch;  // per-SM int32[65536] spill rows of the u16 batched kernel (kept zero)
  cudaEvent_t ov_ev[17] = {};  // overlapped host-input path: start + one per chunk copy
  BinResult hres;  // host side of the last host-returning call (pages reused)
};

// Multi-GPU rank exchange over peer memory (fin_u8.cuh, Xchg): this rank's
// buffer -- int64 slots[2][world][512] | uint32 flags[2][world] | uint32 err
// -- exported by CUDA IPC, the peers' buffers opened, and device arrays of
// the peers' slot / flag pointers for the kernel.
struct ecc_xchg {
  ecc_ctx* ctx = nullptr;
  int rank = 0, world = 1;
  uint32_t epoch = 0;
  void* buf = nullptr;
  size_t flags_off = 0, err_off = 0, bytes = 0;
  std::vector<void*> base;  // [world] opened peer buffers (own: buf)
  void* ptrs = nullptr;     // device: int64_t* slots[world] | uint32_t* flags[world]
  uint32_t* err_host = nullptr;  // mapped pinned word the kernel raises on a peer timeout
  uint32_t* err_dev = nullptr;   // its device alias
  cudaStream_t last = nullptr;   // stream of the last fused launch (status syncs it)
};

namespace {

int bind(ecc_ctx* ctx) {
  if (!ctx) return fail(ECC_EINVAL, "null context");
  CKR(cudaSetDevice(ctx->device));
  return ECC_OK;
}

cudaStream_t pick(ecc_ctx* ctx, void* stream) {
  return stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
}

int check_dtype(ecc_dtype t) {
  if (t != ECC_U8 && t != ECC_U16 && t != ECC_F32)
    return fail(ECC_EINVAL, "unknown dtype " + std::to_string((int)t));
  return ECC_OK;
}

int check_dims(const ecc_dims& d) {
  if (d.w0 < 1 || d.w1 < 1 || d.w2 < 1)
    return fail(ECC_EINVAL, "dims must be >= 1, got " + dims_str(d));
  return ECC_OK;
}

// Resolves (dtype, binmap) to a bin count and an affine map.
int resolve_bins(ecc_dtype dtype, const ecc_binmap* bm, uint64_t* nbins,
                 bool* affine, bool* sorted, AffineMap* am) {
  const int kind = bm ? bm->kind : (dtype == ECC_F32 ? ECC_BIN_SORTED : ECC_BIN_IDENTITY);
  *affine = false;
  *sorted = false;
  if (dtype == ECC_U8 || dtype == ECC_U16) {
    if (kind != ECC_BIN_IDENTITY)
      return fail(ECC_EINVAL, "integer images use the identity bin map");
    *nbins = dtype == ECC_U8 ? 256 : 65536;
    return ECC_OK;
  }
  if (kind == ECC_BIN_SORTED) {
    *sorted = true;
    *nbins = 0;
    return ECC_OK;
  }
  if (kind != ECC_BIN_AFFINE)
    return fail(ECC_EINVAL, "f32 images need an affine or sorted bin map");
  if (!(bm->step > 0.0f) || bm->nbins < 1 || bm->nbins > (1u << 24) || bm->lo != bm->lo)
    return fail(ECC_EINVAL, "invalid affine bin map");
  *affine = true;
  *nbins = bm->nbins;
  am->lo = bm->lo;
  am->step = bm->step;
  am->inv_step = 1.0 / (double)bm->step;
  am->nbins = bm->nbins;
  am->pow2_scale = 0.0f;
  {
    int e = 0;
    const double mant = std::frexp((double)bm->step, &e);
    if (bm->lo == 0.0f && mant == 0.5 && e <= 1 && e > -100 && bm->nbins <= (1u << 22))
      am->pow2_scale = (float)(1.0 / (double)bm->step);
  }
  return ECC_OK;
}

int check_slab(ecc_dims d, uint64_t plane0, uint64_t nplanes, uint64_t own0,
               uint64_t own1) {
  CKI(check_dims(d));
  if (!(own0 < own1) || own1 > d.w0)
    return fail(ECC_EINVAL, "invalid chunk range [" + std::to_string(own0) + ", " +
                                std::to_string(own1) + ") for dims " + dims_str(d));
  const uint64_t need0 = own0 == 0 ? 0 : own0 - 1;
  const uint64_t need1 = std::min<uint64_t>(own1 + 1, d.w0);
  if (plane0 > need0 || plane0 + nplanes < need1)
    return fail(ECC_EINVAL, "slab buffer planes [" + std::to_string(plane0) + ", " +
                                std::to_string(plane0 + nplanes) +
                                ") do not cover the halo range [" + std::to_string(need0) +
                                ", " + std::to_string(need1) + ")");
  return ECC_OK;
}

// Plan validation with the reference's messages (streaming.hpp:186-195):
// bounds[0..nchunks] must be 0 = b0 < b1 < ... < b_n = w0.
int check_plan(const uint64_t* bounds, size_t nchunks, const ecc_dims& dims) {
  if (nchunks == 0 || !bounds) return fail(ECC_EINVAL, "empty chunk plan");
  if (bounds[0] != 0) return fail(ECC_EINVAL, "chunk plan does not cover the image contiguously");
  for (size_t k = 0; k < nchunks; ++k)
    if (bounds[k + 1] <= bounds[k])
      return fail(ECC_EINVAL, "chunk plan does not cover the image contiguously");
  if (bounds[nchunks] != dims.w0)
    return fail(ECC_EINVAL, "chunk plan covers [0, " + std::to_string(bounds[nchunks]) +
                                ") but the source has w0 = " + std::to_string(dims.w0));
  return ECC_OK;
}

Slab make_slab(const void* base, ecc_dims d, uint64_t plane0, uint64_t nplanes,
               uint64_t own0, uint64_t own1) {
  Slab s;
  s.base = base;
  s.plane0 = (int64_t)plane0;
  s.nplanes = (int64_t)nplanes;
  s.w0 = (int64_t)d.w0;
  s.w1 = (int64_t)d.w1;
  s.w2 = (int64_t)d.w2;
  s.own0 = (int64_t)own0;
  s.own1 = (int64_t)own1;
  return s;
}

int read_flags(ecc_ctx* ctx, cudaStream_t st) {
  uint32_t f = 0;
  CKR(cudaMemcpyAsync(&f, ctx->flags.p, 4, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  if (f & kFlagNaN) return fail(ECC_ENAN, "cannot build a value index: NaN input");
  if (f & kFlagBinmap)
    return fail(ECC_EBINMAP, "a value does not lie on the affine bin grid");
  return ECC_OK;
}

// Accumulate one slab into ctx->hist (already zeroed), dispatching to the
// specialised kernels when they cover the shape.
// 3D u8 slabs whose rows are not a multiple of 16 bytes (TMA stride rule)
// or whose base is not 16-byte aligned are copied once into a padded
// device buffer (row pitch rounded up to 16) so they too take the
// bit-sliced kernel; the padding columns lie outside w2 and read as collar.
int pad_for_u8_fast(ecc_ctx* ctx, const Slab& s, ecc_dtype dtype, bool affine, cudaStream_t st,
                    Slab* out) {
  *out = s;
  if (dtype != ECC_U8 || affine) return ECC_OK;
  if (s.w2 == 1) {  // 2D: rows along axis 1 padded to 16 bytes (k_u8_2d.cu)
    if (u8_2d_supported(s)) return ECC_OK;
    Slab p = s;
    p.ppitch = (s.w1 + 15) / 16 * 16;
    Slab probe = p;
    probe.base = nullptr;
    if (!u8_2d_supported(probe)) return ECC_OK;
    CKI(ctx->pad.ensure((size_t)s.nplanes * p.ppitch));
    CKR(cudaMemcpy2DAsync(ctx->pad.p, (size_t)p.ppitch, s.base, (size_t)s.plane_pitch(),
                          (size_t)s.w1, (size_t)s.nplanes, cudaMemcpyDeviceToDevice, st));
    p.base = ctx->pad.p;
    *out = p;
    return ECC_OK;
  }
  if (s.w2 <= 1 || u8_3d_supported(s)) return ECC_OK;
  Slab p = s;
  p.pitch = (s.w2 + 15) / 16 * 16;
  if (!u8_3d_supported(Slab{nullptr, p.plane0, p.nplanes, p.w0, p.w1, p.w2, p.own0, p.own1,
                            p.pitch}))
    return ECC_OK;  // too large for the fast path: stays on the generic kernel
  CKI(ctx->pad.ensure((size_t)s.nplanes * s.w1 * p.pitch));
  CKR(cudaMemcpy2DAsync(ctx->pad.p, (size_t)p.pitch, s.base, (size_t)s.row_pitch(), (size_t)s.w2,
                        (size_t)(s.nplanes * s.w1), cudaMemcpyDeviceToDevice, st));
  p.base = ctx->pad.p;
  *out = p;
  return ECC_OK;
}

// u16 images and affine-quantised f32 images with <= 65536 bins run the
// 16-bit bit-sliced kernels (k_u16_3d.cu, k_u16_2d.cu): f32 slabs are first mapped to bin
// indices (monotone, so the stencil sees the same order), u16 slabs whose
// rows break the 16-byte TMA stride rule are copied to a padded pitch.
int accumulate_keys16(ecc_ctx* ctx, const Slab& s, ecc_dtype dtype, bool affine,
                      const AffineMap& am, uint32_t nbins, int64_t* hist, cudaStream_t st,
                      bool* handled) {
  *handled = false;
  const bool u16 = dtype == ECC_U16 && !affine && nbins == 65536;
  const bool f32 = dtype == ECC_F32 && affine && nbins <= 65536;
  if (!(u16 || f32) || s.w1 > (1 << 30) || s.w2 > (1 << 30) || s.w0 > (1 << 30)) return ECC_OK;
  if (s.w2 == 1) {  // 2D (k_u16_2d.cu): rows along axis 1, pitch a multiple of 8 keys
    Slab k = s;
    if (f32 || !u16_2d_supported(s)) {
      k.ppitch = (s.w1 + 7) / 8 * 8;
      CKI(ctx->keys16.ensure((size_t)s.nplanes * k.ppitch * 2));
      if (f32) {
        CKR(launch_affine_keys(static_cast<const float*>(s.base), (uint64_t)s.nplanes,
                               (uint32_t)s.w1, (uint32_t)k.ppitch, am, ctx->keys16.as<uint16_t>(),
                               ctx->flags.as<uint32_t>(), ctx->sms, st));
        ctx->launches += 1;
      } else {
        CKR(cudaMemcpy2DAsync(ctx->keys16.p, (size_t)k.ppitch * 2, s.base,
                              (size_t)s.plane_pitch() * 2, (size_t)s.w1 * 2, (size_t)s.nplanes,
                              cudaMemcpyDeviceToDevice, st));
      }
      k.base = ctx->keys16.p;
    }
    CKR(launch_u16_2d(k, nbins, hist, ctx->sms, st));
    ctx->launches += 1;
    *handled = true;
    return ECC_OK;
  }
  if (s.w2 < 1) return ECC_OK;
  Slab k = s;
  if (f32 || !u16_3d_supported(s)) {
    k.pitch = (s.w2 + 7) / 8 * 8;
    CKI(ctx->keys16.ensure((size_t)s.nplanes * s.w1 * k.pitch * 2));
    if (f32) {
      CKR(launch_affine_keys(static_cast<const float*>(s.base), (uint64_t)(s.nplanes * s.w1),
                             (uint32_t)s.w2, (uint32_t)k.pitch, am, ctx->keys16.as<uint16_t>(),
                             ctx->flags.as<uint32_t>(), ctx->sms, st));
      ctx->launches += 1;
    } else {
      CKR(cudaMemcpy2DAsync(ctx->keys16.p, (size_t)k.pitch * 2, s.base, (size_t)s.row_pitch() * 2,
                            (size_t)s.w2 * 2, (size_t)(s.nplanes * s.w1),
                            cudaMemcpyDeviceToDevice, st));
    }
    k.base = ctx->keys16.p;
  }
  CKR(launch_u16_3d(k, nbins, hist, ctx->sms, st));
  ctx->launches += 1;
  *handled = true;
  return ECC_OK;
}

int accumulate(ecc_ctx* ctx, const Slab& s0, ecc_dtype dtype, bool affine,
               const AffineMap& am, uint32_t nbins, int64_t* hist, cudaStream_t st) {
  {
    bool done = false;
    CKI(accumulate_keys16(ctx, s0, dtype, affine, am, nbins, hist, st, &done));
    if (done) return ECC_OK;
  }
  Slab s;
  CKI(pad_for_u8_fast(ctx, s0, dtype, affine, st, &s));
  bool handled = false;
  CKR(launch_accumulate_fast(s, (int)dtype, affine, am, hist, nbins,
                             ctx->flags.as<uint32_t>(), ctx->sms, st, &handled));
  if (!handled)
    CKR(launch_generic_accumulate(s, (int)dtype, affine, am, hist, nbins,
                                  ctx->flags.as<uint32_t>(), ctx->sms, st));
  ctx->launches += 1;
  return ECC_OK;
}

// Result of a whole-volume or streamed run, in bin space.
// Whole 3D u8 image in ONE launch (k_u8_3d with the fused last-CTA K3).
bool fusable(ecc_dtype dtype, const Slab& s, bool affine) {
  return dtype == ECC_U8 && !affine && (u8_3d_supported(s) || u8_2d_supported(s));
}

int launch_fused(ecc_ctx* ctx, const Slab& s, uint32_t* bins, int64_t* changes, int64_t* chi,
                 uint64_t* count, cudaStream_t st) {
  if (!ctx->fused.p) {
    CKI(ctx->fused.ensure(256 + 512 * 8));
    CKR(cudaMemsetAsync(ctx->fused.p, 0, 256 + 512 * 8, st));
  }
  U83dFinalize fz{ctx->fused.as<uint32_t>(), bins, changes, chi, count};
  int64_t* ghist = reinterpret_cast<int64_t*>(ctx->fused.as<uint8_t>() + 256);
  if (s.w2 == 1)
    CKR(launch_u8_2d(s, ghist, ctx->sms, st, &fz));
  else
    CKR(launch_u8_3d(s, ghist, nullptr, ctx->sms, st, &fz));
  ctx->launches += 1;
  return ECC_OK;
}

// One device block holds everything a host caller reads back -- the
// occurring-bin count, the error flags and the compacted curve -- so a call
// ends with ONE device-to-host copy and one synchronisation:
//   [0, 8) count | [8, 12) flags | [64, ...) bins u32 | changes i64 | chi i64
struct ResultLayout {
  size_t bins, changes, chi, bytes;
  explicit ResultLayout(uint64_t nbins) {
    bins = 64;
    changes = bins + ((nbins * 4 + 7) & ~7ull);
    chi = changes + nbins * 8;
    bytes = chi + nbins * 8;
  }
};

int result_block(ecc_ctx* ctx, uint64_t nbins, ResultLayout* L) {
  *L = ResultLayout(nbins);
  CKI(ctx->res.ensure(L->bytes));
  CKI(ctx->res_host.ensure(L->bytes));
  return ECC_OK;
}

// The flags are copied into the block, the block comes back in one copy,
// and flag errors are reported with the wording of read_flags().
int fetch_result(ecc_ctx* ctx, const ResultLayout& L, cudaStream_t st, BinResult* out) {
  uint8_t* d = ctx->res.as<uint8_t>();
  uint8_t* h = static_cast<uint8_t*>(ctx->res_host.p);
  if (ctx->flags.p) CKR(cudaMemcpyAsync(d + 8, ctx->flags.p, 4, cudaMemcpyDeviceToDevice, st));
  else CKR(cudaMemsetAsync(d + 8, 0, 4, st));
  CKR(cudaMemcpyAsync(h, d, L.bytes, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  uint64_t m;
  uint32_t f;
  std::memcpy(&m, h, 8);
  std::memcpy(&f, h + 8, 4);
  if (f & kFlagNaN) return fail(ECC_ENAN, "cannot build a value index: NaN input");
  if (f & kFlagBinmap) return fail(ECC_EBINMAP, "a value does not lie on the affine bin grid");
  out->bins.assign(reinterpret_cast<const uint32_t*>(h + L.bins),
                   reinterpret_cast<const uint32_t*>(h + L.bins) + m);
  out->changes.assign(reinterpret_cast<const int64_t*>(h + L.changes),
                      reinterpret_cast<const int64_t*>(h + L.changes) + m);
  out->chi.assign(reinterpret_cast<const int64_t*>(h + L.chi),
                  reinterpret_cast<const int64_t*>(h + L.chi) + m);
  return ECC_OK;
}

// K3 over ctx->hist into the result block, then fetch_result.
int finalize_to_host(ecc_ctx* ctx, uint32_t nbins, cudaStream_t st, BinResult* out) {
  ResultLayout L(nbins);
  CKI(result_block(ctx, nbins, &L));
  uint8_t* d = ctx->res.as<uint8_t>();
  CKI(ctx->finscr.ensure(16ull * (nbins / 1024 + 1)));
  CKR(launch_finalize(ctx->hist.as<int64_t>(), nbins, reinterpret_cast<uint32_t*>(d + L.bins),
                      reinterpret_cast<int64_t*>(d + L.changes),
                      reinterpret_cast<int64_t*>(d + L.chi), reinterpret_cast<uint64_t*>(d),
                      ctx->finscr.p, st));
  ctx->launches += 1;
  return fetch_result(ctx, L, st, out);
}

// General f32 path (build_index_counts, value_index.hpp:159-197, on the
// device): per-voxel int8 changes + order keys, radix argsort by key,
// reduce-by-key into (distinct value, summed change).  Appends the slab's
// (key, sum) runs to `out` (unmerged; caller merges across slabs).
struct ToI64 {
  __host__ __device__ int64_t operator()(int8_t v) const { return v; }
};

// order-key spans up to this many values take the dense histogram (no sort)
constexpr uint64_t kDenseKeySpan = 1ull << 24;
// a dense table fed by at most this many voxels uses the packed one-atomic
// words (count << 32 | sum(change + 8) stays exact: 13 * 2^28 < 2^32)
constexpr uint64_t kPackedMaxVoxels = 1ull << 28;

int merge_runs(ecc_ctx* ctx, cudaStream_t st, uint64_t n, uint64_t* m_out);

// Grows a run buffer to hold `elems` elements of `esz` bytes, keeping its
// first `keep` elements (DevBuf::ensure discards the contents).
int grow_keep(DevBuf* b, uint64_t elems, size_t esz, uint64_t keep, cudaStream_t st) {
  if (elems * esz <= b->cap) return ECC_OK;
  DevBuf nb;
  CKI(nb.ensure(elems * esz));
  if (keep) CKR(cudaMemcpyAsync(nb.p, b->p, keep * esz, cudaMemcpyDeviceToDevice, st));
  CKR(cudaStreamSynchronize(st));
  b->release();
  *b = nb;
  return ECC_OK;
}

// Room for `add` more runs after the `*n_acc` accumulated ones.  When the
// accumulator is full its runs are merged first (merge_local, vcec.hpp:35-66:
// one entry per distinct value), so device memory follows the number of
// distinct values seen so far plus one chunk -- not the image size.
int reserve_runs(ecc_ctx* ctx, cudaStream_t st, uint64_t add, uint64_t* n_acc) {
  const uint64_t cap = std::min(ctx->akeys.cap / 4, ctx->asums.cap / 8);
  if (*n_acc + add <= cap) return ECC_OK;
  if (*n_acc > 0) CKI(merge_runs(ctx, st, *n_acc, n_acc));
  const uint64_t want = std::max(*n_acc + add, 2 * *n_acc);
  CKI(grow_keep(&ctx->akeys, want, 4, *n_acc, st));
  CKI(grow_keep(&ctx->asums, want, 8, *n_acc, st));
  return ECC_OK;
}

// Appends the slab's reduced (order key, change sum) runs to the device
// accumulator ctx->akeys / ctx->asums at offset *n (no host round trip).
int sorted_slab(ecc_ctx* ctx, const Slab& s, cudaStream_t st, uint64_t* n_acc) {
  const uint64_t n64 = (uint64_t)(s.own1 - s.own0) * s.w1 * s.w2;
  if (n64 > 0x7FFFFFFFull)
    return fail(ECC_EINVAL, "chunk exceeds 2^31 voxels; use a finer chunk plan");
  const int n = (int)n64;
  CKI(ctx->keys.ensure(n64 * 4));
  CKI(ctx->keys2.ensure(n64 * 4));
  CKI(ctx->ch8.ensure(n64));
  CKI(ctx->ch8b.ensure(n64));
  CKI(ctx->count.ensure(8));
  CKI(reserve_runs(ctx, st, n64, n_acc));
  const float* owned = static_cast<const float*>(s.base) + (s.own0 - s.plane0) * s.w1 * s.w2;
  // flags words 1, 2: min / max order key -> dense histogram or the bit range
  // the sort must cover
  CKI(ctx->flags.ensure(16));
  uint32_t* mm = ctx->flags.as<uint32_t>() + 1;
  {
    const uint32_t init[2] = {0xFFFFFFFFu, 0u};
    CKR(cudaMemcpyAsync(mm, init, 8, cudaMemcpyHostToDevice, st));
  }
  CKR(launch_key_range(owned, n64, ctx->flags.as<uint32_t>(), mm, ctx->sms, st));
  ctx->launches += 1;
  uint32_t range[2] = {0, 0};
  CKR(cudaMemcpyAsync(range, mm, 8, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  const uint32_t span = n64 ? range[1] - range[0] : 0;
  uint32_t* out_keys = ctx->akeys.as<uint32_t>() + *n_acc;
  int64_t* out_sums = ctx->asums.as<int64_t>() + *n_acc;
  if (n64 >= (1ull << 20) && (uint64_t)span + 1 <= kDenseKeySpan) {
    // dense order-key histogram (see dense_sorted): K3's compaction writes
    // the occurring (key - min, summed change) pairs straight into the run
    // accumulator; the minimum is added back
    const uint32_t nbins = span + 1;
    AffineMap am{};
    am.keyed = 1;
    am.key_lo = range[0];
    am.packed = n64 <= kPackedMaxVoxels;
    const uint64_t hbytes = (am.packed ? 1 : 2) * (uint64_t)nbins * 8;
    CKI(ctx->hist.ensure(hbytes));
    CKI(ctx->sums.ensure((uint64_t)nbins * 8));
    CKI(ctx->finscr.ensure(16ull * (nbins / 1024 + 1)));
    CKR(cudaMemsetAsync(ctx->hist.p, 0, hbytes, st));
    CKR(launch_generic_accumulate(s, ECC_F32, true, am, ctx->hist.as<int64_t>(), nbins,
                                  ctx->flags.as<uint32_t>(), ctx->sms, st));
    CKR(launch_finalize(ctx->hist.as<int64_t>(), nbins, out_keys, out_sums,
                        ctx->sums.as<int64_t>(), ctx->count.as<uint64_t>(), ctx->finscr.p, st,
                        am.packed != 0));
    ctx->launches += 2;
    uint64_t m = 0;
    CKR(cudaMemcpyAsync(&m, ctx->count.p, 8, cudaMemcpyDeviceToHost, st));
    CKR(cudaStreamSynchronize(st));
    CKR(launch_add_key(out_keys, m, mm, ctx->sms, st));
    ctx->launches += 1;
    *n_acc += m;
    return ECC_OK;
  }
  CKR(launch_generic_changes(s, ECC_F32, ctx->ch8.as<int8_t>(), ctx->sms, st));
  CKR(launch_order_keys(owned, n64, ctx->keys.as<uint32_t>(), mm, ctx->sms, st));
  ctx->launches += 2;
  const int bit0 = 0, bit1 = span ? 32 - __builtin_clz(span) : 1;
  size_t t1 = 0, t2 = 0;
  CKR(cub::DeviceRadixSort::SortPairs(nullptr, t1, ctx->keys.as<uint32_t>(),
                                      ctx->keys2.as<uint32_t>(), ctx->ch8.as<int8_t>(),
                                      ctx->ch8b.as<int8_t>(), n, bit0, bit1, st));
  auto vals = thrust::make_transform_iterator(ctx->ch8b.as<const int8_t>(), ToI64());
  CKR(cub::DeviceReduce::ReduceByKey(nullptr, t2, ctx->keys2.as<uint32_t>(), out_keys, vals,
                                     out_sums, ctx->count.as<uint64_t>(), cub::Sum(), n, st));
  CKI(ctx->tmp.ensure(std::max(t1, t2)));
  t1 = ctx->tmp.cap;
  CKR(cub::DeviceRadixSort::SortPairs(ctx->tmp.p, t1, ctx->keys.as<uint32_t>(),
                                      ctx->keys2.as<uint32_t>(), ctx->ch8.as<int8_t>(),
                                      ctx->ch8b.as<int8_t>(), n, bit0, bit1, st));
  t2 = ctx->tmp.cap;
  CKR(cub::DeviceReduce::ReduceByKey(ctx->tmp.p, t2, ctx->keys2.as<uint32_t>(), out_keys, vals,
                                     out_sums, ctx->count.as<uint64_t>(), cub::Sum(), n, st));
  ctx->launches += 2;
  uint64_t m = 0;
  CKR(cudaMemcpyAsync(&m, ctx->count.p, 8, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  CKR(launch_add_key(out_keys, m, mm, ctx->sms, st));  // back to absolute order keys
  ctx->launches += 1;
  *n_acc += m;
  return ECC_OK;
}

// merge_local (vcec.hpp:35-66) of every slab's runs on the device: one more
// sort + reduce-by-key when there were several slabs, then the int64 prefix
// sum (vcec_to_ecc) and one copy back.
// out == nullptr: the curve stays on the device (keys in ctx->akeys, sums
// in ctx->asums, chi in ctx->chi); *m_out gets the point count.
// merge_local of the accumulated runs in place: sort (akeys, asums) by key
// into (keys2, sums2), reduce-by-key back into (akeys, asums); *m_out = the
// number of distinct keys.
int merge_runs(ecc_ctx* ctx, cudaStream_t st, uint64_t n, uint64_t* m_out) {
  if (n > 0x7FFFFFFFull) return fail(ECC_EINVAL, "too many distinct values to merge");
  uint32_t* keys = ctx->akeys.as<uint32_t>();
  int64_t* sums = ctx->asums.as<int64_t>();
  CKI(ctx->keys2.ensure(n * 4));
  CKI(ctx->sums2.ensure(n * 8));
  CKI(ctx->count.ensure(8));
  size_t t1 = 0, t2 = 0;
  CKR(cub::DeviceRadixSort::SortPairs(nullptr, t1, keys, ctx->keys2.as<uint32_t>(), sums,
                                      ctx->sums2.as<int64_t>(), (int)n, 0, 32, st));
  CKR(cub::DeviceReduce::ReduceByKey(nullptr, t2, ctx->keys2.as<uint32_t>(), keys,
                                     ctx->sums2.as<int64_t>(), sums, ctx->count.as<uint64_t>(),
                                     cub::Sum(), (int)n, st));
  CKI(ctx->tmp.ensure(std::max(t1, t2)));
  t1 = ctx->tmp.cap;
  CKR(cub::DeviceRadixSort::SortPairs(ctx->tmp.p, t1, keys, ctx->keys2.as<uint32_t>(), sums,
                                      ctx->sums2.as<int64_t>(), (int)n, 0, 32, st));
  t2 = ctx->tmp.cap;
  CKR(cub::DeviceReduce::ReduceByKey(ctx->tmp.p, t2, ctx->keys2.as<uint32_t>(), keys,
                                     ctx->sums2.as<int64_t>(), sums, ctx->count.as<uint64_t>(),
                                     cub::Sum(), (int)n, st));
  ctx->launches += 2;
  uint64_t m = 0;
  CKR(cudaMemcpyAsync(&m, ctx->count.p, 8, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  *m_out = m;
  return ECC_OK;
}

int sorted_finish(ecc_ctx* ctx, cudaStream_t st, uint64_t n, bool merge, BinResult* out,
                  uint64_t* m_out = nullptr) {
  uint64_t m = n;
  if (merge && n > 0) CKI(merge_runs(ctx, st, n, &m));
  const uint32_t* keys = ctx->akeys.as<uint32_t>();
  const int64_t* sums = ctx->asums.as<int64_t>();
  CKI(ctx->chi.ensure(std::max<uint64_t>(m, 1) * 8));
  if (m > 0) {
    size_t t3 = 0;
    CKR(cub::DeviceScan::InclusiveSum(nullptr, t3, sums, ctx->chi.as<int64_t>(), (int)m, st));
    CKI(ctx->tmp.ensure(t3));
    t3 = ctx->tmp.cap;
    CKR(cub::DeviceScan::InclusiveSum(ctx->tmp.p, t3, sums, ctx->chi.as<int64_t>(), (int)m, st));
    ctx->launches += 1;
  }
  if (m_out) *m_out = m;
  if (!out) return ECC_OK;
  out->keys.resize(m);
  out->changes.resize(m);
  out->chi.resize(m);
  if (m) {
    CKR(cudaMemcpyAsync(out->keys.data(), keys, m * 4, cudaMemcpyDeviceToHost, st));
    CKR(cudaMemcpyAsync(out->changes.data(), sums, m * 8, cudaMemcpyDeviceToHost, st));
    CKR(cudaMemcpyAsync(out->chi.data(), ctx->chi.p, m * 8, cudaMemcpyDeviceToHost, st));
  }
  CKR(cudaStreamSynchronize(st));
  return ECC_OK;
}

float key_to_float(uint32_t k) {
  const uint32_t u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

// Writes thresholds (dtype elements) for the result.
void write_values(ecc_dtype dtype, bool sorted, const AffineMap& am, const BinResult& r,
                  void* out) {
  const size_t m = sorted ? r.keys.size() : r.bins.size();
  for (size_t i = 0; i < m; ++i) {
    if (dtype == ECC_U8)
      static_cast<uint8_t*>(out)[i] = (uint8_t)r.bins[i];
    else if (dtype == ECC_U16)
      static_cast<uint16_t*>(out)[i] = (uint16_t)r.bins[i];
    else if (sorted)
      static_cast<float*>(out)[i] = key_to_float(r.keys[i]);
    else
      static_cast<float*>(out)[i] = affine_value(am, r.bins[i]);
  }
}

// General f32 over a whole resident volume when its order keys span fewer
// than 2^24 values (e.g. smoothed fields): a dense histogram indexed by
// (order key - min key) replaces the radix sort + reduce-by-key -- the
// generic stencil's HIST mode adds each voxel's change and count to its
// key's bin with global int64 atomics, and K3 compacts the occurring keys in
// ascending order, which is exactly build_index_counts' (value, summed
// change) list (value_index.hpp:159-197).  *used = false when the span is
// too wide (the sort path runs instead).  The curve is left in the result
// block (layout L); keys are bins + *key_lo.
// range_ready: flags words 1, 2 already hold the volume's order-key range
// (fused into the smoothing pass that wrote it, ecc_bench_run).
int dense_sorted(ecc_ctx* ctx, const Slab& s, cudaStream_t st, ResultLayout* L, uint32_t* key_lo,
                 bool* used, bool range_ready = false) {
  *used = false;
  const uint64_t n64 = (uint64_t)(s.own1 - s.own0) * s.w1 * s.w2;
  if (n64 < (1ull << 20)) return ECC_OK;  // small volumes: the sort is cheap
  const float* owned = static_cast<const float*>(s.base) + (s.own0 - s.plane0) * s.w1 * s.w2;
  CKI(ctx->flags.ensure(16));
  uint32_t* mm = ctx->flags.as<uint32_t>() + 1;
  if (!range_ready) {
    const uint32_t init[2] = {0xFFFFFFFFu, 0u};
    CKR(cudaMemcpyAsync(mm, init, 8, cudaMemcpyHostToDevice, st));
    CKR(launch_key_range(owned, n64, ctx->flags.as<uint32_t>(), mm, ctx->sms, st));
    ctx->launches += 1;
  }
  uint32_t range[2] = {0, 0};
  CKR(cudaMemcpyAsync(range, mm, 8, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  CKI(read_flags(ctx, st));  // NaN
  const uint64_t span = (uint64_t)(range[1] - range[0]) + 1;
  if (span > kDenseKeySpan) return ECC_OK;
  AffineMap am{};
  am.keyed = 1;
  am.key_lo = range[0];
  am.packed = n64 <= kPackedMaxVoxels;  // one 64-bit atomic per voxel (HistSink)
  const uint32_t nbins = (uint32_t)span;
  const uint64_t hbytes = (am.packed ? 1 : 2) * (uint64_t)nbins * 8;
  CKI(ctx->hist.ensure(hbytes));
  CKR(cudaMemsetAsync(ctx->hist.p, 0, hbytes, st));
  CKR(launch_generic_accumulate(s, ECC_F32, true, am, ctx->hist.as<int64_t>(), nbins,
                                ctx->flags.as<uint32_t>(), ctx->sms, st));
  ctx->launches += 1;
  *L = ResultLayout(nbins);
  CKI(ctx->res.ensure(L->bytes));  // device only: the host reads back just the m points
  uint8_t* d = ctx->res.as<uint8_t>();
  CKI(ctx->finscr.ensure(16ull * (nbins / 1024 + 1)));
  CKR(launch_finalize(ctx->hist.as<int64_t>(), nbins, reinterpret_cast<uint32_t*>(d + L->bins),
                      reinterpret_cast<int64_t*>(d + L->changes),
                      reinterpret_cast<int64_t*>(d + L->chi), reinterpret_cast<uint64_t*>(d),
                      ctx->finscr.p, st, am.packed != 0));
  ctx->launches += 1;
  *key_lo = range[0];
  *used = true;
  return ECC_OK;
}

// Whole device-resident volume -> BinResult.
int run_volume(ecc_ctx* ctx, const void* d_data, ecc_dtype dtype, ecc_dims dims,
               const ecc_binmap* bm, cudaStream_t st, BinResult* res, bool* sorted_out,
               AffineMap* am_out) {
  uint64_t nbins = 0;
  bool affine = false, sorted = false;
  AffineMap am{};
  CKI(resolve_bins(dtype, bm, &nbins, &affine, &sorted, &am));
  *sorted_out = sorted;
  *am_out = am;
  CKI(ctx->flags.ensure(4));
  CKR(cudaMemsetAsync(ctx->flags.p, 0, 4, st));
  const Slab s = make_slab(d_data, dims, 0, dims.w0, 0, dims.w0);
  if (sorted) {
    ResultLayout L(1);
    uint32_t key_lo = 0;
    bool dense = false;
    CKI(dense_sorted(ctx, s, st, &L, &key_lo, &dense));
    if (dense) {
      // read the point count, then only the m compacted points
      const uint8_t* d = ctx->res.as<uint8_t>();
      uint64_t m = 0;
      CKR(cudaMemcpyAsync(&m, d, 8, cudaMemcpyDeviceToHost, st));
      CKR(cudaStreamSynchronize(st));
      res->keys.resize(m);
      res->changes.resize(m);
      res->chi.resize(m);
      if (m) {
        CKR(cudaMemcpyAsync(res->keys.data(), d + L.bins, m * 4, cudaMemcpyDeviceToHost, st));
        CKR(cudaMemcpyAsync(res->changes.data(), d + L.changes, m * 8, cudaMemcpyDeviceToHost, st));
        CKR(cudaMemcpyAsync(res->chi.data(), d + L.chi, m * 8, cudaMemcpyDeviceToHost, st));
        CKR(cudaStreamSynchronize(st));
      }
      for (auto& k : res->keys) k += key_lo;  // bins -> order keys
      return ECC_OK;
    }
    uint64_t n = 0;
    CKI(sorted_slab(ctx, s, st, &n));
    CKI(read_flags(ctx, st));
    return sorted_finish(ctx, st, n, false, res);
  }
  Slab sp;
  CKI(pad_for_u8_fast(ctx, s, dtype, affine, st, &sp));
  if (fusable(dtype, sp, affine)) {
    ResultLayout L(nbins);
    CKI(result_block(ctx, nbins, &L));
    uint8_t* d = ctx->res.as<uint8_t>();
    CKI(launch_fused(ctx, sp, reinterpret_cast<uint32_t*>(d + L.bins),
                     reinterpret_cast<int64_t*>(d + L.changes), reinterpret_cast<int64_t*>(d + L.chi),
                     reinterpret_cast<uint64_t*>(d), st));
    return fetch_result(ctx, L, st, res);
  }
  CKI(ctx->hist.ensure(2 * nbins * 8));
  CKR(cudaMemsetAsync(ctx->hist.p, 0, 2 * nbins * 8, st));
  CKI(accumulate(ctx, s, dtype, affine, am, (uint32_t)nbins, ctx->hist.as<int64_t>(), st));
  CKI(finalize_to_host(ctx, (uint32_t)nbins, st, res));
  return ECC_OK;
}

int stage_input(ecc_ctx* ctx, const void* data, int where, uint64_t bytes,
                cudaStream_t st, const void** d_data) {
  if (where == 1) {
    *d_data = data;
    return ECC_OK;
  }
  if (where != 0) return fail(ECC_EINVAL, "where must be 0 (host) or 1 (device)");
  CKI(ctx->input.ensure(bytes));
  CKR(cudaMemcpyAsync(ctx->input.p, data, bytes, cudaMemcpyHostToDevice, st));
  *d_data = ctx->input.p;
  return ECC_OK;
}

// Spill rows of the u16 batched kernel: one int32[65536] row per SM id
// (%smid < 256 on every part this targets), zeroed once and kept zero by
// the kernel itself.
int batch_scratch(ecc_ctx* ctx, ecc_dtype dtype, cudaStream_t st) {
  if (dtype != ECC_U16 || ctx->bscratch.p) return ECC_OK;
  const size_t bytes = 256ull * 65536 * 4;
  CKI(ctx->bscratch.ensure(bytes));
  CKR(cudaMemsetAsync(ctx->bscratch.p, 0, bytes, st));
  return ECC_OK;
}

// gaussian_kernel (datagen.hpp:66-79), restated on the host with the same
// double arithmetic and libm exp, so the taps are bit-identical.
int gaussian_weights(double sigma, int width, std::vector<double>* w) {
  if (width < 1 || width % 2 == 0)
    return fail(ECC_EINVAL, "Gaussian kernel width must be odd and >= 1");
  if (width > gaussian_max_width())
    return fail(ECC_EINVAL, "Gaussian kernel width " + std::to_string(width) + " exceeds " +
                                std::to_string(gaussian_max_width()));
  w->assign(width, 0.0);
  const int half = width / 2;
  double sum = 0;
  for (int i = -half; i <= half; ++i) {
    const double v = width == 1 ? 1.0 : std::exp(-(double(i) * i) / (2.0 * sigma * sigma));
    (*w)[i + half] = v;
    sum += v;
  }
  for (double& v : *w) v /= sum;
  return ECC_OK;
}

// gaussian_smooth (datagen.hpp:108-122): axes 0, 1, 2 in turn, each skipped
// when its extent or the width is 1; in may equal out.
// mm (optional): the last pass also reduces the result's order-key range
// into mm[0..1] and NaN into ctx->flags; *ranged says whether it could.
int smooth_device(ecc_ctx* ctx, const float* in, float* out, ecc_dims d, double sigma, int width,
                  cudaStream_t st, uint32_t* mm = nullptr, bool* ranged = nullptr) {
  if (ranged) *ranged = false;
  std::vector<double> w;
  CKI(gaussian_weights(sigma, width, &w));
  const uint64_t n = d.w0 * d.w1 * d.w2;
  const uint64_t ext[3] = {d.w0, d.w1, d.w2};
  int axes[3], na = 0;
  for (int a = 0; a < 3; ++a)
    if (ext[a] > 1 && width > 1) axes[na++] = a;
  if (na == 0) {
    if (in != out) CKR(cudaMemcpyAsync(out, in, n * 4, cudaMemcpyDeviceToDevice, st));
    return ECC_OK;
  }
  CKI(ctx->sm_w.ensure(w.size() * 8));
  CKR(cudaMemcpyAsync(ctx->sm_w.p, w.data(), w.size() * 8, cudaMemcpyHostToDevice, st));
  CKI(ctx->sm_tmp[0].ensure(n * 4));
  if (na > 2) CKI(ctx->sm_tmp[1].ensure(n * 4));
  const float* src = in;
  // in place with a single active axis: the pass must not write what it reads
  const bool via_tmp = na == 1 && in == out;
  for (int j = 0; j < na; ++j) {
    float* dst = (j == na - 1 && !via_tmp) ? out : ctx->sm_tmp[j & 1].as<float>();
    const bool last = j == na - 1 && !via_tmp && mm;
    CKR(launch_convolve_axis(src, dst, d.w0, d.w1, d.w2, axes[j], ctx->sm_w.as<double>(), width,
                             st, last ? mm : nullptr, last ? ctx->flags.as<uint32_t>() : nullptr,
                             last ? ranged : nullptr));
    ctx->launches += 1;
    src = dst;
  }
  if (via_tmp) CKR(cudaMemcpyAsync(out, src, n * 4, cudaMemcpyDeviceToDevice, st));
  // (a pageable-source async copy returns once the taps are staged, so `w`
  // may go out of scope here)
  return ECC_OK;
}

}  // namespace

// ===================================================================== ABI
extern "C" {

int ecc_abi_version(void) { return ECC_B200_ABI_VERSION; }

const char* ecc_last_error(void) { return g_err.c_str(); }

int ecc_ctx_create(int device, ecc_ctx** out) {
  if (!out) return fail(ECC_EINVAL, "null output pointer");
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(ECC_ECUDA, std::string("no CUDA device available: ") +
                               (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
  }
  if (device < 0 || device >= ndev)
    return fail(ECC_EINVAL, "device " + std::to_string(device) + " out of range");
  CKR(cudaSetDevice(device));
  auto* ctx = new ecc_ctx();
  ctx->device = device;
  CKR(cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device));
  CKR(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  CKR(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
  *out = ctx;
  return ECC_OK;
}

void ecc_ctx_destroy(ecc_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  for (cudaEvent_t& e : ctx->ov_ev)
    if (e) cudaEventDestroy(e);
  cudaStreamSynchronize(ctx->stream);
  cudaStreamSynchronize(ctx->copy);
  for (DevBuf* b : {&ctx->input, &ctx->hist, &ctx->bins, &ctx->changes, &ctx->chi,
                    &ctx->count, &ctx->flags, &ctx->keys, &ctx->keys2, &ctx->ch8,
                    &ctx->ch8b, &ctx->sums, &ctx->tmp, &ctx->slab[0], &ctx->slab[1], &ctx->slab[2],
                    &ctx->fused, &ctx->bscratch, &ctx->nanidx, &ctx->pad,
                    &ctx->keys16, &ctx->finscr, &ctx->res, &ctx->akeys,
                    &ctx->asums, &ctx->sums2, &ctx->sm_tmp[0], &ctx->sm_tmp[1], &ctx->sm_w})
    b->release();
  ctx->staging[0].release();
  ctx->staging[1].release();
  ctx->host_small.release();
  ctx->res_host.release();
  cudaStreamDestroy(ctx->stream);
  cudaStreamDestroy(ctx->copy);
  delete ctx;
}

void* ecc_ctx_stream(ecc_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

uint64_t ecc_ctx_launch_count(ecc_ctx* ctx) { return ctx ? ctx->launches : 0; }

int ecc_bin_count(ecc_dtype dtype, const ecc_binmap* bm, uint64_t* nbins) {
  CKI(check_dtype(dtype));
  bool a, s;
  AffineMap am;
  return resolve_bins(dtype, bm, nbins, &a, &s, &am);
}

int ecc_accumulate_slab(ecc_ctx* ctx, const void* d_planes, ecc_dtype dtype,
                        ecc_dims image, uint64_t plane0, uint64_t nplanes,
                        uint64_t own0, uint64_t own1, const ecc_binmap* bm,
                        int64_t* d_hist, void* stream) {
  CKI(bind(ctx));
  CKI(check_dtype(dtype));
  CKI(check_slab(image, plane0, nplanes, own0, own1));
  if (!d_planes || !d_hist) return fail(ECC_EINVAL, "null device pointer");
  uint64_t nbins;
  bool affine, sorted;
  AffineMap am{};
  CKI(resolve_bins(dtype, bm, &nbins, &affine, &sorted, &am));
  if (sorted) return fail(ECC_EINVAL, "the sorted bin map has no dense histogram");
  cudaStream_t st = pick(ctx, stream);
  CKI(ctx->flags.ensure(4));
  CKR(cudaMemsetAsync(ctx->flags.p, 0, 4, st));
  const Slab s = make_slab(d_planes, image, plane0, nplanes, own0, own1);
  CKI(accumulate(ctx, s, dtype, affine, am, (uint32_t)nbins, d_hist, st));
  if (affine) CKI(read_flags(ctx, st));
  return ECC_OK;
}

int ecc_compute_changes(ecc_ctx* ctx, const void* d_planes, ecc_dtype dtype,
                        ecc_dims image, uint64_t plane0, uint64_t nplanes,
                        uint64_t own0, uint64_t own1, int8_t* d_out, void* stream) {
  CKI(bind(ctx));
  CKI(check_dtype(dtype));
  CKI(check_slab(image, plane0, nplanes, own0, own1));
  if (!d_planes || !d_out) return fail(ECC_EINVAL, "null device pointer");
  const Slab s = make_slab(d_planes, image, plane0, nplanes, own0, own1);
  bool handled = false;
  CKR(launch_changes_fast(s, (int)dtype, d_out, ctx->sms, pick(ctx, stream), &handled));
  if (!handled) CKR(launch_generic_changes(s, (int)dtype, d_out, ctx->sms, pick(ctx, stream)));
  ctx->launches += 1;
  return ECC_OK;
}

int ecc_curve_device(ecc_ctx* ctx, const void* d_data, ecc_dtype dtype, ecc_dims dims,
                     const ecc_binmap* bm, uint32_t* d_bins, int64_t* d_changes, int64_t* d_chi,
                     uint64_t* d_count, void* stream) {
  CKI(bind(ctx));
  CKI(check_dtype(dtype));
  CKI(check_dims(dims));
  if (!d_data || !d_bins || !d_changes || !d_chi || !d_count)
    return fail(ECC_EINVAL, "null device pointer");
  uint64_t nbins;
  bool affine, sorted;
  AffineMap am{};
  CKI(resolve_bins(dtype, bm, &nbins, &affine, &sorted, &am));
  if (sorted) return fail(ECC_EINVAL, "the sorted bin map has no device-side curve; use ecc_curve");
  cudaStream_t st = pick(ctx, stream);
  const Slab s = make_slab(d_data, dims, 0, dims.w0, 0, dims.w0);
  Slab sp;
  CKI(pad_for_u8_fast(ctx, s, dtype, affine, st, &sp));
  if (fusable(dtype, sp, affine)) return launch_fused(ctx, sp, d_bins, d_changes, d_chi, d_count, st);
  CKI(ctx->flags.ensure(4));
  CKR(cudaMemsetAsync(ctx->flags.p, 0, 4, st));
  CKI(ctx->hist.ensure(2 * nbins * 8));
  CKR(cudaMemsetAsync(ctx->hist.p, 0, 2 * nbins * 8, st));
  CKI(accumulate(ctx, s, dtype, affine, am, (uint32_t)nbins, ctx->hist.as<int64_t>(), st));
  CKI(ctx->finscr.ensure(16ull * (nbins / 1024 + 1)));
  CKR(launch_finalize(ctx->hist.as<int64_t>(), (uint32_t)nbins, d_bins, d_changes, d_chi, d_count,
                      ctx->finscr.p, st));
  ctx->launches += 1;
  if (affine) CKI(read_flags(ctx, st));
  return ECC_OK;
}

int ecc_finalize(ecc_ctx* ctx, const int64_t* d_hist, uint64_t nbins, uint32_t* d_bins,
                 int64_t* d_changes, int64_t* d_chi, uint64_t* d_count, void* stream) {
  CKI(bind(ctx));
  if (!d_hist || !d_bins || !d_changes || !d_chi || !d_count)
    return fail(ECC_EINVAL, "null device pointer");
  if (nbins < 1 || nbins > (1u << 24)) return fail(ECC_EINVAL, "bad bin count");
  CKI(ctx->finscr.ensure(16ull * (nbins / 1024 + 1)));
  CKR(launch_finalize(d_hist, (uint32_t)nbins, d_bins, d_changes, d_chi, d_count, ctx->finscr.p,
                      pick(ctx, stream)));
  ctx->launches += 1;
  return ECC_OK;
}

// A large 3D u8 image in host memory: the H2D copy is split into plane
// chunks on the copy stream and each chunk's K1+K2 runs on the compute
// stream as soon as it and the next chunk (its halo plane) have landed, so
// only the last chunk's kernel and K3 remain after the copy; the image is
// still one resident volume (one TMA descriptor), chunks differ only in
// their owned planes.  Returns handled = false when the shape does not fit.
int overlapped_u8(ecc_ctx* ctx, const void* host, ecc_dims dims, cudaStream_t st, BinResult* r,
                  bool* handled) {
  *handled = false;
  const uint64_t plane = dims.w1 * dims.w2, bytes = dims.w0 * plane;
  if (dims.w2 <= 1 || bytes < (32ull << 20) || dims.w0 < 8) return ECC_OK;
  static const char* env = std::getenv("ECC_B200_OVERLAP_CHUNKS");  // tuning / A-B hook
  const int env_nc = env ? std::atoi(env) : -1;
  if (env_nc == 0) return ECC_OK;
  CKI(ctx->input.ensure(bytes));
  const Slab s = make_slab(ctx->input.p, dims, 0, dims.w0, 0, dims.w0);
  if (!u8_3d_supported(s)) return ECC_OK;
  // 16 MB chunks, at most 8 (measured on C2, 128 MB: 1 chunk 3.31 ms, 2: 2.62,
  // 4: 2.57, 8: 2.56, 16: 3.40 -- many small copies lose DMA efficiency)
  int nc = (int)std::min<uint64_t>(8, std::min<uint64_t>(dims.w0 / 4, bytes >> 24));
  if (env_nc > 0) nc = (int)std::min<uint64_t>(std::min(env_nc, 16), dims.w0);
  nc = std::max(nc, 1);
  for (int k = 0; k <= nc; ++k)
    if (!ctx->ov_ev[k]) CKR(cudaEventCreateWithFlags(&ctx->ov_ev[k], cudaEventDisableTiming));
  // every chunk accumulates into the fused workspace's histogram (zero by
  // invariant); the last chunk's launch also runs K3 (last-CTA ticket) into
  // the result block and re-zeroes the workspace
  if (!ctx->fused.p) {
    CKI(ctx->fused.ensure(256 + 512 * 8));
    CKR(cudaMemsetAsync(ctx->fused.p, 0, 256 + 512 * 8, st));
  }
  int64_t* ghist = reinterpret_cast<int64_t*>(ctx->fused.as<uint8_t>() + 256);
  ResultLayout L(256);
  CKI(result_block(ctx, 256, &L));
  uint8_t* rb = ctx->res.as<uint8_t>();
  U83dFinalize fz{ctx->fused.as<uint32_t>(), reinterpret_cast<uint32_t*>(rb + L.bins),
                  reinterpret_cast<int64_t*>(rb + L.changes), reinterpret_cast<int64_t*>(rb + L.chi),
                  reinterpret_cast<uint64_t*>(rb)};
  // copies start after everything already queued on the compute stream
  CKR(cudaEventRecord(ctx->ov_ev[nc], st));
  CKR(cudaStreamWaitEvent(ctx->copy, ctx->ov_ev[nc], 0));
  std::vector<uint64_t> b(nc + 1);
  // tapered chunks (sizes proportional to nc, nc-1, ..., 1): few copies
  // early, a small last chunk whose kernel is all that trails the copy
  // (C2: 2516 us tapered vs 2533 us equal chunks end to end)
  {
    const uint64_t tot = (uint64_t)nc * (nc + 1) / 2;
    uint64_t acc = 0;
    for (int k = 0; k <= nc; ++k) {
      b[k] = dims.w0 * acc / tot;
      if (k < nc) acc += (uint64_t)(nc - k);
    }
    b[nc] = dims.w0;
    for (int k = 1; k <= nc; ++k)
      if (b[k] <= b[k - 1]) return ECC_OK;  // degenerate split: the one-shot path
  }
  int rc = ECC_OK;
  for (int k = 0; k < nc && rc == ECC_OK; ++k) {
    cudaError_t e = cudaMemcpyAsync(ctx->input.as<uint8_t>() + b[k] * plane,
                                    static_cast<const uint8_t*>(host) + b[k] * plane,
                                    (b[k + 1] - b[k]) * plane, cudaMemcpyHostToDevice, ctx->copy);
    if (e == cudaSuccess) e = cudaEventRecord(ctx->ov_ev[k], ctx->copy);
    if (e != cudaSuccess) rc = fail(ECC_ECUDA, cudaGetErrorString(e));
  }
  for (int k = 0; k < nc && rc == ECC_OK; ++k) {
    cudaError_t e = cudaStreamWaitEvent(st, ctx->ov_ev[k], 0);
    if (e == cudaSuccess && k + 1 < nc) e = cudaStreamWaitEvent(st, ctx->ov_ev[k + 1], 0);
    Slab sk = s;
    sk.own0 = (int64_t)b[k];
    sk.own1 = (int64_t)b[k + 1];
    if (e == cudaSuccess)
      e = launch_u8_3d(sk, ghist, nullptr, ctx->sms, st, k == nc - 1 ? &fz : nullptr);
    if (e != cudaSuccess) rc = fail(ECC_ECUDA, cudaGetErrorString(e));
    ctx->launches += 1;
  }
  if (rc == ECC_OK) rc = fetch_result(ctx, L, st, r);
  if (rc != ECC_OK) {
    // no copy into ctx->input may outlive the call, and the fused workspace
    // must be zero again for the next launch
    cudaStreamSynchronize(ctx->copy);
    cudaStreamSynchronize(st);
    cudaMemset(ctx->fused.p, 0, 256 + 512 * 8);
    return rc;
  }
  *handled = true;
  return ECC_OK;
}

// The same overlap for the other dense maps (u16, affine f32): tapered
// chunks copied on the copy stream, each chunk's K1+K2 on a slab view of the
// resident volume (its planes + halo, so the f32 -> bin key pass covers just
// those planes) as soon as it has landed, K3 after the last.
int overlapped_dense(ecc_ctx* ctx, const void* host, ecc_dtype dtype, ecc_dims dims,
                     const ecc_binmap* bm, cudaStream_t st, BinResult* r, AffineMap* am_out,
                     bool* handled) {
  *handled = false;
  uint64_t nbins = 0;
  bool affine = false, sorted = false;
  AffineMap am{};
  CKI(resolve_bins(dtype, bm, &nbins, &affine, &sorted, &am));
  const uint64_t plane = dims.w1 * dims.w2, eb = esize(dtype), bytes = dims.w0 * plane * eb;
  if (sorted || dtype == ECC_U8 || dims.w2 <= 1 || bytes < (32ull << 20) || dims.w0 < 8)
    return ECC_OK;
  int nc = (int)std::min<uint64_t>(8, std::min<uint64_t>(dims.w0 / 4, bytes >> 24));
  nc = std::max(nc, 1);
  std::vector<uint64_t> b(nc + 1);
  {
    const uint64_t tot = (uint64_t)nc * (nc + 1) / 2;
    uint64_t acc = 0;
    for (int k = 0; k <= nc; ++k) {
      b[k] = dims.w0 * acc / tot;
      if (k < nc) acc += (uint64_t)(nc - k);
    }
    b[nc] = dims.w0;
    for (int k = 1; k <= nc; ++k)
      if (b[k] <= b[k - 1]) return ECC_OK;
  }
  CKI(ctx->input.ensure(bytes));
  for (int k = 0; k <= nc; ++k)
    if (!ctx->ov_ev[k]) CKR(cudaEventCreateWithFlags(&ctx->ov_ev[k], cudaEventDisableTiming));
  CKI(ctx->flags.ensure(16));
  CKI(ctx->hist.ensure(2 * nbins * 8));
  CKR(cudaMemsetAsync(ctx->flags.p, 0, 4, st));
  CKR(cudaMemsetAsync(ctx->hist.p, 0, 2 * nbins * 8, st));
  CKR(cudaEventRecord(ctx->ov_ev[nc], st));
  CKR(cudaStreamWaitEvent(ctx->copy, ctx->ov_ev[nc], 0));
  int rc = ECC_OK;
  for (int k = 0; k < nc && rc == ECC_OK; ++k) {
    cudaError_t e = cudaMemcpyAsync(ctx->input.as<uint8_t>() + b[k] * plane * eb,
                                    static_cast<const uint8_t*>(host) + b[k] * plane * eb,
                                    (b[k + 1] - b[k]) * plane * eb, cudaMemcpyHostToDevice,
                                    ctx->copy);
    if (e == cudaSuccess) e = cudaEventRecord(ctx->ov_ev[k], ctx->copy);
    if (e != cudaSuccess) rc = fail(ECC_ECUDA, cudaGetErrorString(e));
  }
  for (int k = 0; k < nc && rc == ECC_OK; ++k) {
    cudaError_t e = cudaStreamWaitEvent(st, ctx->ov_ev[k], 0);
    if (e == cudaSuccess && k + 1 < nc) e = cudaStreamWaitEvent(st, ctx->ov_ev[k + 1], 0);
    if (e != cudaSuccess) {
      rc = fail(ECC_ECUDA, cudaGetErrorString(e));
      break;
    }
    const uint64_t r0 = b[k] == 0 ? 0 : b[k] - 1;
    const uint64_t r1 = std::min<uint64_t>(b[k + 1] + 1, dims.w0);
    const Slab sk = make_slab(ctx->input.as<uint8_t>() + r0 * plane * eb, dims, r0, r1 - r0, b[k],
                              b[k + 1]);
    rc = accumulate(ctx, sk, dtype, affine, am, (uint32_t)nbins, ctx->hist.as<int64_t>(), st);
  }
  if (rc == ECC_OK && affine) rc = read_flags(ctx, st);
  if (rc == ECC_OK) rc = finalize_to_host(ctx, (uint32_t)nbins, st, r);
  if (rc != ECC_OK) {
    cudaStreamSynchronize(ctx->copy);
    return rc;
  }
  *am_out = am;
  *handled = true;
  return ECC_OK;
}

static int volume_common(ecc_ctx* ctx, const void* data, int where, ecc_dtype dtype,
                         ecc_dims dims, const ecc_binmap* bm, void* values_out,
                         int64_t* series_out, uint64_t cap, uint64_t* n_out, bool want_chi) {
  CKI(bind(ctx));
  CKI(check_dtype(dtype));
  CKI(check_dims(dims));
  if (!data || !values_out || !series_out || !n_out) return fail(ECC_EINVAL, "null pointer");
  cudaStream_t st = ctx->stream;
  const uint64_t bytes = dims.w0 * dims.w1 * dims.w2 * esize(dtype);
  // every path reports the error flags of THIS call (fetch_result copies
  // them into the result block): clear what an earlier rejected call left
  CKI(ctx->flags.ensure(16));
  CKR(cudaMemsetAsync(ctx->flags.p, 0, 4, st));
  BinResult& r = ctx->hres;
  bool sorted = false;
  AffineMap am{};
  bool done = false;
  if (where == 0 && dtype == ECC_U8 && (!bm || bm->kind == ECC_BIN_IDENTITY))
    CKI(overlapped_u8(ctx, data, dims, st, &r, &done));
  else if (where == 0)
    CKI(overlapped_dense(ctx, data, dtype, dims, bm, st, &r, &am, &done));
  if (!done) {
    const void* d_data = nullptr;
    CKI(stage_input(ctx, data, where, bytes, st, &d_data));
    CKI(run_volume(ctx, d_data, dtype, dims, bm, st, &r, &sorted, &am));
  }
  const size_t m = r.changes.size();
  *n_out = m;
  if (m > cap) return fail(ECC_EINVAL, "output capacity " + std::to_string(cap) +
                                           " is below the " + std::to_string(m) + " values");
  write_values(dtype, sorted, am, r, values_out);
  std::memcpy(series_out, want_chi ? r.chi.data() : r.changes.data(), m * 8);
  return ECC_OK;
}

int ecc_vcec(ecc_ctx* ctx, const void* data, int where, ecc_dtype dtype, ecc_dims dims,
             const ecc_binmap* bm, void* values_out, int64_t* changes_out, uint64_t cap,
             uint64_t* n_out) {
  return volume_common(ctx, data, where, dtype, dims, bm, values_out, changes_out, cap,
                       n_out, false);
}

int ecc_curve(ecc_ctx* ctx, const void* data, int where, ecc_dtype dtype, ecc_dims dims,
              const ecc_binmap* bm, void* thresholds_out, int64_t* chi_out, uint64_t cap,
              uint64_t* n_out) {
  return volume_common(ctx, data, where, dtype, dims, bm, thresholds_out, chi_out, cap,
                       n_out, true);
}

// Raw-file fixups done on the device right after each chunk's H2D
// (image.hpp:39-52): byte swap of big-endian f32 and NaN rejection.
struct Fixup {
  bool active = false;
  bool big_endian = false;
};

static int stream_impl(ecc_ctx* ctx, ecc_read_rows_fn read_rows, void* user,
                       ecc_dtype dtype, ecc_dims dims, const uint64_t* bounds,
                       size_t nchunks, const ecc_binmap* bm, ecc_chunk_timing* timings,
                       void* values_out, int64_t* changes_out, uint64_t cap,
                       uint64_t* n_out, Fixup fix) {
  CKI(bind(ctx));
  CKI(check_dtype(dtype));
  if (dims.w0 < 1) return fail(ECC_EINVAL, "w0 must be >= 1");
  CKI(check_dims(dims));
  if (!read_rows || !values_out || !changes_out || !n_out)
    return fail(ECC_EINVAL, "null pointer");
  CKI(check_plan(bounds, nchunks, dims));
  uint64_t nbins = 0;
  bool affine = false, sorted = false;
  AffineMap am{};
  CKI(resolve_bins(dtype, bm, &nbins, &affine, &sorted, &am));

  const auto t0 = std::chrono::steady_clock::now();
  auto since = [&] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  const uint64_t row_bytes = dims.w1 * dims.w2 * esize(dtype);
  uint64_t max_rows = 0;
  for (size_t k = 0; k < nchunks; ++k)
    max_rows = std::max<uint64_t>(max_rows, bounds[k + 1] - bounds[k] + 2);
  max_rows = std::min<uint64_t>(max_rows, dims.w0);
  const uint64_t buf_bytes = max_rows * row_bytes;
  for (int b = 0; b < 2; ++b) {
    CKI(ctx->staging[b].ensure(buf_bytes));
    CKI(ctx->slab[b].ensure(buf_bytes));
  }
  CKI(ctx->flags.ensure(4));
  cudaStream_t st = ctx->stream, cp = ctx->copy;
  CKR(cudaMemsetAsync(ctx->flags.p, 0, 4, st));
  if (!sorted) {
    CKI(ctx->hist.ensure(2 * nbins * 8));
    CKR(cudaMemsetAsync(ctx->hist.p, 0, 2 * nbins * 8, st));
  }
  cudaEvent_t ev0, h2d_done[2], used[2], kb[2], ke[2];
  CKR(cudaEventCreate(&ev0));
  for (int b = 0; b < 2; ++b) {
    CKR(cudaEventCreate(&h2d_done[b]));
    CKR(cudaEventCreate(&used[b]));
    CKR(cudaEventCreate(&kb[b]));
    CKR(cudaEventCreate(&ke[b]));
  }
  if (fix.active) {
    CKI(ctx->nanidx.ensure(8 * nchunks));
    CKR(cudaMemsetAsync(ctx->nanidx.p, 0xFF, 8 * nchunks, st));
  }
  CKR(cudaEventRecord(ev0, st));
  // map device event times onto the host clock of the ChunkTiming fields
  CKR(cudaEventSynchronize(ev0));
  const double t_ev0 = since();
  uint64_t sorted_n = 0;  // (key, sum) runs accumulated on the device
  std::vector<ecc_chunk_timing> tim(nchunks);
  std::vector<double> h2d_end_host(nchunks, 0);
  int rc = ECC_OK;
  bool pending[2] = {false, false};
  size_t pending_k[2] = {0, 0};
  auto harvest = [&](int b) -> int {
    // event timings for the chunk that last used buffer b
    if (!pending[b]) return ECC_OK;
    CKR(cudaEventSynchronize(ke[b]));
    float a = 0, c = 0;
    CKR(cudaEventElapsedTime(&a, ev0, kb[b]));
    CKR(cudaEventElapsedTime(&c, ev0, ke[b]));
    ecc_chunk_timing& t = tim[pending_k[b]];
    t.kernel_begin = t_ev0 + a * 1e-3;
    t.kernel_end = t_ev0 + c * 1e-3;
    pending[b] = false;
    return ECC_OK;
  };
  for (size_t k = 0; k < nchunks && rc == ECC_OK; ++k) {
    const int b = (int)(k & 1);
    const uint64_t own0 = bounds[k], own1 = bounds[k + 1];
    const uint64_t r0 = own0 == 0 ? 0 : own0 - 1;
    const uint64_t r1 = std::min<uint64_t>(own1 + 1, dims.w0);
    // the pinned buffer b was last read by the H2D copy of chunk k-2
    CKR(cudaEventSynchronize(used[b]));
    ecc_chunk_timing& t = tim[k];
    t.begin = own0;
    t.end = own1;
    t.ingest_begin = since();
    char errbuf[512] = {0};
    const int src = read_rows(user, r0, r1, ctx->staging[b].p, errbuf, sizeof errbuf);
    if (src != 0) {
      rc = fail(ECC_ESOURCE, "ingestion of chunk " + std::to_string(k) + " failed: " +
                                 std::string(errbuf[0] ? errbuf : "read_rows failed"));
      break;
    }
    // the device buffer b was last read by the kernel of chunk k-2
    CKR(cudaStreamWaitEvent(cp, ke[b], 0));
    CKR(cudaMemcpyAsync(ctx->slab[b].p, ctx->staging[b].p, (r1 - r0) * row_bytes,
                        cudaMemcpyHostToDevice, cp));
    CKR(cudaEventRecord(used[b], cp));
    CKR(cudaEventRecord(h2d_done[b], cp));
    t.ingest_end = since();
    t.index_begin = t.index_end = t.ingest_end;
    CKI(harvest(b));
    CKR(cudaStreamWaitEvent(st, h2d_done[b], 0));
    CKR(cudaEventRecord(kb[b], st));
    if (fix.active) {
      CKR(launch_fixup(ctx->slab[b].p, (int)dtype, (r1 - r0) * dims.w1 * dims.w2,
                       r0 * dims.w1 * dims.w2, fix.big_endian,
                       ctx->nanidx.as<unsigned long long>() + k, ctx->sms, st));
      ctx->launches += 1;
    }
    const Slab s = make_slab(ctx->slab[b].p, dims, r0, r1 - r0, own0, own1);
    t.merge_begin = since();
    if (sorted) {
      CKI(sorted_slab(ctx, s, st, &sorted_n));
    } else {
      CKI(accumulate(ctx, s, dtype, affine, am, (uint32_t)nbins, ctx->hist.as<int64_t>(), st));
    }
    CKR(cudaEventRecord(ke[b], st));
    t.merge_end = since();
    pending[b] = true;
    pending_k[b] = k;
  }
  for (int b = 0; b < 2 && rc == ECC_OK; ++b) CKI(harvest(b));
  CKR(cudaStreamSynchronize(st));
  CKR(cudaStreamSynchronize(cp));
  for (int b = 0; b < 2; ++b) {
    cudaEventDestroy(h2d_done[b]);
    cudaEventDestroy(used[b]);
    cudaEventDestroy(kb[b]);
    cudaEventDestroy(ke[b]);
  }
  cudaEventDestroy(ev0);
  if (rc != ECC_OK) return rc;
  if (fix.active) {  // the first chunk (in plan order) whose rows held a NaN
    std::vector<unsigned long long> nan(nchunks);
    CKR(cudaMemcpyAsync(nan.data(), ctx->nanidx.p, 8 * nchunks, cudaMemcpyDeviceToHost, st));
    CKR(cudaStreamSynchronize(st));
    for (size_t k = 0; k < nchunks; ++k)
      if (nan[k] != ~0ull)
        return fail(ECC_ESOURCE, "ingestion of chunk " + std::to_string(k) +
                                     " failed: NaN value at linear index " + std::to_string(nan[k]));
  }
  BinResult& r = ctx->hres;
  if (sorted) {
    CKI(read_flags(ctx, st));
    CKI(sorted_finish(ctx, st, sorted_n, nchunks > 1, &r));
  } else {
    CKI(finalize_to_host(ctx, (uint32_t)nbins, st, &r));
  }
  // merge phase = the device-side reduction; report it after the kernel
  for (auto& t : tim) {
    t.merge_begin = t.kernel_end;
    t.merge_end = t.kernel_end;
  }
  if (timings) std::memcpy(timings, tim.data(), nchunks * sizeof(ecc_chunk_timing));
  const size_t m = r.changes.size();
  *n_out = m;
  if (m > cap) return fail(ECC_EINVAL, "output capacity below the number of values");
  write_values(dtype, sorted, am, r, values_out);
  std::memcpy(changes_out, r.changes.data(), m * 8);
  return ECC_OK;
}

int ecc_process_stream(ecc_ctx* ctx, ecc_read_rows_fn read_rows, void* user,
                       ecc_dtype dtype, ecc_dims dims, const uint64_t* bounds,
                       size_t nchunks, const ecc_binmap* bm, ecc_chunk_timing* timings,
                       void* values_out, int64_t* changes_out, uint64_t cap,
                       uint64_t* n_out) {
  return stream_impl(ctx, read_rows, user, dtype, dims, bounds, nchunks, bm, timings, values_out,
                     changes_out, cap, n_out, Fixup{});
}

namespace {
struct FileReader {
  int fd = -1;
  std::string path;
  uint64_t row_bytes = 0;
};

int file_read_rows(void* user, uint64_t r0, uint64_t r1, void* dst, char* errbuf,
                   size_t errlen) {
  auto* f = static_cast<FileReader*>(user);
  uint64_t off = r0 * f->row_bytes, left = (r1 - r0) * f->row_bytes;
  char* p = static_cast<char*>(dst);
  while (left) {
    const ssize_t n = pread(f->fd, p, std::min<uint64_t>(left, 1ull << 30), (off_t)off);
    if (n <= 0) {
      std::snprintf(errbuf, errlen, "read failure on '%s' at row %llu", f->path.c_str(),
                    (unsigned long long)r0);
      return 1;
    }
    p += n;
    off += (uint64_t)n;
    left -= (uint64_t)n;
  }
  return 0;
}
}  // namespace

int ecc_process_file(ecc_ctx* ctx, const char* path, ecc_dtype dtype, ecc_dims dims,
                     int big_endian, const uint64_t* bounds, size_t nchunks,
                     const ecc_binmap* bm, ecc_chunk_timing* timings, void* values_out,
                     int64_t* changes_out, uint64_t cap, uint64_t* n_out) {
  CKI(bind(ctx));
  CKI(check_dtype(dtype));
  CKI(check_dims(dims));
  if (!path) return fail(ECC_EINVAL, "null path");
  FileReader f;
  f.path = path;
  f.row_bytes = dims.w1 * dims.w2 * esize(dtype);
  f.fd = open(path, O_RDONLY);
  if (f.fd < 0) return fail(ECC_ESOURCE, std::string("cannot open '") + path + "'");
  struct stat stt;
  const uint64_t expected = dims.w0 * f.row_bytes;
  if (fstat(f.fd, &stt) != 0) {
    close(f.fd);
    return fail(ECC_ESOURCE, std::string("cannot stat '") + path + "'");
  }
  if ((uint64_t)stt.st_size != expected) {
    close(f.fd);
    return fail(ECC_EINVAL, std::string("size mismatch for '") + path + "': expected " +
                                std::to_string(expected) + " bytes for dims " + dims_str(dims) +
                                ", found " + std::to_string((uint64_t)stt.st_size));
  }
  Fixup fix;
  fix.active = dtype == ECC_F32;  // u8 / u16 files need neither swap nor NaN check
  fix.big_endian = big_endian != 0;
  const int rc = stream_impl(ctx, file_read_rows, &f, dtype, dims, bounds, nchunks, bm, timings,
                             values_out, changes_out, cap, n_out, fix);
  close(f.fd);
  return rc;
}

}  // extern "C"

namespace {

// The pipelined host-DMA loop shared by ecc_process_host and
// ecc_accumulate_host: chunk k's planes + halo are copied (copy stream) from
// the caller's host buffer -- which holds image planes [plane0, plane0 +
// nheld) -- into one of three device slabs while earlier chunks' kernels run
// (compute stream), accumulating into `hist`.  Synchronous.
int host_pipeline(ecc_ctx* ctx, const void* host, uint64_t plane0, uint64_t nheld,
                  ecc_dtype dtype, ecc_dims dims, const uint64_t* bounds, size_t nchunks,
                  bool affine, const AffineMap& am, uint64_t nbins, int64_t* hist,
                  ecc_chunk_timing* timings) {
  const auto t0 = std::chrono::steady_clock::now();
  auto since = [&] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  const uint64_t row_bytes = dims.w1 * dims.w2 * esize(dtype);
  uint64_t max_rows = 0;
  for (size_t k = 0; k < nchunks; ++k) {
    const uint64_t r0 = bounds[k] == 0 ? 0 : bounds[k] - 1;
    const uint64_t r1 = std::min<uint64_t>(bounds[k + 1] + 1, dims.w0);
    if (r0 < plane0 || r1 > plane0 + nheld)
      return fail(ECC_EINVAL, "chunk " + std::to_string(k) + " needs planes [" +
                                  std::to_string(r0) + ", " + std::to_string(r1) +
                                  ") but the host buffer holds [" + std::to_string(plane0) +
                                  ", " + std::to_string(plane0 + nheld) + ")");
    max_rows = std::max<uint64_t>(max_rows, r1 - r0);
  }
  constexpr int NB = 3;  // device slab buffers in flight
  for (int b = 0; b < NB; ++b) CKI(ctx->slab[b].ensure(max_rows * row_bytes));
  cudaStream_t st = ctx->stream, cp = ctx->copy;
  std::vector<cudaEvent_t> ev(4 * nchunks + 1);
  for (auto& e : ev) CKR(cudaEventCreate(&e));
  auto evh0 = [&](size_t k) { return ev[4 * k + 0]; };  // H2D begin
  auto evh1 = [&](size_t k) { return ev[4 * k + 1]; };  // H2D end
  auto evk0 = [&](size_t k) { return ev[4 * k + 2]; };  // kernel begin
  auto evk1 = [&](size_t k) { return ev[4 * k + 3]; };  // kernel end
  cudaEvent_t start = ev[4 * nchunks];
  // copies start after everything already queued on the compute stream
  CKR(cudaEventRecord(start, st));
  CKR(cudaStreamWaitEvent(cp, start, 0));
  const double t_start = since();
  int rc = ECC_OK;
  for (size_t k = 0; k < nchunks && rc == ECC_OK; ++k) {
    const int b = (int)(k % NB);
    const uint64_t own0 = bounds[k], own1 = bounds[k + 1];
    const uint64_t r0 = own0 == 0 ? 0 : own0 - 1;
    const uint64_t r1 = std::min<uint64_t>(own1 + 1, dims.w0);
    cudaError_t e = cudaSuccess;
    if (k >= (size_t)NB) e = cudaStreamWaitEvent(cp, evk1(k - NB), 0);  // buffer reuse
    if (e == cudaSuccess) e = cudaEventRecord(evh0(k), cp);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(ctx->slab[b].p,
                          static_cast<const uint8_t*>(host) + (r0 - plane0) * row_bytes,
                          (r1 - r0) * row_bytes, cudaMemcpyHostToDevice, cp);
    if (e == cudaSuccess) e = cudaEventRecord(evh1(k), cp);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, evh1(k), 0);
    if (e == cudaSuccess) e = cudaEventRecord(evk0(k), st);
    if (e != cudaSuccess) {
      rc = fail(ECC_ECUDA, cudaGetErrorString(e));
      break;
    }
    const Slab s = make_slab(ctx->slab[b].p, dims, r0, r1 - r0, own0, own1);
    rc = accumulate(ctx, s, dtype, affine, am, (uint32_t)nbins, hist, st);
    if (rc == ECC_OK && cudaEventRecord(evk1(k), st) != cudaSuccess)
      rc = fail(ECC_ECUDA, "event record failed");
  }
  const cudaError_t e1 = cudaStreamSynchronize(cp);
  const cudaError_t e2 = cudaStreamSynchronize(st);
  if (rc == ECC_OK && (e1 != cudaSuccess || e2 != cudaSuccess))
    rc = fail(ECC_ECUDA, cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
  if (rc == ECC_OK && timings) {
    for (size_t k = 0; k < nchunks; ++k) {
      float a = 0, b = 0, c = 0, d = 0;
      cudaEventElapsedTime(&a, start, evh0(k));
      cudaEventElapsedTime(&b, start, evh1(k));
      cudaEventElapsedTime(&c, start, evk0(k));
      cudaEventElapsedTime(&d, start, evk1(k));
      ecc_chunk_timing& t = timings[k];
      t.begin = bounds[k];
      t.end = bounds[k + 1];
      t.ingest_begin = t_start + a * 1e-3;
      t.ingest_end = t_start + b * 1e-3;
      t.index_begin = t.index_end = t.ingest_end;
      t.kernel_begin = t_start + c * 1e-3;
      t.kernel_end = t_start + d * 1e-3;
      t.merge_begin = t.merge_end = t.kernel_end;
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return rc;
}

}  // namespace

extern "C" {

int ecc_process_host(ecc_ctx* ctx, const void* host, ecc_dtype dtype, ecc_dims dims,
                     const uint64_t* bounds, size_t nchunks, const ecc_binmap* bm,
                     ecc_chunk_timing* timings, void* values_out, int64_t* changes_out,
                     uint64_t cap, uint64_t* n_out) {
  CKI(bind(ctx));
  CKI(check_dtype(dtype));
  CKI(check_dims(dims));
  if (!host || !values_out || !changes_out || !n_out) return fail(ECC_EINVAL, "null pointer");
  CKI(check_plan(bounds, nchunks, dims));
  uint64_t nbins = 0;
  bool affine = false, sorted = false;
  AffineMap am{};
  CKI(resolve_bins(dtype, bm, &nbins, &affine, &sorted, &am));
  if (sorted)
    return fail(ECC_EINVAL, "the sorted bin map streams through ecc_process_stream");
  // pinned (page-locked or registered) memory is copied by DMA straight from
  // the caller's buffer; pageable memory makes each copy synchronous
  CKI(ctx->flags.ensure(4));
  CKI(ctx->hist.ensure(2 * nbins * 8));
  cudaStream_t st = ctx->stream;
  CKR(cudaMemsetAsync(ctx->flags.p, 0, 4, st));
  CKR(cudaMemsetAsync(ctx->hist.p, 0, 2 * nbins * 8, st));
  CKI(host_pipeline(ctx, host, 0, dims.w0, dtype, dims, bounds, nchunks, affine, am, nbins,
                    ctx->hist.as<int64_t>(), timings));
  if (affine) CKI(read_flags(ctx, st));
  BinResult& r = ctx->hres;
  CKI(finalize_to_host(ctx, (uint32_t)nbins, st, &r));
  const size_t m = r.changes.size();
  *n_out = m;
  if (m > cap) return fail(ECC_EINVAL, "output capacity below the number of values");
  write_values(dtype, false, am, r, values_out);
  std::memcpy(changes_out, r.changes.data(), m * 8);
  return ECC_OK;
}

int ecc_accumulate_host(ecc_ctx* ctx, const void* host_planes, uint64_t plane0,
                        uint64_t nplanes, ecc_dtype dtype, ecc_dims image,
                        const uint64_t* bounds, size_t nchunks, const ecc_binmap* bm,
                        int64_t* d_hist) {
  CKI(bind(ctx));
  CKI(check_dtype(dtype));
  CKI(check_dims(image));
  if (!host_planes || !bounds || !d_hist) return fail(ECC_EINVAL, "null pointer");
  if (nchunks == 0) return fail(ECC_EINVAL, "empty chunk plan");
  for (size_t k = 0; k < nchunks; ++k)
    if (bounds[k + 1] <= bounds[k] || bounds[k + 1] > image.w0)
      return fail(ECC_EINVAL, "chunk bounds must increase within [0, w0]");
  uint64_t nbins = 0;
  bool affine = false, sorted = false;
  AffineMap am{};
  CKI(resolve_bins(dtype, bm, &nbins, &affine, &sorted, &am));
  if (sorted) return fail(ECC_EINVAL, "the sorted bin map has no dense histogram");
  CKI(ctx->flags.ensure(4));
  CKR(cudaMemsetAsync(ctx->flags.p, 0, 4, ctx->stream));
  CKI(host_pipeline(ctx, host_planes, plane0, nplanes, dtype, image, bounds, nchunks, affine, am,
                    nbins, d_hist, nullptr));
  if (affine) CKI(read_flags(ctx, ctx->stream));
  return ECC_OK;
}

int ecc_batch2d(ecc_ctx* ctx, const void* data, int where, ecc_dtype dtype, uint64_t count,
                uint64_t h, uint64_t w, int32_t* chi, uint32_t* presence, void* stream) {
  CKI(bind(ctx));
  CKI(check_dtype(dtype));
  if (dtype == ECC_F32) return fail(ECC_EINVAL, "batched 2D supports u8 and u16 images");
  if (h < 1 || w < 1 || h * w > (1ull << 26))
    return fail(ECC_EINVAL, "batched images must have 1 <= h*w <= 2^26 pixels");
  if (count > 0x7FFFFFFFull) return fail(ECC_EINVAL, "too many images");
  if (!data || !chi || !presence) return fail(ECC_EINVAL, "null pointer");
  cudaStream_t st = pick(ctx, stream);
  const uint64_t nbins = dtype == ECC_U8 ? 256 : 65536;
  if (where == 1) {
    CKI(batch_scratch(ctx, dtype, st));
    CKR(launch_batch2d(data, (int)dtype, count, (int)h, (int)w, chi, presence,
                       ctx->bscratch.as<int32_t>(), st));
    ctx->launches += 1;
    return ECC_OK;
  }
  if (where != 0) return fail(ECC_EINVAL, "where must be 0 (host) or 1 (device)");
  const uint64_t in_bytes = count * h * w * esize(dtype);
  CKI(ctx->input.ensure(in_bytes));
  CKI(ctx->chi.ensure(count * nbins * 4));
  CKI(ctx->bins.ensure(count * nbins / 8));
  CKR(cudaMemcpyAsync(ctx->input.p, data, in_bytes, cudaMemcpyHostToDevice, st));
  CKI(batch_scratch(ctx, dtype, st));
  CKR(launch_batch2d(ctx->input.p, (int)dtype, count, (int)h, (int)w, ctx->chi.as<int32_t>(),
                     ctx->bins.as<uint32_t>(), ctx->bscratch.as<int32_t>(), st));
  ctx->launches += 1;
  CKR(cudaMemcpyAsync(chi, ctx->chi.p, count * nbins * 4, cudaMemcpyDeviceToHost, st));
  CKR(cudaMemcpyAsync(presence, ctx->bins.p, count * nbins / 8, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  return ECC_OK;
}

int ecc_fill_synthetic(ecc_ctx* ctx, void* d_data, ecc_dtype dtype, uint64_t n,
                       uint64_t seed, uint64_t base, void* stream) {
  CKI(bind(ctx));
  CKI(check_dtype(dtype));
  if (!d_data) return fail(ECC_EINVAL, "null device pointer");
  CKR(launch_fill(d_data, (int)dtype, n, seed, base, ctx->sms, pick(ctx, stream)));
  return ECC_OK;
}

int ecc_uniform_noise(ecc_ctx* ctx, float* d_out, uint64_t n, uint64_t seed, void* stream) {
  CKI(bind(ctx));
  if (!d_out) return fail(ECC_EINVAL, "null device pointer");
  CKR(launch_uniform_noise(d_out, n, seed, ctx->sms, pick(ctx, stream)));
  ctx->launches += 1;
  return ECC_OK;
}

int ecc_gaussian_smooth(ecc_ctx* ctx, const float* d_in, float* d_out, ecc_dims dims,
                        double sigma, int width, void* stream) {
  CKI(bind(ctx));
  CKI(check_dims(dims));
  if (!d_in || !d_out) return fail(ECC_EINVAL, "null device pointer");
  return smooth_device(ctx, d_in, d_out, dims, sigma, width, pick(ctx, stream));
}

int ecc_bench_run(ecc_ctx* ctx, ecc_dims dims, uint64_t iterations, uint64_t seed, double sigma,
                  int width, ecc_bench_report* rep) {
  CKI(bind(ctx));
  CKI(check_dims(dims));
  if (!rep) return fail(ECC_EINVAL, "null report");
  if (iterations < 1) return fail(ECC_EINVAL, "bench needs at least one iteration");
  {
    std::vector<double> w;
    CKI(gaussian_weights(sigma, width, &w));
  }
  using clk = std::chrono::steady_clock;
  const auto secs = [](clk::time_point a, clk::time_point b) {
    return std::chrono::duration<double>(b - a).count();
  };
  cudaStream_t st = ctx->stream;
  const uint64_t n = dims.w0 * dims.w1 * dims.w2;
  std::memset(rep, 0, sizeof(*rep));
  rep->iterations = iterations;
  rep->voxels = n;
  CKI(ctx->input.ensure(n * 4));
  float* img = ctx->input.as<float>();
  CKI(ctx->flags.ensure(16));
  const auto tg0 = clk::now();
  CKR(launch_uniform_noise(img, n, seed, ctx->sms, st));
  ctx->launches += 1;
  CKR(cudaStreamSynchronize(st));
  rep->generate_s = secs(tg0, clk::now());
  cudaEvent_t e0, e1, e2;
  CKR(cudaEventCreate(&e0));
  CKR(cudaEventCreate(&e1));
  CKR(cudaEventCreate(&e2));
  double smooth_ms = 0, ecc_ms = 0;
  uint64_t m = 0;
  const uint8_t* last_chi = nullptr;  // device int64 chi of the last curve
  int rc = ECC_OK;
  const Slab s = make_slab(img, dims, 0, dims.w0, 0, dims.w0);
  const auto t0 = clk::now();
  for (uint64_t it = 0; it < iterations && rc == ECC_OK; ++it) {
    // the last smoothing pass also reduces the key range the ECC's dense
    // histogram needs (flags words 1, 2), replacing a separate pass
    {
      static const uint32_t init[4] = {0u, 0xFFFFFFFFu, 0u, 0u};
      cudaMemcpyAsync(ctx->flags.p, init, 16, cudaMemcpyHostToDevice, st);
    }
    bool ranged = false;
    cudaEventRecord(e0, st);
    rc = smooth_device(ctx, img, img, dims, sigma, width, st, ctx->flags.as<uint32_t>() + 1,
                       &ranged);
    if (rc != ECC_OK) break;
    cudaEventRecord(e1, st);
    // process_image + vcec_to_ecc (streaming.hpp:332-338, curve.hpp:28-35)
    // on the sorted f32 path; the curve stays in device memory
    // dense key histogram when the key span allows (no sort), else the sort
    ResultLayout L(1);
    uint32_t key_lo = 0;
    bool dense = false;
    rc = dense_sorted(ctx, s, st, &L, &key_lo, &dense, ranged);
    if (rc == ECC_OK && dense) {
      rc = cudaMemcpyAsync(&m, ctx->res.p, 8, cudaMemcpyDeviceToHost, st) == cudaSuccess
               ? ECC_OK
               : fail(ECC_ECUDA, "count readback failed");
      last_chi = ctx->res.as<uint8_t>() + L.chi;
    } else if (rc == ECC_OK) {
      uint64_t nacc = 0;
      rc = sorted_slab(ctx, s, st, &nacc);
      if (rc == ECC_OK) rc = read_flags(ctx, st);
      if (rc == ECC_OK) rc = sorted_finish(ctx, st, nacc, false, nullptr, &m);
      last_chi = ctx->chi.as<uint8_t>();
    }
    cudaEventRecord(e2, st);
    cudaEventSynchronize(e2);
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, e0, e1);
    cudaEventElapsedTime(&b, e1, e2);
    smooth_ms += a;
    ecc_ms += b;
  }
  rep->total_s = secs(t0, clk::now());
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  CKI(rc);
  const double it = (double)iterations;
  rep->per_iteration_s = (rep->generate_s + rep->total_s) / it;
  rep->ecc_avg_s = ecc_ms * 1e-3 / it;
  rep->smooth_avg_s = smooth_ms * 1e-3 / it;
  rep->ecc_gvox_per_s = ecc_ms > 0 ? (double)n * it / (ecc_ms * 1e-3) / 1e9 : 0;
  rep->last_points = m;
  if (m > 0 && last_chi) {
    CKR(cudaMemcpy(&rep->last_chi_first, last_chi, 8, cudaMemcpyDeviceToHost));
    CKR(cudaMemcpy(&rep->last_chi_last, last_chi + (m - 1) * 8, 8, cudaMemcpyDeviceToHost));
  }
  return ECC_OK;
}

int ecc_batch_format(ecc_ctx* ctx, const int32_t* d_chi, const uint32_t* d_presence,
                     uint64_t count, ecc_dtype dtype, int format, char* out, uint64_t cap,
                     uint64_t* offsets, uint64_t* total) {
  CKI(bind(ctx));
  if (dtype != ECC_U8 && dtype != ECC_U16)
    return fail(ECC_EINVAL, "batched curves have u8 or u16 thresholds");
  if (format != 0 && format != 1) return fail(ECC_EINVAL, "format must be 0 (csv) or 1 (json)");
  if (!d_chi || !d_presence || !offsets || !total) return fail(ECC_EINVAL, "null pointer");
  const uint32_t nbins = dtype == ECC_U8 ? 256 : 65536;
  cudaStream_t st = ctx->stream;
  CKI(ctx->sums.ensure((count + 1) * 8));
  CKI(ctx->sums2.ensure((count + 1) * 8));
  uint64_t* sizes = ctx->sums.as<uint64_t>();
  uint64_t* offs = ctx->sums2.as<uint64_t>();
  CKR(cudaMemsetAsync(sizes + count, 0, 8, st));
  CKR(launch_format_sizes(d_chi, d_presence, count, nbins, format, sizes, st));
  size_t t = 0;
  CKR(cub::DeviceScan::ExclusiveSum(nullptr, t, sizes, offs, (int)(count + 1), st));
  CKI(ctx->tmp.ensure(t));
  t = ctx->tmp.cap;
  CKR(cub::DeviceScan::ExclusiveSum(ctx->tmp.p, t, sizes, offs, (int)(count + 1), st));
  CKR(cudaMemcpyAsync(offsets, offs, (count + 1) * 8, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  ctx->launches += 2;
  *total = offsets[count];
  if (!out) return ECC_OK;  // size query
  if (cap < *total)
    return fail(ECC_EINVAL, "output capacity " + std::to_string(cap) + " is below the " +
                                std::to_string(*total) + " bytes");
  CKI(ctx->keys.ensure(*total));
  CKR(launch_format_write(d_chi, d_presence, count, nbins, format, offs, ctx->keys.as<char>(),
                          st));
  ctx->launches += 1;
  CKR(cudaMemcpyAsync(out, ctx->keys.p, *total, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  return ECC_OK;
}

int ecc_batch_zero_crossings(ecc_ctx* ctx, const int32_t* d_chi, const uint32_t* d_presence,
                             uint64_t count, ecc_dtype dtype, uint32_t* d_out, void* stream) {
  CKI(bind(ctx));
  if (dtype != ECC_U8 && dtype != ECC_U16)
    return fail(ECC_EINVAL, "batched curves have u8 or u16 thresholds");
  if (!d_chi || !d_presence || !d_out) return fail(ECC_EINVAL, "null device pointer");
  CKR(launch_zero_crossings(d_chi, d_presence, count, dtype == ECC_U8 ? 256 : 65536, d_out,
                            pick(ctx, stream)));
  ctx->launches += 1;
  return ECC_OK;
}

int ecc_xchg_create(ecc_ctx* ctx, int rank, int world, ecc_xchg** out, void* handle_out) {
  CKI(bind(ctx));
  if (!out || !handle_out) return fail(ECC_EINVAL, "null pointer");
  if (world < 1 || rank < 0 || rank >= world) return fail(ECC_EINVAL, "bad rank / world");
  auto* x = new ecc_xchg();
  x->ctx = ctx;
  x->rank = rank;
  x->world = world;
  x->flags_off = (size_t)2 * world * 512 * 8;
  x->err_off = x->flags_off + (size_t)2 * world * 4;
  x->bytes = x->err_off + 256;
  cudaError_t e = cudaMalloc(&x->buf, x->bytes);
  if (e == cudaSuccess) e = cudaMemset(x->buf, 0, x->bytes);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, x->buf);
  if (e != cudaSuccess) {
    if (x->buf) cudaFree(x->buf);
    delete x;
    return fail(ECC_ECUDA, std::string("exchange buffer: ") + cudaGetErrorString(e));
  }
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  if (e == cudaSuccess)
    e = cudaHostAlloc(reinterpret_cast<void**>(&x->err_host), 64, cudaHostAllocMapped);
  if (e == cudaSuccess) {
    *x->err_host = 0;
    e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&x->err_dev), x->err_host, 0);
  }
  if (e != cudaSuccess) {
    if (x->err_host) cudaFreeHost(x->err_host);
    cudaFree(x->buf);
    delete x;
    return fail(ECC_ECUDA, std::string("exchange error word: ") + cudaGetErrorString(e));
  }
  std::memcpy(handle_out, &h, 64);
  *out = x;
  return ECC_OK;
}

int ecc_xchg_open(ecc_xchg* x, const void* handles) {
  if (!x || !handles) return fail(ECC_EINVAL, "null pointer");
  CKI(bind(x->ctx));
  x->base.assign(x->world, nullptr);
  for (int r = 0; r < x->world; ++r) {
    if (r == x->rank) {
      x->base[r] = x->buf;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const uint8_t*>(handles) + 64 * r, 64);
    const cudaError_t e = cudaIpcOpenMemHandle(&x->base[r], h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return fail(ECC_ECUDA, "opening rank " + std::to_string(r) + "'s exchange buffer: " +
                                 cudaGetErrorString(e));
  }
  std::vector<void*> p(2 * x->world);
  for (int r = 0; r < x->world; ++r) {
    p[r] = x->base[r];
    p[x->world + r] = static_cast<uint8_t*>(x->base[r]) + x->flags_off;
  }
  if (!x->ptrs) CKR(cudaMalloc(&x->ptrs, p.size() * sizeof(void*)));
  CKR(cudaMemcpy(x->ptrs, p.data(), p.size() * sizeof(void*), cudaMemcpyHostToDevice));
  return ECC_OK;
}

void ecc_xchg_destroy(ecc_xchg* x) {
  if (!x) return;
  cudaSetDevice(x->ctx->device);
  cudaDeviceSynchronize();
  for (int r = 0; r < (int)x->base.size(); ++r)
    if (r != x->rank && x->base[r]) cudaIpcCloseMemHandle(x->base[r]);
  if (x->ptrs) cudaFree(x->ptrs);
  if (x->buf) cudaFree(x->buf);
  if (x->err_host) cudaFreeHost(x->err_host);
  delete x;
}

int ecc_xchg_status(ecc_xchg* x) {
  if (!x) return fail(ECC_EINVAL, "null exchange");
  CKI(bind(x->ctx));
  CKR(cudaStreamSynchronize(x->last ? x->last : x->ctx->stream));
  if (*reinterpret_cast<volatile uint32_t*>(x->err_host))
    return fail(ECC_ECUDA, "rank exchange timed out: a peer never published its histogram");
  return ECC_OK;
}

int ecc_curve_sharded(ecc_ctx* ctx, ecc_xchg* x, const void* d_planes, ecc_dims image,
                      uint64_t plane0, uint64_t nplanes, uint64_t own0, uint64_t own1,
                      uint32_t* d_bins, int64_t* d_changes, int64_t* d_chi, uint64_t* d_count,
                      void* stream) {
  CKI(bind(ctx));
  CKI(check_dims(image));
  CKI(check_slab(image, plane0, nplanes, own0, own1));
  if (!x || !x->ptrs) return fail(ECC_EINVAL, "exchange not opened");
  // a peer timed out in an earlier launch: this rank's step count is out of
  // step with its peers, so no later curve could be trusted
  if (*reinterpret_cast<volatile uint32_t*>(x->err_host))
    return fail(ECC_ECUDA, "rank exchange timed out: a peer never published its histogram");
  if (!d_planes || !d_bins || !d_changes || !d_chi || !d_count)
    return fail(ECC_EINVAL, "null device pointer");
  const Slab s = make_slab(d_planes, image, plane0, nplanes, own0, own1);
  if (!u8_3d_supported(s) || own1 <= own0)
    return fail(ECC_EINVAL, "the fused sharded curve takes 3D u8 slabs with 16-byte rows");
  cudaStream_t st = pick(ctx, stream);
  if (!ctx->fused.p) {
    CKI(ctx->fused.ensure(256 + 512 * 8));
    CKR(cudaMemsetAsync(ctx->fused.p, 0, 256 + 512 * 8, st));
  }
  U83dFinalize fz{ctx->fused.as<uint32_t>(), d_bins, d_changes, d_chi, d_count};
  fz.world = x->world;
  fz.rank = x->rank;
  fz.epoch = ++x->epoch;
  fz.slots = static_cast<int64_t* const*>(x->ptrs);
  fz.flags = reinterpret_cast<uint32_t* const*>(static_cast<void**>(x->ptrs) + x->world);
  fz.my_slots = static_cast<const int64_t*>(x->buf);
  fz.my_flags = reinterpret_cast<const uint32_t*>(static_cast<uint8_t*>(x->buf) + x->flags_off);
  fz.err = x->err_dev;
  x->last = st;
  CKR(launch_u8_3d(s, reinterpret_cast<int64_t*>(ctx->fused.as<uint8_t>() + 256), nullptr,
                   ctx->sms, st, &fz));
  ctx->launches += 1;
  return ECC_OK;
}

}  // extern "C"

// ===================================================================== padded chunks
// The reference's chunk-level API on the device (ecc_chunk_*, ecc_value_index,
// ecc_merge_local; see ecc_b200.h).  The PaddedChunk storage is uploaded as
// is and turned into a key image (k_chunk_keys), so the stencil sees exactly
// the stored extended values, collar and padding rows included.
namespace {

size_t ext_size(ecc_dtype t) { return t == ECC_U8 ? 2 : 4; }
int ext_type(ecc_dtype t) { return t == ECC_U8 ? 0 : (t == ECC_U16 ? 1 : 2); }

int check_chunk(const ecc_chunk& c, uint64_t r0, uint64_t r1) {
  CKI(check_dims(c.image));
  if (!(c.begin < c.end) || c.end > c.image.w0)
    return fail(ECC_EINVAL, "invalid chunk range [" + std::to_string(c.begin) + ", " +
                                std::to_string(c.end) + ") for dims " + dims_str(c.image));
  if (r0 > r1 || r1 > c.end - c.begin)
    return fail(ECC_EINVAL, "rows [" + std::to_string(r0) + ", " + std::to_string(r1) +
                                ") are outside the chunk's " + std::to_string(c.end - c.begin) +
                                " owned rows");
  return ECC_OK;
}

// Padded rows [r0, r1 + 2) -> key image in ctx->keys; *s describes it with
// owned rows r0..r1-1 (key-image planes 1..np-2) and the collar not owned.
// as3d: evaluate a 2D chunk with the 3D stencil over its padded axis 2 (the
// reference's introduced() is dimension-free: offsets along axis 2 meet the
// collar).
int chunk_keyimage(ecc_ctx* ctx, const void* padded, ecc_dtype dtype, const ecc_chunk& c,
                   uint64_t r0, uint64_t r1, cudaStream_t st, Slab* s, bool as3d = false) {
  const bool is2d = c.image.w2 == 1 && !as3d;
  const uint64_t w1p = c.image.w1 + 2, w2p = c.image.w2 + 2, plane = w1p * w2p;
  const uint64_t np = r1 - r0 + 2;
  const size_t es = ext_size(dtype);
  CKI(ctx->input.ensure(np * plane * es));
  CKR(cudaMemcpyAsync(ctx->input.p, static_cast<const char*>(padded) + r0 * plane * es,
                      np * plane * es, cudaMemcpyHostToDevice, st));
  const uint64_t w2k = is2d ? 1 : w2p;
  CKI(ctx->keys.ensure(np * w1p * w2k * 4));
  CKR(launch_chunk_keys(ctx->input.p, ext_type(dtype), np, w1p, w2p, is2d, false,
                        ctx->keys.as<uint32_t>(), ctx->sms, st));
  ctx->launches += 1;
  Slab k{};
  k.base = ctx->keys.p;
  k.plane0 = 0;
  k.nplanes = (int64_t)np;
  k.w0 = (int64_t)np;
  k.w1 = (int64_t)w1p;
  k.w2 = (int64_t)w2k;
  k.own0 = 1;
  k.own1 = (int64_t)np - 1;
  k.oj0 = 1;
  k.oj1 = (int64_t)w1p - 1;
  if (!is2d) {
    k.ok0 = 1;
    k.ok1 = (int64_t)w2p - 1;
  }
  *s = k;
  return ECC_OK;
}

int check_ptr(const void* p, const char* what) {
  if (!p) return fail(ECC_EINVAL, std::string("null ") + what);
  return ECC_OK;
}

// Sort + reduce-by-key of (ctx->keys2[0..n), ctx->ch8[0..n)) into
// (ctx->akeys, ctx->asums); *m = distinct keys.
int reduce_keys(ecc_ctx* ctx, uint64_t n, cudaStream_t st, uint64_t* m) {
  if (n > 0x7FFFFFFFull) return fail(ECC_EINVAL, "value list exceeds 2^31 entries");
  CKI(ctx->keys.ensure(n * 4));
  CKI(ctx->ch8b.ensure(n));
  CKI(ctx->akeys.ensure(n * 4));
  CKI(ctx->asums.ensure(n * 8));
  CKI(ctx->count.ensure(8));
  size_t t1 = 0, t2 = 0;
  auto vals = thrust::make_transform_iterator(ctx->ch8b.as<const int8_t>(), ToI64());
  CKR(cub::DeviceRadixSort::SortPairs(nullptr, t1, ctx->keys2.as<uint32_t>(), ctx->keys.as<uint32_t>(),
                                      ctx->ch8.as<int8_t>(), ctx->ch8b.as<int8_t>(), (int)n, 0, 32,
                                      st));
  CKR(cub::DeviceReduce::ReduceByKey(nullptr, t2, ctx->keys.as<uint32_t>(), ctx->akeys.as<uint32_t>(),
                                     vals, ctx->asums.as<int64_t>(), ctx->count.as<uint64_t>(),
                                     cub::Sum(), (int)n, st));
  CKI(ctx->tmp.ensure(std::max(t1, t2)));
  t1 = ctx->tmp.cap;
  CKR(cub::DeviceRadixSort::SortPairs(ctx->tmp.p, t1, ctx->keys2.as<uint32_t>(),
                                      ctx->keys.as<uint32_t>(), ctx->ch8.as<int8_t>(),
                                      ctx->ch8b.as<int8_t>(), (int)n, 0, 32, st));
  t2 = ctx->tmp.cap;
  CKR(cub::DeviceReduce::ReduceByKey(ctx->tmp.p, t2, ctx->keys.as<uint32_t>(),
                                     ctx->akeys.as<uint32_t>(), vals, ctx->asums.as<int64_t>(),
                                     ctx->count.as<uint64_t>(), cub::Sum(), (int)n, st));
  ctx->launches += 2;
  CKR(cudaMemcpyAsync(m, ctx->count.p, 8, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  return ECC_OK;
}

// (akeys, asums)[0..m) -> host values of dtype (keys decoded by `decode`) and sums.
int emit_keys(ecc_ctx* ctx, ecc_dtype dtype, uint64_t m, int decode, void* values_out,
              int64_t* sums_out, uint64_t cap, uint64_t* n_out, cudaStream_t st) {
  *n_out = m;
  if (m > cap) return fail(ECC_EINVAL, "output capacity " + std::to_string(cap) + " < " +
                                           std::to_string(m) + " distinct values");
  std::vector<uint32_t> keys(m);
  if (m) CKR(cudaMemcpyAsync(keys.data(), ctx->akeys.p, m * 4, cudaMemcpyDeviceToHost, st));
  if (m && sums_out)
    CKR(cudaMemcpyAsync(sums_out, ctx->asums.p, m * 8, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  for (uint64_t i = 0; i < m; ++i) {
    uint32_t k = keys[i];
    if (decode == 1) k -= 32768u;            // int16 extended u8
    else if (decode == 2) k ^= 0x80000000u;  // int32 extended u16
    if (dtype == ECC_U8) static_cast<uint8_t*>(values_out)[i] = (uint8_t)k;
    else if (dtype == ECC_U16) static_cast<uint16_t*>(values_out)[i] = (uint16_t)k;
    else static_cast<float*>(values_out)[i] = key_to_float(k);
  }
  return ECC_OK;
}

int read_flag_errors(ecc_ctx* ctx, cudaStream_t st, const char* binmap_msg) {
  uint32_t f = 0;
  CKR(cudaMemcpyAsync(&f, ctx->flags.p, 4, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  if (f & kFlagNaN) return fail(ECC_ENAN, "cannot build a value index: NaN input");
  if (f & kFlagBinmap) return fail(ECC_EBINMAP, binmap_msg);
  return ECC_OK;
}

}  // namespace

int ecc_chunk_changes(ecc_ctx* ctx, const void* padded, ecc_dtype dtype, ecc_chunk c,
                      uint64_t row_begin, uint64_t row_end, int8_t* out) {
  CKI(bind(ctx));
  CKI(check_dtype(dtype));
  CKI(check_ptr(padded, "padded chunk"));
  CKI(check_chunk(c, row_begin, row_end));
  const uint64_t n = (row_end - row_begin) * c.image.w1 * c.image.w2;
  if (n == 0) return ECC_OK;
  CKI(check_ptr(out, "output"));
  cudaStream_t st = ctx->stream;
  Slab s;
  CKI(chunk_keyimage(ctx, padded, dtype, c, row_begin, row_end, st, &s));
  CKI(ctx->ch8.ensure(n));
  AffineMap am{};
  CKR(launch_keyimage(s, 2, am, nullptr, 0, nullptr, ctx->ch8.p, ctx->sms, st));
  ctx->launches += 1;
  CKR(cudaMemcpyAsync(out, ctx->ch8.p, n, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  return ECC_OK;
}

int ecc_chunk_faces(ecc_ctx* ctx, const void* padded, ecc_dtype dtype, ecc_chunk c,
                    uint64_t row_begin, uint64_t row_end, uint32_t* out) {
  CKI(bind(ctx));
  CKI(check_dtype(dtype));
  CKI(check_ptr(padded, "padded chunk"));
  CKI(check_chunk(c, row_begin, row_end));
  const uint64_t n = (row_end - row_begin) * c.image.w1 * c.image.w2;
  if (n == 0) return ECC_OK;
  CKI(check_ptr(out, "output"));
  cudaStream_t st = ctx->stream;
  Slab s;
  CKI(chunk_keyimage(ctx, padded, dtype, c, row_begin, row_end, st, &s, true));
  CKI(ctx->keys2.ensure(n * 4));
  AffineMap am{};
  CKR(launch_keyimage(s, 3, am, nullptr, 0, nullptr, ctx->keys2.p, ctx->sms, st));
  ctx->launches += 1;
  CKR(cudaMemcpyAsync(out, ctx->keys2.p, n * 4, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  return ECC_OK;
}

int ecc_chunk_accumulate(ecc_ctx* ctx, const void* padded, ecc_dtype dtype, ecc_chunk c,
                         uint64_t row_begin, uint64_t row_end, const float* index_values,
                         uint64_t nbins, int64_t* hist_out) {
  CKI(bind(ctx));
  CKI(check_dtype(dtype));
  CKI(check_ptr(padded, "padded chunk"));
  CKI(check_ptr(hist_out, "histogram"));
  CKI(check_chunk(c, row_begin, row_end));
  AffineMap am{};
  if (!index_values) {
    if (dtype == ECC_F32) return fail(ECC_EINVAL, "f32 chunks are binned by a value index");
    const uint64_t want = dtype == ECC_U8 ? 256 : 65536;
    if (nbins != want)
      return fail(ECC_EINVAL, "identity bins of this dtype number " + std::to_string(want));
    am.key_lo = dtype == ECC_U8 ? 32768u : 0x80000000u;  // the key image's encoding
    am.key_mask = (uint32_t)(want - 1);
  } else {
    if (nbins == 0 || nbins > 0x7FFFFFFFull)
      return fail(ECC_EINVAL, "a value index needs 1 .. 2^31 bins");
  }
  std::fill(hist_out, hist_out + nbins, 0);
  if (row_begin == row_end) return ECC_OK;
  cudaStream_t st = ctx->stream;
  CKI(ctx->flags.ensure(16));
  CKR(cudaMemsetAsync(ctx->flags.p, 0, 16, st));
  if (index_values) {
    // the table in key space: order keys of the index values (value_index.hpp:95-99)
    CKI(ctx->bins.ensure(nbins * 4));
    CKI(ctx->sums2.ensure(nbins * 4));
    CKR(cudaMemcpyAsync(ctx->sums2.p, index_values, nbins * 4, cudaMemcpyHostToDevice, st));
    CKR(launch_value_keys(ctx->sums2.p, (int)ECC_F32, nbins, ctx->bins.as<uint32_t>(),
                          ctx->flags.as<uint32_t>(), ctx->sms, st));
    ctx->launches += 1;
    am.table = ctx->bins.as<uint32_t>();
    am.table_n = (uint32_t)nbins;
  }
  Slab s;
  CKI(chunk_keyimage(ctx, padded, dtype, c, row_begin, row_end, st, &s));
  CKI(ctx->hist.ensure(2 * nbins * 8));
  CKR(cudaMemsetAsync(ctx->hist.p, 0, 2 * nbins * 8, st));
  CKR(launch_keyimage(s, 0, am, ctx->hist.as<int64_t>(), (uint32_t)nbins,
                      ctx->flags.as<uint32_t>(), nullptr, ctx->sms, st));
  ctx->launches += 1;
  CKI(read_flag_errors(ctx, st, "value not present in index (internal consistency bug)"));
  CKR(cudaMemcpyAsync(hist_out, ctx->hist.p, nbins * 8, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  return ECC_OK;
}

int ecc_value_index(ecc_ctx* ctx, ecc_dtype dtype, const void* values, uint64_t n,
                    const int8_t* changes, void* values_out, int64_t* sums_out, uint64_t cap,
                    uint64_t* n_out) {
  CKI(bind(ctx));
  CKI(check_dtype(dtype));
  CKI(check_ptr(n_out, "count output"));
  *n_out = 0;
  if (n == 0) return fail(ECC_EINVAL, "cannot build a value index: empty input");
  CKI(check_ptr(values, "values"));
  CKI(check_ptr(values_out, "values output"));
  cudaStream_t st = ctx->stream;
  CKI(ctx->flags.ensure(16));
  CKR(cudaMemsetAsync(ctx->flags.p, 0, 16, st));
  CKI(ctx->input.ensure(n * esize(dtype)));
  CKR(cudaMemcpyAsync(ctx->input.p, values, n * esize(dtype), cudaMemcpyHostToDevice, st));
  CKI(ctx->keys2.ensure(n * 4));
  CKI(ctx->ch8.ensure(n));
  CKR(launch_value_keys(ctx->input.p, (int)dtype, n, ctx->keys2.as<uint32_t>(),
                        ctx->flags.as<uint32_t>(), ctx->sms, st));
  ctx->launches += 1;
  if (changes) CKR(cudaMemcpyAsync(ctx->ch8.p, changes, n, cudaMemcpyHostToDevice, st));
  else CKR(cudaMemsetAsync(ctx->ch8.p, 0, n, st));
  CKI(read_flag_errors(ctx, st, "value not present in index"));
  uint64_t m = 0;
  CKI(reduce_keys(ctx, n, st, &m));
  return emit_keys(ctx, dtype, m, 0, values_out, changes ? sums_out : nullptr, cap, n_out, st);
}

int ecc_chunk_index_counts(ecc_ctx* ctx, const void* padded, ecc_dtype dtype, ecc_chunk c,
                           const int8_t* changes, void* values_out, int64_t* sums_out,
                           uint64_t cap, uint64_t* n_out) {
  CKI(bind(ctx));
  CKI(check_dtype(dtype));
  CKI(check_ptr(padded, "padded chunk"));
  CKI(check_ptr(n_out, "count output"));
  CKI(check_ptr(values_out, "values output"));
  *n_out = 0;
  CKI(check_chunk(c, 0, c.end - c.begin));
  const bool is2d = c.image.w2 == 1;
  const uint64_t len = c.end - c.begin, w1p = c.image.w1 + 2, w2p = c.image.w2 + 2;
  const uint64_t n = len * c.image.w1 * c.image.w2;
  if (n > 0xFFFFFFFFull) return fail(ECC_EINVAL, "chunk exceeds 2^32 voxels; use a finer chunk plan");
  cudaStream_t st = ctx->stream;
  const size_t es = ext_size(dtype);
  CKI(ctx->input.ensure((len + 2) * w1p * w2p * es));
  CKR(cudaMemcpyAsync(ctx->input.p, padded, (len + 2) * w1p * w2p * es, cudaMemcpyHostToDevice, st));
  CKI(ctx->keys2.ensure(n * 4));
  CKI(ctx->ch8.ensure(n));
  CKR(launch_chunk_keys(ctx->input.p, ext_type(dtype), len + 2, w1p, w2p, is2d, true,
                        ctx->keys2.as<uint32_t>(), ctx->sms, st));
  ctx->launches += 1;
  if (changes) CKR(cudaMemcpyAsync(ctx->ch8.p, changes, n, cudaMemcpyHostToDevice, st));
  else CKR(cudaMemsetAsync(ctx->ch8.p, 0, n, st));
  uint64_t m = 0;
  CKI(reduce_keys(ctx, n, st, &m));
  const int decode = dtype == ECC_U8 ? 1 : (dtype == ECC_U16 ? 2 : 0);
  return emit_keys(ctx, dtype, m, decode, values_out, changes ? sums_out : nullptr, cap, n_out, st);
}

int ecc_merge_local(ecc_ctx* ctx, ecc_dtype dtype, const void* gvals, const int64_t* gchg,
                    uint64_t gn, const int64_t* local, uint64_t nlocal, const void* ivals,
                    uint64_t in, void* out_vals, int64_t* out_chg, uint64_t cap,
                    uint64_t* n_out) {
  CKI(bind(ctx));
  CKI(check_dtype(dtype));
  CKI(check_ptr(n_out, "count output"));
  *n_out = 0;
  if ((gn && (!gvals || !gchg)) || (in && (!ivals || !local)) || !out_vals || !out_chg)
    return fail(ECC_EINVAL, "null merge_local argument");
  const uint64_t want = dtype == ECC_U8 ? 256 : (dtype == ECC_U16 ? 65536 : in);
  if (nlocal != want)
    return fail(ECC_EINVAL, "local VCEC length does not match the index bin count");
  const uint64_t n = gn + in;
  if (n == 0) return ECC_OK;
  if (n > 0x7FFFFFFFull) return fail(ECC_EINVAL, "too many distinct values to merge");
  cudaStream_t st = ctx->stream;
  CKI(ctx->flags.ensure(16));
  CKR(cudaMemsetAsync(ctx->flags.p, 0, 16, st));
  const size_t es = esize(dtype);
  CKI(ctx->input.ensure(n * es));
  CKI(ctx->akeys.ensure(n * 4));
  CKI(ctx->asums.ensure(n * 8));
  CKI(ctx->sums.ensure(std::max<uint64_t>(nlocal, 1) * 8));
  if (gn) {
    CKR(cudaMemcpyAsync(ctx->input.p, gvals, gn * es, cudaMemcpyHostToDevice, st));
    CKR(cudaMemcpyAsync(ctx->asums.p, gchg, gn * 8, cudaMemcpyHostToDevice, st));
  }
  if (in) {
    CKR(cudaMemcpyAsync(ctx->input.as<uint8_t>() + gn * es, ivals, in * es, cudaMemcpyHostToDevice,
                        st));
    CKR(cudaMemcpyAsync(ctx->sums.p, local, nlocal * 8, cudaMemcpyHostToDevice, st));
  }
  CKR(launch_value_keys(ctx->input.p, (int)dtype, n, ctx->akeys.as<uint32_t>(),
                        ctx->flags.as<uint32_t>(), ctx->sms, st));
  CKR(launch_gather_local(ctx->akeys.as<uint32_t>() + gn, dtype != ECC_F32, in,
                          ctx->sums.as<int64_t>(), nlocal, ctx->asums.as<int64_t>() + gn,
                          ctx->flags.as<uint32_t>(), ctx->sms, st));
  ctx->launches += 2;
  CKI(read_flag_errors(ctx, st, "value not present in index (internal consistency bug)"));
  uint64_t m = 0;
  CKI(merge_runs(ctx, st, n, &m));
  return emit_keys(ctx, dtype, m, 0, out_vals, out_chg, cap, n_out, st);
}

// ===================================================================== host-buffer helpers
int ecc_uniform_noise_host(ecc_ctx* ctx, float* out, uint64_t n, uint64_t seed) {
  CKI(bind(ctx));
  if (n == 0) return ECC_OK;
  if (!out) return fail(ECC_EINVAL, "null output");
  cudaStream_t st = ctx->stream;
  CKI(ctx->input.ensure(n * 4));
  CKR(launch_uniform_noise(ctx->input.as<float>(), n, seed, ctx->sms, st));
  ctx->launches += 1;
  CKR(cudaMemcpyAsync(out, ctx->input.p, n * 4, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  return ECC_OK;
}

int ecc_gaussian_smooth_host(ecc_ctx* ctx, const float* in, float* out, ecc_dims dims,
                             double sigma, int width) {
  CKI(bind(ctx));
  CKI(check_dims(dims));
  if (!in || !out) return fail(ECC_EINVAL, "null host pointer");
  cudaStream_t st = ctx->stream;
  const uint64_t n = dims.w0 * dims.w1 * dims.w2;
  CKI(ctx->input.ensure(n * 4));
  CKR(cudaMemcpyAsync(ctx->input.p, in, n * 4, cudaMemcpyHostToDevice, st));
  CKI(smooth_device(ctx, ctx->input.as<float>(), ctx->input.as<float>(), dims, sigma, width, st));
  CKR(cudaMemcpyAsync(out, ctx->input.p, n * 4, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  return ECC_OK;
}

int ecc_fixup_f32_host(ecc_ctx* ctx, float* data, uint64_t n, uint64_t base, int big_endian) {
  CKI(bind(ctx));
  if (n == 0) return ECC_OK;
  if (!data) return fail(ECC_EINVAL, "null host pointer");
  cudaStream_t st = ctx->stream;
  CKI(ctx->input.ensure(n * 4));
  CKI(ctx->nanidx.ensure(8));
  CKR(cudaMemsetAsync(ctx->nanidx.p, 0xFF, 8, st));
  CKR(cudaMemcpyAsync(ctx->input.p, data, n * 4, cudaMemcpyHostToDevice, st));
  CKR(launch_fixup(ctx->input.p, ECC_F32, n, base, big_endian != 0,
                   ctx->nanidx.as<unsigned long long>(), ctx->sms, st));
  ctx->launches += 1;
  unsigned long long first = ~0ull;
  CKR(cudaMemcpyAsync(&first, ctx->nanidx.p, 8, cudaMemcpyDeviceToHost, st));
  if (big_endian) CKR(cudaMemcpyAsync(data, ctx->input.p, n * 4, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  if (first != ~0ull) return fail(ECC_ENAN, "NaN value at linear index " + std::to_string(first));
  return ECC_OK;
}

// ===================================================================== one curve's text
namespace {
struct ToU64 {
  __host__ __device__ uint64_t operator()(uint32_t v) const { return v; }
};
}  // namespace

int ecc_format_curve(ecc_ctx* ctx, ecc_dtype dtype, const void* thresholds, const int64_t* chi,
                     uint64_t n, int where, int mode, char* out, uint64_t cap,
                     uint64_t* size_out) {
  CKI(bind(ctx));
  CKI(check_dtype(dtype));
  if (!size_out) return fail(ECC_EINVAL, "null size output");
  if (mode < 0 || mode > 2) return fail(ECC_EINVAL, "format mode must be 0 (CSV), 1 (JSON) or 2 (VCEC CSV)");
  if (n && (!thresholds || !chi)) return fail(ECC_EINVAL, "null curve arrays");
  if (n > 0x7FFFFFFFull) return fail(ECC_EINVAL, "curve exceeds 2^31 points");
  static const char* kHead[3] = {"threshold,euler_characteristic\n", "[", "value,change\n"};
  static const char* kTail[3] = {"", "]\n", ""};
  const uint64_t head = std::strlen(kHead[mode]), tail = std::strlen(kTail[mode]);
  cudaStream_t st = ctx->stream;
  const void* t = thresholds;
  const int64_t* c = chi;
  const size_t es = esize(dtype);
  if (n && where == 0) {
    CKI(ctx->input.ensure(n * es));
    CKI(ctx->asums.ensure(n * 8));
    CKR(cudaMemcpyAsync(ctx->input.p, thresholds, n * es, cudaMemcpyHostToDevice, st));
    CKR(cudaMemcpyAsync(ctx->asums.p, chi, n * 8, cudaMemcpyHostToDevice, st));
    t = ctx->input.p;
    c = ctx->asums.as<int64_t>();
  }
  uint64_t body = 0;
  if (n) {
    CKI(ctx->keys2.ensure(n * 4));
    CKI(ctx->sums2.ensure((n + 1) * 8));
    CKR(launch_point_sizes(mode, t, (int)dtype, c, n, ctx->keys2.as<uint32_t>(), ctx->sms, st));
    auto sz = thrust::make_transform_iterator(ctx->keys2.as<const uint32_t>(), ToU64());
    size_t tb = 0;
    CKR(cub::DeviceScan::ExclusiveSum(nullptr, tb, sz, ctx->sums2.as<uint64_t>(), (int)n + 0, st));
    CKI(ctx->tmp.ensure(tb));
    tb = ctx->tmp.cap;
    CKR(cub::DeviceScan::ExclusiveSum(ctx->tmp.p, tb, sz, ctx->sums2.as<uint64_t>(), (int)n, st));
    uint64_t last_off = 0;
    uint32_t last_sz = 0;
    CKR(cudaMemcpyAsync(&last_off, ctx->sums2.as<uint64_t>() + (n - 1), 8, cudaMemcpyDeviceToHost, st));
    CKR(cudaMemcpyAsync(&last_sz, ctx->keys2.as<uint32_t>() + (n - 1), 4, cudaMemcpyDeviceToHost, st));
    CKR(cudaStreamSynchronize(st));
    ctx->launches += 2;
    body = last_off + last_sz;
  }
  const uint64_t total = head + body + tail;
  *size_out = total;
  if (total > cap || !out)
    return fail(ECC_EINVAL, "output capacity " + std::to_string(cap) + " < " +
                                std::to_string(total) + " bytes");
  std::memcpy(out, kHead[mode], head);
  if (n) {
    CKI(ctx->res.ensure(body));
    CKR(launch_point_write(mode, t, (int)dtype, c, n, ctx->sums2.as<uint64_t>(), 0,
                           ctx->res.as<char>(), ctx->sms, st));
    ctx->launches += 1;
    CKR(cudaMemcpyAsync(out + head, ctx->res.p, body, cudaMemcpyDeviceToHost, st));
    CKR(cudaStreamSynchronize(st));
  }
  std::memcpy(out + head + body, kTail[mode], tail);
  return ECC_OK;
}
