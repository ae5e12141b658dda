// internal.h -- launchers shared between the kernel translation units and
// the C ABI (capi.cu).  Not installed; the public boundary is
// include/ecc_b200.h.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "ecc_common.cuh"

namespace eccb {

// Opt kernel FN in to `bytes` of dynamic shared memory, once per device (the
// attribute is per device; a process may drive several GPUs, one context
// each).
template <auto FN>
inline void smem_optin(int bytes) {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(done.load(std::memory_order_relaxed) & bit)) {
    cudaFuncSetAttribute(FN, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done.fetch_or(bit);
  }
}

// Allow kernel FN non-portable cluster sizes (up to 16 CTAs), once per device.
template <auto FN>
inline void cluster16_optin() {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(done.load(std::memory_order_relaxed) & bit)) {
    cudaFuncSetAttribute(FN, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    done.fetch_or(bit);
  }
}

// Workspace of the fused single-launch curve (k_u8_3d.cu): `ticket` and the
// 512-entry int64 histogram must be zero before the launch and are zero
// again after it.
struct U83dFinalize {
  uint32_t* ticket;
  uint32_t* bins;
  int64_t* changes;
  int64_t* chi;
  uint64_t* count;
  // multi-GPU: fused rank exchange over peer memory (fin_u8.cuh, Xchg)
  int world = 1, rank = 0;
  uint32_t epoch = 0;
  int64_t* const* slots = nullptr;   // device array [world] of peers' slot buffers
  uint32_t* const* flags = nullptr;  // device array [world] of peers' flag arrays
  const int64_t* my_slots = nullptr;
  const uint32_t* my_flags = nullptr;
  uint32_t* err = nullptr;
};
bool u8_3d_supported(const Slab& s);
bool u16_3d_supported(const Slab& s);
bool u8_2d_supported(const Slab& s);
bool u16_2d_supported(const Slab& s);
cudaError_t launch_u16_2d(const Slab& s, uint32_t nbins, int64_t* ghist, int sms, cudaStream_t st);
cudaError_t launch_u8_2d(const Slab& s, int64_t* ghist, int sms, cudaStream_t st,
                         const U83dFinalize* fz = nullptr);
cudaError_t launch_u16_3d(const Slab& s, uint32_t nbins, int64_t* ghist, int sms, cudaStream_t st);
cudaError_t launch_affine_keys(const float* v, uint64_t rows, uint32_t w2, uint32_t pitch,
                               const AffineMap& am, uint16_t* keys, uint32_t* flags, int sms,
                               cudaStream_t st);
cudaError_t launch_u8_3d(const Slab& s, int64_t* ghist, int8_t* chg, int sms, cudaStream_t st,
                         const U83dFinalize* fz = nullptr);

cudaError_t launch_generic_accumulate(const Slab& s, int dtype, bool affine,
                                      const AffineMap& am, int64_t* ghist,
                                      uint32_t nbins, uint32_t* flags, int sms,
                                      cudaStream_t st);
cudaError_t launch_generic_changes(const Slab& s, int dtype, int8_t* out, int sms,
                                   cudaStream_t st);
// PaddedChunk storage -> uint32 key image (etype 0 int16, 1 int32, 2 float)
cudaError_t launch_chunk_keys(const void* padded, int etype, uint64_t np, uint64_t w1p,
                              uint64_t w2p, bool is2d, bool interior, uint32_t* keys, int sms,
                              cudaStream_t st);
// generic kernels over a key image; mode 0 histogram, 2 changes, 3 faces
cudaError_t launch_keyimage(const Slab& s, int mode, const AffineMap& am, int64_t* ghist,
                            uint32_t nbins, uint32_t* flags, void* out, int sms, cudaStream_t st);
cudaError_t launch_value_keys(const void* v, int dtype, uint64_t n, uint32_t* keys,
                              uint32_t* flags, int sms, cudaStream_t st);
cudaError_t launch_gather_local(const uint32_t* keys, bool by_value, uint64_t n,
                                const int64_t* local, uint64_t nlocal, int64_t* sums,
                                uint32_t* flags, int sms, cudaStream_t st);
// per owned voxel, the mask of FaceOffsets it introduces (tourney.cuh faces3)
cudaError_t launch_generic_faces(const Slab& s, int dtype, uint32_t* out, int sms,
                                 cudaStream_t st);
// sorted f32 path: key range (+ NaN flag), keys minus the minimum, and the
// minimum added back to the reduced keys
cudaError_t launch_key_range(const float* v, uint64_t n, uint32_t* flags, uint32_t* mm, int sms,
                             cudaStream_t st);
cudaError_t launch_order_keys(const float* v, uint64_t n, uint32_t* keys, const uint32_t* mm,
                              int sms, cudaStream_t st);
cudaError_t launch_add_key(uint32_t* keys, uint64_t n, const uint32_t* mm, int sms,
                           cudaStream_t st);
// K3; `scratch` (16 bytes per 1024 bins) enables the multi-CTA version for
// large bin counts.
// packed: the generic kernels' one-atomic dense table (HistSink)
cudaError_t launch_finalize(const int64_t* hist, uint32_t nbins, uint32_t* bins,
                            int64_t* changes, int64_t* chi, uint64_t* count, void* scratch,
                            cudaStream_t st, bool packed = false);
cudaError_t launch_uniform_noise(float* d, uint64_t n, uint64_t seed, int sms, cudaStream_t st);
int gaussian_max_width();
// mm / flags (optional): the pass also reduces its outputs' order-key range
// (mm[0] min, mm[1] max, NaN -> flags) when it is the pipelined contiguous
// pass; *ranged says whether it did
cudaError_t launch_convolve_axis(const float* in, float* out, uint64_t w0, uint64_t w1,
                                 uint64_t w2, int axis, const double* d_weights, int width,
                                 cudaStream_t st, uint32_t* mm = nullptr,
                                 uint32_t* flags = nullptr, bool* ranged = nullptr);
// batched curve serialisation (k_format.cu)
cudaError_t launch_format_sizes(const int32_t* chi, const uint32_t* pres, uint64_t count,
                                uint32_t nbins, int json, uint64_t* sizes, cudaStream_t st);
cudaError_t launch_format_write(const int32_t* chi, const uint32_t* pres, uint64_t count,
                                uint32_t nbins, int json, const uint64_t* offsets, char* out,
                                cudaStream_t st);
cudaError_t launch_zero_crossings(const int32_t* chi, const uint32_t* pres, uint64_t count,
                                  uint32_t nbins, uint32_t* zc, cudaStream_t st);
// one sparse curve's text (k_format.cu): per-point byte counts, then the write
cudaError_t launch_point_sizes(int mode, const void* t, int dtype, const int64_t* c, uint64_t n,
                               uint32_t* sizes, int sms, cudaStream_t st);
cudaError_t launch_point_write(int mode, const void* t, int dtype, const int64_t* c, uint64_t n,
                               const uint64_t* offsets, uint64_t head, char* out, int sms,
                               cudaStream_t st);
cudaError_t launch_fill(void* d, int dtype, uint64_t n, uint64_t seed,
                        uint64_t base, int sms, cudaStream_t st);

}  // namespace eccb
