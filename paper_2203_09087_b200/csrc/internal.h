// internal.h -- launchers shared between the kernel translation units and
// the C ABI (capi.cu).  Not installed; the public boundary is
// include/ecc_b200.h.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ecc_common.cuh"

namespace eccb {

cudaError_t launch_generic_accumulate(const Slab& s, int dtype, bool affine,
                                      const AffineMap& am, int64_t* ghist,
                                      uint32_t nbins, uint32_t* flags, int sms,
                                      cudaStream_t st);
cudaError_t launch_generic_changes(const Slab& s, int dtype, int8_t* out, int sms,
                                   cudaStream_t st);
cudaError_t launch_order_keys(const float* v, uint64_t n, uint32_t* keys,
                              uint32_t* flags, int sms, cudaStream_t st);
cudaError_t launch_finalize(const int64_t* hist, uint32_t nbins, uint32_t* bins,
                            int64_t* changes, int64_t* chi, uint64_t* count,
                            cudaStream_t st);
cudaError_t launch_fill(void* d, int dtype, uint64_t n, uint64_t seed,
                        uint64_t base, int sms, cudaStream_t st);

}  // namespace eccb
