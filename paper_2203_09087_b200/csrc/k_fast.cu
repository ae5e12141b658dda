// k_fast.cu -- dispatch of u8 slabs to the bit-sliced kernels
// (k_u8_3d.cu, k_u8_2d.cu); returns handled = false when the generic kernel
// (k_generic.cu) must run.  16-bit keys are dispatched in capi.cu
// (accumulate_keys16), since they may need a conversion pass first.
#include "internal.h"

namespace eccb {

cudaError_t launch_accumulate_fast(const Slab& s, int dtype, bool affine,
                                   const AffineMap& am, int64_t* ghist,
                                   uint32_t nbins, uint32_t* flags, int sms,
                                   cudaStream_t st, bool* handled) {
  (void)am;
  (void)flags;
  *handled = false;
  if (dtype == 0 && !affine && nbins == 256 && u8_3d_supported(s)) {
    *handled = true;
    return launch_u8_3d(s, ghist, nullptr, sms, st);
  }
  if (dtype == 0 && !affine && nbins == 256 && u8_2d_supported(s)) {
    *handled = true;
    return launch_u8_2d(s, ghist, sms, st);
  }
  return cudaSuccess;
}

cudaError_t launch_changes_fast(const Slab& s, int dtype, int8_t* out, int sms, cudaStream_t st,
                                bool* handled) {
  *handled = false;
  if (dtype == 0 && u8_3d_supported(s)) {
    *handled = true;
    return launch_u8_3d(s, nullptr, out, sms, st);
  }
  return cudaSuccess;
}

}  // namespace eccb
