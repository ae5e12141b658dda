// k_fast.cu -- dispatch to the shape-specialised kernels; returns
// handled = false when the generic kernel (k_generic.cu) must run.
#include "internal.h"

namespace eccb {

bool wide_supported(const Slab& s, int dtype, bool affine, uint32_t nbins);
cudaError_t launch_wide(const Slab& s, int dtype, bool affine, const AffineMap& am, int64_t* ghist,
                        uint32_t nbins, uint32_t* flags, int sms, cudaStream_t st);


cudaError_t launch_accumulate_fast(const Slab& s, int dtype, bool affine,
                                   const AffineMap& am, int64_t* ghist,
                                   uint32_t nbins, uint32_t* flags, int sms,
                                   cudaStream_t st, bool* handled) {
  *handled = false;
  if (dtype == 0 && !affine && nbins == 256 && u8_3d_supported(s)) {
    *handled = true;
    return launch_u8_3d(s, ghist, nullptr, sms, st);
  }
  if (wide_supported(s, dtype, affine, nbins)) {
    *handled = true;
    return launch_wide(s, dtype, affine, am, ghist, nbins, flags, sms, st);
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
