// ecc/context.hpp -- the C++ side of the drop-in's device access: one GPU
// context per device behind the C ABI of ecc_b200.h, the dtype mapping,
// f32 bin maps and error translation to ecc::error.  Every header of the
// drop-in that does voxel work reaches the GPU through this.
//
// Link with paper_2203_09087_b200/lib/libecc_b200.so.  There is no CPU
// fallback: without the library or a GPU every call throws ecc::error.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "ecc/common.hpp"
#include "ecc_b200.h"

namespace ecc {

// Value -> histogram bin map for f32 images (ecc_binmap).  u8/u16 always use
// the identity map.  `sorted()` is the reference's general path (distinct
// values found by sort + reduce-by-key, value_index.hpp:159-197, on the
// device); `affine(n, lo, step)` is the exact quantised map BASELINE config 4
// uses (every value must equal lo + k * step, 0 <= k < n, else ecc::error).
struct BinMap {
  ecc_binmap raw{ECC_BIN_SORTED, 0, 0.0f, 0.0f};
  static BinMap sorted() { return BinMap{}; }
  static BinMap identity() { return BinMap{{ECC_BIN_IDENTITY, 0, 0.0f, 0.0f}}; }
  static BinMap affine(std::uint32_t n, float lo, float step) {
    return BinMap{{ECC_BIN_AFFINE, n, lo, step}};
  }
};

namespace detail {

inline void check(int rc) {
  if (rc != ECC_OK) throw error(ecc_last_error());
}

template <class T>
struct dtype_of;
template <>
struct dtype_of<std::uint8_t> {
  static constexpr ecc_dtype value = ECC_U8;
};
template <>
struct dtype_of<std::uint16_t> {
  static constexpr ecc_dtype value = ECC_U16;
};
template <>
struct dtype_of<float> {
  static constexpr ecc_dtype value = ECC_F32;
};

template <class T>
const ecc_binmap* binmap_for(const BinMap* bm, ecc_binmap& storage) {
  if constexpr (dtype_of<T>::value == ECC_F32) {
    storage = bm ? bm->raw : BinMap::sorted().raw;
  } else {
    storage = BinMap::identity().raw;
  }
  return &storage;
}

inline ecc_dims cdims(const Dims& d) { return ecc_dims{d.w0, d.w1, d.w2}; }

}  // namespace detail

// One CUDA context (stream, scratch, pinned staging) on one GPU.
class Context {
 public:
  explicit Context(int device = 0) { detail::check(ecc_ctx_create(device, &ctx_)); }
  ~Context() { ecc_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  ecc_ctx* get() const { return ctx_; }
  void* stream() const { return ecc_ctx_stream(ctx_); }
  std::uint64_t launch_count() const { return ecc_ctx_launch_count(ctx_); }

  // Process-wide default context of `device` (created on first use); the
  // reference-shaped free functions (process_image, ...) run on it.
  static Context& on(int device = 0) {
    static std::mutex m;
    static std::vector<std::unique_ptr<Context>> all;
    std::lock_guard<std::mutex> lock(m);
    if (device < 0) throw error("device " + std::to_string(device) + " out of range");
    if (all.size() <= static_cast<std::size_t>(device)) all.resize(device + 1);
    if (!all[device]) all[device] = std::make_unique<Context>(device);
    return *all[device];
  }

 private:
  ecc_ctx* ctx_ = nullptr;
};

}  // namespace ecc
