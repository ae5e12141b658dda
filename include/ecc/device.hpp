// ecc/device.hpp -- the C++ side of the drop-in: one GPU context per device
// behind the C ABI of ecc_b200.h, the dtype mapping, error translation to
// ecc::error, and the GPU entry points the reference has no name for
// (device-resident curves, batched 2D, slab kernels).
//
// Link with paper_2203_09087_b200/lib/libecc_b200.so.  There is no CPU
// fallback: without the library or a GPU every call throws ecc::error.
#pragma once

#include <cstdint>
#include <algorithm>
#include <memory>
#include <type_traits>
#include <mutex>
#include <string>
#include <vector>

#include "ecc/common.hpp"
#include "ecc/curve.hpp"
#include "ecc/vcec.hpp"
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

namespace device {

// Host image -> curve (H2D, K1+K2+K3 on the GPU, D2H of the curve).
template <class T>
EccCurve<T> curve(const T* values, const Dims& dims, const BinMap* bm = nullptr,
                  Context& ctx = Context::on(0)) {
  ecc_binmap b;
  const auto* pb = detail::binmap_for<T>(bm, b);
  std::uint64_t cap = 0;
  if (b.kind == ECC_BIN_SORTED)
    cap = std::min<std::uint64_t>(dims.voxel_count(), 1ull << 22);
  else
    detail::check(ecc_bin_count(detail::dtype_of<T>::value, pb, &cap));
  for (;;) {
    EccCurve<T> c;
    c.thresholds.resize(cap);
    c.chi.resize(cap);
    std::uint64_t n = 0;
    const int rc = ecc_curve(ctx.get(), values, 0, detail::dtype_of<T>::value, detail::cdims(dims),
                             pb, c.thresholds.data(), c.chi.data(), cap, &n);
    if (rc != ECC_OK && n > cap) {  // sorted path with more distinct values
      cap = n;
      continue;
    }
    detail::check(rc);
    c.thresholds.resize(n);
    c.chi.resize(n);
    return c;
  }
}

// Same for the VCEC.
template <class T>
GlobalVcec<T> vcec(const T* values, const Dims& dims, const BinMap* bm = nullptr,
                   Context& ctx = Context::on(0)) {
  ecc_binmap b;
  const auto* pb = detail::binmap_for<T>(bm, b);
  std::uint64_t cap = 0;
  if (b.kind == ECC_BIN_SORTED)
    cap = std::min<std::uint64_t>(dims.voxel_count(), 1ull << 22);
  else
    detail::check(ecc_bin_count(detail::dtype_of<T>::value, pb, &cap));
  for (;;) {
    GlobalVcec<T> v;
    v.values.resize(cap);
    v.changes.resize(cap);
    std::uint64_t n = 0;
    const int rc = ecc_vcec(ctx.get(), values, 0, detail::dtype_of<T>::value, detail::cdims(dims),
                            pb, v.values.data(), v.changes.data(), cap, &n);
    if (rc != ECC_OK && n > cap) {
      cap = n;
      continue;
    }
    detail::check(rc);
    v.values.resize(n);
    v.changes.resize(n);
    return v;
  }
}

// Device-resident image (d_values in HBM) -> curve in device buffers; one
// fused launch for 3D u8 volumes (ecc_curve_device).
template <class T>
void curve_on_device(const T* d_values, const Dims& dims, std::uint32_t* d_bins,
                     std::int64_t* d_changes, std::int64_t* d_chi, std::uint64_t* d_count,
                     const BinMap* bm = nullptr, void* stream = nullptr,
                     Context& ctx = Context::on(0)) {
  ecc_binmap b;
  detail::check(ecc_curve_device(ctx.get(), d_values, detail::dtype_of<T>::value,
                                 detail::cdims(dims), detail::binmap_for<T>(bm, b), d_bins,
                                 d_changes, d_chi, d_count, stream));
}

// Batched 2D (no reference equivalent): `count` h x w images
// back to back -> dense chi[count][nbins] (int32) + presence bitmaps.
template <class T>
void batch2d(const T* images, std::uint64_t count, std::uint64_t h, std::uint64_t w,
             std::vector<std::int32_t>& chi, std::vector<std::uint32_t>& presence,
             Context& ctx = Context::on(0)) {
  static_assert(!std::is_same_v<T, float>, "batched 2D takes u8 / u16 images");
  const std::uint64_t nbins = std::is_same_v<T, std::uint8_t> ? 256 : 65536;
  chi.resize(count * nbins);
  presence.resize(count * nbins / 32);
  detail::check(ecc_batch2d(ctx.get(), images, 0, detail::dtype_of<T>::value, count, h, w,
                            chi.data(), presence.data(), nullptr));
}

// Occurring points of one dense batched curve row.
template <class T>
EccCurve<T> batch_row_curve(const std::int32_t* chi_row, const std::uint32_t* presence_row,
                            std::uint64_t nbins) {
  EccCurve<T> c;
  for (std::uint64_t t = 0; t < nbins; ++t)
    if ((presence_row[t >> 5] >> (t & 31)) & 1u) {
      c.thresholds.push_back(static_cast<T>(t));
      c.chi.push_back(chi_row[t]);
    }
  return c;
}

}  // namespace device
}  // namespace ecc
