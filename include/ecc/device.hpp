// ecc/device.hpp -- the GPU entry points the reference has no name for
// (device-resident curves, batched 2D, slab kernels) over the context of
// ecc/context.hpp.
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
#include "ecc/context.hpp"
#include "ecc/curve.hpp"
#include "ecc/vcec.hpp"
#include "ecc_b200.h"

namespace ecc {

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

// write_curve's CSV / JSON text (curve.hpp:87-121) of one curve, formatted on
// the GPU (f32 thresholds as std::to_chars' shortest round-trip text):
// byte-identical to ecc::write_curve, for large curves.
template <class T>
std::string format_curve(const EccCurve<T>& c, CurveFormat format, Context& ctx = Context::on(0)) {
  std::uint64_t n = 0;
  const int mode = format == CurveFormat::json ? 1 : 0;
  const int rc = ecc_format_curve(ctx.get(), detail::dtype_of<T>::value, c.thresholds.data(),
                                  c.chi.data(), c.size(), 0, mode, nullptr, 0, &n);
  if (rc != ECC_OK && n == 0) detail::check(rc);
  std::string out(n, '\0');
  detail::check(ecc_format_curve(ctx.get(), detail::dtype_of<T>::value, c.thresholds.data(),
                                 c.chi.data(), c.size(), 0, mode, out.data(), n, &n));
  return out;
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
