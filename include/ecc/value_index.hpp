// ecc/value_index.hpp -- drop-in for the reference's value_index.hpp
// (value_index.hpp:13-197): ValueIndex<float> / ValueIndex<uint8_t>,
// build_index, the float order keys and build_index_counts.
//
// Building an index (sort + unique of a chunk's values) and the
// per-value aggregation of build_index_counts (the reference's radix argsort
// + run walk) run on the device as a radix sort + reduce-by-key
// (ecc_value_index / ecc_chunk_index_counts).  The index itself is the
// reference's host container: ascending distinct values, bin_of a binary
// search over them.
#pragma once

#include <algorithm>
#include <bit>
#include <cstdint>
#include <span>
#include <vector>

#include "ecc/chunk.hpp"
#include "ecc/common.hpp"
#include "ecc/context.hpp"

namespace ecc {

namespace detail {

// Order-preserving map from floats to uint32 (value_index.hpp:95-99): -0.0
// and +0.0 share a key.  The kernels use the same map (ecc_common.cuh).
inline std::uint32_t float_order_key(float f) {
  auto u = std::bit_cast<std::uint32_t>(f);
  if (u == 0x80000000u) u = 0;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Its inverse, -0.0 canonicalised to +0.0 (value_index.hpp:102-105).
inline float float_from_order_key(std::uint32_t k) {
  const std::uint32_t u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  return std::bit_cast<float>(u);
}

// Distinct values of `values` (and their summed changes) on the device.
template <class T>
std::vector<T> device_distinct(std::span<const T> values, const std::int8_t* changes,
                               std::vector<std::int64_t>* sums, Context& ctx) {
  std::uint64_t cap = std::min<std::uint64_t>(values.size(), 1ull << 20), n = 0;
  for (;;) {
    std::vector<T> out(cap);
    if (sums) sums->resize(cap);
    const int rc = ecc_value_index(ctx.get(), dtype_of<T>::value, values.data(), values.size(),
                                   changes, out.data(), sums ? sums->data() : nullptr, cap, &n);
    if (rc != ECC_OK && n > cap) {
      cap = n;
      continue;
    }
    check(rc);
    out.resize(n);
    if (sums) sums->resize(n);
    return out;
  }
}

}  // namespace detail

template <class T>
class ValueIndex;

// Sorted distinct floats; bin b holds value b (value_index.hpp:23-58).
template <>
class ValueIndex<float> {
 public:
  static ValueIndex build(std::span<const float> values, Context& ctx = Context::on(0)) {
    if (values.empty()) throw error("cannot build a value index: empty input");
    return from_sorted_unique(detail::device_distinct<float>(values, nullptr, nullptr, ctx));
  }
  static ValueIndex from_sorted_unique(std::vector<float> sorted) {
    ValueIndex idx;
    idx.values_ = std::move(sorted);
    return idx;
  }
  std::size_t bin_count() const { return values_.size(); }
  std::size_t bin_of(float v) const {
    auto it = std::lower_bound(values_.begin(), values_.end(), v);
    if (it == values_.end() || *it != v)
      throw error("value not present in index (internal consistency bug)");
    return static_cast<std::size_t>(it - values_.begin());
  }
  std::span<const float> distinct_values() const { return values_; }
  float value_of_bin(std::size_t b) const { return values_[b]; }

 private:
  std::vector<float> values_;
};

// 256 identity bins plus the list of occurring values (value_index.hpp:60-85).
template <>
class ValueIndex<std::uint8_t> {
 public:
  static ValueIndex build(std::span<const std::uint8_t> values, Context& ctx = Context::on(0)) {
    if (values.empty()) throw error("cannot build a value index: empty input");
    ValueIndex idx;
    idx.occurring_ = detail::device_distinct<std::uint8_t>(values, nullptr, nullptr, ctx);
    return idx;
  }
  std::size_t bin_count() const { return 256; }
  std::size_t bin_of(std::uint8_t v) const { return v; }
  std::span<const std::uint8_t> distinct_values() const { return occurring_; }
  std::uint8_t value_of_bin(std::size_t b) const { return static_cast<std::uint8_t>(b); }

 private:
  std::vector<std::uint8_t> occurring_;
};

template <class T>
ValueIndex<T> build_index(std::span<const T> values) {
  return ValueIndex<T>::build(values);
}

// A chunk's index plus its per-bin VCEC counts (value_index.hpp:150-157).
struct IndexedCounts {
  ValueIndex<float> index;
  std::vector<std::int64_t> counts;
};

// `changes` holds the per-voxel change of every owned voxel of the chunk in
// owned row-major order (compute_changes); the result lists the chunk's
// distinct values ascending with their summed changes
// (value_index.hpp:159-197), computed on the device.
inline IndexedCounts build_index_counts(const PaddedChunk<float>& chunk,
                                        std::span<const std::int8_t> changes,
                                        Context& ctx = Context::on(0)) {
  const std::uint64_t n = chunk.owned_voxels();
  if (changes.size() != n)
    throw error("change buffer does not match the chunk's owned voxel count");
  if (n > 0xFFFFFFFFull) throw error("chunk exceeds 2^32 voxels; use a finer chunk plan");
  std::uint64_t cap = std::min<std::uint64_t>(n, 1ull << 20), m = 0;
  for (;;) {
    std::vector<float> vals(cap);
    IndexedCounts out;
    out.counts.resize(cap);
    const int rc = ecc_chunk_index_counts(ctx.get(), chunk.data(), ECC_F32, chunk.descriptor(),
                                          changes.data(), vals.data(), out.counts.data(), cap, &m);
    if (rc != ECC_OK && m > cap) {
      cap = m;
      continue;
    }
    detail::check(rc);
    vals.resize(m);
    out.counts.resize(m);
    out.index = ValueIndex<float>::from_sorted_unique(std::move(vals));
    return out;
  }
}

}  // namespace ecc
