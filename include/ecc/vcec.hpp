// ecc/vcec.hpp -- drop-in for GlobalVcec and merge_local (reference
// vcec.hpp:15-66).
//
// process_image never calls merge_local: its merge is the device histogram
// (one int64 bin per value, summed by every CTA / chunk / GPU) and K3's
// compaction of the occurring bins.  merge_local is the reference's
// lower-level entry point for callers that hold a chunk histogram; it runs
// as a device sort + reduce-by-key of the global entries and the chunk's
// occurring values (ecc_merge_local).
#pragma once

#include <algorithm>
#include <cstdint>
#include <numeric>
#include <span>
#include <vector>

#include "ecc/common.hpp"
#include "ecc/context.hpp"
#include "ecc/value_index.hpp"

namespace ecc {

// Map from grayscale value to the signed change in the Euler characteristic:
// ascending occurring values (zero-change values that occur are kept) and
// their int64 changes.  Sums to 1 over any complete image.
template <class T>
struct GlobalVcec {
  std::vector<T> values;
  std::vector<std::int64_t> changes;

  std::size_t size() const { return values.size(); }
  std::int64_t total() const {
    return std::accumulate(changes.begin(), changes.end(), std::int64_t{0});
  }
  std::int64_t change_for(T v) const {
    auto it = std::lower_bound(values.begin(), values.end(), v);
    if (it == values.end() || *it != v) return 0;
    return changes[static_cast<std::size_t>(it - values.begin())];
  }
};

// Folds a chunk-local histogram into the global VCEC: for every value the
// chunk's index lists as occurring, global[value] += local[bin_of(value)],
// inserting new values (zero changes included).
template <class T, class C>
void merge_local(GlobalVcec<T>& global, std::span<const C> local, const ValueIndex<T>& index,
                 Context& ctx = Context::on(0)) {
  if (local.size() != index.bin_count())
    throw error("local VCEC length does not match the index bin count");
  const auto incoming = index.distinct_values();
  std::vector<std::int64_t> loc(local.begin(), local.end());
  const std::uint64_t cap = global.size() + incoming.size();
  std::vector<T> values(cap);
  std::vector<std::int64_t> changes(cap);
  std::uint64_t n = 0;
  detail::check(ecc_merge_local(ctx.get(), detail::dtype_of<T>::value, global.values.data(),
                                global.changes.data(), global.size(), loc.data(), loc.size(),
                                incoming.data(), incoming.size(), values.data(), changes.data(),
                                cap, &n));
  values.resize(n);
  changes.resize(n);
  global.values = std::move(values);
  global.changes = std::move(changes);
}

}  // namespace ecc
