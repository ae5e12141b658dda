// ecc/vcec.hpp -- drop-in for GlobalVcec (reference vcec.hpp:15-31).
//
// The reference builds it with merge_local (vcec.hpp:35-66), a host sorted
// merge per chunk.  Here the merge is the device histogram (one int64 bin
// per value, summed by every CTA / every chunk / every GPU) and K3's
// compaction of the occurring bins; GlobalVcec is only the result type.
#pragma once

#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

#include "ecc/common.hpp"

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

}  // namespace ecc
