// ecc/kernel.hpp -- drop-in for the reference's kernel.hpp
// (kernel.hpp:14-277): FaceOffset / earlier, introduced / voxel_contribution,
// LocalVcec, accumulate_chunk, compute_changes and accumulate_dense_u8 on a
// PaddedChunk.
//
// Every voxel evaluation runs on the GPU: the chunk's padded storage is
// uploaded as it is and the tournament stencil (csrc/tourney.cuh) produces
// the per-voxel changes (ecc_chunk_changes), the introduced-face masks
// (ecc_chunk_faces) or the per-bin change sums (ecc_chunk_accumulate).  The
// definitions the reference states as code -- earlier()'s order rule and the
// face-dimension signs -- are restated here as the contract the device
// kernels are tested against.
#pragma once

#include <array>
#include <cstdint>
#include <span>
#include <type_traits>
#include <vector>

#include "ecc/chunk.hpp"
#include "ecc/common.hpp"
#include "ecc/context.hpp"
#include "ecc/value_index.hpp"

namespace ecc {

// Offset from a voxel to one of its faces, each component in {-1, 0, +1};
// the face dimension is d minus the number of nonzero components.
using FaceOffset = std::array<int, 3>;

// True iff the voxel at v + s comes before v in row-major order: the first
// nonzero component (axis 0 first) is negative (kernel.hpp:18-27).  Ties
// between equal values go to the earlier voxel.
inline bool earlier(const FaceOffset& s) {
  for (int i = 0; i < 3; ++i) {
    if (s[i] < 0) return true;
    if (s[i] > 0) return false;
  }
  throw error("earlier() requires a nonzero offset");
}

namespace detail {

template <class T>
constexpr ecc_dtype chunk_dtype() {
  return dtype_of<T>::value;
}

inline void check_owned(const Coord& v, const Dims& d, std::uint64_t begin, std::uint64_t end) {
  if (v[0] < begin || v[0] >= end || v[1] >= d.w1 || v[2] >= d.w2)
    throw error("voxel (" + std::to_string(v[0]) + "," + std::to_string(v[1]) + "," +
                std::to_string(v[2]) + ") is not an owned voxel of chunk rows [" +
                std::to_string(begin) + ", " + std::to_string(end) + ")");
}

// Introduced-face mask of one owned voxel (bit (o0+1)*9 + (o1+1)*3 + o2+1).
template <class T>
std::uint32_t face_mask(const PaddedChunk<T>& chunk, const Coord& v, Context& ctx) {
  const Dims& d = chunk.image_dims();
  check_owned(v, d, chunk.begin(), chunk.end());
  const std::uint64_t r = v[0] - chunk.begin();
  std::vector<std::uint32_t> row(d.w1 * d.w2);
  check(ecc_chunk_faces(ctx.get(), chunk.data(), chunk_dtype<T>(), chunk.descriptor(), r, r + 1,
                        row.data()));
  return row[v[1] * d.w2 + v[2]];
}

}  // namespace detail

// True iff voxel v introduces the face with offset o: v is the minimum of
// the voxels containing that face, ties to the lower row-major index,
// collar sentinels never defeating v (kernel.hpp:29-55).
template <class T>
bool introduced(const PaddedChunk<T>& chunk, const Coord& v, const FaceOffset& o,
                Context& ctx = Context::on(0)) {
  if (o[0] == 0 && o[1] == 0 && o[2] == 0) throw error("introduced() requires a nonzero offset");
  for (int i = 0; i < 3; ++i)
    if (o[i] < -1 || o[i] > 1) throw error("face offsets are in {-1, 0, +1}");
  const int bit = (o[0] + 1) * 9 + (o[1] + 1) * 3 + (o[2] + 1);
  return (detail::face_mask(chunk, v, ctx) >> bit) & 1u;
}

// Signed change of the Euler characteristic contributed by one owned voxel:
// (-1)^d for the voxel plus (-1)^dim(face) per introduced face
// (kernel.hpp:57-74).
template <class T>
int voxel_contribution(const PaddedChunk<T>& chunk, const Coord& v, Context& ctx = Context::on(0)) {
  const Dims& d = chunk.image_dims();
  detail::check_owned(v, d, chunk.begin(), chunk.end());
  const std::uint64_t r = v[0] - chunk.begin();
  std::vector<std::int8_t> row(d.w1 * d.w2);
  detail::check(ecc_chunk_changes(ctx.get(), chunk.data(), detail::chunk_dtype<T>(),
                                  chunk.descriptor(), r, r + 1, row.data()));
  return row[v[1] * d.w2 + v[2]];
}

using LocalVcec = std::vector<std::int64_t>;

// Chunk-local histogram of Euler changes, one counter per bin of the index
// (kernel.hpp:226-239): the device stencil + per-bin sums.
template <class T>
LocalVcec accumulate_chunk(const PaddedChunk<T>& chunk, const ValueIndex<T>& index,
                           Context& ctx = Context::on(0)) {
  LocalVcec counts(index.bin_count(), 0);
  if constexpr (std::is_same_v<T, float>) {
    detail::check(ecc_chunk_accumulate(ctx.get(), chunk.data(), ECC_F32, chunk.descriptor(), 0,
                                       chunk.owned_len(), index.distinct_values().data(),
                                       index.bin_count(), counts.data()));
  } else {
    detail::check(ecc_chunk_accumulate(ctx.get(), chunk.data(), detail::chunk_dtype<T>(),
                                       chunk.descriptor(), 0, chunk.owned_len(), nullptr,
                                       index.bin_count(), counts.data()));
  }
  return counts;
}

// Per-voxel changes of rows [row_begin, row_end) in owned row-major order,
// written at their owned linear index (kernel.hpp:241-265).
template <class T>
void compute_changes(const PaddedChunk<T>& chunk, std::uint64_t row_begin, std::uint64_t row_end,
                     std::span<std::int8_t> changes, Context& ctx = Context::on(0)) {
  const Dims& d = chunk.image_dims();
  const std::uint64_t off = row_begin * d.w1 * d.w2;
  if (row_end < row_begin || off + (row_end - row_begin) * d.w1 * d.w2 > changes.size())
    throw error("change buffer is smaller than the requested rows");
  detail::check(ecc_chunk_changes(ctx.get(), chunk.data(), detail::chunk_dtype<T>(),
                                  chunk.descriptor(), row_begin, row_end, changes.data() + off));
}

// 8-bit fast path: the center value is the bin (kernel.hpp:267-277).
template <class C>
void accumulate_dense_u8(const PaddedChunk<std::uint8_t>& chunk, std::uint64_t row_begin,
                         std::uint64_t row_end, std::span<C> counts,
                         Context& ctx = Context::on(0)) {
  if (counts.size() < 256) throw error("accumulate_dense_u8 needs 256 counters");
  std::vector<std::int64_t> h(256);
  detail::check(ecc_chunk_accumulate(ctx.get(), chunk.data(), ECC_U8, chunk.descriptor(),
                                     row_begin, row_end, nullptr, 256, h.data()));
  for (int b = 0; b < 256; ++b) counts[b] += static_cast<C>(h[b]);
}

}  // namespace ecc
