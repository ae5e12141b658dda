// ecc/streaming.hpp -- drop-in for the reference streaming engine
// (streaming.hpp:21-338): ChunkRange / ChunkPlan / ChunkTarget /
// plan_chunks (same ceil split and budget formula), ChunkTiming /
// EngineReport / EngineOptions, and process_image for a ChunkSource or an
// in-memory Image.
//
// process_image runs on the GPU: ecc_process_stream (csrc/capi.cu) pulls the
// plan's chunks (owned rows + one halo row per side) through read_rows into
// pinned staging, copies them to HBM on a copy stream while the previous
// chunk's stencil + histogram kernel runs, and finishes with the device
// compaction.  Exceptions from read_rows surface as
// "ingestion of chunk k failed: <what>" (streaming.hpp:250-259); invalid
// plans throw the reference's messages (streaming.hpp:186-195).
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "ecc/chunk.hpp"
#include "ecc/common.hpp"
#include "ecc/device.hpp"
#include "ecc/image.hpp"
#include "ecc/vcec.hpp"

namespace ecc {

struct ChunkRange {
  std::uint64_t begin = 0;
  std::uint64_t end = 0;
  std::uint64_t len() const { return end - begin; }
  bool operator==(const ChunkRange&) const = default;
};

struct ChunkPlan {
  std::vector<ChunkRange> ranges;
  std::size_t chunk_count() const { return ranges.size(); }
};

struct ChunkTarget {
  static ChunkTarget count(std::uint64_t c) {
    ChunkTarget t;
    t.chunks = c;
    return t;
  }
  static ChunkTarget memory_budget(std::uint64_t bytes) {
    ChunkTarget t;
    t.budget_bytes = bytes;
    return t;
  }
  std::optional<std::uint64_t> chunks;
  std::optional<std::uint64_t> budget_bytes;
};

namespace detail {

// Ceil split of [0, w0) into at most c ranges (the reference's even_plan).
inline ChunkPlan even_plan(std::uint64_t w0, std::uint64_t c) {
  c = std::max<std::uint64_t>(1, std::min(c, w0));
  const std::uint64_t len = (w0 + c - 1) / c;
  ChunkPlan plan;
  for (std::uint64_t a = 0; a < w0; a += len) plan.ranges.push_back({a, std::min(a + len, w0)});
  return plan;
}

}  // namespace detail

template <class T>
ChunkPlan plan_chunks(const Dims& dims, const ChunkTarget& target) {
  if (dims.w0 < 1) throw error("w0 must be >= 1");
  if (target.chunks) return detail::even_plan(dims.w0, *target.chunks);
  if (!target.budget_bytes) throw error("chunk target needs a count or a memory budget");
  const std::uint64_t plane = padded_chunk_bytes<T>(dims, 1) / 3;
  const std::uint64_t minimum = 2 * padded_chunk_bytes<T>(dims, 1);
  if (*target.budget_bytes < minimum)
    throw error("memory budget " + std::to_string(*target.budget_bytes) +
                " bytes is below the minimum feasible " + std::to_string(minimum) +
                " bytes (two single-row padded chunks)");
  const std::uint64_t len = *target.budget_bytes / (2 * plane) - 2;
  return detail::even_plan(dims.w0, (dims.w0 + len - 1) / len);
}

struct ChunkTiming {
  ChunkRange range;
  double ingest_begin = 0, ingest_end = 0;  // seconds since engine start
  double index_begin = 0, index_end = 0;
  double kernel_begin = 0, kernel_end = 0;
  double merge_begin = 0, merge_end = 0;
};

struct EngineReport {
  std::vector<ChunkTiming> chunks;
  double read_s = 0, index_s = 0, kernel_s = 0, merge_s = 0;
  std::uint64_t peak_chunk_bytes = 0;
};

struct EngineOptions {
  unsigned workers = 1;  // accepted for API compatibility; the GPU sets its own parallelism
  std::chrono::milliseconds ingest_delay{0};  // test hook, as in the reference
  int device = 0;                             // extension: which GPU
  std::optional<BinMap> bins;                 // extension: f32 bin map (default sorted)
};

namespace detail {

template <class T>
struct StreamCall {
  ChunkSource<T>* src;
  std::chrono::milliseconds delay;
  std::exception_ptr err;
};

template <class T>
int read_rows_tramp(void* user, std::uint64_t r0, std::uint64_t r1, void* dst, char* errbuf,
                    std::size_t errlen) {
  auto* call = static_cast<StreamCall<T>*>(user);
  try {
    if (call->delay.count() > 0) std::this_thread::sleep_for(call->delay);
    call->src->read_rows(r0, r1, static_cast<T*>(dst));
    return 0;
  } catch (const std::exception& e) {
    std::snprintf(errbuf, errlen, "%s", e.what());
  } catch (...) {
    std::snprintf(errbuf, errlen, "unknown exception");
  }
  call->err = std::current_exception();
  return 1;
}

}  // namespace detail

// EngineReport from the per-chunk timings: phase sums and the bytes of the
// pinned staging the driver holds (two buffers of the largest chunk's rows
// plus its halo rows -- the GPU counterpart of the reference's <= 2 resident
// padded chunks, and what is registered with chunk_memory()).
inline std::uint64_t staging_bytes(const ChunkPlan& plan, const Dims& dims, std::size_t elem) {
  std::uint64_t rows = 0;
  for (const auto& r : plan.ranges) rows = std::max(rows, r.len() + 2);
  return 2 * std::min(rows, dims.w0) * dims.w1 * dims.w2 * elem;
}

inline void fill_report(EngineReport* report, const std::vector<ecc_chunk_timing>& tim,
                        std::uint64_t staging) {
  if (!report) return;
  report->chunks.clear();
  report->read_s = report->index_s = report->kernel_s = report->merge_s = 0;
  for (const auto& t : tim) {
    ChunkTiming c;
    c.range = {t.begin, t.end};
    c.ingest_begin = t.ingest_begin;
    c.ingest_end = t.ingest_end;
    c.index_begin = t.index_begin;
    c.index_end = t.index_end;
    c.kernel_begin = t.kernel_begin;
    c.kernel_end = t.kernel_end;
    c.merge_begin = t.merge_begin;
    c.merge_end = t.merge_end;
    report->read_s += c.ingest_end - c.ingest_begin;
    report->index_s += c.index_end - c.index_begin;
    report->kernel_s += c.kernel_end - c.kernel_begin;
    report->merge_s += c.merge_end - c.merge_begin;
    report->chunks.push_back(c);
  }
  report->peak_chunk_bytes = staging;
}

template <class T>
GlobalVcec<T> process_image(ChunkSource<T>& source, const ChunkPlan& plan,
                            const EngineOptions& opt = {}, EngineReport* report = nullptr) {
  const Dims dims = source.dims();
  if (plan.ranges.empty()) throw error("empty chunk plan");
  std::uint64_t expected = 0;
  for (const auto& r : plan.ranges) {
    if (r.begin != expected || r.end <= r.begin)
      throw error("chunk plan does not cover the image contiguously");
    expected = r.end;
  }
  if (expected != dims.w0)
    throw error("chunk plan covers [0, " + std::to_string(expected) +
                ") but the source has w0 = " + std::to_string(dims.w0));
  std::vector<std::uint64_t> bounds{0};
  for (const auto& r : plan.ranges) bounds.push_back(r.end);
  Context& ctx = Context::on(opt.device);
  ecc_binmap b;
  const BinMap* bm = opt.bins ? &*opt.bins : nullptr;
  const ecc_binmap* pb = detail::binmap_for<T>(bm, b);
  std::uint64_t cap = 0;
  if (b.kind == ECC_BIN_SORTED)
    cap = std::min<std::uint64_t>(dims.voxel_count(), 1ull << 22);
  else
    detail::check(ecc_bin_count(detail::dtype_of<T>::value, pb, &cap));
  std::vector<ecc_chunk_timing> tim(plan.ranges.size());
  const std::uint64_t staging = staging_bytes(plan, dims, sizeof(T));
  const TrackedBytes held(staging);
  for (;;) {
    GlobalVcec<T> out;
    out.values.resize(cap);
    out.changes.resize(cap);
    std::uint64_t n = 0;
    detail::StreamCall<T> call{&source, opt.ingest_delay, nullptr};
    const int rc = ecc_process_stream(ctx.get(), &detail::read_rows_tramp<T>, &call,
                                      detail::dtype_of<T>::value, detail::cdims(dims),
                                      bounds.data(), plan.ranges.size(), pb, tim.data(),
                                      out.values.data(), out.changes.data(), cap, &n);
    if (rc != ECC_OK && n > cap) {
      cap = n;
      continue;
    }
    detail::check(rc);
    out.values.resize(n);
    out.changes.resize(n);
    fill_report(report, tim, staging);
    return out;
  }
}

// A FileSource streams through the GPU file path (ecc_process_file): chunked
// pread into pinned staging, f32 byte swap + NaN rejection on the device,
// the reference's error wording.
template <class T>
GlobalVcec<T> process_image(FileSource<T>& source, const ChunkPlan& plan,
                            const EngineOptions& opt = {}, EngineReport* report = nullptr) {
  const Dims dims = source.dims();
  if (plan.ranges.empty()) throw error("empty chunk plan");
  std::vector<std::uint64_t> bounds{plan.ranges.front().begin};
  for (const auto& r : plan.ranges) bounds.push_back(r.end);
  Context& ctx = Context::on(opt.device);
  ecc_binmap b;
  const BinMap* bm = opt.bins ? &*opt.bins : nullptr;
  const ecc_binmap* pb = detail::binmap_for<T>(bm, b);
  std::uint64_t cap = 0;
  if (b.kind == ECC_BIN_SORTED)
    cap = std::min<std::uint64_t>(dims.voxel_count(), 1ull << 22);
  else
    detail::check(ecc_bin_count(detail::dtype_of<T>::value, pb, &cap));
  std::vector<ecc_chunk_timing> tim(plan.ranges.size());
  const std::uint64_t staging = staging_bytes(plan, dims, sizeof(T));
  const TrackedBytes held(staging);
  for (;;) {
    GlobalVcec<T> out;
    out.values.resize(cap);
    out.changes.resize(cap);
    std::uint64_t n = 0;
    const int rc = ecc_process_file(ctx.get(), source.path().c_str(), detail::dtype_of<T>::value,
                                    detail::cdims(dims), source.options().big_endian ? 1 : 0,
                                    bounds.data(), plan.ranges.size(), pb, tim.data(),
                                    out.values.data(), out.changes.data(), cap, &n);
    if (rc != ECC_OK && n > cap) {
      cap = n;
      continue;
    }
    detail::check(rc);
    out.values.resize(n);
    out.changes.resize(n);
    fill_report(report, tim, staging);
    return out;
  }
}

// Convenience wrapper for whole in-memory images (streaming.hpp:332-338).
template <class T>
GlobalVcec<T> process_image(const Image<T>& image, const ChunkPlan& plan,
                            const EngineOptions& opt = {}, EngineReport* report = nullptr) {
  MemorySource<T> source(image);
  return process_image(source, plan, opt, report);
}

}  // namespace ecc
