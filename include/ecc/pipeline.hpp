// ecc/pipeline.hpp -- the reference's in-memory benchmark pipeline
// (proj/include/ecc/pipeline.hpp:212-291, datagen.hpp:57-122), GPU-resident.
//
//   BenchReport, bench_run(dims, iterations, seed, sigma, width)
//     uniform noise once, then `iterations` x {gaussian_smooth; ECC}, every
//     step on the GPU (ecc_bench_run), same report fields and to_string().
//   device::uniform_noise / device::gaussian_smooth
//     the generator and the separable Gaussian smoothing on device buffers,
//     bit-identical to the reference's host versions.
//
//   RunReport, ComputeConfig, compute_file(path, cfg)
//     one end-to-end run over a raw volume file (pipeline.hpp:23-133):
//     FileSource -> process_image on the GPU file path -> vcec_to_ecc ->
//     optional curve / VCEC files; same fields, plan and GVox/s definition.
//
// batch_run (glob + CLI orchestration) is not mirrored.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <fstream>
#include <optional>
#include <sstream>
#include <string>
#include <thread>

#include "ecc/common.hpp"
#include "ecc/curve.hpp"
#include "ecc/datagen.hpp"
#include "ecc/device.hpp"
#include "ecc/image.hpp"
#include "ecc/streaming.hpp"
#include "ecc_b200.h"

namespace ecc {

struct BenchReport {
  std::uint64_t iterations = 0;
  std::uint64_t voxels = 0;
  double generate_s = 0;
  double total_s = 0;          // smoothing + ECC loop, including one-time costs
  double per_iteration_s = 0;  // (generate_s + total_s) / iterations
  double ecc_avg_s = 0;        // device time per ECC (CUDA events)
  double smooth_avg_s = 0;     // device time per smoothing (CUDA events)
  double ecc_gvox_per_s = 0;
  std::uint64_t last_points = 0;     // not in the reference: the last curve's size
  std::int64_t last_chi_first = 0;   // and its first / last chi
  std::int64_t last_chi_last = 0;

  std::string to_string() const {
    std::ostringstream os;
    os << "iterations:       " << iterations << "\n"
       << "voxels:           " << voxels << "\n"
       << "generate:         " << generate_s << " s\n"
       << "loop total:       " << total_s << " s\n"
       << "per iteration:    " << per_iteration_s << " s\n"
       << "ECC avg:          " << ecc_avg_s << " s\n"
       << "smoothing avg:    " << smooth_avg_s << " s\n"
       << "ECC GVox/s:       " << ecc_gvox_per_s << "\n";
    return os.str();
  }
};

inline BenchReport bench_run(const Dims& dims, std::uint64_t iterations, std::uint64_t seed = 1,
                             double sigma = 2.0, int width = 13,
                             Context& ctx = Context::on(0)) {
  ecc_bench_report r{};
  detail::check(ecc_bench_run(ctx.get(), detail::cdims(dims), iterations, seed, sigma, width, &r));
  BenchReport b;
  b.iterations = r.iterations;
  b.voxels = r.voxels;
  b.generate_s = r.generate_s;
  b.total_s = r.total_s;
  b.per_iteration_s = r.per_iteration_s;
  b.ecc_avg_s = r.ecc_avg_s;
  b.smooth_avg_s = r.smooth_avg_s;
  b.ecc_gvox_per_s = r.ecc_gvox_per_s;
  b.last_points = r.last_points;
  b.last_chi_first = r.last_chi_first;
  b.last_chi_last = r.last_chi_last;
  return b;
}

// Per-phase times of one compute run (pipeline.hpp:23-48): the engine's
// ChunkTiming sums (CUDA-event device times for the kernel phase) and the
// wall time of the whole call.
struct RunReport {
  std::uint64_t voxels = 0;
  std::size_t chunk_count = 0;
  std::size_t curve_points = 0;
  std::int64_t final_chi = 0;
  double read_s = 0, index_s = 0, kernel_s = 0, merge_s = 0, total_s = 0;

  double gvox_per_s() const {
    return kernel_s > 0 ? static_cast<double>(voxels) / kernel_s / 1e9 : 0.0;
  }

  std::string to_string() const {
    std::ostringstream os;
    os << "voxels:        " << voxels << "\n"
       << "chunks:        " << chunk_count << "\n"
       << "curve points:  " << curve_points << "\n"
       << "final chi:     " << final_chi << "\n"
       << "disk read:     " << read_s << " s\n"
       << "index build:   " << index_s << " s\n"
       << "kernel:        " << kernel_s << " s\n"
       << "merge:         " << merge_s << " s\n"
       << "total:         " << total_s << " s\n"
       << "kernel GVox/s: " << gvox_per_s() << "\n";
    return os.str();
  }
};

struct ComputeConfig {
  std::optional<Dims> dims;       // falls back to the sidecar
  std::optional<ValueKind> kind;  // falls back to the sidecar
  bool big_endian = false;
  std::optional<std::uint64_t> chunks;
  std::optional<std::uint64_t> memory_budget;
  unsigned workers = std::max(1u, std::thread::hardware_concurrency());
  CurveFormat format = CurveFormat::csv;
  std::optional<std::string> curve_out;
  std::optional<std::string> vcec_out;
  std::chrono::milliseconds ingest_delay{0};
};

namespace detail {

template <class T>
RunReport compute_file_typed(const std::string& input, const Dims& dims,
                             const ComputeConfig& cfg) {
  const auto t0 = std::chrono::steady_clock::now();
  FileSource<T> source(input, dims, RawOptions{cfg.big_endian});
  const ChunkTarget target =
      cfg.memory_budget
          ? ChunkTarget::memory_budget(*cfg.memory_budget)
          : ChunkTarget::count(cfg.chunks ? *cfg.chunks : std::max<std::uint64_t>(2, cfg.workers));
  const ChunkPlan plan = plan_chunks<T>(dims, target);
  EngineOptions opt;
  opt.workers = cfg.workers;
  opt.ingest_delay = cfg.ingest_delay;
  EngineReport er;
  GlobalVcec<T> vcec = process_image<T>(source, plan, opt, &er);
  RunReport report;
  report.voxels = dims.voxel_count();
  report.chunk_count = plan.chunk_count();
  report.read_s = er.read_s;
  report.index_s = er.index_s;
  report.kernel_s = er.kernel_s;
  report.merge_s = er.merge_s;
  if (cfg.vcec_out) {
    std::ofstream out(*cfg.vcec_out, std::ios::binary | std::ios::trunc);
    if (!out) throw error("cannot open '" + *cfg.vcec_out + "' for writing");
    write_vcec(vcec, out);
  }
  EccCurve<T> curve = vcec_to_ecc(std::move(vcec));
  report.curve_points = curve.size();
  report.final_chi = curve.chi.empty() ? 0 : curve.chi.back();
  if (cfg.curve_out) write_curve(curve, cfg.format, *cfg.curve_out);
  report.total_s =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return report;
}

}  // namespace detail

// One end-to-end compute run over a raw volume file (pipeline.hpp:115-133).
inline RunReport compute_file(const std::string& input, const ComputeConfig& cfg) {
  Dims dims;
  ValueKind kind;
  if (cfg.dims && cfg.kind) {
    dims = *cfg.dims;
    kind = *cfg.kind;
  } else {
    const auto meta = read_sidecar(input);
    if (!meta) throw error("no dims/dtype given and no sidecar found for '" + input + "'");
    dims = cfg.dims.value_or(meta->dims);
    kind = cfg.kind.value_or(meta->kind);
  }
  if (kind == ValueKind::u8) return detail::compute_file_typed<std::uint8_t>(input, dims, cfg);
  if (kind == ValueKind::u16) return detail::compute_file_typed<std::uint16_t>(input, dims, cfg);
  return detail::compute_file_typed<float>(input, dims, cfg);
}

namespace device {

// uniform_noise (datagen.hpp:57-62) into a device buffer of dims.voxel_count() floats.
inline void uniform_noise(float* d_out, const Dims& dims, std::uint64_t seed,
                          void* stream = nullptr, Context& ctx = Context::on(0)) {
  detail::check(ecc_uniform_noise(ctx.get(), d_out, dims.voxel_count(), seed, stream));
}

// gaussian_smooth (datagen.hpp:108-122) of a device buffer; d_in may equal d_out.
inline void gaussian_smooth(const float* d_in, float* d_out, const Dims& dims, double sigma,
                            int width, void* stream = nullptr, Context& ctx = Context::on(0)) {
  detail::check(ecc_gaussian_smooth(ctx.get(), d_in, d_out, detail::cdims(dims), sigma, width,
                                    stream));
}

}  // namespace device
}  // namespace ecc
