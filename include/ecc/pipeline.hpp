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
// compute_file / batch_run (file + CLI orchestration) are not mirrored:
// process_image(FileSource<T>&, plan) covers their hot path.
#pragma once

#include <cstdint>
#include <sstream>
#include <string>

#include "ecc/common.hpp"
#include "ecc/device.hpp"
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
