// ecc/datagen.hpp -- drop-in for the synthetic-input part of the reference's
// datagen.hpp (datagen.hpp:48-122): GenKind / GenSpec, uniform_noise,
// gaussian_kernel and gaussian_smooth, computed on the device and returned
// as host images, bit-identical to the reference's host versions
// (csrc/k_pipeline.cu; the taps are the reference's formula with libm exp).
// generate_grf (Box-Muller through libm log / cos) is not reproducible to
// the bit on the GPU and is not mirrored.
#pragma once

#include <cmath>
#include <cstdint>
#include <vector>

#include "ecc/common.hpp"
#include "ecc/context.hpp"
#include "ecc/image.hpp"

namespace ecc {

enum class GenKind { uniform, grf };

struct GenSpec {
  Dims dims;
  std::uint64_t seed = 0;
  GenKind kind = GenKind::uniform;
  double sigma = 4.0;  // GRF smoothness, in voxels
  int levels = 1024;   // GRF quantisation level count
  int width = 0;       // Gaussian kernel width; 0 = derived from sigma
};

// counter_uniform(seed, i) for every voxel (datagen.hpp:57-62), on the device.
inline Image<float> uniform_noise(const GenSpec& spec, Context& ctx = Context::on(0)) {
  Image<float> img{spec.dims, std::vector<float>(spec.dims.voxel_count())};
  detail::check(ecc_uniform_noise_host(ctx.get(), img.values.data(), img.values.size(), spec.seed));
  return img;
}

namespace detail {

// Normalised sampled Gaussian taps (datagen.hpp:66-79).
inline std::vector<double> gaussian_kernel(double sigma, int width) {
  if (width < 1 || width % 2 == 0) throw error("Gaussian kernel width must be odd and >= 1");
  std::vector<double> w(width);
  const int half = width / 2;
  double sum = 0;
  for (int i = -half; i <= half; ++i) {
    const double v = width == 1 ? 1.0 : std::exp(-(double(i) * i) / (2.0 * sigma * sigma));
    w[i + half] = v;
    sum += v;
  }
  for (double& v : w) v /= sum;
  return w;
}

}  // namespace detail

// Separable Gaussian smoothing with edge clamping (datagen.hpp:108-122), on
// the device.
inline Image<float> gaussian_smooth(const Image<float>& image, double sigma, int width,
                                    Context& ctx = Context::on(0)) {
  Image<float> out{image.dims, std::vector<float>(image.values.size())};
  detail::check(ecc_gaussian_smooth_host(ctx.get(), image.values.data(), out.values.data(),
                                         detail::cdims(image.dims), sigma, width));
  return out;
}

}  // namespace ecc
