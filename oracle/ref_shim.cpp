// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Exposes the UNMODIFIED reference engine (header-only C++20 library under
// /root/reference/proj/include, compiled in place by oracle/Makefile) through
// a few extern "C" entry points, so tests and bench.py's reference arm can
// call it through ctypes.  The reference sources are never copied into this
// repository; the build output goes to oracle/_ref/ (git-ignored).
//
// Calls mirror the reference's own test helpers: run_engine / engine_curve
// (proj/tests/test_util.hpp:58-72) = plan_chunks + process_image +
// vcec_to_ecc; naive_ecc (oracle.hpp:80-107) is the brute-force oracle.
#include <cstdint>
#include <cstring>
#include <sstream>
#include <string>
#include <thread>

#include "ecc/curve.hpp"
#include "ecc/datagen.hpp"
#include "ecc/oracle.hpp"
#include "ecc/pipeline.hpp"
#include "ecc/streaming.hpp"

namespace {

thread_local std::string g_err;

// ChunkSource over a caller-owned buffer (chunk.hpp:131-152 contract).
template <class T>
class PtrSource final : public ecc::ChunkSource<T> {
 public:
  PtrSource(const T* p, ecc::Dims d) : p_(p), d_(d) {}
  ecc::Dims dims() const override { return d_; }
  void read_rows(std::uint64_t r0, std::uint64_t r1, T* dst) override {
    const std::uint64_t row = d_.w1 * d_.w2;
    std::memcpy(dst, p_ + r0 * row, (r1 - r0) * row * sizeof(T));
  }

 private:
  const T* p_;
  ecc::Dims d_;
};

template <class T>
std::int64_t run(const T* img, std::uint64_t w0, std::uint64_t w1,
                 std::uint64_t w2, std::uint64_t chunks, unsigned workers,
                 T* values, std::int64_t* changes, double* phases) {
  try {
    const ecc::Dims d{w0, w1, w2};
    PtrSource<T> src(img, d);
    if (workers == 0) workers = std::max(1u, std::thread::hardware_concurrency());
    if (chunks == 0) chunks = std::max<std::uint64_t>(2, workers);
    const auto plan = ecc::plan_chunks<T>(d, ecc::ChunkTarget::count(chunks));
    ecc::EngineOptions opt;
    opt.workers = workers;
    ecc::EngineReport rep;
    const auto vcec = ecc::process_image<T>(src, plan, opt, &rep);
    for (std::size_t i = 0; i < vcec.size(); ++i) {
      values[i] = vcec.values[i];
      changes[i] = vcec.changes[i];
    }
    if (phases) {
      phases[0] = rep.read_s;
      phases[1] = rep.index_s;
      phases[2] = rep.kernel_s;
      phases[3] = rep.merge_s;
    }
    return static_cast<std::int64_t>(vcec.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

template <class T>
std::int64_t naive(const T* img, std::uint64_t w0, std::uint64_t w1,
                   std::uint64_t w2, T* thresholds, std::int64_t* chi) {
  try {
    ecc::Image<T> im{{w0, w1, w2}, std::vector<T>(img, img + w0 * w1 * w2)};
    const auto c = ecc::naive_ecc(im);
    for (std::size_t i = 0; i < c.size(); ++i) {
      thresholds[i] = c.thresholds[i];
      chi[i] = c.chi[i];
    }
    return static_cast<std::int64_t>(c.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

template <class T>
std::int64_t csv(const T* thresholds, const std::int64_t* chi, std::uint64_t m,
                 char* out, std::uint64_t cap) {
  ecc::EccCurve<T> c;
  c.thresholds.assign(thresholds, thresholds + m);
  c.chi.assign(chi, chi + m);
  std::ostringstream os;
  ecc::write_curve(c, ecc::CurveFormat::csv, os);
  const std::string s = os.str();
  if (s.size() > cap) return -static_cast<std::int64_t>(s.size());
  std::memcpy(out, s.data(), s.size());
  return static_cast<std::int64_t>(s.size());
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

unsigned ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

std::uint64_t ref_counter_hash(std::uint64_t seed, std::uint64_t i) {
  return ecc::rng::counter_hash(seed, i);
}

// process_image + (caller) vcec_to_ecc through the reference engine.
std::int64_t ref_vcec_u8(const std::uint8_t* img, std::uint64_t w0,
                         std::uint64_t w1, std::uint64_t w2,
                         std::uint64_t chunks, unsigned workers,
                         std::uint8_t* values, std::int64_t* changes,
                         double* phases) {
  return run<std::uint8_t>(img, w0, w1, w2, chunks, workers, values, changes,
                           phases);
}

std::int64_t ref_vcec_f32(const float* img, std::uint64_t w0, std::uint64_t w1,
                          std::uint64_t w2, std::uint64_t chunks,
                          unsigned workers, float* values,
                          std::int64_t* changes, double* phases) {
  return run<float>(img, w0, w1, w2, chunks, workers, values, changes, phases);
}

std::int64_t ref_naive_u8(const std::uint8_t* img, std::uint64_t w0,
                          std::uint64_t w1, std::uint64_t w2,
                          std::uint8_t* thresholds, std::int64_t* chi) {
  return naive<std::uint8_t>(img, w0, w1, w2, thresholds, chi);
}

std::int64_t ref_naive_f32(const float* img, std::uint64_t w0, std::uint64_t w1,
                           std::uint64_t w2, float* thresholds,
                           std::int64_t* chi) {
  return naive<float>(img, w0, w1, w2, thresholds, chi);
}

// write_curve CSV bytes (curve.hpp:87-103), for the Appendix-B hashes.
std::int64_t ref_curve_csv_u8(const std::uint8_t* t, const std::int64_t* chi,
                              std::uint64_t m, char* out, std::uint64_t cap) {
  return csv<std::uint8_t>(t, chi, m, out, cap);
}

std::int64_t ref_curve_csv_f32(const float* t, const std::int64_t* chi,
                               std::uint64_t m, char* out, std::uint64_t cap) {
  return csv<float>(t, chi, m, out, cap);
}

// Pipeline pieces (datagen.hpp:57-62, 108-122; pipeline.hpp:236-291).
void ref_uniform_noise(std::uint64_t w0, std::uint64_t w1, std::uint64_t w2,
                       std::uint64_t seed, float* out) {
  ecc::GenSpec spec;
  spec.dims = {w0, w1, w2};
  spec.seed = seed;
  const auto img = ecc::uniform_noise(spec);
  std::memcpy(out, img.values.data(), img.values.size() * sizeof(float));
}

int ref_gaussian_smooth(const float* in, std::uint64_t w0, std::uint64_t w1,
                        std::uint64_t w2, double sigma, int width, float* out) {
  try {
    ecc::Image<float> im{{w0, w1, w2}, std::vector<float>(in, in + w0 * w1 * w2)};
    const auto sm = ecc::gaussian_smooth(im, sigma, width);
    std::memcpy(out, sm.values.data(), sm.values.size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// bench_run; r = {generate_s, total_s, per_iteration_s, ecc_avg_s,
// smooth_avg_s, ecc_gvox_per_s}
int ref_bench_run(std::uint64_t w0, std::uint64_t w1, std::uint64_t w2,
                  std::uint64_t iterations, std::uint64_t seed, double sigma,
                  int width, double* r) {
  try {
    const auto rep = ecc::bench_run({w0, w1, w2}, iterations, seed, sigma, width);
    r[0] = rep.generate_s;
    r[1] = rep.total_s;
    r[2] = rep.per_iteration_s;
    r[3] = rep.ecc_avg_s;
    r[4] = rep.smooth_avg_s;
    r[5] = rep.ecc_gvox_per_s;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
