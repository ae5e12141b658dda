// e2e_c -- end-to-end latency of ecc_curve through the C ABI alone (no
// Python): host image in (pageable or pinned), curve out, per call
//   H2D + fused kernel(s) + one D2H + sync.
//   e2e_c            -> C1 (256^2 u8) and C2 (512^3 u8), pinned inputs
// Development tool (tools/); synthetic inputs from the oracle's
// generator.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#include "ecc_b200.h"

extern "C" void ecc_oracle_fill_u8(uint8_t*, uint64_t, uint64_t, uint64_t);

static void run(ecc_ctx* ctx, const char* name, ecc_dims d, int reps) {
  const uint64_t n = d.w0 * d.w1 * d.w2;
  uint8_t* img = nullptr;
  cudaMallocHost(&img, n);
  ecc_oracle_fill_u8(img, n, 1, 0);
  std::vector<uint8_t> t(256);
  std::vector<int64_t> chi(256);
  uint64_t m = 0;
  std::vector<double> us;
  for (int i = 0; i < reps + 5; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    if (ecc_curve(ctx, img, 0, ECC_U8, d, nullptr, t.data(), chi.data(), 256, &m) != 0) {
      std::printf("error: %s\n", ecc_last_error());
      return;
    }
    const double dt = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    if (i >= 5) us.push_back(dt);
  }
  std::sort(us.begin(), us.end());
  double mean = 0;
  for (double x : us) mean += x;
  mean /= us.size();
  std::printf("{\"config\": \"%s\", \"points\": %llu, \"chi_last\": %lld, \"e2e_us_mean\": %.2f, "
              "\"e2e_us_median\": %.2f, \"e2e_us_min\": %.2f, \"gvox_s\": %.3f}\n",
              name, (unsigned long long)m, (long long)chi[m - 1], mean, us[us.size() / 2], us[0],
              n / (mean * 1e-6) / 1e9);
  cudaFreeHost(img);
}

int main() {
  ecc_ctx* ctx = nullptr;
  if (ecc_ctx_create(0, &ctx) != 0) {
    std::printf("error: %s\n", ecc_last_error());
    return 1;
  }
  run(ctx, "C1 256^2 u8 (C ABI, pinned host input)", ecc_dims{256, 256, 1}, 2000);
  run(ctx, "C2 512^3 u8 (C ABI, pinned host input)", ecc_dims{512, 512, 512}, 50);
  ecc_ctx_destroy(ctx);
  return 0;
}
