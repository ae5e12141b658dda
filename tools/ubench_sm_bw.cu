// Per-SM streaming bandwidth: f32 -> u16 conversion (the affine key pass's
// access pattern) by one CTA per SM on a limited number of SMs, U float4
// loads in flight per thread.  Tooling for the C4 design.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubsm tools/ubench_sm_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(384, 1) conv(const float4* __restrict__ src, uint2* __restrict__ dst, uint64_t n4) {
  extern __shared__ char pad[];
  if (threadIdx.x == 100000) pad[0] = 0;
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * nt < n4; i += U * nt) {
    float4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = __ldcs(src + i + u * nt);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t a = (uint32_t)(x[u].x * 65536.f), b = (uint32_t)(x[u].y * 65536.f);
      const uint32_t c = (uint32_t)(x[u].z * 65536.f), d = (uint32_t)(x[u].w * 65536.f);
      dst[i + u * nt] = make_uint2(a | (b << 16), c | (d << 16));
    }
  }
}

template <int U>
void run(const float4* s, uint2* d, uint64_t n4, int sms) {
  cudaFuncSetAttribute(conv<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  conv<U><<<sms, 384, 200 * 1024>>>(s, d, n4);
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) conv<U><<<sms, 384, 200 * 1024>>>(s, d, n4);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 3;
  const double bytes = n4 * 24.0;
  printf("U=%2d sms=%3d  %.3f ms  %.0f GB/s total  %.1f GB/s per SM\n", U, sms, ms, bytes / ms / 1e6,
         bytes / ms / 1e6 / sms);
}

int main() {
  const uint64_t n = 1ull << 28;  // 1 GiB of f32
  float4* s;
  uint2* d;
  cudaMalloc(&s, n * 4);
  cudaMalloc(&d, n * 2);
  cudaMemset(s, 0, n * 4);
  for (int sms : {16, 24, 32, 48, 148}) {
    run<8>(s, d, n / 4, sms);
    run<16>(s, d, n / 4, sms);
    run<32>(s, d, n / 4, sms);
  }
  return 0;
}
