// Microbenchmarks for the histogram-update primitives the ECC kernels are
// built from (B200, sm_100a). Not product code: it measures the hardware
// rates that DESIGN.md's kernel choices rest on.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench tools/ubench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, \
             __LINE__);                                                    \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

constexpr int ITERS = 256;

// 1) ATOMS, 256 bins x 32 lane-private copies (bank = lane): conflict-free.
__global__ void k_atoms_private(uint32_t* out, uint32_t seed) {
  __shared__ uint32_t h[256 * 32];
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) h[i] = 0;
  __syncthreads();
  uint32_t lane = threadIdx.x & 31;
  uint32_t x = hash32(seed ^ (blockIdx.x * blockDim.x + threadIdx.x));
#pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    x = x * 1664525u + 1013904223u;
    uint32_t bin = x >> 24;
    atomicAdd(&h[bin * 32 + lane], (1u << 20) + (x & 7));
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = h[lane + 32 * (seed & 255)];
}

// 2) ATOMS into one shared 256-bin histogram: random bank conflicts.
__global__ void k_atoms_shared256(uint32_t* out, uint32_t seed) {
  __shared__ uint32_t h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  uint32_t x = hash32(seed ^ (blockIdx.x * blockDim.x + threadIdx.x));
#pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    x = x * 1664525u + 1013904223u;
    atomicAdd(&h[x >> 24], (1u << 20) + (x & 7));
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = h[seed & 255];
}

// 3) ATOMS into a 32768-bin (128 KB) shared histogram, random.
__global__ void k_atoms_big(uint32_t* out, uint32_t seed) {
  extern __shared__ uint32_t h[];
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) h[i] = 0;
  __syncthreads();
  uint32_t x = hash32(seed ^ (blockIdx.x * blockDim.x + threadIdx.x));
#pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    x = x * 1664525u + 1013904223u;
    atomicAdd(&h[x >> 17], (1u << 16) + (x & 7));
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = h[seed & 32767];
}

// 4) RED.global into a 65536-bin int32 histogram (L2-resident), random.
__global__ void k_red_global(uint32_t* hist, uint32_t mask, uint32_t seed) {
  uint32_t x = hash32(seed ^ (blockIdx.x * blockDim.x + threadIdx.x));
#pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    x = x * 1664525u + 1013904223u;
    atomicAdd(&hist[(x >> 8) & mask], 1u);
  }
}

// 5) DSMEM: cluster of 2, each CTA owns 32768 bins; every update goes to the
// CTA chosen by one hash bit (half remote).
__global__ void __cluster_dims__(2, 1, 1) k_dsmem(uint32_t* out, uint32_t seed) {
  extern __shared__ uint32_t h[];
  cg::cluster_group cluster = cg::this_cluster();
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) h[i] = 0;
  cluster.sync();
  uint32_t x = hash32(seed ^ (blockIdx.x * blockDim.x + threadIdx.x));
#pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    x = x * 1664525u + 1013904223u;
    uint32_t* dst = cluster.map_shared_rank(h, (x >> 31) & 1);
    atomicAdd(&dst[(x >> 16) & 32767], 1u);
  }
  cluster.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = h[seed & 32767];
}

// 6) Streaming read bandwidth: 16-B loads, xor-reduce.
__global__ void k_read(const uint4* __restrict__ p, size_t n, uint32_t* out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// 7) LOP3 issue rate: pure ALU chain (8 independent chains per thread).
__global__ void k_lop3(uint32_t* out, uint32_t seed) {
  uint32_t a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = hash32(seed + threadIdx.x * 8 + j);
  for (int i = 0; i < 4096; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t r;
      asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(a[j]), "r"(a[(j + 1) & 7]), "r"(a[(j + 3) & 7]));
      a[j] = r;
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc ^= a[j];
  if (acc == 0x12345678u) out[0] = acc;
}

template <class F>
float time_ms(F f, int reps = 5) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  printf("SMs %d, max clock %d kHz\n", sms, clk);
  uint32_t* out;
  CK(cudaMalloc(&out, 1 << 24));
  const double ghz = clk / 1e6;

  for (int threads : {256, 512, 1024}) {
    int blocks = sms * (2048 / threads) * 4;
    double ops = double(blocks) * threads * ITERS;
    float ms = time_ms([&] { k_atoms_private<<<blocks, threads>>>(out, 7); });
    printf("ATOMS lane-private 256x32 (blk %d): %.1f Gop/s = %.2f lanes/clk/SM\n",
           threads, ops / ms / 1e6, ops / (ms * 1e-3) / sms / (ghz * 1e9));
    ms = time_ms([&] { k_atoms_shared256<<<blocks, threads>>>(out, 7); });
    printf("ATOMS shared 256 (blk %d): %.1f Gop/s = %.2f lanes/clk/SM\n", threads,
           ops / ms / 1e6, ops / (ms * 1e-3) / sms / (ghz * 1e9));
  }
  {
    CK(cudaFuncSetAttribute(k_atoms_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
    int threads = 1024, blocks = sms * 4;
    double ops = double(blocks) * threads * ITERS;
    float ms = time_ms([&] { k_atoms_big<<<blocks, threads, 131072>>>(out, 7); });
    printf("ATOMS 32768-bin random: %.1f Gop/s = %.2f lanes/clk/SM\n", ops / ms / 1e6,
           ops / (ms * 1e-3) / sms / (ghz * 1e9));
  }
  {
    uint32_t* hist;
    CK(cudaMalloc(&hist, size_t(1) << 30));
    for (uint32_t mask : {0xFFFFu, 0xFFFFFu, 0xFFFFFFu}) {
      int threads = 512, blocks = sms * 16;
      double ops = double(blocks) * threads * ITERS;
      float ms = time_ms([&] { k_red_global<<<blocks, threads>>>(hist, mask, 9); });
      printf("RED.global random over %u bins: %.1f Gop/s\n", mask + 1, ops / ms / 1e6);
    }
    CK(cudaFree(hist));
  }
  {
    CK(cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
    int threads = 1024, blocks = sms;  // even
    double ops = double(blocks) * threads * ITERS;
    float ms = time_ms([&] { k_dsmem<<<blocks, threads, 131072>>>(out, 7); });
    printf("DSMEM cluster2 atomics (half remote): %.1f Gop/s = %.2f lanes/clk/SM\n",
           ops / ms / 1e6, ops / (ms * 1e-3) / sms / (ghz * 1e9));
  }
  {
    size_t bytes = size_t(2) << 30;
    uint4* p;
    CK(cudaMalloc(&p, bytes));
    CK(cudaMemset(p, 1, bytes));
    for (int bpsm : {2, 4, 8}) {
      float ms = time_ms([&] { k_read<<<sms * bpsm, 512>>>(p, bytes / 16, out); });
      printf("read BW (blocks %d x 512): %.1f GB/s\n", sms * bpsm, bytes / ms / 1e6);
    }
    CK(cudaFree(p));
  }
  {
    int threads = 512, blocks = sms * 4;
    double ops = double(blocks) * threads * 4096 * 8;
    float ms = time_ms([&] { k_lop3<<<blocks, threads>>>(out, 3); });
    printf("LOP3: %.1f Tlane-op/s = %.2f warp-instr/clk/SM\n", ops / ms / 1e9,
           ops / 32 / (ms * 1e-3) / sms / (ghz * 1e9));
  }
  return 0;
}
