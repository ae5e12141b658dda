// Instruction-throughput microbenchmarks for the bit-sliced ECC stencil
// (B200, sm_100a).  Not product code: measures which SASS ops share the
// ALU pipe and what an SM sustains per clock, plus shared-memory histogram
// update variants and TMA box start-coordinate rules.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench2 tools/ubench2.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e = (x);                                                                       \
    if (e != cudaSuccess) {                                                                    \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);           \
      exit(1);                                                                                 \
    }                                                                                          \
  } while (0)

constexpr int NI = 2048;  // loop iterations
constexpr int NC = 8;     // independent chains

// Each OP macro updates a[j] from a[j], a[j+1], a[j+3] (8 chains).
#define BODY(EXPR)                                                   \
  _Pragma("unroll") for (int j = 0; j < NC; ++j) {                   \
    uint32_t x = a[j], y = a[(j + 1) & 7], z = a[(j + 3) & 7], r;    \
    EXPR;                                                            \
    a[j] = r;                                                        \
  }

template <int OP>
__global__ void k_op(uint32_t* out, uint32_t seed) {
  uint32_t a[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) a[j] = seed * (threadIdx.x + 1) * (j + 3);
  for (int i = 0; i < NI; ++i) {
    if (OP == 0) BODY(asm volatile("lop3.b32 %0,%1,%2,%3,0x96;" : "=r"(r) : "r"(x), "r"(y), "r"(z)))
    if (OP == 1) BODY(asm volatile("mad.lo.u32 %0,%1,%2,%3;" : "=r"(r) : "r"(x), "r"(y), "r"(z)))
    if (OP == 2) BODY(asm volatile("shf.l.wrap.b32 %0,%1,%2,%3;" : "=r"(r) : "r"(x), "r"(y), "r"(z)))
    if (OP == 3) BODY(asm volatile("prmt.b32 %0,%1,%2,%3;" : "=r"(r) : "r"(x), "r"(y), "r"(z)))
    if (OP == 4) BODY(asm volatile("add.u32 %0,%1,%2;" : "=r"(r) : "r"(x), "r"(y)); r += z)
    if (OP == 5) BODY(asm volatile("{.reg .b32 t; add.u32 t,%1,%2; xor.b32 %0,t,%3;}" : "=r"(r) : "r"(x), "r"(y), "r"(z)))
    // LOP3 + IMAD interleaved (co-issue test): half the chains each
    if (OP == 6) {
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        uint32_t x = a[j], y = a[(j + 1) & 7], z = a[(j + 3) & 7], r;
        if (j & 1)
          asm volatile("mad.lo.u32 %0,%1,%2,%3;" : "=r"(r) : "r"(x), "r"(y), "r"(z));
        else
          asm volatile("lop3.b32 %0,%1,%2,%3,0x96;" : "=r"(r) : "r"(x), "r"(y), "r"(z));
        a[j] = r;
      }
    }
    if (OP == 7) BODY(asm volatile("{.reg .b32 t; fma.rn.f16x2 %0,%1,%2,%3;}" : "=r"(r) : "r"(x), "r"(y), "r"(z)))
    if (OP == 8) BODY(asm volatile("min.u16x2 %0,%1,%2;" : "=r"(r) : "r"(x), "r"(y)); r ^= z)
    if (OP == 9) BODY(asm volatile("shr.b32 %0,%1,%2;" : "=r"(r) : "r"(x), "r"(y)); r |= z)
    if (OP == 10) BODY(asm volatile("mul.hi.u32 %0,%1,%2;" : "=r"(r) : "r"(x), "r"(y)); r += z)
    if (OP == 11) BODY(asm volatile("{.reg .pred p; setp.lt.u32 p,%1,%2; selp.b32 %0,%3,%1,p;}" : "=r"(r) : "r"(x), "r"(y), "r"(z)))
    if (OP == 12) BODY(asm volatile("fma.rn.f32 %0,%1,%2,%3;" : "=r"(r) : "r"(x), "r"(y), "r"(z)))
    if (OP == 13) BODY(asm volatile("popc.b32 %0,%1;" : "=r"(r) : "r"(x)); r += y)
    if (OP == 14) BODY(asm volatile("shfl.sync.down.b32 %0,%1,1,0x1f,0xffffffff;" : "=r"(r) : "r"(x)); r ^= y)
    if (OP == 15) BODY(asm volatile("vadd4.u32.u32.u32.add %0,%1,%2,%3;" : "=r"(r) : "r"(x), "r"(y), "r"(z)))
  }
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < NC; ++j) acc ^= a[j];
  if (acc == 0x12345678u) out[0] = acc;
}

const char* kName[] = {"LOP3", "IMAD", "SHF.wrap", "PRMT", "IADD(+IADD)", "IADD+LOP3 pair",
                       "LOP3|IMAD mix", "HFMA2", "VIMNMX u16x2(+LOP)", "SHR(+LOP)", "IMAD.HI(+IADD)",
                       "ISETP+SEL", "FFMA", "POPC(+IADD)", "SHFL(+LOP)", "VADD4"};

// ---------------- histogram update variants (256-value x 16-change joint table)
constexpr int HI = 512;
__device__ __forceinline__ uint32_t lcg(uint32_t& x) { return x = x * 1664525u + 1013904223u; }

// V: 0 = ATOMS.ADD 1 to joint (c<<8|v) table, all lanes
//    1 = same with ~41% of lanes predicated off
//    2 = ATOMS.ADD of (c+8)|1<<16 into a 256-bin table
//    3 = lane-private RMW LDS+STS into [v][lane]
//    4 = red.shared (no return)
template <int V>
__global__ void k_hist(uint32_t* out, uint32_t seed) {
  extern __shared__ uint32_t h[];
  const int words = (V == 3) ? 256 * 32 * (blockDim.x / 32) : 4096;
  for (int i = threadIdx.x; i < words; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = seed ^ (threadIdx.x * 0x9E3779B9u);
#pragma unroll 8
  for (int i = 0; i < HI; ++i) {
    const uint32_t r = lcg(x);
    const uint32_t v = r >> 24, c = (r >> 8) & 15;
    if (V == 0) atomicAdd(&h[(c << 8) | v], 1u);
    if (V == 1) {
      if (((r >> 12) & 127) < 75) atomicAdd(&h[(c << 8) | v], 1u);
    }
    if (V == 2) atomicAdd(&h[v], c | 65536u);
    if (V == 3) {
      uint32_t* p = &h[(warp * 256 + v) * 32 + lane];
      *(volatile uint32_t*)p = *(volatile uint32_t*)p + c;
    }
    if (V == 4) asm volatile("red.shared.add.u32 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&h[(c << 8) | v])) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = h[seed & 255];
}

// ---------------- TMA start-coordinate probe
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k_tma(const __grid_constant__ CUtensorMap map, int c0, int c1, int* out) {
  __shared__ alignas(128) uint8_t buf[32 * 32];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(1024) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su(buf)),
        "l"((uint64_t)&map), "r"(c0), "r"(c1), "r"(0), "r"(su(&bar))
        : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                 : "=r"(done) : "r"(su(&bar)) : "memory");
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = buf[i];
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

template <int OP>
void run_op(uint32_t* out, int sms, double ghz) {
  const int threads = 512, blocks = sms * 4;
  const double warp_instr = double(blocks) * (threads / 32) * NI * NC;
  float ms = time_ms([&] { k_op<OP><<<blocks, threads>>>(out, 3); });
  printf("%-22s %.2f warp-instr(loop body)/clk/SM\n", kName[OP], warp_instr / (ms * 1e-3) / sms / (ghz * 1e9));
}

template <int V>
void run_hist(uint32_t* out, int sms, double ghz, const char* name) {
  const int threads = 512, blocks = sms * 2;
  const size_t smem = (V == 3) ? 256 * 32 * 8 * 4 / 2 : 4096 * 4;
  const int thr = (V == 3) ? 128 : threads;
  CK(cudaFuncSetAttribute(k_hist<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const double upd = double(blocks) * thr * HI;
  float ms = time_ms([&] { k_hist<V><<<blocks, thr, smem>>>(out, 7); });
  printf("hist %-40s %.2f lane-updates/clk/SM\n", name, upd / (ms * 1e-3) / sms / (ghz * 1e9));
}

int main() {
  int sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  const double ghz = clk / 1e6;
  printf("SMs %d, max clock %.3f GHz (rates assume max clock)\n", sms, ghz);
  uint32_t* out;
  CK(cudaMalloc(&out, 1 << 24));
  run_op<0>(out, sms, ghz); run_op<1>(out, sms, ghz); run_op<2>(out, sms, ghz);
  run_op<3>(out, sms, ghz); run_op<4>(out, sms, ghz); run_op<5>(out, sms, ghz);
  run_op<6>(out, sms, ghz); run_op<7>(out, sms, ghz); run_op<8>(out, sms, ghz);
  run_op<9>(out, sms, ghz); run_op<10>(out, sms, ghz); run_op<11>(out, sms, ghz);
  run_op<12>(out, sms, ghz); run_op<13>(out, sms, ghz); run_op<14>(out, sms, ghz);
  run_op<15>(out, sms, ghz);
  run_hist<0>(out, sms, ghz, "ATOMS joint 4096, all lanes");
  run_hist<1>(out, sms, ghz, "ATOMS joint 4096, 59% lanes (per issued)");
  run_hist<2>(out, sms, ghz, "ATOMS 256 packed inc");
  run_hist<3>(out, sms, ghz, "lane-private LDS+STS RMW");
  run_hist<4>(out, sms, ghz, "RED.shared joint 4096");

  // TMA: 3D u8 tensor 256 x 64 x 2, box 32 x 32 x 1, probe odd / negative starts
  void* p;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  uint8_t* d;
  CK(cudaMalloc(&d, 256 * 64 * 2));
  uint8_t hbuf[256 * 64 * 2];
  for (int i = 0; i < 256 * 64 * 2; ++i) hbuf[i] = (uint8_t)(i * 7 + (i >> 8));
  CK(cudaMemcpy(d, hbuf, sizeof hbuf, cudaMemcpyHostToDevice));
  CUtensorMap map;
  cuuint64_t dims[3] = {256, 64, 2};
  cuuint64_t st[2] = {256, 256 * 64};
  cuuint32_t box[3] = {32, 32, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("tma encode rc=%d\n", (int)r);
  int* dout;
  CK(cudaMalloc(&dout, 4096));
  int hout[1024];
  const int starts[][2] = {{0, 0}, {29, 3}, {-1, -1}, {237, 40}, {1, 0}, {-5, 60}};
  for (auto& s : starts) {
    k_tma<<<1, 128>>>(map, s[0], s[1], dout);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("tma start (%d,%d): %s\n", s[0], s[1], cudaGetErrorString(e));
      return 0;
    }
    CK(cudaMemcpy(hout, dout, 4096, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int y = 0; y < 32; ++y)
      for (int z = 0; z < 32; ++z) {
        const int gz = s[0] + z, gy = s[1] + y;
        const int want = (gz < 0 || gz >= 256 || gy < 0 || gy >= 64) ? 0 : hbuf[gy * 256 + gz];
        bad += hout[y * 32 + z] != want;
      }
    printf("tma start (%d,%d): %s, mismatches %d\n", s[0], s[1], "ok", bad);
  }
  return 0;
}
