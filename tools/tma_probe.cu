// Probe: which TMA issue patterns run on this box (debug aid, not product).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__device__ __forceinline__ uint32_t su(const void* p){return (uint32_t)__cvta_generic_to_shared(p);}
template<int MODE>
__global__ void k(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, int* out, int a0, int a1, int a2){
  __shared__ alignas(128) uint8_t buf[64*32];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x==0){ asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;"::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;":::"memory");
    asm volatile("fence.proxy.async.shared::cta;":::"memory"); }
  __syncthreads();
  const CUtensorMap* m = (MODE & 1) ? gmap : &map;
  const int bytes = (MODE & 4) ? 64*32 : 48*32;
  if (threadIdx.x==0){
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"::"r"(su(&bar)),"r"(bytes):"memory");
    int c0 = a0, c1 = a1;
    if (MODE & 2)
      asm volatile("cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(su(buf)),"l"((uint64_t)m),"r"(c0),"r"(c1),"r"(a2),"r"(su(&bar)):"memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(su(buf)),"l"((uint64_t)m),"r"(c0),"r"(c1),"r"(a2),"r"(su(&bar)):"memory");
  }
  uint32_t done=0; while(!done){ asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}":"=r"(done):"r"(su(&bar)):"memory"); }
  if (threadIdx.x < 32) out[threadIdx.x] = buf[threadIdx.x*48 + 10];
}
int A0,A1,A2;
template<int M> void run(CUtensorMap map, CUtensorMap* gm, int* out){
  k<M><<<1,128>>>(map,gm,out,A0,A1,A2); cudaError_t e = cudaDeviceSynchronize();
  int h[32]; cudaMemcpy(h,out,128,cudaMemcpyDeviceToHost);
  printf("mode %d c=(%d,%d,%d): %s v=%d %d\n", M, A0, A1, A2, cudaGetErrorString(e), h[0], h[5]);
}
int main(int argc, char** argv){
  int mode = atoi(argv[1]); A0 = atoi(argv[2]); A1 = atoi(argv[3]); A2 = atoi(argv[4]);
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled",&p,cudaEnableDefault,&q);
  auto enc=(PFN_cuTensorMapEncodeTiled_v12000)p;
  uint8_t* d; cudaMalloc(&d, 64*64*4); cudaMemset(d, 7, 64*64*4);
  CUtensorMap map; cuuint64_t dims[3]={64,64,4}; cuuint64_t st[2]={64,64*64};
  cuuint32_t box[3]={(mode&4)?64u:48u,32,1}, es[3]={1,1,1};
  CUresult r=enc(&map,CU_TENSOR_MAP_DATA_TYPE_UINT8,3,d,dims,st,box,es,CU_TENSOR_MAP_INTERLEAVE_NONE,CU_TENSOR_MAP_SWIZZLE_NONE,
     (mode&16)?CU_TENSOR_MAP_L2_PROMOTION_NONE:CU_TENSOR_MAP_L2_PROMOTION_L2_128B,CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d q=%d\n",(int)r,(int)q);
  CUtensorMap* gm; cudaMalloc(&gm, sizeof(map)); cudaMemcpy(gm,&map,sizeof(map),cudaMemcpyHostToDevice);
  int* out; cudaMalloc(&out, 128);
  switch(mode & 15){
    case 0: run<0>(map,gm,out); break; case 1: run<1>(map,gm,out); break;
    case 2: run<2>(map,gm,out); break; case 4: run<4>(map,gm,out); break;
    case 8: run<8>(map,gm,out); break; case 12: run<12>(map,gm,out); break;
  }
  return 0;
}
