// Random 4-byte loads per warp lane: how fast when the target region is L1-resident,
// L2-resident, or a shared-memory table?  Sizes the "summary in shared memory"
// and "small column ranges" ideas.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint32_t x){ x ^= x>>16; x*=0x7feb352dU; x^=x>>15; x*=0x846ca68bU; x^=x>>16; return x; }
template<int U, int MODE>  // MODE 0: ld.global (L1-cached), 1: ld.global.cg (L2 only), 2: shared
__global__ void k(const uint32_t* bm, uint32_t mask, int iters, uint32_t* sink){
  extern __shared__ uint32_t sm[];
  if (MODE == 2) { for (uint32_t i = threadIdx.x; i <= mask; i += blockDim.x) sm[i] = bm[i]; __syncthreads(); }
  uint32_t t = blockIdx.x*blockDim.x+threadIdx.x;
  uint32_t acc=0, x = t * 0x9E3779B9u;
  for(int i=0;i<iters;i++){
    uint32_t v[U];
    #pragma unroll
    for(int j=0;j<U;j++){ x = hsh(x + j); uint32_t a;
      if (MODE == 0) asm volatile("ld.global.u32 %0, [%1];" : "=r"(a) : "l"(bm + (x & mask)));
      else if (MODE == 1) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(a) : "l"(bm + (x & mask)));
      else a = sm[x & mask];
      v[j]=a; }
    #pragma unroll
    for(int j=0;j<U;j++) acc ^= v[j];
  }
  if(acc==0x12345) sink[0]=acc;
}
int main(){
  const size_t words = 64u<<20;
  uint32_t* bm; cudaMalloc(&bm, words*4); cudaMemset(bm, 0, words*4);
  uint32_t* sink; cudaMalloc(&sink,4);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  const int iters = 256;
  #define RUN(U, MODE, KB, G, B) { size_t smem = MODE==2 ? (size_t)KB*1024 : 0; \
    cudaFuncSetAttribute(k<U,MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    for(int r=0;r<3;r++){ cudaEventRecord(e0); k<U,MODE><<<G,B,smem>>>(bm, (uint32_t)(KB*256-1), iters, sink); cudaEventRecord(e1); cudaEventSynchronize(e1);} \
    cudaEventElapsedTime(&ms,e0,e1); double n = (double)G*B*iters*U; printf("mode %d U=%2d region %6d KB grid=%4d block=%d: %.1f G loads/s (%.2f per clk per SM at 1.965 GHz)\n", MODE, U, KB, G, B, n/ms/1e6, n/ms/1e6/148/1.965); }
  RUN(8,0,16,296,512) RUN(8,0,32,296,512) RUN(8,0,64,296,512) RUN(8,0,128,296,512) RUN(8,0,256,296,512) RUN(8,0,1024,296,512) RUN(8,0,8192,296,512) RUN(8,0,32768,296,512)
  RUN(8,1,64,296,512) RUN(8,1,8192,296,512)
  RUN(8,2,16,296,512) RUN(8,2,32,296,512) RUN(8,2,64,296,512)
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
