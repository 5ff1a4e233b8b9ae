// Random 4-byte loads from an L2-resident bitmap (8 MB, like the frontier plane):
// the ceiling of the bottom-up frontier probes, at several loads-in-flight per thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint32_t x){ x ^= x>>16; x*=0x7feb352dU; x^=x>>15; x*=0x846ca68bU; x^=x>>16; return x; }
template<int U>
__global__ void k(const uint32_t* bm, uint32_t mask, int iters, uint32_t* sink){
  uint32_t t = blockIdx.x*blockDim.x+threadIdx.x;
  uint32_t acc=0, x = t * 0x9E3779B9u;
  for(int i=0;i<iters;i++){
    uint32_t v[U];
    #pragma unroll
    for(int j=0;j<U;j++){ x = hsh(x + j); uint32_t a; asm volatile("ld.global.u32 %0, [%1];" : "=r"(a) : "l"(bm + (x & mask))); v[j]=a; }
    #pragma unroll
    for(int j=0;j<U;j++) acc ^= v[j];
  }
  if(acc==0x12345) sink[0]=acc;
}
int main(){
  const size_t words = 2u<<20;  // 8 MB
  uint32_t* bm; cudaMalloc(&bm, words*4); cudaMemset(bm, 0, words*4);
  uint32_t* sink; cudaMalloc(&sink,4);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  const int iters = 256;
  #define RUN(U, G, B) { for(int r=0;r<3;r++){ cudaEventRecord(e0); k<U><<<G,B>>>(bm, words-1, iters, sink); cudaEventRecord(e1); cudaEventSynchronize(e1);} \
    cudaEventElapsedTime(&ms,e0,e1); double n = (double)G*B*iters*U; printf("U=%2d grid=%5d block=%d: %.1f G loads/s\n", U, G, B, n/ms/1e6); }
  RUN(1, 148*4, 512) RUN(4, 148*4, 512) RUN(8, 148*4, 512) RUN(16, 148*4, 512) RUN(8, 148*2, 512) RUN(16, 148*2, 512) RUN(32, 148*2, 512)
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
