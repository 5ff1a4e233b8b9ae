// random 32B sector reads: fully random vs clustered in 2MB pages vs clustered in 64KB
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t hsh(uint64_t x){ x ^= x>>33; x*=0xff51afd7ed558ccdULL; x^=x>>33; x*=0xc4ceb9fe1a85ec53ULL; x^=x>>33; return x; }
// each warp-iteration: pick a random "region" of 2^rb bytes; lanes read random 32B sectors inside it
__global__ void k(const uint4* buf, int lognbytes, int rb, int64_t iters, uint32_t* sink){
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x*(int64_t)blockDim.x+threadIdx.x)>>5, nw=((int64_t)gridDim.x*blockDim.x)>>5;
  uint32_t acc=0;
  for(int64_t i=w;i<iters;i+=nw*4){
    uint4 v[4][2];
    #pragma unroll
    for(int j=0;j<4;j++){
      uint64_t h = hsh(i + j*nw);
      uint64_t region = (h >> 20) & ((1ull << (lognbytes - rb)) - 1);
      uint64_t off = (hsh(h + lane) & ((1ull << (rb - 5)) - 1));   // sector index within region
      uint64_t sec = (region << (rb - 5)) + off;
      v[j][0] = __ldcs(buf + sec*2); v[j][1] = __ldcs(buf + sec*2 + 1);
    }
    #pragma unroll
    for(int j=0;j<4;j++) acc ^= v[j][0].x ^ v[j][1].w;
  }
  if(acc==0x12345) sink[0]=acc;
}
int main(){
  size_t bytes = 8ull<<30;
  uint4* buf; cudaMalloc(&buf, bytes); cudaMemset(buf,1,bytes);
  uint32_t* sink; cudaMalloc(&sink,4);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms; int64_t iters = 4<<20;  // warp-iterations -> 32 sectors each
  for (int rb : {33, 30, 27, 24, 21, 18, 16, 13}) {
    for(int rep=0;rep<2;rep++){ cudaEventRecord(e0); k<<<148*8,256>>>(buf, 33, rb, iters, sink); cudaEventRecord(e1); cudaEventSynchronize(e1);}
    cudaEventElapsedTime(&ms,e0,e1);
    printf("random 32B sectors, clustered per warp in %8.0f KB regions of 8 GB: %.1f GB/s\n", (double)(1ull<<rb)/1024, iters*32*32.0/ms/1e6);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
