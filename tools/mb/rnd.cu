// random-access DRAM throughput on B200: each lane reads G bytes (16B loads) at random G-aligned offsets
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t hsh(uint64_t x){ x ^= x>>33; x*=0xff51afd7ed558ccdULL; x^=x>>33; x*=0xc4ceb9fe1a85ec53ULL; x^=x>>33; return x; }
template<int G>
__global__ void k(const uint4* buf, uint64_t nunits, int64_t nops, uint32_t* sink){
  int64_t t = blockIdx.x*(int64_t)blockDim.x+threadIdx.x, nt=(int64_t)gridDim.x*blockDim.x;
  uint32_t acc=0;
  for(int64_t i=t;i<nops;i+=nt*4){
    uint4 v[4][G/16];
    #pragma unroll
    for(int j=0;j<4;j++){ uint64_t u = hsh(i+j*nt)&(nunits-1); 
      #pragma unroll
      for(int q=0;q<G/16;q++) v[j][q]=__ldcs(buf+u*(G/16)+q); }
    #pragma unroll
    for(int j=0;j<4;j++)
      #pragma unroll
      for(int q=0;q<G/16;q++) acc ^= v[j][q].x ^ v[j][q].w;
  }
  if(acc==0x12345) sink[0]=acc;
}
__global__ void seq(const uint4* buf, int64_t n, uint32_t* sink){
  int64_t t = blockIdx.x*(int64_t)blockDim.x+threadIdx.x, nt=(int64_t)gridDim.x*blockDim.x;
  uint32_t acc=0;
  for(int64_t i=t;i<n;i+=nt){ uint4 v=__ldcs(buf+i); acc^=v.x^v.w; }
  if(acc==0x12345) sink[0]=acc;
}
int main(){
  size_t bytes = 8ull<<30;
  uint4* buf; cudaMalloc(&buf, bytes); cudaMemset(buf,1,bytes);
  uint32_t* sink; cudaMalloc(&sink,4);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for(int rep=0;rep<2;rep++){ cudaEventRecord(e0); seq<<<148*8,256>>>(buf, bytes/16, sink); cudaEventRecord(e1); cudaEventSynchronize(e1);}
  cudaEventElapsedTime(&ms,e0,e1); printf("sequential read: %.1f GB/s\n", bytes/ms/1e6);
  int64_t nops = 64<<20;
  #define RUN(G) for(int grid: {148*8, 148*16}) { for(int rep=0;rep<2;rep++){ cudaEventRecord(e0); k<G><<<grid,256>>>(buf, bytes/G, nops, sink); cudaEventRecord(e1); cudaEventSynchronize(e1);} \
     cudaEventElapsedTime(&ms,e0,e1); printf("random %3d B units, grid %d: %.1f GB/s useful, %.1f M units/ms\n", G, grid, nops*(double)G/ms/1e6, nops/ms/1e3); }
  RUN(16) RUN(32) RUN(64) RUN(128)
  for (size_t sz : {256ull<<20, 512ull<<20, 1ull<<30, 2ull<<30, 4ull<<30, 8ull<<30}) {
    for(int rep=0;rep<2;rep++){ cudaEventRecord(e0); k<32><<<148*8,256>>>(buf, sz/32, nops, sink); cudaEventRecord(e1); cudaEventSynchronize(e1);}
    cudaEventElapsedTime(&ms,e0,e1); printf("random 32 B units over %5zu MB: %.1f GB/s\n", sz>>20, nops*32.0/ms/1e6);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
