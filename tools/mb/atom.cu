// microbenchmark: random L2 ops throughput on B200
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint64_t x){ x ^= x>>33; x*=0xff51afd7ed558ccdULL; x^=x>>33; x*=0xc4ceb9fe1a85ec53ULL; x^=x>>33; return (uint32_t)x; }
template<int OP>
__global__ void k(uint32_t* buf, uint32_t mask, int64_t nops, uint32_t* sink){
  int64_t t = blockIdx.x*(int64_t)blockDim.x+threadIdx.x, nt=(int64_t)gridDim.x*blockDim.x;
  uint32_t acc=0;
  for(int64_t i=t;i<nops;i+=nt*8){
    uint32_t a[8];
    #pragma unroll
    for(int j=0;j<8;j++) a[j]=hsh(i+j*nt)&mask;
    #pragma unroll
    for(int j=0;j<8;j++){
      if(i+j*nt>=nops) break;
      if(OP==0) atomicOr(buf+(a[j]>>5), 1u<<(a[j]&31));
      else if(OP==1) atomicMin(buf+a[j], (uint32_t)i);
      else if(OP==2) acc += __ldg(buf+(a[j]>>5));
      else if(OP==3) acc += buf[a[j]>>5];
    }
  }
  if(acc==0x12345) sink[0]=acc;
}
int main(){
  uint32_t* buf; cudaMalloc(&buf, 1ull<<30); cudaMemset(buf,0,1ull<<30);
  uint32_t* sink; cudaMalloc(&sink,4);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int64_t nops=256<<20;
  struct {const char* name; int op; uint32_t mask;} cs[]={
    {"RED.OR bitmap 8MB (2^26 bits)",0,(1u<<26)-1},
    {"RED.MIN 16MB (2^22 words)",1,(1u<<22)-1},
    {"RED.MIN 256MB (2^26 words)",1,(1u<<26)-1},
    {"LDG.nc bitmap 8MB",2,(1u<<26)-1},
    {"LDG bitmap 8MB",3,(1u<<26)-1},
    {"RED.OR bitmap 64KB",0,(1u<<19)-1},
  };
  for(auto& c: cs){
    for(int grid : {148*4, 148*8}){
      for(int rep=0;rep<2;rep++){
        cudaEventRecord(e0);
        if(c.op==0) k<0><<<grid,256>>>(buf,c.mask,nops,sink);
        if(c.op==1) k<1><<<grid,256>>>(buf,c.mask,nops,sink);
        if(c.op==2) k<2><<<grid,256>>>(buf,c.mask,nops,sink);
        if(c.op==3) k<3><<<grid,256>>>(buf,c.mask,nops,sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms,e0,e1);
        if(rep) printf("%-32s grid %5d: %.3f ms  %.1f Gop/s\n", c.name, grid, ms, nops/ms/1e6);
      }
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
