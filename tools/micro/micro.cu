// Microbenchmarks that inform the ESI kernel design on B200 (sm_100a).
// Not part of the product path.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__global__ void rd128(const int4* __restrict__ p, size_t n, int* out){
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x; size_t st = (size_t)gridDim.x*blockDim.x;
  int acc=0;
  for(; i+3*st<n; i+=4*st){ int4 a=__ldcs(p+i), b=__ldcs(p+i+st), c=__ldcs(p+i+2*st), d=__ldcs(p+i+3*st); acc ^= a.x^b.y^c.z^d.w; }
  for(; i<n; i+=st){ int4 a=__ldcs(p+i); acc^=a.x; }
  if(acc==0x12345) out[0]=acc;
}
__global__ void rdL2(const int4* __restrict__ p, size_t n, int reps, int* out){
  int acc=0;
  for(int r=0;r<reps;r++){
    size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x; size_t st = (size_t)gridDim.x*blockDim.x;
    for(; i<n; i+=st){ int4 a=__ldcg(p+i); acc^=a.x^a.w; }
  }
  if(acc==0x12345) out[0]=acc;
}
__global__ void wr128(int4* __restrict__ p, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x; size_t st = (size_t)gridDim.x*blockDim.x;
  for(; i<n; i+=st){ __stcs(p+i, make_int4(i,i,i,i)); }
}
__global__ void matchk(int iters, int mod, int* out){
  unsigned v = threadIdx.x*2654435761u + blockIdx.x; int acc=0;
  for(int i=0;i<iters;i++){ unsigned key=(v>>7)%mod; unsigned m=__match_any_sync(0xffffffffu,key); acc+=__popc(m); v=v*1664525u+1013904223u; }
  if(acc==0x12345) out[0]=acc;
}
__global__ void satom(int iters, int* out){
  __shared__ int h[1024];
  for(int i=threadIdx.x;i<1024;i+=blockDim.x) h[i]=0; __syncthreads();
  unsigned v = threadIdx.x*2654435761u + blockIdx.x; int acc=0;
  for(int i=0;i<iters;i++){ acc+=atomicAdd(&h[(v>>9)&1023],1); v=v*1664525u+1013904223u; }
  if(acc==0x12345) out[0]=acc;
}
__global__ void empty(){}
__global__ void gbar(int iters, unsigned* ctr){
  cg::grid_group g = cg::this_grid();
  for(int i=0;i<iters;i++) g.sync();
}
int main(){
  int dev=0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr,dev));
  printf("dev %s SMs %d L2 %d MB smem/SM %zu clk %d kHz memclk %d kHz bus %d\n", pr.name, pr.multiProcessorCount, pr.l2CacheSize>>20, pr.sharedMemPerMultiprocessor, pr.clockRate, pr.memoryClockRate, pr.memoryBusWidth);
  int nsm=pr.multiProcessorCount;
  size_t bytes = (size_t)4<<30; int4* buf; CK(cudaMalloc(&buf, bytes)); int* out; CK(cudaMalloc(&out,64));
  size_t n = bytes/16; cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  wr128<<<nsm*8,512>>>(buf,n); CK(cudaDeviceSynchronize());
  for(int bpm : {4,8,16}) for(int thr: {256,512}){
    rd128<<<nsm*bpm,thr>>>(buf,n,out);
    cudaEventRecord(a); for(int r=0;r<5;r++) rd128<<<nsm*bpm,thr>>>(buf,n,out); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    printf("HBM read LDG.128 grid %dx%d: %.1f GB/s\n", nsm*bpm, thr, 5.0*bytes/ms/1e6);
  }
  cudaEventRecord(a); for(int r=0;r<5;r++) wr128<<<nsm*8,512>>>(buf,n); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
  printf("HBM write STG.128: %.1f GB/s\n", 5.0*bytes/ms/1e6);
  cudaEventRecord(a); for(int r=0;r<5;r++) cudaMemcpyAsync(buf, (char*)buf+bytes/2, bytes/2, cudaMemcpyDeviceToDevice); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
  printf("D2D memcpy (r+w): %.1f GB/s\n", 5.0*bytes/ms/1e6);
  for(size_t mb : {8, 32, 64, 96}){
    size_t nn = mb<<20; nn/=16; int reps=20;
    rdL2<<<nsm*8,512>>>(buf,nn,1,out);
    cudaEventRecord(a); rdL2<<<nsm*8,512>>>(buf,nn,reps,out); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    printf("L2 re-read %zu MB x%d: %.1f GB/s\n", mb, reps, (double)reps*nn*16/ms/1e6);
  }
  for(int mod : {1, 32, 720, 1<<20}){
    int it=4096; matchk<<<nsm*8,512>>>(it,mod,out);
    cudaEventRecord(a); matchk<<<nsm*8,512>>>(it,mod,out); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    double warpops = (double)nsm*8*16*it; printf("match_any mod %d: %.3f warp-ops/clk/SM (%.2f G warp-ops/s)\n", mod, warpops/(ms*1e-3)/nsm/(pr.clockRate*1e3), warpops/ms/1e6);
  }
  { int it=4096; satom<<<nsm*8,512>>>(it,out);
    cudaEventRecord(a); satom<<<nsm*8,512>>>(it,out); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    double warpops = (double)nsm*8*16*it; printf("smem atomicAdd spread: %.3f warp-ops/clk/SM\n", warpops/(ms*1e-3)/nsm/(pr.clockRate*1e3)); }
  for(int r=0;r<100;r++) empty<<<1,32>>>(); CK(cudaDeviceSynchronize());
  cudaEventRecord(a); for(int r=0;r<1000;r++) empty<<<nsm*4,256>>>(); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
  printf("empty kernel back-to-back (stream): %.2f us/launch\n", ms);
  { cudaStream_t s; cudaStreamCreate(&s); cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal); for(int r=0;r<1000;r++) empty<<<nsm*4,256,0,s>>>(); cudaStreamEndCapture(s,&g); CK(cudaGraphInstantiate(&ge,g,0));
    cudaGraphLaunch(ge,s); cudaStreamSynchronize(s);
    cudaEventRecord(a,s); cudaGraphLaunch(ge,s); cudaEventRecord(b,s); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    printf("empty kernel in graph: %.2f us/launch\n", ms); }
  for(int bpm: {4,6,8}){ int it=200; int nb=nsm*bpm; void* args[]={&it,&out};
    CK(cudaLaunchCooperativeKernel((void*)gbar, nb, 128, args, 0, 0)); CK(cudaDeviceSynchronize());
    cudaEventRecord(a); cudaLaunchCooperativeKernel((void*)gbar, nb, 128, args, 0, 0); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    printf("grid.sync with %d CTAs: %.2f us\n", nb, ms*1000/it); }
  return 0;
}
