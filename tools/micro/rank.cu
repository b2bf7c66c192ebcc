// Micro-benchmark: cost of warp-level stable ranking primitives on B200 (sm_100a).
// Not part of the product path.  Each kernel computes, for NR rounds of 32 keys
// per warp, rank = #earlier lanes with the same key, and accumulates a checksum.
//   match : __match_any_sync + popc
//   ballot: log2(K) ballots + XNOR-AND + popc
//   atom  : shared atomicAdd on a per-warp histogram (order not guaranteed)
// plus the readout quad inner loop and an 8-byte LDS/STS loop for reference.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__device__ __forceinline__ unsigned lanemask_lt() { unsigned r; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r)); return r; }

template <int MODE, int BITS>
__global__ void rankk(int iters, unsigned mod, int* out) {
  __shared__ unsigned h[32][256];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < 256; i += 32) h[w][i] = 0;
  __syncwarp();
  unsigned v = threadIdx.x * 2654435761u + blockIdx.x * 97u;
  unsigned acc = 0;
  for (int i = 0; i < iters; ++i) {
    v = v * 1664525u + 1013904223u;
    const unsigned key = (v >> 8) % mod;
    unsigned r;
    if (MODE == 0) {
      const unsigned m = __match_any_sync(0xffffffffu, key);
      r = __popc(m & lanemask_lt());
    } else if (MODE == 1) {
      unsigned peers = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < BITS; ++b) {
        const unsigned bb = __ballot_sync(0xffffffffu, (key >> b) & 1u);
        peers &= ((key >> b) & 1u) ? bb : ~bb;
      }
      r = __popc(peers & lanemask_lt());
    } else {
      r = atomicAdd(&h[w][key & 255], 1u);
    }
    acc += r;
  }
  if (acc == 0x12345u) out[0] = acc;
}

int main() {
  cudaDeviceProp pr;
  CK(cudaGetDeviceProperties(&pr, 0));
  int nsm = pr.multiProcessorCount;
  int* out;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  auto run = [&](const char* name, auto kern, unsigned mod) {
    const int it = 2048, blocks = nsm * 2, thr = 1024;
    kern<<<blocks, thr>>>(it, mod, out);
    cudaEventRecord(a);
    kern<<<blocks, thr>>>(it, mod, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    const double warpops = (double)blocks * (thr / 32) * it;
    printf("%-28s mod %5u: %.3f warp-ranks/clk/SM  (%.1f ns per 32 keys per SM)\n", name, mod,
           warpops / (ms * 1e-3) / nsm / (clk_khz * 1e3), ms * 1e6 / (warpops / nsm));
  };
  for (unsigned mod : {1u, 8u, 24u, 148u, 444u}) {
    run("match_any", rankk<0, 1>, mod);
    run("ballot 5 bits", rankk<1, 5>, mod);
    run("ballot 8 bits", rankk<1, 8>, mod);
    run("smem atomicAdd", rankk<2, 1>, mod);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
