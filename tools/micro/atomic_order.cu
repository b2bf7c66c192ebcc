// Does a warp-wide shared-memory atomicAdd resolve same-address lanes in ascending
// lane order on this GPU?  Compares atomic ranks with ballot-derived stable ranks.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k(int iters, int mod, unsigned long long* bad, unsigned long long* total) {
  __shared__ unsigned h[8][1024];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < 1024; i += 32) h[warp][i] = 0;
  __syncwarp();
  unsigned v = (blockIdx.x * 977 + threadIdx.x) * 2654435761u;
  unsigned long long nb = 0, nt = 0;
  for (int it = 0; it < iters; ++it) {
    v = v * 1664525u + 1013904223u;
    unsigned key = (v >> 9) % mod;
    if (((v >> 3) & 7) == 0) key = 0;  // extra collisions
    unsigned mask_lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(mask_lt));
    unsigned peers = 0xffffffffu;
    for (int b = 0; b < 10; ++b) {
      unsigned bb = __ballot_sync(0xffffffffu, (key >> b) & 1);
      peers &= ((key >> b) & 1) ? bb : ~bb;
    }
    unsigned before = h[warp][key];
    __syncwarp();
    unsigned r = atomicAdd(&h[warp][key], 1u);
    __syncwarp();
    unsigned expect = before + __popc(peers & mask_lt);
    nb += (r != expect);
    nt += 1;
    if ((it & 63) == 63) { for (int i = lane; i < 1024; i += 32) h[warp][i] = 0; __syncwarp(); }
  }
  atomicAdd(bad, nb);
  atomicAdd(total, nt);
}
int main() {
  unsigned long long *bad, *tot;
  cudaMalloc(&bad, 8); cudaMalloc(&tot, 8);
  for (int mod : {2, 4, 16, 64, 256, 1000}) {
    cudaMemset(bad, 0, 8); cudaMemset(tot, 0, 8);
    k<<<148 * 4, 256>>>(4096, mod, bad, tot);
    unsigned long long hb, ht;
    cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&ht, tot, 8, cudaMemcpyDeviceToHost);
    printf("mod %5d: %llu of %llu lane-ops out of lane order\n", mod, hb, ht);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
