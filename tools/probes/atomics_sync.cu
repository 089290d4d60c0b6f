// Probe: (1) same-address atomicAdd throughput (one counter, many warps);
// (2) cooperative grid.sync cost at full residency; (3) a warp-aggregated
// append of N items to one counter.  Numbers feed DESIGN.md §4.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void same_addr(unsigned* c, int per_warp) {
  if ((threadIdx.x & 31) == 0)
    for (int i = 0; i < per_warp; i++) atomicAdd(c, 1u);
}
__global__ void spread_addr(unsigned* c, int per_warp) {
  unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if ((threadIdx.x & 31) == 0)
    for (int i = 0; i < per_warp; i++) atomicAdd(c + (w % 4096) * 32, 1u);
}
__global__ void syncs(unsigned* c, int n) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < n; i++) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) *c = n;
}

int main() {
  unsigned* c; cudaMalloc(&c, 4096 * 32 * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int blocks : {148, 1184, 4096}) {
    for (int pw : {1, 8}) {
      cudaMemset(c, 0, 4); same_addr<<<blocks, 256>>>(c, pw); cudaDeviceSynchronize();
      cudaEventRecord(a); same_addr<<<blocks, 256>>>(c, pw); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      long n = (long)blocks * 8 * pw;
      printf("same-address atomics: %ld ops in %.2f us -> %.2f ns/op\n", n, ms * 1e3, ms * 1e6 / n);
      cudaEventRecord(a); spread_addr<<<blocks, 256>>>(c, pw); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("spread atomics (4096 addrs): %ld ops in %.2f us\n", n, ms * 1e3);
    }
  }
  int dev = 0, per_sm = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  for (int threads : {256, 512}) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, syncs, threads, 0);
    for (int mult : {1, per_sm}) {
      int blocks = p.multiProcessorCount * mult;
      for (int n : {1, 100}) {
        void* args[] = {&c, &n};
        cudaLaunchCooperativeKernel((void*)syncs, blocks, threads, args, 0, 0); cudaDeviceSynchronize();
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)syncs, blocks, threads, args, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("grid.sync x%d: %d blocks x %d threads: %.2f us total (%.2f us/sync incl. launch)\n", n, blocks, threads, ms * 1e3, ms * 1e3 / n);
      }
    }
  }
  return 0;
}
