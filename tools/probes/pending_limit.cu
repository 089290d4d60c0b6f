// Probe: what does cudaDeviceSetLimit(cudaLimitDevRuntimePendingLaunchCount, v)
// actually grant on sm_100, and how many fire-and-forget launches fit?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void leaf(int* c) { if (threadIdx.x == 0) atomicAdd(c, 1); }
__global__ void storm(int* c, int* err, int per_thread) {
  for (int i = 0; i < per_thread; i++) {
    leaf<<<1, 32, 0, cudaStreamFireAndForget>>>(c);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { atomicAdd(err, 1); return; }
  }
}
int main() {
  int *c, *err; cudaMalloc(&c, 4); cudaMalloc(&err, 4);
  for (size_t v : {(size_t)2048, (size_t)1 << 20, (size_t)1 << 21, (size_t)3 << 20, (size_t)1 << 22, (size_t)1 << 23}) {
    cudaError_t e = cudaDeviceSetLimit(cudaLimitDevRuntimePendingLaunchCount, v);
    size_t got = 0; cudaDeviceGetLimit(&got, cudaLimitDevRuntimePendingLaunchCount);
    size_t fr, tot; cudaMemGetInfo(&fr, &tot);
    printf("set %zu -> %s, got %zu, free %.1f GB\n", v, cudaGetErrorString(e), got, fr / 1e9);
    for (int launches : {1 << 20, 3 << 20}) {
      cudaMemset(c, 0, 4); cudaMemset(err, 0, 4);
      storm<<<launches / 256 / 4, 256>>>(c, err, 4);
      cudaError_t s = cudaDeviceSynchronize();
      int hc, he; cudaMemcpy(&hc, c, 4, cudaMemcpyDeviceToHost); cudaMemcpy(&he, err, 4, cudaMemcpyDeviceToHost);
      printf("   storm %d launches: done %d, failed threads %d, %s\n", launches, hc, he, cudaGetErrorString(s));
    }
  }
  return 0;
}
