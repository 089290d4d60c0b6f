// Device-wide barrier latency on B200: the library's generation barrier
// (common.cuh soft_grid_sync), cooperative groups' grid.sync(), and a
// monotonic 64-bit arrival counter (one release atomic per block, acquire
// polls until the round's target).  Standalone:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o barrier_probe barrier_probe.cu && ./barrier_probe
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long gns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void gen_sync(unsigned* count, unsigned* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g0;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g0) : "l"(gen) : "memory");
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      *reinterpret_cast<volatile unsigned*>(count) = 0;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      unsigned g;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
        if (g == g0) __nanosleep(20);
      } while (g == g0);
    }
  }
  __syncthreads();
}

template <bool SLEEP>
__device__ __forceinline__ void mono_sync(unsigned long long* count) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long old;
    asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(count) : "memory");
    const unsigned long long target = (old / gridDim.x + 1) * gridDim.x;
    unsigned long long seen;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(seen) : "l"(count) : "memory");
      if (SLEEP && seen < target) __nanosleep(20);
    } while (seen < target);
  }
  __syncthreads();
}

// red (no return) arrival + acquire polls
__device__ __forceinline__ void mono_red_sync(unsigned long long* count, unsigned long long& target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(count) : "memory");
    target += gridDim.x;
    unsigned long long seen;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(seen) : "l"(count) : "memory");
    } while (seen < target);
  }
  __syncthreads();
}

__global__ void k_gen(unsigned* w, int iters, unsigned long long* out) {
  const unsigned long long t0 = gns();
  for (int i = 0; i < iters; i++) gen_sync(w, w + 32);
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = gns() - t0;
}
__global__ void k_cg(int iters, unsigned long long* out) {
  const unsigned long long t0 = gns();
  for (int i = 0; i < iters; i++) cg::this_grid().sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = gns() - t0;
}
template <bool SLEEP>
__global__ void k_mono(unsigned long long* c, int iters, unsigned long long* out) {
  const unsigned long long t0 = gns();
  for (int i = 0; i < iters; i++) mono_sync<SLEEP>(c);
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = gns() - t0;
}
__global__ void k_red(unsigned long long* c, int iters, unsigned long long* out) {
  unsigned long long target = 0;
  const unsigned long long t0 = gns();
  for (int i = 0; i < iters; i++) mono_red_sync(c, target);
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = gns() - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* w;
  unsigned long long *c, *out;
  cudaMalloc(&w, 4096);
  cudaMalloc(&c, 4096);
  cudaMalloc(&out, 64);
  const int iters = 2000;
  const int shapes[][2] = {{8, 256}, {2, 512}, {1, 1024}};
  for (auto& sh : shapes) {
    const int blocks = sh[0] * sms, threads = sh[1];
    for (int rep = 0; rep < 2; rep++) {
      unsigned long long ns[5] = {};
      int it = iters;
      cudaMemset(w, 0, 4096);
      k_gen<<<blocks, threads>>>(w, it, out);
      cudaMemcpy(&ns[0], out, 8, cudaMemcpyDeviceToHost);
      void* args[] = {&it, &out};
      cudaLaunchCooperativeKernel((const void*)k_cg, blocks, threads, args, 0, 0);
      cudaMemcpy(&ns[1], out, 8, cudaMemcpyDeviceToHost);
      cudaMemset(c, 0, 4096);
      k_mono<true><<<blocks, threads>>>(c, it, out);
      cudaMemcpy(&ns[2], out, 8, cudaMemcpyDeviceToHost);
      cudaMemset(c, 0, 4096);
      k_mono<false><<<blocks, threads>>>(c, it, out);
      cudaMemcpy(&ns[3], out, 8, cudaMemcpyDeviceToHost);
      cudaMemset(c, 0, 4096);
      k_red<<<blocks, threads>>>(c, it, out);
      cudaMemcpy(&ns[4], out, 8, cudaMemcpyDeviceToHost);
      cudaError_t e = cudaDeviceSynchronize();
      printf("%4d x %4d: generation %.3f us  cg %.3f us  mono+sleep %.3f us  mono spin %.3f us  red spin %.3f us  (%s)\n",
             blocks, threads, ns[0] / 1e3 / iters, ns[1] / 1e3 / iters, ns[2] / 1e3 / iters, ns[3] / 1e3 / iters,
             ns[4] / 1e3 / iters, cudaGetErrorString(e));
    }
  }
  return 0;
}
