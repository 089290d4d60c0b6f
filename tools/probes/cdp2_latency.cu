// CDP2 launch-latency probe (sm_100a): is the ~67 us device-launch latency seen in
// cdp2_probe a function of the pending-launch limit, of warm-up, or intrinsic?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -rdc=true -O2 -o cdp2_latency cdp2_latency.cu -lcudadevrt
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void empty_k(int* c) { if (c && threadIdx.x == 0 && blockIdx.x == 0) c[7] = 1; }
__global__ void faf_parent(int* c) { if (threadIdx.x == 0) empty_k<<<1, 32, 0, cudaStreamFireAndForget>>>(c); }
__global__ void tail_parent(int* c) { if (threadIdx.x == 0) empty_k<<<1, 32, 0, cudaStreamTailLaunch>>>(c); }
__global__ void faf_big(int* c) { if (threadIdx.x == 0) empty_k<<<1184, 256, 0, cudaStreamFireAndForget>>>(c); }
__global__ void named_parent(int* c) {
  if (threadIdx.x == 0) {
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    empty_k<<<1, 32, 0, s>>>(c);
    cudaStreamDestroy(s);
  }
}
__global__ void chain(int* c, int lim) { c[0]++; if (c[0] < lim) chain<<<1, 1, 0, cudaStreamTailLaunch>>>(c, lim); }
__global__ void fchain(int* c, int lim) { c[0]++; if (c[0] < lim) fchain<<<1, 1, 0, cudaStreamFireAndForget>>>(c, lim); }

template <class F> float timeit(F f, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); CK(cudaDeviceSynchronize());
  cudaEventRecord(a); for (int i = 0; i < reps; i++) f(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b); return ms * 1000.f / reps;
}

int main() {
  int* d; CK(cudaMalloc(&d, 64)); CK(cudaMemset(d, 0, 64));
  for (size_t lim : {(size_t)2048, (size_t)1 << 16, (size_t)1 << 20}) {
    CK(cudaDeviceSetLimit(cudaLimitDevRuntimePendingLaunchCount, lim));
    printf("pending limit %zu\n", lim);
    printf("  host empty kernel, back-to-back: %.2f us\n", timeit([&] { empty_k<<<1, 32>>>(d); }, 200));
    printf("  host empty kernel, synced each:  %.2f us\n", timeit([&] { empty_k<<<1, 32>>>(d); cudaDeviceSynchronize(); }, 50));
    printf("  parent+FAF child, back-to-back:  %.2f us\n", timeit([&] { faf_parent<<<1, 32>>>(d); }, 200));
    printf("  parent+tail child, back-to-back: %.2f us\n", timeit([&] { tail_parent<<<1, 32>>>(d); }, 200));
    printf("  parent+FAF 1184x256 child:       %.2f us\n", timeit([&] { faf_big<<<1, 32>>>(d); }, 200));
    printf("  parent+named-stream child:       %.2f us\n", timeit([&] { named_parent<<<1, 32>>>(d); }, 50));
    printf("  tail chain x100 per link:        %.2f us\n", timeit([&] { cudaMemsetAsync(d, 0, 4); chain<<<1, 1>>>(d, 100); }, 5) / 100);
    printf("  FAF chain x20 per link:          %.2f us\n", timeit([&] { cudaMemsetAsync(d, 0, 4); fchain<<<1, 1>>>(d, 20); }, 5) / 20);
  }
  return 0;
}
