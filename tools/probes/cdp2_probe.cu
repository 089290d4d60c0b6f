// CDP2 semantics probe for sm_100a: answers the questions DESIGN.md depends on.
//  Q1 does a tail-launched grid run after the launching grid's fire-and-forget children?
//  Q2 does it also wait for grandchildren?
//  Q3 how long can a tail-launch chain get (does it nest)?
//  Q4 how deep can a fire-and-forget chain nest?
//  Q5 device-launch throughput (one launch per thread / per block).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -rdc=true -O2 -o cdp2_probe cdp2_probe.cu -lcudadevrt
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ void spin(long long cyc) { long long t = clock64(); while (clock64() - t < cyc) {} }

__global__ void q1_child(volatile int* f) { spin(2000000); f[0] = 1; __threadfence(); }
__global__ void q1_grandchild(volatile int* f) { spin(2000000); f[2] = 1; __threadfence(); }
__global__ void q1_child2(volatile int* f) { q1_grandchild<<<1, 1, 0, cudaStreamFireAndForget>>>((int*)f); }
__global__ void q1_post(volatile int* f) { f[1] = f[0]; f[3] = f[2]; }
__global__ void q1_parent(int* f) {
  q1_child<<<1, 1, 0, cudaStreamFireAndForget>>>(f);
  q1_child2<<<1, 1, 0, cudaStreamFireAndForget>>>(f);
  q1_post<<<1, 1, 0, cudaStreamTailLaunch>>>(f);
}

__global__ void q3_chain(int* c, int lim) {
  c[0] = c[0] + 1;
  if (c[0] < lim) {
    q3_chain<<<1, 1, 0, cudaStreamTailLaunch>>>(c, lim);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) c[1] = (int)e;
  }
}

__global__ void q4_nest(int* c, int d, int lim) {
  atomicMax(c, d);
  if (d < lim) {
    q4_nest<<<1, 1, 0, cudaStreamFireAndForget>>>(c, d + 1, lim);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess && c[1] == 0) c[1] = (int)e * 1000 + d;
  }
}
// tail chain where each link also FAF-launches a child: does the FAF depth accumulate along the chain?
__global__ void q6_leaf(int* c) { atomicAdd(c + 2, 1); }
__global__ void q6_chain(int* c, int lim) {
  q6_leaf<<<1, 1, 0, cudaStreamFireAndForget>>>(c);
  cudaError_t e0 = cudaGetLastError();
  if (e0 != cudaSuccess && c[1] == 0) c[1] = (int)e0 * 1000 + c[0];
  c[0] = c[0] + 1;
  if (c[0] < lim) {
    q6_chain<<<1, 1, 0, cudaStreamTailLaunch>>>(c, lim);
  }
}
// chain: FAF child does the tail launch of the next level (level-synchronous recursion shape)
__global__ void q7_level(int* c, int d, int lim);
__global__ void q7_next(int* c, int d, int lim) {
  q7_level<<<1, 1, 0, cudaStreamFireAndForget>>>(c, d, lim);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && c[1] == 0) c[1] = (int)e * 1000 + d;
}
__global__ void q7_level(int* c, int d, int lim) {
  atomicMax(c, d);
  if (d < lim) q7_next<<<1, 1, 0, cudaStreamTailLaunch>>>(c, d + 1, lim);
}

__global__ void q5_child(int* c) { if (threadIdx.x == 0) atomicAdd(c, 1); }
__global__ void q5_parent(int* c, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) q5_child<<<1, 32, 0, cudaStreamFireAndForget>>>(c);
}
__global__ void q5_parent_block(int* c) {
  if (threadIdx.x == 0) q5_child<<<1, 32, 0, cudaStreamFireAndForget>>>(c);
}

int main() {
  int* d; CK(cudaMalloc(&d, 64)); int h[8];
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("dev %s sms %d cc %d.%d l2 %d MB smem/sm %zu\n", p.name, p.multiProcessorCount, p.major, p.minor, p.l2CacheSize >> 20, p.sharedMemPerMultiprocessor);
  size_t v; CK(cudaDeviceGetLimit(&v, cudaLimitDevRuntimePendingLaunchCount)); printf("default pending launch count %zu\n", v);
  CK(cudaMemset(d, 0, 64)); q1_parent<<<1, 1>>>(d); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost));
  printf("Q1 tail-after-child=%d tail-after-grandchild=%d\n", h[1], h[3]);
  for (int lim : {10, 100, 1000, 10000}) {
    CK(cudaMemset(d, 0, 64)); q3_chain<<<1, 1>>>(d, lim); cudaError_t e = cudaDeviceSynchronize(); CK(cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost));
    printf("Q3 tail chain lim %d reached %d err %d sync %s\n", lim, h[0], h[1], cudaGetErrorString(e));
  }
  for (int lim : {10, 20, 23, 24, 25, 30}) {
    CK(cudaMemset(d, 0, 64)); q4_nest<<<1, 1>>>(d, 1, lim); cudaError_t e = cudaDeviceSynchronize(); CK(cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost));
    printf("Q4 FAF nest lim %d reached %d err %d sync %s\n", lim, h[0], h[1], cudaGetErrorString(e));
    cudaGetLastError();
  }
  for (int lim : {30, 100}) {
    CK(cudaMemset(d, 0, 64)); q6_chain<<<1, 1>>>(d, lim); cudaError_t e = cudaDeviceSynchronize(); CK(cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost));
    printf("Q6 tail chain+FAF lim %d links %d leaves %d err %d sync %s\n", lim, h[0], h[2], h[1], cudaGetErrorString(e));
  }
  for (int lim : {10, 23, 30, 100}) {
    CK(cudaMemset(d, 0, 64)); q7_level<<<1, 1>>>(d, 1, lim); cudaError_t e = cudaDeviceSynchronize(); CK(cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost));
    printf("Q7 tail->FAF level chain lim %d reached %d err %d sync %s\n", lim, h[0], h[1], cudaGetErrorString(e));
    cudaGetLastError();
  }
  CK(cudaDeviceSetLimit(cudaLimitDevRuntimePendingLaunchCount, 1 << 20));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int n : {1024, 16384, 65536, 262144}) {
    for (int rep = 0; rep < 2; rep++) {
      CK(cudaMemset(d, 0, 64)); cudaEventRecord(a); q5_parent<<<(n + 255) / 256, 256>>>(d, n); cudaEventRecord(b); cudaError_t e = cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, a, b); CK(cudaMemcpy(h, d, 4, cudaMemcpyDeviceToHost));
      printf("Q5 per-thread launches n=%d done=%d %.3f ms (%.1f ns/launch) %s\n", n, h[0], ms, ms * 1e6 / n, cudaGetErrorString(e));
    }
  }
  for (int nb : {148, 1024, 4096, 16384}) {
    for (int rep = 0; rep < 2; rep++) {
      CK(cudaMemset(d, 0, 64)); cudaEventRecord(a); q5_parent_block<<<nb, 256>>>(d); cudaEventRecord(b); cudaError_t e = cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, a, b); CK(cudaMemcpy(h, d, 4, cudaMemcpyDeviceToHost));
      printf("Q5 per-block launches nb=%d done=%d %.3f ms (%.1f ns/launch) %s\n", nb, h[0], ms, ms * 1e6 / nb, cudaGetErrorString(e));
    }
  }
  // single FAF launch latency: parent<<<1,1>>> launching 1 child, repeated
  for (int rep = 0; rep < 3; rep++) {
    CK(cudaMemset(d, 0, 64)); cudaEventRecord(a); q5_parent<<<1, 32>>>(d, 1); cudaEventRecord(b); CK(cudaDeviceSynchronize());
    float ms; cudaEventElapsedTime(&ms, a, b); printf("Q5 one-launch round trip %.2f us\n", ms * 1e3);
  }
  for (int rep = 0; rep < 3; rep++) {
    CK(cudaMemset(d, 0, 64)); cudaEventRecord(a); q3_chain<<<1, 1>>>(d, 1000); cudaEventRecord(b); CK(cudaDeviceSynchronize());
    float ms; cudaEventElapsedTime(&ms, a, b); printf("Q3 tail chain 1000: %.2f us per link\n", ms * 1e3 / 1000);
  }
  return 0;
}
