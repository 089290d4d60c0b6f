// How many thread-block clusters of the SpMV drain's shape (1024 threads,
// ~130 KB dynamic shared memory) can be co-resident on this B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* p) { extern __shared__ float s[]; if (threadIdx.x == 1u << 30) p[0] = s[0]; }
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 131072 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8}) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(sms / cs * cs);
    lc.blockDim = dim3(1024);
    lc.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    lc.attrs = at; lc.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (const void*)k, &lc);
    printf("cluster %d: max active clusters %d (= %d CTAs of %d SMs) %s\n", cs, n, n * cs, sms, cudaGetErrorString(e));
  }
  return 0;
}
