// Launch floor of the bench's timing method (512 MB memset flush, event pair,
// one or two launches) for kernel shapes like the SpMV drain's.  Standalone:
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o /tmp/floor floor_probe.cu && /tmp/floor
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void empty_k() {}
__global__ void empty_dyn() { extern __shared__ float s[]; if (threadIdx.x == 1u << 30) s[0] = 0; }
__global__ void pdl_first() { asm volatile("griddepcontrol.launch_dependents;"); }
__global__ void pdl_second() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* flush = nullptr;
  CK(cudaMalloc(&flush, 512u << 20));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  CK(cudaFuncSetAttribute(empty_dyn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  auto launch_pdl = [&](const void* fn, dim3 g, dim3 b, size_t smem, bool pdl) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = g; lc.blockDim = b; lc.dynamicSmemBytes = smem; lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at; lc.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelExC(&lc, fn, nullptr);
  };
  struct Case { const char* name; int kind; };
  const Case cases[] = {
    {"nothing (event pair only)", 0},
    {"empty <<<1, 32>>>", 1},
    {"empty <<<148, 1024>>>", 2},
    {"empty <<<148, 1024, 128 KB>>>", 3},
    {"empty <<<148, 1024, 200 KB>>>", 4},
    {"<<<148,256>>> + PDL <<<148,1024,128 KB>>>", 5},
    {"<<<148,256>>> + plain <<<148,1024,128 KB>>>", 6},
    {"graph: <<<148,256>>> + <<<148,1024,128 KB>>>", 7},
  };
  cudaGraphExec_t gexec = nullptr;
  {
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
    pdl_first<<<sms, 256, 0, s>>>();
    launch_pdl((const void*)empty_dyn, dim3(sms), dim3(1024), 128 * 1024, false);
    CK(cudaStreamEndCapture(s, &graph));
    CK(cudaGraphInstantiate(&gexec, graph, 0));
  }
  for (const Case& c : cases) {
    for (int flush_on = 1; flush_on >= 0; flush_on--) {
      std::vector<float> ts;
      for (int r = 0; r < 40; r++) {
        if (flush_on) cudaMemsetAsync(flush, r & 0xff, 512u << 20, s);
        cudaEventRecord(e0, s);
        switch (c.kind) {
          case 1: empty_k<<<1, 32, 0, s>>>(); break;
          case 2: empty_k<<<sms, 1024, 0, s>>>(); break;
          case 3: empty_dyn<<<sms, 1024, 128 * 1024, s>>>(); break;
          case 4: empty_dyn<<<sms, 1024, 200 * 1024, s>>>(); break;
          case 5: pdl_first<<<sms, 256, 0, s>>>();
                  launch_pdl((const void*)pdl_second, dim3(sms), dim3(1024), 128 * 1024, true); break;
          case 6: pdl_first<<<sms, 256, 0, s>>>();
                  launch_pdl((const void*)empty_dyn, dim3(sms), dim3(1024), 128 * 1024, false); break;
          case 7: cudaGraphLaunch(gexec, s); break;
          default: break;
        }
        cudaEventRecord(e1, s);
        CK(cudaStreamSynchronize(s));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 5) ts.push_back(ms * 1e3f);
      }
      std::sort(ts.begin(), ts.end());
      float mean = 0;
      for (float t : ts) mean += t;
      mean /= ts.size();
      printf("%-46s flush %d: mean %6.2f us  median %6.2f  min %6.2f\n", c.name, flush_on, mean, ts[ts.size() / 2], ts[0]);
    }
  }
  return 0;
}
