// PageRank (the paper's PR benchmark; SPEC.md:454 oracle "PR = one-or-more
// power iterations with damping 0.85"; :468 fixed iteration count).
//
// A PR power iteration is an SpMV over the transposed graph: with
// P[v][u] = 1 / outdeg(u) for every edge u -> v,
//   r'[v] = (1 - d) / n + d * ((P r)[v] + D / n),   D = sum of r over dangling u.
// So PR runs the SpMV consolidation variants (spmv.cu) on P, one SpMV per
// iteration, plus one small update kernel that also accumulates the next
// dangling mass.  P is built once per graph on the host (counting sort by
// destination, rows sorted by source) and kept resident.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <vector>

#include "ctx.h"

struct dpc_prgraph {
  dpc_ctx* ctx = nullptr;
  dpc_dgraph* pt = nullptr;      // P = transposed graph, values 1 / outdeg(source)
  int64_t n = 0;
  unsigned* dangling = nullptr;  // ids of vertices without out-edges
  int64_t ndangling = 0;
  double* dmass = nullptr;       // [3] dangling mass, rotated by iteration (read / accumulate / clear)
  unsigned char* dflag = nullptr; // 1 for a dangling vertex (no out-edge)
};

namespace dpc {
namespace pr {

__global__ void __launch_bounds__(256) init_kernel(float* r, unsigned n, double* dmass, double d0) {
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) r[i] = 1.0f / static_cast<float>(n);
  if (i == 0) dmass[0] = d0, dmass[1] = 0.0, dmass[2] = 0.0;
}

// One kernel per iteration after the SpMV (y = P r):
//   r[v] = (1-d)/n + d (y[v] + D/n),  D = dmass[it % 3]
// and, for the next iteration, the dangling mass of the new ranks into
// dmass[(it + 1) % 3]; dmass[(it + 2) % 3] (last read one iteration ago) is
// cleared for the one after.  Replaces a clear launch and a pass over the
// dangling list per iteration.
__global__ void __launch_bounds__(256) update_kernel(float* __restrict__ r, const float* __restrict__ y, unsigned n,
                                                      double damping, double* dmass,
                                                      const unsigned char* __restrict__ dflag, int it) {
  const double dn = dmass[it % 3] / n;
  const double base = (1.0 - damping) / n;
  if (blockIdx.x == 0 && threadIdx.x == 0) dmass[(it + 2) % 3] = 0.0;
  double s = 0.0;
  for (unsigned v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const float nr = static_cast<float>(base + damping * (static_cast<double>(y[v]) + dn));
    r[v] = nr;
    if (dflag[v]) s += nr;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s != 0.0) atomicAdd(dmass + (it + 1) % 3, s);
}

}  // namespace pr
}  // namespace dpc

using namespace dpc;

extern "C" {

dpc_status dpc_pr_upload(dpc_ctx* ctx, const dpc_csr* G, dpc_prgraph** out) {
  clear_error();
  if (!ctx || !G || !out) return fail(DPC_E_INVALID, "NULL argument");
  dpc_status st = dpc_csr_validate(G);
  if (st != DPC_OK) return st;
  if (G->ncols && G->ncols != G->n) return fail(DPC_E_INVALID, "PageRank needs a square graph");
  const int64_t n = G->n, m = G->m;
  // P = transpose with values 1 / outdeg(source), rows (destinations) sorted by source
  std::vector<int64_t> rp(static_cast<size_t>(n) + 1, 0);
  for (int64_t k = 0; k < m; k++) rp[static_cast<size_t>(G->col[k]) + 1]++;
  for (int64_t v = 0; v < n; v++) rp[v + 1] += rp[v];
  std::vector<int32_t> col(static_cast<size_t>(m));
  std::vector<float> val(static_cast<size_t>(m));
  std::vector<int64_t> fill(rp.begin(), rp.end() - 1);
  std::vector<unsigned> dang;
  for (int64_t u = 0; u < n; u++) {
    const int64_t b = G->rowptr[u], e = G->rowptr[u + 1];
    if (e == b) dang.push_back(static_cast<unsigned>(u));
    const float inv = e > b ? 1.0f / static_cast<float>(e - b) : 0.0f;
    for (int64_t k = b; k < e; k++) {
      const int64_t at = fill[G->col[k]]++;
      col[at] = static_cast<int32_t>(u);
      val[at] = inv;
    }
  }
  dpc_csr* P = nullptr;
  st = dpc_csr_create(n, m, rp.data(), col.data(), nullptr, val.data(), &P);
  if (st != DPC_OK) return st;
  auto* h = new (std::nothrow) dpc_prgraph();
  if (!h) {
    dpc_csr_free(P);
    return fail(DPC_E_OOM, "prgraph allocation failed");
  }
  h->ctx = ctx;
  h->n = n;
  st = dpc_dgraph_upload(ctx, P, &h->pt);
  dpc_csr_free(P);
  if (st != DPC_OK) {
    dpc_pr_free(h);
    return st;
  }
  h->ndangling = static_cast<int64_t>(dang.size());
  cudaError_t e = cudaMalloc(&h->dangling, sizeof(unsigned) * std::max<size_t>(dang.size(), 1));
  if (e == cudaSuccess) e = cudaMalloc(&h->dmass, sizeof(double) * 3);
  if (e == cudaSuccess) e = cudaMalloc(&h->dflag, static_cast<size_t>(std::max<int64_t>(n, 1)));
  if (e == cudaSuccess && !dang.empty())
    e = cudaMemcpy(h->dangling, dang.data(), sizeof(unsigned) * dang.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    std::vector<unsigned char> fl(static_cast<size_t>(std::max<int64_t>(n, 1)), 0);
    for (unsigned v : dang) fl[v] = 1;
    e = cudaMemcpy(h->dflag, fl.data(), fl.size(), cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    dpc_pr_free(h);
    return cuda_fail(e, "dpc_pr_upload");
  }
  *out = h;
  return DPC_OK;
}

void dpc_pr_free(dpc_prgraph* h) {
  if (!h) return;
  if (h->pt) dpc_dgraph_free(h->pt);
  if (h->dangling) cudaFree(h->dangling);
  if (h->dmass) cudaFree(h->dmass);
  if (h->dflag) cudaFree(h->dflag);
  delete h;
}

float* dpc_pr_rank(dpc_prgraph* h) { return h && h->pt ? h->pt->x : nullptr; }

dpc_status dpc_pr_device(dpc_ctx* ctx, dpc_prgraph* h, int32_t iters, double damping,
                         const dpc_launch_cfg* cfg, dpc_metrics* met) {
  clear_error();
  if (!ctx || !h) return fail(DPC_E_INVALID, "NULL argument");
  if (iters < 0 || !(damping >= 0.0 && damping <= 1.0)) return fail(DPC_E_INVALID, "bad iters / damping");
  const unsigned n = static_cast<unsigned>(h->n);
  if (n == 0) return DPC_OK;
  cudaStream_t s = ctx->stream;
  dpc_dgraph* pt = h->pt;
  const unsigned nb = std::max(1u, (n + 255) / 256), gb = std::min(nb, 8u * static_cast<unsigned>(ctx->sms));
  pr::init_kernel<<<nb, 256, 0, s>>>(pt->x, n, h->dmass, static_cast<double>(h->ndangling) / n);
  DPC_CUDA(cudaGetLastError());
  for (int32_t it = 0; it < iters; it++) {
    dpc_status st = dpc_spmv_device(ctx, pt, pt->x, pt->y, cfg, met);  // y = P r
    if (st != DPC_OK) return st;
    pr::update_kernel<<<gb, 256, 0, s>>>(pt->x, pt->y, n, damping, h->dmass, h->dflag, it);
    DPC_CUDA(cudaGetLastError());
  }
  // the SpMV calls counted their own launch; here: init + one update per iteration
  if (met) met->host_launches += 1 + static_cast<int64_t>(iters);
  return DPC_OK;
}

dpc_status dpc_run_pagerank(dpc_ctx* ctx, const dpc_csr* G, int32_t iters, double damping, float* rank,
                            const dpc_launch_cfg* cfg, dpc_metrics* met) {
  clear_error();
  if (!ctx || !G || !rank) return fail(DPC_E_INVALID, "NULL argument");
  dpc_prgraph* h = nullptr;
  dpc_status st = dpc_pr_upload(ctx, G, &h);
  if (st != DPC_OK) return st;
  if (met) std::memset(met, 0, sizeof(*met));
  st = dpc_pr_device(ctx, h, iters, damping, cfg, met);
  if (st == DPC_OK) st = flush_check(ctx, h->pt);  // asynchronous SpMV runs: their fault check
  if (st == DPC_OK && G->n > 0) st = dpc_copy_d2h(ctx, rank, h->pt->x, sizeof(float) * static_cast<size_t>(G->n));
  dpc_pr_free(h);
  return st;
}

}  // extern "C"
