// Multi-GPU layer (BASELINE config 5): one process per GPU,
// 1-D row partition, NCCL over NVLink 5 / NVSwitch for the vector exchange.
//
// SpMV step on rank p (rows and x entries [p*R, (p+1)*R)):
//   ncclAllGather(x_local -> x_full)     [R floats in, R*world out, NVLink]
//   y_local = A_local x_full              [grid-consolidated SpMV, spmv.cu]
// Both are enqueued on the context stream, so the gather and the SpMV are
// ordered without a host round trip.  The communicator is created from a
// unique id the caller broadcasts (torch.distributed / MPI / files).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <vector>

#include "ctx.h"

struct dpc_comm {
  ncclComm_t nccl = nullptr;
  int rank = 0;
  int world = 1;
  dpc_ctx* ctx = nullptr;
  unsigned* d_counts = nullptr;   // world x world send counts (SSSP exchange)
  unsigned* h_counts = nullptr;   // pinned mirror
  unsigned* d_scalar = nullptr;   // all-reduce scratch
  unsigned* h_scalar = nullptr;
};

namespace dpc {
static dpc_status nccl_fail(ncclResult_t r, const char* what) {
  return fail(DPC_E_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}
}  // namespace dpc

#define DPC_NCCL(call)                                         \
  do {                                                         \
    ncclResult_t _r = (call);                                  \
    if (_r != ncclSuccess) return ::dpc::nccl_fail(_r, #call); \
  } while (0)

using namespace dpc;

extern "C" {

dpc_status dpc_comm_unique_id(uint8_t id[128]) {
  clear_error();
  if (!id) return fail(DPC_E_INVALID, "id is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  ncclUniqueId u;
  DPC_NCCL(ncclGetUniqueId(&u));
  std::memcpy(id, &u, sizeof(u));
  return DPC_OK;
}

dpc_status dpc_comm_init(dpc_ctx* ctx, int32_t rank, int32_t world, const uint8_t id[128],
                         dpc_comm** out) {
  clear_error();
  if (!ctx || !id || !out) return fail(DPC_E_INVALID, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(DPC_E_INVALID, "bad rank / world");
  DPC_CUDA(cudaSetDevice(ctx->device));
  auto* c = new (std::nothrow) dpc_comm();
  if (!c) return fail(DPC_E_OOM, "comm allocation failed");
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclResult_t r = ncclCommInitRank(&c->nccl, world, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  c->rank = rank;
  c->world = world;
  c->ctx = ctx;
  *out = c;
  return DPC_OK;
}

void dpc_comm_destroy(dpc_comm* c) {
  if (!c) return;
  if (c->nccl) ncclCommDestroy(c->nccl);
  if (c->d_counts) cudaFree(c->d_counts);
  if (c->d_scalar) cudaFree(c->d_scalar);
  if (c->h_counts) cudaFreeHost(c->h_counts);
  if (c->h_scalar) cudaFreeHost(c->h_scalar);
  delete c;
}

int32_t dpc_comm_rank(dpc_comm* c) { return c ? c->rank : -1; }
int32_t dpc_comm_world(dpc_comm* c) { return c ? c->world : 0; }

dpc_status dpc_partition_rows(const dpc_csr* g, int32_t world, int64_t* bounds) {
  clear_error();
  if (!g || !bounds || world < 1) return fail(DPC_E_INVALID, "bad arguments");
  if (!g->rowptr) return fail(DPC_E_INVALID, "rowptr is NULL");
  bounds[0] = 0;
  int64_t r = 0;
  for (int32_t p = 1; p < world; p++) {
    const int64_t target = g->m * p / world;
    r = std::lower_bound(g->rowptr + r, g->rowptr + g->n + 1, target) - g->rowptr;
    bounds[p] = std::min<int64_t>(r, g->n);
  }
  bounds[world] = g->n;
  return DPC_OK;
}

dpc_status dpc_multi_spmv(dpc_ctx* ctx, dpc_comm* comm, dpc_dgraph* local, const float* d_x_local,
                          float* d_y_local, const dpc_launch_cfg* cfg, dpc_metrics* met) {
  clear_error();
  if (!ctx || !comm || !local || !d_x_local || !d_y_local) return fail(DPC_E_INVALID, "NULL argument");
  if (local->ncols != local->n * comm->world)
    return fail(DPC_E_INVALID, "local block must have R rows and R * world columns");
  DPC_NCCL(ncclAllGather(d_x_local, local->x, static_cast<size_t>(local->n), ncclFloat, comm->nccl,
                         ctx->stream));
  return dpc_spmv_device(ctx, local, local->x, d_y_local, cfg, met);
}

// Vertex-partitioned SSSP over NCCL (BASELINE config 5): the dpc_msssp_*
// steps (sssp.cu) with the exchange done by grouped ncclSend / ncclRecv of
// {vertex, distance} pairs over NVLink, the per-owner counts by one
// ncclAllGather, and the stop test by an ncclAllReduce of |F_it+1|.
dpc_status dpc_multi_sssp(dpc_ctx* ctx, dpc_comm* comm, dpc_dgraph* local, int64_t n_global, int64_t source,
                          const dpc_launch_cfg* cfg, dpc_metrics* met) {
  clear_error();
  if (!ctx || !comm || !local) return fail(DPC_E_INVALID, "NULL argument");
  const int P = comm->world, me = comm->rank;
  const int64_t R = (n_global + P - 1) / P;
  cudaStream_t s = ctx->stream;
  if (!comm->d_counts) {
    DPC_CUDA(cudaMalloc(&comm->d_counts, sizeof(unsigned) * 64 * 64));
    DPC_CUDA(cudaMallocHost(&comm->h_counts, sizeof(unsigned) * 64 * 64));
    DPC_CUDA(cudaMalloc(&comm->d_scalar, sizeof(unsigned) * 2));
    DPC_CUDA(cudaMallocHost(&comm->h_scalar, sizeof(unsigned) * 2));
  }
  dpc_status st = dpc_msssp_begin(ctx, local, me * R, R, n_global, P, source, cfg);
  if (st != DPC_OK) return st;
  std::vector<uint32_t> sc(static_cast<size_t>(P));
  for (int64_t it = 0; it <= n_global; it++) {
    st = dpc_msssp_relax(ctx, local, sc.data());
    if (st != DPC_OK) return st;
    // every rank learns the full count matrix (row q = what q sends)
    DPC_NCCL(ncclAllGather(dpc_msssp_send_counts(local), comm->d_counts, static_cast<size_t>(P), ncclUint32,
                           comm->nccl, s));
    DPC_CUDA(cudaMemcpyAsync(comm->h_counts, comm->d_counts, sizeof(unsigned) * P * P, cudaMemcpyDeviceToHost, s));
    DPC_CUDA(cudaStreamSynchronize(s));
    // the receive area must hold what every peer queued for this rank
    // (bounded by the peers' edge counts, not this rank's)
    uint64_t incoming = 0;
    for (int q = 0; q < P; q++)
      if (q != me) incoming += comm->h_counts[q * P + me];
    void* rbuf = nullptr;
    st = dpc_msssp_recv_reserve(ctx, local, incoming, &rbuf);
    if (st != DPC_OK) return st;
    uint2* recv = static_cast<uint2*>(rbuf);
    uint64_t total = 0;
    DPC_NCCL(ncclGroupStart());
    for (int q = 0; q < P; q++) {
      if (q == me) continue;
      const size_t out = comm->h_counts[me * P + q], in = comm->h_counts[q * P + me];
      if (out) DPC_NCCL(ncclSend(dpc_msssp_send_buffer(local, q), 2 * out, ncclUint32, q, comm->nccl, s));
      if (in) DPC_NCCL(ncclRecv(recv + total, 2 * in, ncclUint32, q, comm->nccl, s));
      total += in;
    }
    DPC_NCCL(ncclGroupEnd());
    uint32_t next = 0;
    st = dpc_msssp_apply(ctx, local, recv, total, &next);
    if (st != DPC_OK) return st;
    comm->h_scalar[0] = next;
    DPC_CUDA(cudaMemcpyAsync(comm->d_scalar, comm->h_scalar, sizeof(unsigned), cudaMemcpyHostToDevice, s));
    DPC_NCCL(ncclAllReduce(comm->d_scalar, comm->d_scalar + 1, 1, ncclUint32, ncclSum, comm->nccl, s));
    DPC_CUDA(cudaMemcpyAsync(comm->h_scalar + 1, comm->d_scalar + 1, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    DPC_CUDA(cudaStreamSynchronize(s));
    if (comm->h_scalar[1] == 0) break;
  }
  return dpc_msssp_end(ctx, local, met);
}

}  // extern "C"
