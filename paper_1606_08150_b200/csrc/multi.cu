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

#include "ctx.h"

struct dpc_comm {
  ncclComm_t nccl = nullptr;
  int rank = 0;
  int world = 1;
  dpc_ctx* ctx = nullptr;
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

}  // extern "C"
