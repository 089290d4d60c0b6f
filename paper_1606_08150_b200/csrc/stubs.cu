// Temporary: entry points not yet implemented in this round.
#include "ctx.h"
using namespace dpc;
extern "C" {
dpc_status dpc_comm_unique_id(uint8_t*) { return fail(DPC_E_INVALID, "multi-GPU not implemented yet"); }
dpc_status dpc_comm_init(dpc_ctx*, int32_t, int32_t, const uint8_t*, dpc_comm**) { return fail(DPC_E_INVALID, "multi-GPU not implemented yet"); }
void dpc_comm_destroy(dpc_comm*) {}
dpc_status dpc_partition_rows(const dpc_csr*, int32_t, int64_t*) { return fail(DPC_E_INVALID, "not implemented yet"); }
dpc_status dpc_multi_spmv(dpc_ctx*, dpc_comm*, dpc_dgraph*, int64_t, int64_t, int64_t, int32_t, const dpc_launch_cfg*, dpc_metrics*) { return fail(DPC_E_INVALID, "not implemented yet"); }
}
