// Host-side definitions of the opaque ABI handles (dpc_ctx, dpc_dgraph,
// dpc_dtree) shared by the CUDA translation units.  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"
#include "dpc.h"
#include "dpc_internal.h"

struct dpc_ctx {
  int device = 0;
  int sms = 148;
  int max_threads_per_sm = 2048;
  int smem_per_sm = 233472;  // shared memory per SM (bytes)
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[64] = {};
  size_t pending_limit = 0;  // current cudaLimitDevRuntimePendingLaunchCount
  void* flush_buf = nullptr;
  size_t flush_bytes = 0;
  int coop = 0;  // cooperative launch supported
  // pipelined host-vector runs (dpc_spmv_host_batch): copy-in / copy-out
  // streams and per-slot events, created on first use
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t pev[9] = {};
  unsigned* p2p_fault = nullptr;  // dpc_p2p_barrier timeout flag
};

// Device-resident graph plus every buffer its apps need.
struct dpc_dgraph {
  dpc_ctx* ctx = nullptr;
  int64_t n = 0, m = 0;
  int64_t ncols = 0;           // columns (= n for square graphs); x has ncols entries
  unsigned* rowptr = nullptr;  // n+1 (uint32; m < 2^32)
  int* col = nullptr;
  int* w = nullptr;
  float* val = nullptr;
  float* x = nullptr;
  float* y = nullptr;
  unsigned* dist = nullptr;
  int* color = nullptr;
  // frontier / worklist buffers (SSSP, GC)
  unsigned* front[2] = {nullptr, nullptr};
  unsigned* stamp = nullptr;  // SSSP dedup stamp / GC pending counts
  uint2* sssp_fbe = nullptr;  // SSSP level form: {row start, row end} beside each light-list entry (2 x n)
  unsigned* gc_state = nullptr;  // GC heavy-vertex bitmaps (36 words per pool slot)
  size_t gc_state_slots = 0;
  void* trace = nullptr;          // per-vertex timestamps of the last traced run (DPC_TRACE=1)
  void* gc_q = nullptr;           // GC async task queue (+ 64 B of counters)
  void* gc_prio = nullptr;        // GC largest-log-degree-first priorities (8 B per vertex)
  size_t gc_q_cap = 0;
  unsigned* gc_hstate = nullptr;  // GC async heavy-vertex states
  size_t gc_hstate_cap = 0;
  int* gc_hcol = nullptr;         // GC async: adjacency split per vertex, higher-priority neighbours first
  unsigned* gc_hsplit = nullptr;  // GC async: number of higher-priority neighbours per vertex
  unsigned* ctr = nullptr;    // per-iteration counters (app-specific layout, 64 B)
  void* ctr_host = nullptr;   // pinned mirror of ctr
  dpc::dev::RunHeader* hdr = nullptr;  // device counters
  dpc::dev::RunHeader* hdr_host = nullptr;  // pinned mirror
  bool hdr_clean = false;  // the last run (SpMV stream) left the header zeroed itself
  bool check_pending = false;  // an asynchronous run awaits its fault check
  bool hdr_copied = false;     // ... and its header copy is already enqueued
  void* batch_buf = nullptr;  // dpc_spmv_host_batch_contig: two slots of grouped x / y vectors
  size_t batch_bytes = 0;
  float* x2 = nullptr;     // second x / y slot of the pipelined host-vector path
  float* y2 = nullptr;
  // consolidation pool
  dpc::dev::Item* items = nullptr;
  unsigned cap = 0;
  // stream-balanced drain (SpMV grid): per-item stream offsets and the
  // item index at every kMark-th stream position
  unsigned* soff = nullptr;
  size_t soff_cap = 0;
  // SpMV hot-column cache plan (column per slot) and per-run x values
  // partitioned SSSP (dpc_msssp_*): remote-distance filter, send / receive
  // pair buffers, per-owner counters, step state
  unsigned* ms_rdist = nullptr;
  void* ms_send = nullptr;
  void* ms_recv = nullptr;
  unsigned* ms_cnt = nullptr;
  size_t ms_n = 0, ms_cap = 0;
  size_t ms_rcap = 0;  // pairs the receive area holds (grown by dpc_msssp_recv_reserve)
  void* ms_state = nullptr;
  // SpMV grid plan (spmv_plan.cu): per 128-nonzero window row-start bits and
  // open segment, the row of each non-empty row, a self-resetting barrier
  unsigned* plan_mask = nullptr;
  unsigned* plan_sin = nullptr;
  unsigned* plan_segrow = nullptr;
  unsigned* plan_bar = nullptr;
  unsigned plan_nwin = 0;
  unsigned* plan8 = nullptr;  // G = 8 window plan (64 B per 256 nonzeros)
  unsigned* plan8_segrow = nullptr;
  unsigned plan8_nwin = 0;
  // hot-column x cache of the plan form: col re-encoded (hot columns as
  // slot | 0x80000000), the column of each slot, per-call x at the slots
  int* plan8h_col = nullptr;
  int* plan8h_hot = nullptr;
  float* plan8h_xh = nullptr;
  unsigned plan8h_nhot4 = 0;
  unsigned plan8h_cap = 0;  // slot capacity the plan was built for (0: none)
  void* sst_items = nullptr;  // SSSP frontier stream form: 2 x (n + 1) items
  size_t sst_cap = 0;
  int* xhot_col = nullptr;
  float* xhot_val = nullptr;
  int xhot_log = 0;
  // host copies used to size pools: degree array
  std::vector<int64_t> host_rowptr;
  std::map<std::pair<int, int>, uint64_t> need_cache;
  int64_t max_deg = 0;
};

struct dpc_dtree {
  dpc_ctx* ctx = nullptr;
  int64_t n = 0;
  int root = 0;
  int depth = 0;
  int* parent = nullptr;
  unsigned* cstart = nullptr;  // n+1
  int* clist = nullptr;
  int* result = nullptr;
  unsigned* level_nodes = nullptr;   // nodes in visit order (level by level)
  unsigned* level_off = nullptr;     // per-level offsets (device, depth+2)
  dpc::dev::RunHeader* hdr = nullptr;
  dpc::dev::RunHeader* hdr_host = nullptr;
  dpc::dev::Item* items = nullptr;
  unsigned cap = 0;
  unsigned* off_host = nullptr;      // pinned level offsets
  int64_t max_children = 0;
  int64_t root_children = 0;
  int64_t internal = 0;              // nodes with >= 1 child
  unsigned group = 1;                // lanes per work item (mean fan-out)
  unsigned* pend = nullptr;          // persistent grid: pending internal children per node
  bool check_pending = false;        // an asynchronous run's header copy awaits its fault check
};

namespace dpc {

// CUDA error -> dpc_status with a message naming the call site.
dpc_status cuda_fail(cudaError_t e, const char* what);
#define DPC_CUDA(call)                                         \
  do {                                                         \
    cudaError_t _e = (call);                                   \
    if (_e != cudaSuccess) return ::dpc::cuda_fail(_e, #call); \
  } while (0)

// Resolved launch configuration for one run.
struct Cfg {
  int variant;
  unsigned threshold;
  unsigned parent_threads;
  unsigned child_threads;
  unsigned child_blocks;  // cap (0 = none)
  unsigned chunk;
  int grid_persistent;  // grid variant as one cooperative persistent kernel
  unsigned flags;       // raw dpc_launch_cfg.flags (bits >= 8: experiment switches)
};

dpc_status resolve_cfg(dpc_ctx* ctx, int app, const dpc_launch_cfg* in, Cfg* out);

// Ensures the device runtime pending-launch pool can hold `need` launches.
// A large pool slows every device launch (tools/probes: 15 us -> 28 us per
// link), so it is set back to the default for the consolidated variants.
dpc_status ensure_pending_limit(dpc_ctx* ctx, size_t need);

// Pool slots needed for (threshold, chunk): sum over rows with
// deg > threshold of ceil(deg / chunk).  Cached per graph.
uint64_t pool_need(dpc_dgraph* g, unsigned threshold, unsigned chunk);
// Sizes the pending-launch pool for the worst case of one parent grid.
dpc_status ensure_pending_for(dpc_ctx* ctx, dpc_dgraph* g, int variant, unsigned threshold,
                              unsigned parent_threads);
dpc_status ensure_pool(dpc_dgraph* g, uint64_t need);

dpc_status begin_run(dpc_ctx* ctx, dpc::dev::RunHeader* hdr);
// Reports the fault of the graph's last asynchronous run (one launched
// without metrics), if any: synchronises, reads its header (copied by the
// run or here) and maps the fault bits.  Every graph entry point calls it
// first, so a fault is never lost behind a later run (dpc.h: dpc_dgraph_check).
dpc_status flush_check(dpc_ctx* ctx, dpc_dgraph* g);
// Marks a run launched without metrics whose header is NOT copied back:
// flush_check will copy it.
inline void defer_check(dpc_dgraph* g) {
  g->check_pending = true;
  g->hdr_copied = false;
}
// Frees the partitioned-SSSP step state of a graph (sssp.cu).
void sssp_state_free(void* state);
// SpMV grid variant with the cached per-matrix window plan (spmv_plan.cu).
dpc_status spmv_plan_build(dpc_ctx* ctx, dpc_dgraph* g);
// *launches += the host-side kernel launches of the call (1, or 2 with the hot-column gather).
dpc_status spmv_plan_run(dpc_ctx* ctx, dpc_dgraph* g, const float* d_x, float* d_y, int flags, int* launches);
// SSSP / BFS grid variant, frontier stream form (sssp_stream.cu).
dpc_status sssp_stream_run(dpc_ctx* ctx, dpc_dgraph* g, int32_t source, bool unit, bool coop,
                           int64_t* host_launches, int64_t* levels, dpc_metrics* met);
// Maps the device-side fault bits of a run header to a status + message.
dpc_status check_header(const dpc::dev::RunHeader* h);
dpc_status finish_metrics(dpc_ctx* ctx, dpc::dev::RunHeader* hdr, dpc::dev::RunHeader* hdr_host,
                          dpc_metrics* met);

}  // namespace dpc
