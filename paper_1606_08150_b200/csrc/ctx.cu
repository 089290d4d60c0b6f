// Context, device-resident handles, launch-configuration policy and the
// host-buffer run wrappers of libdpc.so.
//
// Policy replaced here:
//  - KC_X (config.hpp:68-75) keeps its meaning — B = max(1, B_occ / X) — but
//    B_occ comes from the B200 (148 SMs, 2048 threads/SM) and the defaults for
//    (threshold, chunk, X) come from the measured sweep (tools/sweep_launch.py ->
//    profiles/r02_launch_cfg.json -> launch_table.inc), not from the occupancy
//    calculator.
//  - per-buffer sizing (memplan.hpp:61-168, const = 4) is replaced by exact
//    counts: the pool holds sum over rows with deg > threshold of
//    ceil(deg / chunk) items, the most any parent pass can insert.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <new>

#include "ctx.h"

using dpc::dev::Item;
using dpc::dev::RunHeader;

namespace dpc {

dpc_status cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();  // clear sticky-free errors
  dpc_status st = (e == cudaErrorMemoryAllocation) ? DPC_E_OOM : DPC_E_CUDA;
  return fail(st, std::string(what) + ": " + cudaGetErrorString(e));
}

// Measured defaults (tools/sweep.py; see DESIGN.md §Launch configuration).
// Index: [app][variant].  Fields: threshold, parent_threads, child_threads,
// child_blocks, kc_x, chunk, flags.
struct Default {
  int threshold, parent_threads, child_threads, child_blocks, kc_x, chunk, flags;
};
#include "launch_table.inc"

dpc_status resolve_cfg(dpc_ctx* ctx, int app, const dpc_launch_cfg* in, Cfg* out) {
  dpc_launch_cfg c;
  int variant = in ? in->variant : DPC_GRID;
  if (variant < DPC_FLAT || variant > DPC_GRID) return fail(DPC_E_INVALID, "unknown variant");
  if (app < 0 || app > DPC_APP_TREE_HEIGHT) return fail(DPC_E_INVALID, "unknown app");
  dpc_launch_cfg_default(app, variant, &c);
  if (in) {
    if (in->threshold >= 0) c.threshold = in->threshold;
    if (in->parent_threads > 0) c.parent_threads = in->parent_threads;
    if (in->child_threads > 0) c.child_threads = in->child_threads;
    if (in->child_blocks > 0) c.child_blocks = in->child_blocks;
    if (in->kc_x >= 0) c.kc_x = in->kc_x;
    if (in->chunk > 0) c.chunk = in->chunk;
    c.flags = in->flags;
  }
  auto ok_threads = [](int t) { return t >= 32 && t <= 1024 && t % 32 == 0; };
  if (!ok_threads(c.parent_threads) || !ok_threads(c.child_threads))
    return fail(DPC_E_INVALID, "thread counts must be multiples of 32 in [32, 1024]");
  if (c.chunk < 32) return fail(DPC_E_INVALID, "chunk must be >= 32 edges");
  out->variant = variant;
  out->threshold = static_cast<unsigned>(c.threshold);
  out->parent_threads = static_cast<unsigned>(c.parent_threads);
  out->child_threads = static_cast<unsigned>(c.child_threads);
  out->chunk = static_cast<unsigned>(c.chunk);
  out->grid_persistent = !(c.flags & DPC_CFG_GRID_CDP);
  out->flags = static_cast<unsigned>(c.flags);
  // KC_X: B = max(1, B_occ / X); X = 0 selects "1-1" (no cap).
  unsigned b_occ = static_cast<unsigned>(ctx->sms) *
                   static_cast<unsigned>(ctx->max_threads_per_sm / c.child_threads);
  if (c.child_blocks > 0) out->child_blocks = static_cast<unsigned>(c.child_blocks);
  else if (c.kc_x > 0) out->child_blocks = std::max(1u, b_occ / static_cast<unsigned>(c.kc_x));
  else out->child_blocks = 0;
  return DPC_OK;
}

dpc_status ensure_pending_limit(dpc_ctx* ctx, size_t need) {
  size_t want = std::max<size_t>(2048, need);
  if (want == ctx->pending_limit) return DPC_OK;
  size_t cur = 0;  // another context of this process may have changed it
  if (cudaDeviceGetLimit(&cur, cudaLimitDevRuntimePendingLaunchCount) == cudaSuccess && cur == want) {
    ctx->pending_limit = want;
    return DPC_OK;
  }
  DPC_CUDA(cudaStreamSynchronize(ctx->stream));
  DPC_CUDA(cudaDeviceSetLimit(cudaLimitDevRuntimePendingLaunchCount, want));
  ctx->pending_limit = want;
  return DPC_OK;
}

uint64_t pool_need(dpc_dgraph* g, unsigned threshold, unsigned chunk) {
  auto key = std::make_pair(static_cast<int>(threshold), static_cast<int>(chunk));
  auto it = g->need_cache.find(key);
  if (it != g->need_cache.end()) return it->second;
  uint64_t need = 0;
  for (int64_t v = 0; v < g->n; v++) {
    uint64_t d = static_cast<uint64_t>(g->host_rowptr[v + 1] - g->host_rowptr[v]);
    if (d > threshold) need += (d + chunk - 1) / chunk;
  }
  g->need_cache[key] = need;
  return need;
}

dpc_status ensure_pending_for(dpc_ctx* ctx, dpc_dgraph* g, int variant, unsigned threshold,
                              unsigned parent_threads) {
  // Outstanding device launches one parent grid can create: basic = one per
  // heavy vertex, warp = one per warp holding one, block = one per block.
  const uint64_t heavy = pool_need(g, threshold, 1u << 30);
  const uint64_t items = static_cast<uint64_t>(g->n);
  uint64_t need = 1;
  if (variant == DPC_BASIC) need = heavy;
  else if (variant == DPC_WARP) need = std::min<uint64_t>(heavy, (items + 31) / 32);
  else if (variant == DPC_BLOCK) need = std::min<uint64_t>(heavy, (items + parent_threads - 1) / parent_threads);
  return ensure_pending_limit(ctx, static_cast<size_t>(need) + 1024);
}

dpc_status ensure_pool(dpc_dgraph* g, uint64_t need) {
  if (need < 1) need = 1;
  if (need > 0xffffffffull) return fail(DPC_E_OVERFLOW, "consolidation pool exceeds 2^32 items");
  if (need <= g->cap) return DPC_OK;
  DPC_CUDA(cudaStreamSynchronize(g->ctx->stream));
  if (g->items) cudaFree(g->items);
  g->items = nullptr;
  g->cap = 0;
  DPC_CUDA(cudaMalloc(&g->items, sizeof(Item) * need));
  g->cap = static_cast<unsigned>(need);
  return DPC_OK;
}

dpc_status check_header(const RunHeader* h) {
  if (h->overflow & 2u)
    return fail(DPC_E_CUDA, std::string("a device-side (CDP2) launch failed: ") +
                                cudaGetErrorString(static_cast<cudaError_t>(h->aux0)));
  if (h->overflow & 8u)
    return fail(DPC_E_INVALID, "coloring needs a symmetric graph (the worklist drained with uncolored vertices)");
  if (h->overflow & dpc::dev::kFaultBarrier)
    return fail(DPC_E_DEADLOCK, "device-wide barrier timed out after 2 s (the grid was not co-resident: "
                                "another context or MPS client on the GPU?)");
  if (h->overflow & 4u) return fail(DPC_E_DEADLOCK, "worklist made no progress for 2 s (lost task)");
  if (h->overflow & 1u) return fail(DPC_E_OVERFLOW, "consolidation pool overflow");
  return DPC_OK;
}

dpc_status flush_check(dpc_ctx* ctx, dpc_dgraph* g) {
  if (!g->check_pending) return DPC_OK;
  g->check_pending = false;
  if (!g->hdr_copied)
    DPC_CUDA(cudaMemcpyAsync(g->hdr_host, g->hdr, sizeof(RunHeader), cudaMemcpyDeviceToHost, ctx->stream));
  g->hdr_copied = false;
  DPC_CUDA(cudaStreamSynchronize(ctx->stream));
  const dpc_status st = check_header(g->hdr_host);
  if (st != DPC_OK) g->hdr_clean = false;  // the next run re-zeroes the header
  return st;
}

dpc_status begin_run(dpc_ctx* ctx, RunHeader* hdr) {
  DPC_CUDA(cudaMemsetAsync(hdr, 0, sizeof(RunHeader), ctx->stream));
  return DPC_OK;
}

dpc_status finish_metrics(dpc_ctx* ctx, RunHeader* hdr, RunHeader* hdr_host, dpc_metrics* met) {
  DPC_CUDA(cudaMemcpyAsync(hdr_host, hdr, sizeof(RunHeader), cudaMemcpyDeviceToHost, ctx->stream));
  DPC_CUDA(cudaStreamSynchronize(ctx->stream));
  dpc_status st = check_header(hdr_host);
  if (st != DPC_OK) return st;
  if (met) {
    met->child_launch_count += hdr_host->launches;
    met->buffer_items_inserted += hdr_host->aux1;
    met->pool_peak = std::max<int64_t>(met->pool_peak, hdr_host->count);
    met->overflow = static_cast<int32_t>(hdr_host->overflow);
  }
  return DPC_OK;
}

}  // namespace dpc

using namespace dpc;

extern "C" {

dpc_status dpc_launch_cfg_default(int32_t app, int32_t variant, dpc_launch_cfg* cfg) {
  if (!cfg) return fail(DPC_E_INVALID, "cfg is NULL");
  if (app < 0 || app > DPC_APP_TREE_HEIGHT || variant < DPC_FLAT || variant > DPC_GRID)
    return fail(DPC_E_INVALID, "unknown app or variant");
  const Default& d = kDefaults[app][variant];
  cfg->variant = variant;
  cfg->threshold = d.threshold;
  cfg->parent_threads = d.parent_threads;
  cfg->child_threads = d.child_threads;
  cfg->child_blocks = d.child_blocks;
  cfg->kc_x = d.kc_x;
  cfg->chunk = d.chunk;
  cfg->flags = d.flags;
  return DPC_OK;
}

dpc_status dpc_ctx_create(int32_t device, dpc_ctx** out) {
  clear_error();
  if (!out) return fail(DPC_E_INVALID, "out is NULL");
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(DPC_E_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  if (device < 0 || device >= count) return fail(DPC_E_INVALID, "device index out of range");
  cudaDeviceProp p;
  DPC_CUDA(cudaGetDeviceProperties(&p, device));
  if (p.major != 10) return fail(DPC_E_CUDA, "libdpc is built for sm_100a (B200); device is sm_" +
                                                 std::to_string(p.major * 10 + p.minor));
  DPC_CUDA(cudaSetDevice(device));
  auto* c = new (std::nothrow) dpc_ctx();
  if (!c) return fail(DPC_E_OOM, "ctx allocation failed");
  c->device = device;
  c->sms = p.multiProcessorCount;
  c->max_threads_per_sm = p.maxThreadsPerMultiProcessor;
  c->smem_per_sm = static_cast<int>(p.sharedMemPerMultiprocessor);
  c->coop = p.cooperativeLaunch;
  e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  for (int i = 0; e == cudaSuccess && i < 64; i++) e = cudaEventCreate(&c->ev[i]);
  if (e == cudaSuccess) {
    c->flush_bytes = std::max<size_t>(2 * static_cast<size_t>(p.l2CacheSize), 256u << 20);
    e = cudaMalloc(&c->flush_buf, c->flush_bytes);
  }
  // the device limits are per process: a second context keeps what an
  // earlier one raised (never lowers them)
  size_t pending = 0, heap = 0;
  if (e == cudaSuccess) e = cudaDeviceGetLimit(&pending, cudaLimitDevRuntimePendingLaunchCount);
  if (e == cudaSuccess && pending < 2048) {
    e = cudaDeviceSetLimit(cudaLimitDevRuntimePendingLaunchCount, 2048);
    pending = 2048;
  }
  // device heap for the allocator-study variants (DPC_CFG_ALLOC_MALLOC): it
  // can only be sized before the first kernel that calls malloc
  if (e == cudaSuccess) e = cudaDeviceGetLimit(&heap, cudaLimitMallocHeapSize);
  if (e == cudaSuccess && heap < (size_t{512} << 20)) {
    if (cudaDeviceSetLimit(cudaLimitMallocHeapSize, size_t{512} << 20) != cudaSuccess)
      cudaGetLastError();  // heap already in use: keep its size (malloc overflow is reported per run)
  }
  if (e != cudaSuccess) {
    dpc_ctx_destroy(c);
    return cuda_fail(e, "dpc_ctx_create");
  }
  c->pending_limit = pending;
  *out = c;
  return DPC_OK;
}

void dpc_ctx_destroy(dpc_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& ev : c->ev)
    if (ev) cudaEventDestroy(ev);
  if (c->flush_buf) cudaFree(c->flush_buf);
  for (auto& ev : c->pev)
    if (ev) cudaEventDestroy(ev);
  if (c->p2p_fault) cudaFree(c->p2p_fault);
  if (c->h2d) cudaStreamDestroy(c->h2d);
  if (c->d2h) cudaStreamDestroy(c->d2h);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

void* dpc_ctx_stream(dpc_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }
int32_t dpc_ctx_sm_count(dpc_ctx* c) { return c ? c->sms : 0; }

dpc_status dpc_ctx_event_record(dpc_ctx* c, int32_t slot) {
  if (!c || slot < 0 || slot >= 64) return fail(DPC_E_INVALID, "bad ctx or event slot");
  DPC_CUDA(cudaEventRecord(c->ev[slot], c->stream));
  return DPC_OK;
}

dpc_status dpc_ctx_event_elapsed(dpc_ctx* c, int32_t a, int32_t b, float* ms) {
  if (!c || !ms || a < 0 || a >= 64 || b < 0 || b >= 64) return fail(DPC_E_INVALID, "bad arguments");
  DPC_CUDA(cudaEventSynchronize(c->ev[b]));
  DPC_CUDA(cudaEventElapsedTime(ms, c->ev[a], c->ev[b]));
  return DPC_OK;
}

dpc_status dpc_ctx_synchronize(dpc_ctx* c) {
  if (!c) return fail(DPC_E_INVALID, "ctx is NULL");
  DPC_CUDA(cudaStreamSynchronize(c->stream));
  return DPC_OK;
}

dpc_status dpc_ctx_flush_l2(dpc_ctx* c) {
  if (!c) return fail(DPC_E_INVALID, "ctx is NULL");
  DPC_CUDA(cudaMemsetAsync(c->flush_buf, 0x5a, c->flush_bytes, c->stream));
  return DPC_OK;
}

void* dpc_dev_alloc(dpc_ctx* c, size_t bytes) {
  if (!c) return nullptr;
  void* p = nullptr;
  cudaSetDevice(c->device);
  if (cudaMalloc(&p, bytes ? bytes : 1) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void dpc_dev_free(dpc_ctx* c, void* p) {
  if (c && p) {
    cudaStreamSynchronize(c->stream);
    cudaFree(p);
  }
}

void* dpc_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void dpc_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

dpc_status dpc_copy_h2d(dpc_ctx* c, void* dst, const void* src, size_t bytes) {
  if (!c) return fail(DPC_E_INVALID, "ctx is NULL");
  DPC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
  DPC_CUDA(cudaStreamSynchronize(c->stream));
  return DPC_OK;
}

dpc_status dpc_dev_memset(dpc_ctx* c, void* dst, int32_t value, size_t bytes) {
  if (!c) return fail(DPC_E_INVALID, "ctx is NULL");
  DPC_CUDA(cudaMemsetAsync(dst, value, bytes, c->stream));
  return DPC_OK;
}

dpc_status dpc_copy_d2h(dpc_ctx* c, void* dst, const void* src, size_t bytes) {
  if (!c) return fail(DPC_E_INVALID, "ctx is NULL");
  DPC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
  DPC_CUDA(cudaStreamSynchronize(c->stream));
  return DPC_OK;
}

// ---------------- device-resident graph ----------------

void dpc_dgraph_free(dpc_dgraph* g) {
  if (!g) return;
  if (g->ctx) {
    cudaSetDevice(g->ctx->device);
    cudaStreamSynchronize(g->ctx->stream);
  }
  void* bufs[] = {g->rowptr, g->col,      g->w,        g->val,   g->x,    g->y,
                  g->dist,   g->color,    g->front[0], g->front[1], g->stamp, g->hdr,
                  g->items, g->ctr, g->gc_state, g->soff, g->xhot_col, g->xhot_val,
                  g->ms_rdist, g->ms_send, g->ms_recv, g->ms_cnt, g->gc_q, g->gc_hstate, g->trace, g->gc_hcol, g->gc_hsplit,
                  g->x2, g->y2, g->sst_items, g->plan_mask, g->plan_sin, g->plan_segrow, g->plan_bar,
                  g->plan8, g->plan8_segrow, g->plan8h_col, g->plan8h_hot, g->plan8h_xh, g->gc_prio, g->batch_buf, g->sssp_fbe};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (g->ms_state) dpc::sssp_state_free(g->ms_state);
  if (g->hdr_host) cudaFreeHost(g->hdr_host);
  if (g->ctr_host) cudaFreeHost(g->ctr_host);
  delete g;
}

dpc_status dpc_dgraph_upload(dpc_ctx* c, const dpc_csr* h, dpc_dgraph** out) {
  clear_error();
  if (!c || !out) return fail(DPC_E_INVALID, "NULL argument");
  dpc_status st = dpc_csr_validate(h);
  if (st != DPC_OK) return st;
  if (h->m >= (int64_t{1} << 32)) return fail(DPC_E_INVALID, "edgeCount must be < 2^32 on device");
  auto* g = new (std::nothrow) dpc_dgraph();
  if (!g) return fail(DPC_E_OOM, "dgraph allocation failed");
  g->ctx = c;
  g->n = h->n;
  g->m = h->m;
  g->ncols = h->ncols ? h->ncols : h->n;
  const size_t n = static_cast<size_t>(h->n), m = static_cast<size_t>(h->m);
  const size_t nx = std::max<size_t>(static_cast<size_t>(g->ncols), 1);
  auto cleanup = [&](cudaError_t e, const char* w) {
    dpc_dgraph_free(g);
    return cuda_fail(e, w);
  };
  cudaError_t e;
  std::vector<unsigned> rp32(n + 1);
  g->host_rowptr.assign(h->rowptr, h->rowptr + n + 1);
  for (size_t i = 0; i <= n; i++) rp32[i] = static_cast<unsigned>(h->rowptr[i]);
  for (size_t i = 0; i < n; i++) g->max_deg = std::max<int64_t>(g->max_deg, h->rowptr[i + 1] - h->rowptr[i]);
  const size_t nv = std::max<size_t>(n, 1), mv = std::max<size_t>(m, 1);
  if ((e = cudaMalloc(&g->rowptr, sizeof(unsigned) * (n + 1))) != cudaSuccess) return cleanup(e, "cudaMalloc rowptr");
  if ((e = cudaMalloc(&g->col, sizeof(int) * (mv + 4))) != cudaSuccess) return cleanup(e, "cudaMalloc col");
  if (h->w && (e = cudaMalloc(&g->w, sizeof(int) * (mv + 4))) != cudaSuccess) return cleanup(e, "cudaMalloc w");
  if (h->val && (e = cudaMalloc(&g->val, sizeof(float) * (mv + 4))) != cudaSuccess) return cleanup(e, "cudaMalloc val");
  if ((e = cudaMalloc(&g->x, sizeof(float) * nx)) != cudaSuccess) return cleanup(e, "cudaMalloc x");
  if ((e = cudaMalloc(&g->y, sizeof(float) * nv)) != cudaSuccess) return cleanup(e, "cudaMalloc y");
  if ((e = cudaMalloc(&g->dist, sizeof(unsigned) * nv)) != cudaSuccess) return cleanup(e, "cudaMalloc dist");
  if ((e = cudaMalloc(&g->color, sizeof(int) * nv)) != cudaSuccess) return cleanup(e, "cudaMalloc color");
  if ((e = cudaMalloc(&g->front[0], sizeof(unsigned) * nv)) != cudaSuccess) return cleanup(e, "cudaMalloc front");
  if ((e = cudaMalloc(&g->front[1], sizeof(unsigned) * nv)) != cudaSuccess) return cleanup(e, "cudaMalloc front");
  if ((e = cudaMalloc(&g->stamp, sizeof(unsigned) * nv)) != cudaSuccess) return cleanup(e, "cudaMalloc stamp");
  if ((e = cudaMalloc(&g->hdr, sizeof(RunHeader) * 2)) != cudaSuccess) return cleanup(e, "cudaMalloc hdr");
  if ((e = cudaMallocHost(&g->hdr_host, sizeof(RunHeader) * 2)) != cudaSuccess) return cleanup(e, "cudaMallocHost hdr");
  cudaStream_t s = c->stream;
  e = cudaMemcpyAsync(g->rowptr, rp32.data(), sizeof(unsigned) * (n + 1), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && m) e = cudaMemcpyAsync(g->col, h->col, sizeof(int) * m, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && m && h->w) e = cudaMemcpyAsync(g->w, h->w, sizeof(int) * m, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && m && h->val) e = cudaMemcpyAsync(g->val, h->val, sizeof(float) * m, cudaMemcpyHostToDevice, s);
  // 16 bytes of zero padding past the last nonzero: vector loads of the last
  // aligned group may touch it (stream_drain widens rows to 16 bytes)
  if (e == cudaSuccess) e = cudaMemsetAsync(g->col + m, 0, 4 * sizeof(int), s);
  if (e == cudaSuccess && g->w) e = cudaMemsetAsync(g->w + m, 0, 4 * sizeof(int), s);
  if (e == cudaSuccess && g->val) e = cudaMemsetAsync(g->val + m, 0, 4 * sizeof(float), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(g->x, 0, sizeof(float) * nx, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(g->y, 0, sizeof(float) * nv, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(g->hdr, 0, sizeof(RunHeader) * 2, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cleanup(e, "dpc_dgraph_upload copy");
  *out = g;
  return DPC_OK;
}

dpc_status dpc_dgraph_phase_ns(dpc_dgraph* g, uint64_t out[3]) {
  if (!g || !out) return fail(DPC_E_INVALID, "NULL argument");
  for (int i = 0; i < 3; i++) out[i] = g->hdr_host->t[i];
  return DPC_OK;
}

dpc_status dpc_dgraph_trace(dpc_dgraph* g, uint64_t* out, int64_t n) {
  if (!g || !out || n < 0 || n > 3 * g->n) return fail(DPC_E_INVALID, "bad arguments");
  if (!g->trace) return fail(DPC_E_INVALID, "no traced run (set DPC_TRACE=1)");
  DPC_CUDA(cudaMemcpy(out, g->trace, sizeof(uint64_t) * static_cast<size_t>(n), cudaMemcpyDeviceToHost));
  return DPC_OK;
}

float* dpc_dgraph_x(dpc_dgraph* g) { return g ? g->x : nullptr; }
float* dpc_dgraph_y(dpc_dgraph* g) { return g ? g->y : nullptr; }
uint32_t* dpc_dgraph_dist(dpc_dgraph* g) { return g ? g->dist : nullptr; }
int32_t* dpc_dgraph_color(dpc_dgraph* g) { return g ? g->color : nullptr; }

// ---------------- host-buffer runs ----------------

dpc_status dpc_spmv_host(dpc_ctx* c, dpc_dgraph* g, const float* x, float* y,
                         const dpc_launch_cfg* cfg, dpc_metrics* met) {
  clear_error();
  if (!c || !g || !x || !y) return fail(DPC_E_INVALID, "NULL argument");
  const size_t xbytes = sizeof(float) * static_cast<size_t>(g->ncols);
  const size_t ybytes = sizeof(float) * static_cast<size_t>(g->n);
  DPC_CUDA(cudaMemcpyAsync(g->x, x, xbytes, cudaMemcpyHostToDevice, c->stream));
  dpc_status st = dpc_spmv_device(c, g, g->x, g->y, cfg, met);
  if (st != DPC_OK) return st;
  DPC_CUDA(cudaMemcpyAsync(y, g->y, ybytes, cudaMemcpyDeviceToHost, c->stream));
  DPC_CUDA(cudaStreamSynchronize(c->stream));
  return flush_check(c, g);  // a device-side fault voids y
}

// Pipelined host-vector SpMV over `count` independent vectors (serving
// form of dpc_spmv_host): two device x / y slots; copy-in on one stream,
// the SpMV on the context stream, copy-out on a third, so vector i+1's
// host->device copy and vector i-1's device->host copy overlap vector i's
// kernel on the two copy engines.  Every vector still crosses PCIe both ways.
dpc_status dpc_spmv_host_batch(dpc_ctx* c, dpc_dgraph* g, const float* const* xs, float* const* ys,
                               int64_t count, const dpc_launch_cfg* cfg, dpc_metrics* met) {
  clear_error();
  if (!c || !g || !xs || !ys || count < 0) return fail(DPC_E_INVALID, "bad arguments");
  for (int64_t i = 0; i < count; i++)
    if (!xs[i] || !ys[i]) return fail(DPC_E_INVALID, "NULL vector in batch");
  DPC_CUDA(cudaSetDevice(c->device));
  if (!c->h2d) {
    DPC_CUDA(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
    DPC_CUDA(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    for (auto& ev : c->pev) DPC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  const size_t xbytes = sizeof(float) * static_cast<size_t>(g->ncols);
  const size_t ybytes = sizeof(float) * static_cast<size_t>(g->n);
  if (!g->x2) {
    DPC_CUDA(cudaMalloc(&g->x2, xbytes + 16));
    DPC_CUDA(cudaMalloc(&g->y2, ybytes + 16));
  }
  float* dx[2] = {g->x, g->x2};
  float* dy[2] = {g->y, g->y2};
  // pev: [0,1] x ready  [2,3] x free  [4,5] y ready  [6,7] y free  [8] start
  cudaEvent_t* e = c->pev;
  DPC_CUDA(cudaEventRecord(e[8], c->stream));
  DPC_CUDA(cudaStreamWaitEvent(c->h2d, e[8], 0));
  DPC_CUDA(cudaStreamWaitEvent(c->d2h, e[8], 0));
  for (int64_t i = 0; i < count; i++) {
    const int s = static_cast<int>(i & 1);
    if (i >= 2) DPC_CUDA(cudaStreamWaitEvent(c->h2d, e[2 + s], 0));
    DPC_CUDA(cudaMemcpyAsync(dx[s], xs[i], xbytes, cudaMemcpyHostToDevice, c->h2d));
    DPC_CUDA(cudaEventRecord(e[s], c->h2d));
    DPC_CUDA(cudaStreamWaitEvent(c->stream, e[s], 0));
    if (i >= 2) DPC_CUDA(cudaStreamWaitEvent(c->stream, e[6 + s], 0));
    dpc_status st = dpc_spmv_device(c, g, dx[s], dy[s], cfg, i + 1 == count ? met : nullptr);
    if (st != DPC_OK) {  // no copy may still touch the caller's host vectors
      cudaStreamSynchronize(c->h2d);
      cudaStreamSynchronize(c->d2h);
      return st;
    }
    DPC_CUDA(cudaEventRecord(e[2 + s], c->stream));
    DPC_CUDA(cudaEventRecord(e[4 + s], c->stream));
    DPC_CUDA(cudaStreamWaitEvent(c->d2h, e[4 + s], 0));
    DPC_CUDA(cudaMemcpyAsync(ys[i], dy[s], ybytes, cudaMemcpyDeviceToHost, c->d2h));
    DPC_CUDA(cudaEventRecord(e[6 + s], c->d2h));
  }
  // the context stream (and its timing events) is ordered after the last copy-out
  DPC_CUDA(cudaEventRecord(e[8], c->d2h));
  DPC_CUDA(cudaStreamWaitEvent(c->stream, e[8], 0));
  DPC_CUDA(cudaStreamSynchronize(c->d2h));
  return flush_check(c, g);  // a device-side fault of any vector voids the batch
}

dpc_status dpc_spmv_host_batch_contig(dpc_ctx* c, dpc_dgraph* g, const float* xs, float* ys, int64_t count,
                                      int64_t group, const dpc_launch_cfg* cfg, dpc_metrics* met) {
  clear_error();
  if (!c || !g || (count > 0 && (!xs || !ys)) || count < 0 || group < 0) return fail(DPC_E_INVALID, "bad arguments");
  if (count == 0) return DPC_OK;
  DPC_CUDA(cudaSetDevice(c->device));
  if (!c->h2d) {
    DPC_CUDA(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
    DPC_CUDA(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    for (auto& ev : c->pev) DPC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  const size_t nx = static_cast<size_t>(g->ncols), ny = static_cast<size_t>(g->n);
  const size_t vbytes = sizeof(float) * (nx + ny);
  // default: ~32 MB per copy (config 2, 128-vector batch: 2 / 4 / 8 / 16 / 32
  // vectors per copy -> 0.114 / 0.102 / 0.102 / 0.104 / 0.117 ms per vector;
  // tools/probes/lab_r02/e2e_contig.py)
  int64_t G = group ? group : std::max<int64_t>(1, static_cast<int64_t>((size_t{32} << 20) / std::max<size_t>(vbytes / 2, 1)));
  G = std::min<int64_t>(G, count);
  // two slots of G vectors: x part then y part (16-byte aligned vectors when n, ncols are multiples of 4)
  const size_t slot_x = sizeof(float) * nx * static_cast<size_t>(G), slot_y = sizeof(float) * ny * static_cast<size_t>(G);
  if (g->batch_bytes < 2 * (slot_x + slot_y)) {
    DPC_CUDA(cudaStreamSynchronize(c->stream));
    if (g->batch_buf) cudaFree(g->batch_buf);
    g->batch_buf = nullptr;
    g->batch_bytes = 0;
    DPC_CUDA(cudaMalloc(&g->batch_buf, 2 * (slot_x + slot_y)));
    g->batch_bytes = 2 * (slot_x + slot_y);
  }
  auto* base = static_cast<unsigned char*>(g->batch_buf);
  float* dx[2] = {reinterpret_cast<float*>(base), reinterpret_cast<float*>(base + slot_x)};
  float* dy[2] = {reinterpret_cast<float*>(base + 2 * slot_x), reinterpret_cast<float*>(base + 2 * slot_x + slot_y)};
  // pev: [0,1] x ready  [2,3] x free  [4,5] y ready  [6,7] y free  [8] start
  cudaEvent_t* e = c->pev;
  DPC_CUDA(cudaEventRecord(e[8], c->stream));
  DPC_CUDA(cudaStreamWaitEvent(c->h2d, e[8], 0));
  DPC_CUDA(cudaStreamWaitEvent(c->d2h, e[8], 0));
  const int64_t ngroups = (count + G - 1) / G;
  for (int64_t k = 0; k < ngroups; k++) {
    const int s = static_cast<int>(k & 1);
    const int64_t v0 = k * G, nv = std::min<int64_t>(G, count - v0);
    if (k >= 2) DPC_CUDA(cudaStreamWaitEvent(c->h2d, e[2 + s], 0));
    DPC_CUDA(cudaMemcpyAsync(dx[s], xs + static_cast<size_t>(v0) * nx, sizeof(float) * nx * static_cast<size_t>(nv),
                             cudaMemcpyHostToDevice, c->h2d));
    DPC_CUDA(cudaEventRecord(e[s], c->h2d));
    DPC_CUDA(cudaStreamWaitEvent(c->stream, e[s], 0));
    if (k >= 2) DPC_CUDA(cudaStreamWaitEvent(c->stream, e[6 + s], 0));
    for (int64_t v = 0; v < nv; v++) {
      dpc_status st = dpc_spmv_device(c, g, dx[s] + static_cast<size_t>(v) * nx, dy[s] + static_cast<size_t>(v) * ny,
                                      cfg, (k + 1 == ngroups && v + 1 == nv) ? met : nullptr);
      if (st != DPC_OK) {  // no copy may still touch the caller's host vectors
        cudaStreamSynchronize(c->h2d);
        cudaStreamSynchronize(c->d2h);
        return st;
      }
    }
    DPC_CUDA(cudaEventRecord(e[2 + s], c->stream));
    DPC_CUDA(cudaEventRecord(e[4 + s], c->stream));
    DPC_CUDA(cudaStreamWaitEvent(c->d2h, e[4 + s], 0));
    DPC_CUDA(cudaMemcpyAsync(ys + static_cast<size_t>(v0) * ny, dy[s], sizeof(float) * ny * static_cast<size_t>(nv),
                             cudaMemcpyDeviceToHost, c->d2h));
    DPC_CUDA(cudaEventRecord(e[6 + s], c->d2h));
  }
  DPC_CUDA(cudaEventRecord(e[8], c->d2h));
  DPC_CUDA(cudaStreamWaitEvent(c->stream, e[8], 0));
  DPC_CUDA(cudaStreamSynchronize(c->d2h));
  return flush_check(c, g);  // a device-side fault of any vector voids the batch
}

dpc_status dpc_run_spmv(dpc_ctx* c, const dpc_csr* A, const float* x, float* y,
                        const dpc_launch_cfg* cfg, dpc_metrics* met) {
  clear_error();
  if (!c || !A || !x || !y) return fail(DPC_E_INVALID, "NULL argument");
  if (!A->val) return fail(DPC_E_INVALID, "SpMV needs matrix values (val)");
  dpc_dgraph* g = nullptr;
  dpc_status st = dpc_dgraph_upload(c, A, &g);
  if (st != DPC_OK) return st;
  if (met) std::memset(met, 0, sizeof(*met));
  st = dpc_spmv_host(c, g, x, y, cfg, met);
  dpc_dgraph_free(g);
  return st;
}

dpc_status dpc_run_sssp(dpc_ctx* c, const dpc_csr* G, int32_t source, uint32_t* dist,
                        const dpc_launch_cfg* cfg, dpc_metrics* met) {
  clear_error();
  if (!c || !G || !dist) return fail(DPC_E_INVALID, "NULL argument");
  if (!G->w) return fail(DPC_E_INVALID, "SSSP needs edge weights (w)");
  for (int64_t k = 0; k < G->m; k++)
    if (G->w[k] < 0) return fail(DPC_E_INVALID, "SSSP weights must be >= 0");
  dpc_dgraph* g = nullptr;
  dpc_status st = dpc_dgraph_upload(c, G, &g);
  if (st != DPC_OK) return st;
  if (met) std::memset(met, 0, sizeof(*met));
  st = dpc_sssp_device(c, g, source, cfg, met);
  if (st == DPC_OK) st = flush_check(c, g);  // asynchronous run: its fault check
  if (st == DPC_OK) st = dpc_copy_d2h(c, dist, g->dist, sizeof(unsigned) * static_cast<size_t>(G->n));
  dpc_dgraph_free(g);
  return st;
}

dpc_status dpc_run_bfs(dpc_ctx* c, const dpc_csr* G, int32_t source, uint32_t* level,
                       const dpc_launch_cfg* cfg, dpc_metrics* met) {
  clear_error();
  if (!c || !G || !level) return fail(DPC_E_INVALID, "NULL argument");
  dpc_dgraph* g = nullptr;
  dpc_status st = dpc_dgraph_upload(c, G, &g);
  if (st != DPC_OK) return st;
  if (met) std::memset(met, 0, sizeof(*met));
  st = dpc_bfs_device(c, g, source, cfg, met);
  if (st == DPC_OK) st = flush_check(c, g);
  if (st == DPC_OK) st = dpc_copy_d2h(c, level, g->dist, sizeof(unsigned) * static_cast<size_t>(G->n));
  dpc_dgraph_free(g);
  return st;
}

dpc_status dpc_run_color(dpc_ctx* c, const dpc_csr* G, uint64_t seed, int32_t* color,
                         int32_t* ncolors, const dpc_launch_cfg* cfg, dpc_metrics* met) {
  clear_error();
  if (!c || !G || !color) return fail(DPC_E_INVALID, "NULL argument");
  dpc_dgraph* g = nullptr;
  dpc_status st = dpc_dgraph_upload(c, G, &g);
  if (st != DPC_OK) return st;
  dpc_metrics local{};
  dpc_metrics* mp = met ? met : &local;
  std::memset(mp, 0, sizeof(*mp));
  st = dpc_color_device(c, g, seed, cfg, mp);
  if (st == DPC_OK) st = flush_check(c, g);
  if (st == DPC_OK) st = dpc_copy_d2h(c, color, g->color, sizeof(int) * static_cast<size_t>(G->n));
  if (st == DPC_OK) {
    // Jones-Plassmann counts down higher-priority neighbours through the
    // reverse arcs: an uncolored vertex means the input was not symmetric.
    for (int64_t v = 0; v < G->n; v++)
      if (color[v] < 0) {
        st = fail(DPC_E_INVALID, "coloring needs a symmetric graph (vertex " + std::to_string(v) +
                                     " has an arc without its reverse)");
        break;
      }
  }
  if (st == DPC_OK && ncolors) *ncolors = mp->result_count;
  dpc_dgraph_free(g);
  return st;
}

static dpc_status run_tree(dpc_ctx* c, const dpc_tree* t, int which, int32_t* out,
                           const dpc_launch_cfg* cfg, dpc_metrics* met) {
  clear_error();
  if (!c || !t || !out) return fail(DPC_E_INVALID, "NULL argument");
  dpc_dtree* d = nullptr;
  dpc_status st = dpc_dtree_upload(c, t, &d);
  if (st != DPC_OK) return st;
  if (met) std::memset(met, 0, sizeof(*met));
  st = dpc_tree_device(c, d, which, cfg, met);
  if (st == DPC_OK) st = dpc_dtree_check(c, d);  // asynchronous run: its fault check
  if (st == DPC_OK) st = dpc_copy_d2h(c, out, d->result, sizeof(int) * static_cast<size_t>(t->n));
  dpc_dtree_free(d);
  return st;
}

dpc_status dpc_run_tree_desc(dpc_ctx* c, const dpc_tree* t, int32_t* desc,
                             const dpc_launch_cfg* cfg, dpc_metrics* met) {
  return run_tree(c, t, DPC_APP_TREE_DESC, desc, cfg, met);
}

dpc_status dpc_run_tree_height(dpc_ctx* c, const dpc_tree* t, int32_t* height,
                               const dpc_launch_cfg* cfg, dpc_metrics* met) {
  return run_tree(c, t, DPC_APP_TREE_HEIGHT, height, cfg, met);
}

}  // extern "C"
