// SSSP (integer weights, uint32 distances) in five variants — the paper's
// Fig. 1(b) irregular loop: each frontier vertex relaxes its
// out-edges inline when deg <= threshold, otherwise the edges become child
// work (a CDP2 child per vertex in basic-dp, consolidated chunk items in the
// warp / block / grid variants).
//
// Algorithm: data-driven Bellman-Ford.  Iteration i relaxes the out-edges of
// every vertex in frontier F_i with atomicMin on dist[]; a vertex whose
// distance drops is appended once (stamp dedup) to F_{i+1}.  Distances reach
// the unique fixpoint = shortest distances, so every variant and every
// schedule is bit-exact against Dijkstra (oracle/oracle.c).
//
// Iteration control: flat / basic / warp / block / grid-CDP run one parent
// grid per iteration from a host loop that reads |F_{i+1}| (device children
// complete before the parent grid does, so the stream order is the barrier).
// The persistent grid variant runs all iterations inside one cooperative
// kernel: insert phase, device-wide barrier, drain phase, barrier — the
// paper's custom global barrier with zero launches.
//
// Frontier appends go through a shared-memory BlockQueue and reach the
// global frontier with one atomic per block (same-address global atomics
// serialise at ~0.7 ns each, tools/probes/atomics_sync).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "ctx.h"

namespace cg = cooperative_groups;

namespace dpc {
namespace sssp {

using dev::Item;
using dev::kFull;
using dev::Pool;
using dev::RunHeader;

constexpr unsigned kInf = 0xffffffffu;
constexpr unsigned kQueue = 2048;  // shared-memory frontier queue per block
using Queue = dev::BlockQueue<kQueue>;

// Per-iteration counters (device): frontier sizes and pool bump pointers,
// triple-buffered by iteration so no reset has to race a reader.
struct Ctr {
  unsigned fsize[3];
  unsigned pool[3];
  unsigned iters;
  unsigned pad[9];
};

struct Args {
  const unsigned* __restrict__ rowptr;
  const int* __restrict__ col;
  const int* __restrict__ w;
  unsigned* dist;
  unsigned* stamp;
  unsigned* front0;
  unsigned* front1;
  Ctr* ctr;
  Pool pool;
  RunHeader* hdr;
  unsigned n;
  unsigned threshold;
  unsigned chunk;
  unsigned child_threads;
  unsigned child_blocks;
  unsigned it;     // iteration index (host-loop variants)
  unsigned fsize;  // |F_it| (host-loop variants)
};

// Per-block state every relaxing kernel carries in shared memory.
struct Block {
  Queue q;
  unsigned long long work;
};

__device__ __forceinline__ unsigned* cur_front(const Args& a, unsigned it) {
  return (it & 1) ? a.front1 : a.front0;
}
__device__ __forceinline__ unsigned* next_front(const Args& a, unsigned it) {
  return (it & 1) ? a.front0 : a.front1;
}
__device__ __forceinline__ unsigned* next_count(const Args& a, unsigned it) {
  return &a.ctr->fsize[(it + 1) % 3];
}

__device__ __forceinline__ void block_begin(Block& s) {
  s.q.init();
  if (threadIdx.x == 0) s.work = 0;
  __syncthreads();
}

// Publishes the block's frontier appends and edge count.  All threads call.
__device__ __forceinline__ void block_end(const Args& a, unsigned it, Block& s) {
  s.q.flush(next_count(a, it), next_front(a, it));
  if (threadIdx.x == 0 && s.work) {
    atomicAdd(&a.hdr->work, s.work);
    s.work = 0;
  }
  __syncthreads();
}

__device__ __forceinline__ void relax(const Args& a, unsigned it, Block& s, unsigned v,
                                      unsigned nd) {
  if (nd < __ldcg(a.dist + v)) {
    unsigned old = atomicMin(a.dist + v, nd);
    if (nd < old && atomicExch(a.stamp + v, it + 1) != it + 1)
      s.q.push(v, next_count(a, it), next_front(a, it));
  }
}

__device__ __forceinline__ void relax_edge(const Args& a, unsigned it, Block& s, unsigned du,
                                           unsigned k) {
  unsigned long long nd = static_cast<unsigned long long>(du) + static_cast<unsigned>(__ldg(a.w + k));
  if (nd < kInf) relax(a, it, s, static_cast<unsigned>(__ldg(a.col + k)), static_cast<unsigned>(nd));
}

__device__ __forceinline__ void relax_serial(const Args& a, unsigned it, Block& s, unsigned du,
                                             unsigned b, unsigned e) {
  for (unsigned k = b; k < e; k++) relax_edge(a, it, s, du, k);
}

// Warp-cooperative relaxation of edges [b, e) of a vertex at distance du.
__device__ __forceinline__ void relax_warp(const Args& a, unsigned it, Block& s, unsigned du,
                                           unsigned b, unsigned e) {
  for (unsigned k = b + dev::lane_id(); k < e; k += 32) relax_edge(a, it, s, du, k);
}

__device__ __forceinline__ void drain_items(const Args& a, unsigned it, Block& s, const Item* items,
                                            unsigned count, unsigned gwarp, unsigned nwarps) {
  for (unsigned i = gwarp; i < count; i += nwarps) {
    Item t = items[i];
    unsigned e = min(t.begin + a.chunk, __ldg(a.rowptr + t.v + 1));
    unsigned du = __ldcg(a.dist + t.v);
    relax_warp(a, it, s, du, t.begin, e);
  }
}

__global__ void __launch_bounds__(256) init_kernel(Args a, unsigned source) {
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < a.n) {
    a.dist[i] = i == source ? 0u : kInf;
    a.stamp[i] = 0;
  }
  if (i == 0) {
    a.front0[0] = source;
    a.ctr->fsize[0] = 1;
    a.ctr->fsize[1] = a.ctr->fsize[2] = 0;
    a.ctr->pool[0] = a.ctr->pool[1] = a.ctr->pool[2] = 0;
    a.ctr->iters = 0;
  }
}

// Warp-cooperative inline relaxation of the light vertices held by the 32
// lanes (the parent's "else work(item)"): their edges are concatenated and
// swept 32 at a time; each lane locates its edge's vertex by a shuffle binary
// search.  All lanes call; dl = this lane's light degree (0 otherwise).
__device__ __forceinline__ void warp_light_relax(const Args& a, unsigned it, Block& s, unsigned b,
                                                 unsigned du, unsigned dl) {
  const unsigned lane = dev::lane_id();
  const unsigned incl = dev::warp_incl_scan(dl);
  const unsigned total = __shfl_sync(kFull, incl, 31);
  const unsigned lo = incl - dl;
  for (unsigned base = 0; base < total; base += 32) {
    const unsigned j = base + lane;
    unsigned l = 0;
#pragma unroll
    for (unsigned st = 16; st > 0; st >>= 1) {
      unsigned c = l + st;
      if (__shfl_sync(kFull, lo, c) <= j) l = c;
    }
    const unsigned bl = __shfl_sync(kFull, b, l), lol = __shfl_sync(kFull, lo, l);
    const unsigned dul = __shfl_sync(kFull, du, l);
    if (j < total) relax_edge(a, it, s, dul, bl + (j - lol));
  }
}

// Prework shared by the DP parents: returns the vertex's chunk count when its
// edges are child work; light vertices are relaxed inline (warp-cooperative).
// All lanes call.  Adds the vertex degree to the block's work counter.
__device__ __forceinline__ unsigned prework(const Args& a, unsigned it, Block& s, unsigned i,
                                            unsigned fsize, unsigned* u, unsigned* b, unsigned* e,
                                            unsigned* du) {
  unsigned want = 0, dl = 0, deg = 0;
  if (i < fsize) {
    *u = cur_front(a, it)[i];
    *b = __ldg(a.rowptr + *u);
    *e = __ldg(a.rowptr + *u + 1);
    *du = __ldcg(a.dist + *u);
    deg = *e - *b;
    if (deg > a.threshold) want = dev::nchunks(deg, a.chunk);
    else dl = deg;
  }
  dev::block_add_u64(&s.work, deg);
  warp_light_relax(a, it, s, *b, *du, dl);
  return want;
}

__global__ void __launch_bounds__(256) cons_child(Args a, const Item* items, unsigned count) {
  __shared__ Block s;
  block_begin(s);
  drain_items(a, a.it, s, items, count, (blockIdx.x * blockDim.x + threadIdx.x) >> 5,
              (gridDim.x * blockDim.x) >> 5);
  block_end(a, a.it, s);
}

__global__ void __launch_bounds__(256) flat_kernel(Args a) {
  __shared__ Block s;
  block_begin(s);
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned deg = 0;
  if (i < a.fsize) {
    unsigned u = cur_front(a, a.it)[i];
    unsigned b = __ldg(a.rowptr + u), e = __ldg(a.rowptr + u + 1);
    deg = e - b;
    relax_serial(a, a.it, s, __ldcg(a.dist + u), b, e);
  }
  dev::block_add_u64(&s.work, deg);
  block_end(a, a.it, s);
}

// Fig. 1(b) child: one edge per thread.
__global__ void __launch_bounds__(256) basic_child(Args a, unsigned du, unsigned b, unsigned e) {
  __shared__ Block s;
  block_begin(s);
  unsigned k = b + blockIdx.x * blockDim.x + threadIdx.x;
  if (k < e) relax_edge(a, a.it, s, du, k);
  block_end(a, a.it, s);
}

__global__ void __launch_bounds__(256) basic_parent(Args a) {
  __shared__ Block s;
  block_begin(s);
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned deg = 0, b = 0, du = 0, dl = 0;
  if (i < a.fsize) {
    unsigned u = cur_front(a, a.it)[i];
    b = __ldg(a.rowptr + u);
    unsigned e = __ldg(a.rowptr + u + 1);
    du = __ldcg(a.dist + u);
    deg = e - b;
    if (deg > a.threshold) {
      basic_child<<<dev::ceil_div(deg, a.child_threads), a.child_threads, 0,
                    cudaStreamFireAndForget>>>(a, du, b, e);
      dev::note_launch(a.hdr);
    } else {
      dl = deg;
    }
  }
  dev::block_add_u64(&s.work, deg);
  warp_light_relax(a, a.it, s, b, du, dl);
  block_end(a, a.it, s);
}

__device__ __forceinline__ unsigned clamp_count(const Args& a, unsigned base, unsigned total) {
  if (base >= a.pool.cap) return 0;
  return min(total, a.pool.cap - base);
}

__global__ void __launch_bounds__(256) warp_parent(Args a) {
  __shared__ Block s;
  block_begin(s);
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x, u = 0, b = 0, e = 0, du = 0;
  unsigned want = prework(a, a.it, s, i, a.fsize, &u, &b, &e, &du);
  unsigned bbase, btotal;
  unsigned at = dev::block_reserve(&a.ctr->pool[a.it % 3], want, &bbase, &btotal);
  if (want) {
    dev::write_chunks(a.pool, a.hdr, at, u, b, e, a.chunk);
    __threadfence();
  }
  const unsigned wbase = __shfl_sync(kFull, at, 0), wtotal = dev::warp_sum(want);
  if (wtotal) {
    unsigned leader = __ffs(__ballot_sync(kFull, want != 0)) - 1;
    __syncwarp();
    if (dev::lane_id() == leader) {
      unsigned cnt = clamp_count(a, wbase, wtotal);
      if (cnt) {
        cons_child<<<dev::child_blocks(cnt, a.child_threads, a.child_blocks), a.child_threads, 0,
                     cudaStreamFireAndForget>>>(a, a.pool.items + wbase, cnt);
        dev::note_launch(a.hdr);
      }
    }
  }
  block_end(a, a.it, s);
}

__global__ void __launch_bounds__(256) block_parent(Args a) {
  __shared__ Block s;
  block_begin(s);
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x, u = 0, b = 0, e = 0, du = 0;
  unsigned want = prework(a, a.it, s, i, a.fsize, &u, &b, &e, &du);
  unsigned bbase, btotal;
  unsigned at = dev::block_reserve(&a.ctr->pool[a.it % 3], want, &bbase, &btotal);
  if (want) {
    dev::write_chunks(a.pool, a.hdr, at, u, b, e, a.chunk);
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0 && btotal) {
    unsigned cnt = clamp_count(a, bbase, btotal);
    if (cnt) {
      cons_child<<<dev::child_blocks(cnt, a.child_threads, a.child_blocks), a.child_threads, 0,
                   cudaStreamFireAndForget>>>(a, a.pool.items + bbase, cnt);
      dev::note_launch(a.hdr);
    }
  }
  block_end(a, a.it, s);
}

__global__ void __launch_bounds__(256) grid_parent(Args a) {
  __shared__ Block s;
  block_begin(s);
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x, u = 0, b = 0, e = 0, du = 0;
  unsigned want = prework(a, a.it, s, i, a.fsize, &u, &b, &e, &du);
  unsigned bbase, btotal;
  unsigned at = dev::block_reserve(&a.ctr->pool[a.it % 3], want, &bbase, &btotal);
  if (want) {
    dev::write_chunks(a.pool, a.hdr, at, u, b, e, a.chunk);
    __threadfence();
  }
  block_end(a, a.it, s);  // this block's inline pushes are published first
  if (dev::grid_last_block(&a.hdr->ticket) && threadIdx.x == 0) {
    unsigned cnt = min(*reinterpret_cast<volatile unsigned*>(&a.ctr->pool[a.it % 3]), a.pool.cap);
    if (cnt) {
      cons_child<<<dev::child_blocks(cnt, a.child_threads, a.child_blocks), a.child_threads, 0,
                   cudaStreamFireAndForget>>>(a, a.pool.items, cnt);
      dev::note_launch(a.hdr);
    }
  }
}

// Zeroes the counters of iteration it+2 (== it-1 mod 3: consumed already)
// and records the pool high-water mark.
__device__ __forceinline__ void rotate(const Args& a, unsigned it) {
  unsigned used = a.ctr->pool[it % 3];
  atomicAdd(&a.hdr->aux1, used);
  atomicMax(&a.hdr->count, used);
  a.ctr->fsize[(it + 2) % 3] = 0;
  a.ctr->pool[(it + 2) % 3] = 0;
}

__global__ void __launch_bounds__(32) rotate_kernel(Args a) {
  if (threadIdx.x == 0) rotate(a, a.it);
}

__global__ void __launch_bounds__(256) grid_persistent(Args a, unsigned max_iters) {
  __shared__ Block s;
  cg::grid_group grid = cg::this_grid();
  const unsigned stride = gridDim.x * blockDim.x;
  const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x;
  block_begin(s);
  unsigned it = 0;
  for (; it < max_iters; it++) {
    const unsigned fs = *reinterpret_cast<volatile unsigned*>(&a.ctr->fsize[it % 3]);
    if (fs == 0) break;
    for (unsigned base = blockIdx.x * blockDim.x; base < fs; base += stride) {
      unsigned i = base + threadIdx.x, u = 0, b = 0, e = 0, du = 0;
      unsigned want = prework(a, it, s, i, fs, &u, &b, &e, &du);
      unsigned bbase, btotal;
      unsigned at = dev::block_reserve(&a.ctr->pool[it % 3], want, &bbase, &btotal);
      if (want) dev::write_chunks(a.pool, a.hdr, at, u, b, e, a.chunk);
    }
    grid.sync();
    unsigned cnt = min(*reinterpret_cast<volatile unsigned*>(&a.ctr->pool[it % 3]), a.pool.cap);
    drain_items(a, it, s, a.pool.items, cnt, gtid >> 5, stride >> 5);
    block_end(a, it, s);
    if (gtid == 0) rotate(a, it);
    grid.sync();
  }
  if (gtid == 0) a.ctr->iters = it;
}

}  // namespace sssp

static int coop_blocks_sssp(dpc_ctx* ctx, const void* fn, int threads) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0) != cudaSuccess) {
    cudaGetLastError();
    per_sm = 1;
  }
  return std::max(1, per_sm) * ctx->sms;
}

}  // namespace dpc

using namespace dpc;

extern "C" dpc_status dpc_sssp_device(dpc_ctx* ctx, dpc_dgraph* g, int32_t source,
                                      const dpc_launch_cfg* cfg, dpc_metrics* met) {
  clear_error();
  if (!ctx || !g) return fail(DPC_E_INVALID, "NULL argument");
  if (g->m > 0 && !g->w) return fail(DPC_E_INVALID, "graph was uploaded without weights (w)");
  if (g->ncols != g->n) return fail(DPC_E_INVALID, "SSSP needs a square graph (not a row slice)");
  if (source < 0 || source >= g->n) return fail(DPC_E_INVALID, "source out of range");
  Cfg c;
  dpc_status st = resolve_cfg(ctx, DPC_APP_SSSP, cfg, &c);
  if (st != DPC_OK) return st;
  if (c.parent_threads != 256 || c.child_threads > 256)
    return fail(DPC_E_INVALID, "SSSP kernels are built for parent_threads = 256, child_threads <= 256");
  if (!g->ctr) {
    DPC_CUDA(cudaMalloc(&g->ctr, sizeof(sssp::Ctr)));
    DPC_CUDA(cudaMallocHost(&g->ctr_host, sizeof(sssp::Ctr)));
  }
  sssp::Args a;
  a.rowptr = g->rowptr;
  a.col = g->col;
  a.w = g->w;
  a.dist = g->dist;
  a.stamp = g->stamp;
  a.front0 = g->front[0];
  a.front1 = g->front[1];
  a.ctr = reinterpret_cast<sssp::Ctr*>(g->ctr);
  a.hdr = g->hdr;
  a.n = static_cast<unsigned>(g->n);
  a.threshold = c.threshold;
  a.chunk = c.chunk;
  a.child_threads = c.child_threads;
  a.child_blocks = c.child_blocks;
  a.it = 0;
  a.fsize = 1;
  if (c.variant != DPC_FLAT && c.variant != DPC_BASIC) {
    st = ensure_pool(g, pool_need(g, c.threshold, c.chunk));
    if (st != DPC_OK) return st;
  }
  a.pool = dev::Pool{g->items, g->cap};
  st = ensure_pending_for(ctx, g, c.variant, c.threshold, c.parent_threads);
  if (st != DPC_OK) return st;
  st = begin_run(ctx, g->hdr);
  if (st != DPC_OK) return st;
  cudaStream_t s = ctx->stream;
  const unsigned nb = std::max(1u, dev::ceil_div(a.n, 256u));
  sssp::init_kernel<<<nb, 256, 0, s>>>(a, static_cast<unsigned>(source));
  DPC_CUDA(cudaGetLastError());
  int64_t host_launches = 1, iters = 0;
  auto* ctr_host = reinterpret_cast<sssp::Ctr*>(g->ctr_host);
  if (c.variant == DPC_GRID && c.grid_persistent) {
    int blocks = coop_blocks_sssp(ctx, reinterpret_cast<const void*>(sssp::grid_persistent), 256);
    unsigned max_iters = a.n + 1;
    void* args[] = {&a, &max_iters};
    DPC_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(sssp::grid_persistent),
                                         dim3(blocks), dim3(256), args, 0, s));
    host_launches += 1;
    DPC_CUDA(cudaMemcpyAsync(ctr_host, a.ctr, sizeof(sssp::Ctr), cudaMemcpyDeviceToHost, s));
    DPC_CUDA(cudaStreamSynchronize(s));
    iters = ctr_host->iters;
  } else {
    unsigned fsize = 1;
    for (unsigned it = 0; fsize > 0 && it <= a.n; it++) {
      a.it = it;
      a.fsize = fsize;
      const unsigned pb = std::max(1u, dev::ceil_div(fsize, 256u));
      switch (c.variant) {
        case DPC_FLAT: sssp::flat_kernel<<<pb, 256, 0, s>>>(a); break;
        case DPC_BASIC: sssp::basic_parent<<<pb, 256, 0, s>>>(a); break;
        case DPC_WARP: sssp::warp_parent<<<pb, 256, 0, s>>>(a); break;
        case DPC_BLOCK: sssp::block_parent<<<pb, 256, 0, s>>>(a); break;
        default: sssp::grid_parent<<<pb, 256, 0, s>>>(a); break;
      }
      sssp::rotate_kernel<<<1, 32, 0, s>>>(a);
      host_launches += 2;
      DPC_CUDA(cudaGetLastError());
      DPC_CUDA(cudaMemcpyAsync(&ctr_host->fsize[(it + 1) % 3], &a.ctr->fsize[(it + 1) % 3],
                               sizeof(unsigned), cudaMemcpyDeviceToHost, s));
      DPC_CUDA(cudaStreamSynchronize(s));
      fsize = ctr_host->fsize[(it + 1) % 3];
      iters = it + 1;
    }
  }
  if (met) {
    met->host_launches += host_launches;
    met->iterations += iters;
    st = finish_metrics(ctx, g->hdr, g->hdr_host, met);
    if (st != DPC_OK) return st;
    met->edges_processed += static_cast<int64_t>(g->hdr_host->work);
    met->buffer_items_inserted = g->hdr_host->aux1;
    return DPC_OK;
  }
  DPC_CUDA(cudaMemcpyAsync(g->hdr_host, g->hdr, sizeof(dev::RunHeader), cudaMemcpyDeviceToHost, s));
  DPC_CUDA(cudaStreamSynchronize(s));
  return check_header(g->hdr_host);
}
