// SpMV y = A x (fp32, CSR) in five variants — the irregular-loop app of
// PAPER.md:79-88 with "neighbors" = the nonzeros of a row.
//
//   flat   : thread per row, serial loop (the paper's no-dp)
//   basic  : thread per row; rows with deg > threshold launch
//            child<<<ceil(deg/T), T>>> via CDP2 (Fig. 1(a)/(b))
//   warp   : heavy rows -> chunk items in a warp-owned pool slice; one child
//            launch per warp by the first inserting lane (transform.hpp:729-735)
//   block  : block-owned slice, __syncthreads, thread 0 launches
//            (transform.hpp:736-744)
//   grid   : global worklist + last-block election -> one child launch
//            (transform.hpp:745-777; sim.hpp:1708-1717), or one persistent
//            cooperative kernel with a device-wide barrier between the insert
//            and drain phases (PAPER.md:244-250 custom global barrier).
//
// The consolidated child (drain_loop MultiBlock, transform.hpp:564-598) is
// replaced by a load-balanced drain: heavy rows are split at insertion into
// chunk items of <= `chunk` nonzeros, and the child maps one warp per item with
// 16-byte vector loads of col/val.  Partial sums of a row's
// chunks are combined with fp32 atomics into y[row] (zeroed by the parent).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "ctx.h"

namespace cg = cooperative_groups;

namespace dpc {
namespace spmv {

using dev::Item;
using dev::kFull;
using dev::Pool;
using dev::RunHeader;

struct Args {
  const unsigned* __restrict__ rowptr;
  const int* __restrict__ col;
  const float* __restrict__ val;
  const float* __restrict__ x;
  float* __restrict__ y;
  unsigned n;
  Pool pool;
  RunHeader* hdr;
  unsigned threshold;
  unsigned chunk;
  unsigned child_threads;
  unsigned child_blocks;  // cap, 0 = none
};

__device__ __forceinline__ int4 ldg_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// Thread-serial row sum (flat variant and the parents' inline "work").
// Blocked 4-way accumulation keeps fp32 error ~(256 + len/256) ulp.
__device__ __forceinline__ float row_serial(const Args& a, unsigned b, unsigned e) {
  float total = 0.f;
  for (unsigned blk = b; blk < e; blk += 256) {
    unsigned be = min(e, blk + 256);
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    unsigned k = blk;
    for (; k + 3 < be; k += 4) {
      s0 += __ldg(a.val + k) * __ldg(a.x + __ldg(a.col + k));
      s1 += __ldg(a.val + k + 1) * __ldg(a.x + __ldg(a.col + k + 1));
      s2 += __ldg(a.val + k + 2) * __ldg(a.x + __ldg(a.col + k + 2));
      s3 += __ldg(a.val + k + 3) * __ldg(a.x + __ldg(a.col + k + 3));
    }
    for (; k < be; k++) s0 += __ldg(a.val + k) * __ldg(a.x + __ldg(a.col + k));
    total += (s0 + s1) + (s2 + s3);
  }
  return total;
}

// Warp-cooperative dot of nonzeros [b, e): scalar head to 16-byte alignment,
// int4/float4 body, scalar tail; returns the warp total in every lane.
__device__ __forceinline__ float warp_range_dot(const Args& a, unsigned b, unsigned e) {
  const unsigned lane = dev::lane_id();
  float s = 0.f;
  const unsigned al = min(e, (b + 3u) & ~3u);
  if (b + lane < al) {
    unsigned k = b + lane;
    s = __ldg(a.val + k) * __ldg(a.x + __ldg(a.col + k));
  }
  const unsigned nv = (e - al) >> 2;
  const int4* c4 = reinterpret_cast<const int4*>(a.col + al);
  const float4* v4 = reinterpret_cast<const float4*>(a.val + al);
  float s1 = 0.f;
  unsigned j = lane;
  for (; j + 32 < nv; j += 64) {
    int4 c0 = ldg_stream(c4 + j), c1 = ldg_stream(c4 + j + 32);
    float4 v0 = ldg_stream(v4 + j), v1 = ldg_stream(v4 + j + 32);
    s += v0.x * __ldg(a.x + c0.x) + v0.y * __ldg(a.x + c0.y) + v0.z * __ldg(a.x + c0.z) +
         v0.w * __ldg(a.x + c0.w);
    s1 += v1.x * __ldg(a.x + c1.x) + v1.y * __ldg(a.x + c1.y) + v1.z * __ldg(a.x + c1.z) +
          v1.w * __ldg(a.x + c1.w);
  }
  if (j < nv) {
    int4 c0 = ldg_stream(c4 + j);
    float4 v0 = ldg_stream(v4 + j);
    s += v0.x * __ldg(a.x + c0.x) + v0.y * __ldg(a.x + c0.y) + v0.z * __ldg(a.x + c0.z) +
         v0.w * __ldg(a.x + c0.w);
  }
  const unsigned t = al + (nv << 2);
  if (t + lane < e) {
    unsigned k = t + lane;
    s1 += __ldg(a.val + k) * __ldg(a.x + __ldg(a.col + k));
  }
  return dev::warp_sum(s + s1);
}

// Drains chunk items [0, count) with one warp per item (grid-stride).
__device__ __forceinline__ void drain_items(const Args& a, const Item* items, unsigned count,
                                            unsigned gwarp, unsigned nwarps) {
  for (unsigned i = gwarp; i < count; i += nwarps) {
    Item it = items[i];
    unsigned e = min(it.begin + a.chunk, __ldg(a.rowptr + it.v + 1));
    float s = warp_range_dot(a, it.begin, e);
    if (dev::lane_id() == 0) atomicAdd(a.y + it.v, s);
  }
}

// <child>_cons: the consolidated child kernel (buffer-draining form).
__global__ void __launch_bounds__(256) cons_child(Args a, const Item* items, unsigned count) {
  const unsigned nw = (gridDim.x * blockDim.x) >> 5;
  const unsigned gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  drain_items(a, items, count, gw, nw);
}

__global__ void __launch_bounds__(256) flat_kernel(Args a) {
  unsigned row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row < a.n) a.y[row] = row_serial(a, __ldg(a.rowptr + row), __ldg(a.rowptr + row + 1));
}

// Fig. 1 basic-dp child: one nonzero per thread, block reduction, one atomic.
__global__ void __launch_bounds__(256) basic_child(Args a, unsigned row, unsigned b, unsigned e) {
  __shared__ float s_part[32];
  unsigned k = b + blockIdx.x * blockDim.x + threadIdx.x;
  float v = k < e ? __ldg(a.val + k) * __ldg(a.x + __ldg(a.col + k)) : 0.f;
  v = dev::warp_sum(v);
  if (dev::lane_id() == 0) s_part[dev::warp_in_block()] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? s_part[threadIdx.x] : 0.f;
    t = dev::warp_sum(t);
    if (threadIdx.x == 0) atomicAdd(a.y + row, t);
  }
}

__global__ void __launch_bounds__(256) basic_parent(Args a) {
  unsigned row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= a.n) return;
  unsigned b = __ldg(a.rowptr + row), e = __ldg(a.rowptr + row + 1);
  if (e - b > a.threshold) {
    a.y[row] = 0.f;
    basic_child<<<dev::ceil_div(e - b, a.child_threads), a.child_threads, 0,
                  cudaStreamFireAndForget>>>(a, row, b, e);
    dev::note_launch(a.hdr);
  } else {
    a.y[row] = row_serial(a, b, e);
  }
}

// Common parent prework for the consolidated variants: inline light rows,
// zero heavy rows' y, return how many chunk items this thread inserts.
__device__ __forceinline__ unsigned parent_prework(const Args& a, unsigned row, unsigned* b,
                                                   unsigned* e) {
  if (row >= a.n) return 0;
  *b = __ldg(a.rowptr + row);
  *e = __ldg(a.rowptr + row + 1);
  if (*e - *b > a.threshold) {
    a.y[row] = 0.f;
    return dev::nchunks(*e - *b, a.chunk);
  }
  a.y[row] = row_serial(a, *b, *e);
  return 0;
}

__device__ __forceinline__ unsigned clamp_count(const Args& a, unsigned base, unsigned total) {
  if (base >= a.pool.cap) return 0;
  return min(total, a.pool.cap - base);
}

__global__ void __launch_bounds__(256) warp_parent(Args a) {
  unsigned row = blockIdx.x * blockDim.x + threadIdx.x, b = 0, e = 0;
  unsigned want = parent_prework(a, row, &b, &e);
  unsigned wbase, wtotal;
  unsigned at = dev::warp_reserve(&a.hdr->count, want, &wbase, &wtotal);
  if (want) {
    dev::write_chunks(a.pool, a.hdr, at, row, b, e, a.chunk);
    __threadfence();
  }
  if (wtotal) {
    unsigned leader = __ffs(__ballot_sync(kFull, want != 0)) - 1;  // a live inserting lane
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
}

__global__ void __launch_bounds__(256) block_parent(Args a) {
  __shared__ unsigned s_base;
  unsigned row = blockIdx.x * blockDim.x + threadIdx.x, b = 0, e = 0;
  unsigned want = parent_prework(a, row, &b, &e);
  unsigned btotal;
  unsigned off = dev::block_excl_scan(want, &btotal);
  if (threadIdx.x == 0 && btotal) s_base = atomicAdd(&a.hdr->count, btotal);
  __syncthreads();
  if (want) {
    dev::write_chunks(a.pool, a.hdr, s_base + off, row, b, e, a.chunk);
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0 && btotal) {
    unsigned cnt = clamp_count(a, s_base, btotal);
    if (cnt) {
      cons_child<<<dev::child_blocks(cnt, a.child_threads, a.child_blocks), a.child_threads, 0,
                   cudaStreamFireAndForget>>>(a, a.pool.items + s_base, cnt);
      dev::note_launch(a.hdr);
    }
  }
}

__global__ void __launch_bounds__(256) grid_parent(Args a) {
  unsigned row = blockIdx.x * blockDim.x + threadIdx.x, b = 0, e = 0;
  unsigned want = parent_prework(a, row, &b, &e);
  unsigned wbase, wtotal;
  unsigned at = dev::warp_reserve(&a.hdr->count, want, &wbase, &wtotal);
  if (want) {
    dev::write_chunks(a.pool, a.hdr, at, row, b, e, a.chunk);
    __threadfence();
  }
  if (dev::grid_last_block(&a.hdr->ticket) && threadIdx.x == 0) {
    unsigned cnt = min(*reinterpret_cast<volatile unsigned*>(&a.hdr->count), a.pool.cap);
    if (cnt) {
      cons_child<<<dev::child_blocks(cnt, a.child_threads, a.child_blocks), a.child_threads, 0,
                   cudaStreamFireAndForget>>>(a, a.pool.items, cnt);
      dev::note_launch(a.hdr);
    }
  }
}

// Grid-level consolidation as one persistent cooperative kernel: insert
// phase, device-wide barrier, drain phase.  Zero device launches.
__global__ void __launch_bounds__(256) grid_persistent(Args a) {
  cg::grid_group grid = cg::this_grid();
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned base = blockIdx.x * blockDim.x; base < a.n; base += stride) {
    unsigned row = base + threadIdx.x, b = 0, e = 0;
    unsigned want = parent_prework(a, row, &b, &e);
    unsigned wbase, wtotal;
    unsigned at = dev::warp_reserve(&a.hdr->count, want, &wbase, &wtotal);
    if (want) dev::write_chunks(a.pool, a.hdr, at, row, b, e, a.chunk);
  }
  grid.sync();
  unsigned cnt = min(*reinterpret_cast<volatile unsigned*>(&a.hdr->count), a.pool.cap);
  drain_items(a, a.pool.items, cnt, (blockIdx.x * blockDim.x + threadIdx.x) >> 5, stride >> 5);
}

}  // namespace spmv

static int coop_blocks(dpc_ctx* ctx, const void* fn, int threads) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0) != cudaSuccess) {
    cudaGetLastError();
    per_sm = 1;
  }
  return std::max(1, per_sm) * ctx->sms;
}

}  // namespace dpc

using namespace dpc;

extern "C" dpc_status dpc_spmv_device(dpc_ctx* ctx, dpc_dgraph* g, const float* d_x, float* d_y,
                                      const dpc_launch_cfg* cfg, dpc_metrics* met) {
  clear_error();
  if (!ctx || !g || !d_x || !d_y) return fail(DPC_E_INVALID, "NULL argument");
  if (g->m > 0 && !g->val) return fail(DPC_E_INVALID, "graph was uploaded without values (val)");
  Cfg c;
  dpc_status st = resolve_cfg(ctx, DPC_APP_SPMV, cfg, &c);
  if (st != DPC_OK) return st;
  if (c.parent_threads != 256 || c.child_threads > 256)
    return fail(DPC_E_INVALID, "SpMV kernels are built for parent_threads = 256, child_threads <= 256");
  spmv::Args a;
  a.rowptr = g->rowptr;
  a.col = g->col;
  a.val = g->val;
  a.x = d_x;
  a.y = d_y;
  a.n = static_cast<unsigned>(g->n);
  a.hdr = g->hdr;
  a.threshold = c.threshold;
  a.chunk = c.chunk;
  a.child_threads = c.child_threads;
  a.child_blocks = c.child_blocks;
  if (c.variant != DPC_FLAT && c.variant != DPC_BASIC) {
    st = ensure_pool(g, pool_need(g, c.threshold, c.chunk));
    if (st != DPC_OK) return st;
  }
  a.pool = dev::Pool{g->items, g->cap};
  st = ensure_pending_for(ctx, g, c.variant, c.threshold, c.parent_threads);
  if (st != DPC_OK) return st;
  st = begin_run(ctx, g->hdr);
  if (st != DPC_OK) return st;
  const unsigned blocks = std::max(1u, dev::ceil_div(a.n, 256u));
  cudaStream_t s = ctx->stream;
  if (a.n > 0) {
    switch (c.variant) {
      case DPC_FLAT: spmv::flat_kernel<<<blocks, 256, 0, s>>>(a); break;
      case DPC_BASIC: spmv::basic_parent<<<blocks, 256, 0, s>>>(a); break;
      case DPC_WARP: spmv::warp_parent<<<blocks, 256, 0, s>>>(a); break;
      case DPC_BLOCK: spmv::block_parent<<<blocks, 256, 0, s>>>(a); break;
      case DPC_GRID:
        if (c.grid_persistent) {
          int nb = coop_blocks(ctx, reinterpret_cast<const void*>(spmv::grid_persistent), 256);
          void* args[] = {&a};
          DPC_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(spmv::grid_persistent),
                                               dim3(nb), dim3(256), args, 0, s));
        } else {
          spmv::grid_parent<<<blocks, 256, 0, s>>>(a);
        }
        break;
    }
    DPC_CUDA(cudaGetLastError());
  }
  if (met) {
    met->host_launches += 1;
    met->edges_processed += g->m;
    met->iterations += 1;
    return finish_metrics(ctx, g->hdr, g->hdr_host, met);
  }
  return DPC_OK;
}
