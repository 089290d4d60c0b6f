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

#include <map>
#include <mutex>

#include "common.cuh"
#include "ctx.h"

namespace cg = cooperative_groups;

namespace dpc {
namespace spmv {

using dev::Item;
using dev::kFull;
using dev::Pool;
using dev::RunHeader;

// Timing probes that skip or fake part of the work (wrong results by design:
// no drain, no y store, synthetic columns, confined gathers, parent-only
// phases) exist only in a probe build (-DDPC_TIMING_PROBES=1); the product
// library compiles them out, so no dpc_launch_cfg.flags value reaches them.
#ifndef DPC_TIMING_PROBES
#define DPC_TIMING_PROBES 0
#endif
constexpr bool kProbes = DPC_TIMING_PROBES != 0;

// Resident 256-thread blocks per SM requested from ptxas for the drain
// kernels (latency-bound gathers want warps in flight: 8 -> 64 warps/SM).
#ifndef DPC_SPMV_MIN_BLOCKS
#define DPC_SPMV_MIN_BLOCKS 8
#endif
constexpr int kMinBlocks = DPC_SPMV_MIN_BLOCKS;

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
  unsigned xflags;        // experiment switches (dpc_launch_cfg.flags >> 24), 0 in production
  unsigned coop;          // launched cooperatively (grid.sync) vs normal launch + soft barrier
  // fused multi-GPU SpMV (dpc_multi_spmv_fused): x is distributed, entry i
  // lives on rank i / rows at offset i % rows and is read straight from the
  // owner's memory (NVLink peer loads); nullptr = local x
  const float* const* xpeer;
  float* xpull;           // pull mode: the owners' slices are copied here (= x) before the barrier
  unsigned rshift;        // log2(rows) when rows is a power of two, else ~0u
  unsigned rows;
  unsigned ncols;         // x entries (pull mode)
};

__device__ __forceinline__ float peer_x(const Args& a, unsigned idx) {
  const unsigned o = a.rshift != ~0u ? idx >> a.rshift : idx / a.rows;
  const unsigned l = a.rshift != ~0u ? idx & (a.rows - 1u) : idx - o * a.rows;
  return __ldg(a.xpeer[o] + l);
}

__device__ __forceinline__ float ld_weak_f(const float* p) {
  float r;
  asm volatile("ld.global.ca.f32 %0, [%1];" : "=f"(r) : "l"(p) : "memory");
  return r;
}

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

// Drains chunk items [0, count).  A warp takes a batch of 32 items (one
// descriptor per lane, so the item and rowptr loads are paid once per batch),
// then streams two items at a time with every lane owning two nonzeros of
// each: eight independent loads in flight per lane before the x gathers.
// Per-item overhead is what bounds the drain (most heavy rows are short,
// 33..1024 nonzeros), so it is amortised instead of vectorising the body.
__device__ __forceinline__ void drain_items(const Args& a, const Item* items, unsigned count,
                                            unsigned gwarp, unsigned nwarps) {
  const unsigned lane = dev::lane_id();
  // this warp owns items gwarp, gwarp + nwarps, ... (strided, so the
  // consecutive chunks of one hub row land on different warps)
  const unsigned mine = count > gwarp ? (count - gwarp + nwarps - 1) / nwarps : 0;
  for (unsigned r0 = 0; r0 < mine; r0 += 32) {
    unsigned v = 0, b = 0, e = 0;
    if (r0 + lane < mine) {
      Item t = items[(r0 + lane) * nwarps + gwarp];
      v = t.v;
      b = t.begin;
      e = min(b + a.chunk, __ldg(a.rowptr + v + 1));
    }
    const unsigned nb = min(32u, mine - r0);
    for (unsigned p = 0; p < nb; p += 2) {
      const unsigned q = p + 1 < nb ? p + 1 : p;
      const unsigned v0 = __shfl_sync(kFull, v, p), b0 = __shfl_sync(kFull, b, p);
      const unsigned e0 = __shfl_sync(kFull, e, p);
      const unsigned v1 = __shfl_sync(kFull, v, q), b1 = __shfl_sync(kFull, b, q);
      const unsigned e1 = q != p ? __shfl_sync(kFull, e, q) : b1;
      const unsigned n0 = e0 - b0, n1 = e1 - b1, nm = max(n0, n1);
      float s0 = 0.f, s1 = 0.f;
      for (unsigned o = lane; o < nm; o += 64) {
        const bool p00 = o < n0, p01 = o + 32 < n0, p10 = o < n1, p11 = o + 32 < n1;
        int c00 = 0, c01 = 0, c10 = 0, c11 = 0;
        float w00 = 0.f, w01 = 0.f, w10 = 0.f, w11 = 0.f;
        if (p00) c00 = __ldg(a.col + b0 + o), w00 = __ldg(a.val + b0 + o);
        if (p01) c01 = __ldg(a.col + b0 + o + 32), w01 = __ldg(a.val + b0 + o + 32);
        if (p10) c10 = __ldg(a.col + b1 + o), w10 = __ldg(a.val + b1 + o);
        if (p11) c11 = __ldg(a.col + b1 + o + 32), w11 = __ldg(a.val + b1 + o + 32);
        float x00 = p00 ? __ldg(a.x + c00) : 0.f, x01 = p01 ? __ldg(a.x + c01) : 0.f;
        float x10 = p10 ? __ldg(a.x + c10) : 0.f, x11 = p11 ? __ldg(a.x + c11) : 0.f;
        s0 += w00 * x00 + w01 * x01;
        s1 += w10 * x10 + w11 * x11;
      }
      s0 = dev::warp_sum(s0);
      s1 = dev::warp_sum(s1);
      if (lane == 0) {
        atomicAdd(a.y + v0, s0);
        if (q != p) atomicAdd(a.y + v1, s1);
      }
    }
  }
}

// <child>_cons: the consolidated child kernel (buffer-draining form).
__global__ void __launch_bounds__(256, kMinBlocks) cons_child(Args a, const Item* items,
                                                              unsigned count) {
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

__device__ __forceinline__ float warp_light_rows(const Args& a, unsigned b, unsigned dl);

__global__ void __launch_bounds__(256) basic_parent(Args a) {
  unsigned row = blockIdx.x * blockDim.x + threadIdx.x, b = 0, e = 0, dl = 0;
  bool heavy = false;
  if (row < a.n) {
    b = __ldg(a.rowptr + row);
    e = __ldg(a.rowptr + row + 1);
    heavy = e - b > a.threshold;
    if (!heavy) dl = e - b;
  }
  if (heavy) {
    a.y[row] = 0.f;
    basic_child<<<dev::ceil_div(e - b, a.child_threads), a.child_threads, 0,
                  cudaStreamFireAndForget>>>(a, row, b, e);
    dev::note_launch(a.hdr);
  }
  float s = warp_light_rows(a, b, dl);
  if (row < a.n && !heavy) a.y[row] = s;
}

// Warp-cooperative inline work ("else work(item)" of Fig. 1) for the light
// rows owned by the 32 lanes of a warp.  The lanes' light nonzeros are
// concatenated (heavy rows contribute nothing) and swept 32 at a time: every
// lane finds the row of its element by a 5-step shuffle binary search, the
// products are summed per row with a segmented shuffle scan, and the segment
// head hands the partial to the owning lane.  Same result as the thread's
// serial loop, without the per-thread serial latency chain.  All lanes call;
// `dl` is this lane's light degree (0 for heavy / out-of-range rows).
__device__ __forceinline__ float warp_light_rows(const Args& a, unsigned b, unsigned dl) {
  const unsigned lane = dev::lane_id();
  const unsigned incl = dev::warp_incl_scan(dl);
  const unsigned total = __shfl_sync(kFull, incl, 31);
  const unsigned lo = incl - dl;  // my row's start in the concatenation
  float acc = 0.f;
  for (unsigned base = 0; base < total; base += 32) {
    const unsigned j = base + lane;
    unsigned l = 0;
#pragma unroll
    for (unsigned s = 16; s > 0; s >>= 1) {
      unsigned c = l + s;
      if (__shfl_sync(kFull, lo, c) <= j) l = c;
    }
    const unsigned bl = __shfl_sync(kFull, b, l), lol = __shfl_sync(kFull, lo, l);
    float v = 0.f;
    if (j < total) {
      unsigned k = bl + (j - lol);
      v = __ldg(a.val + k) * __ldg(a.x + __ldg(a.col + k));
    }
    // segmented suffix sum over lanes holding the same row
#pragma unroll
    for (unsigned s = 1; s < 32; s <<= 1) {
      float ov = __shfl_down_sync(kFull, v, s);
      unsigned ol = __shfl_down_sync(kFull, l, s);
      if (lane + s < 32 && ol == l) v += ov;
    }
    // the owner lane picks up its segment's sum from the segment head
    unsigned head = (lo > base ? lo : base) - base;
    bool mine = dl > 0 && lo < base + 32 && lo + dl > base;
    float got = __shfl_sync(kFull, v, head & 31u);
    if (mine) acc += got;
  }
  return acc;
}

__device__ __forceinline__ int ld_stream_i(const int* p) {
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ float ld_stream_f(const float* p) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}

// Segmented dot product over a warp: lane i owns the nonzero segment
// [b_i, b_i + len_i); returns sum(val * x[col]) over lane i's segment.  The
// concatenated segments are swept U*32 elements per step: all U col/val
// loads of a step are issued before any x gather (memory-level parallelism),
// col/val bypass L1 (x keeps it), each element finds its owner with a 5-step
// shuffle binary search and partial sums reach the owner through a segmented
// shuffle reduction.  Balanced however the lengths are distributed.
template <int U>
__device__ __forceinline__ float warp_segments_dot(const Args& a, unsigned b, unsigned len) {
  const unsigned lane = dev::lane_id();
  const unsigned incl = dev::warp_incl_scan(len);
  const unsigned total = __shfl_sync(kFull, incl, 31);
  const unsigned lo = incl - len;
  float acc = 0.f;
  for (unsigned base = 0; base < total; base += 32 * U) {
    unsigned l[U];
    int c[U];
    float w[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const unsigned j = base + u * 32 + lane;
      unsigned s = 0;
#pragma unroll
      for (unsigned st = 16; st > 0; st >>= 1) {
        unsigned cand = s + st;
        if (__shfl_sync(kFull, lo, cand) <= j) s = cand;
      }
      l[u] = s;
      const unsigned k = __shfl_sync(kFull, b, s) + (j - __shfl_sync(kFull, lo, s));
      const bool ok = j < total;
      c[u] = ok ? ld_stream_i(a.col + k) : 0;
      w[u] = ok ? ld_stream_f(a.val + k) : 0.f;
    }
    float p[U];
#pragma unroll
    for (int u = 0; u < U; u++) p[u] = w[u] * __ldg(a.x + c[u]);
#pragma unroll
    for (int u = 0; u < U; u++) {
      float v = p[u];
      const unsigned lu = l[u];
#pragma unroll
      for (unsigned s = 1; s < 32; s <<= 1) {
        float ov = __shfl_down_sync(kFull, v, s);
        unsigned ol = __shfl_down_sync(kFull, lu, s);
        if (lane + s < 32 && ol == lu) v += ov;
      }
      const unsigned j0 = base + u * 32;
      const unsigned first = lo > j0 ? lo : j0;
      const bool mine = len > 0 && lo < j0 + 32 && lo + len > j0;
      const float got = __shfl_sync(kFull, v, (first - j0) & 31u);
      if (mine) acc += got;
    }
  }
  return acc;
}

// Light rows of a 32-row tile through the segmented sweep (4 elements per lane
// per step covers the typical tile in one step).  All lanes call.
__device__ __forceinline__ unsigned parent_prework_stream(const Args& a, unsigned row, unsigned* b,
                                                          unsigned* e) {
  unsigned dl = 0, want = 0;
  if (row < a.n) {
    *b = __ldg(a.rowptr + row);
    *e = __ldg(a.rowptr + row + 1);
    if (*e - *b > a.threshold) {
      a.y[row] = 0.f;
      want = dev::nchunks(*e - *b, a.chunk);
    } else {
      dl = *e - *b;
    }
  }
  float s = warp_segments_dot<4>(a, *b, dl);
  if (row < a.n && !want) a.y[row] = s;
  return want;
}

// Drain through the segmented sweep: a warp's batch of up to 32 items (lane i
// holds item i) is one concatenated stream, 8 elements per lane per step.
__device__ __forceinline__ void drain_items_stream(const Args& a, const Item* items, unsigned count,
                                                   unsigned gwarp, unsigned nwarps) {
  const unsigned lane = dev::lane_id();
  const unsigned mine = count > gwarp ? (count - gwarp + nwarps - 1) / nwarps : 0;
  for (unsigned r0 = 0; r0 < mine; r0 += 32) {
    unsigned v = 0, b = 0, len = 0;
    if (r0 + lane < mine) {
      Item t = items[(r0 + lane) * nwarps + gwarp];
      v = t.v;
      b = t.begin;
      len = min(b + a.chunk, __ldg(a.rowptr + v + 1)) - b;
    }
    float s = warp_segments_dot<8>(a, b, len);
    if (len) atomicAdd(a.y + v, s);
  }
}

// Common parent prework for the DP variants: zero heavy rows' y, do the light
// rows' inline work warp-cooperatively, return how many chunk items this
// thread inserts.  All lanes call.
__device__ __forceinline__ unsigned parent_prework(const Args& a, unsigned row, unsigned* b,
                                                   unsigned* e) {
  unsigned dl = 0, want = 0;
  if (row < a.n) {
    *b = __ldg(a.rowptr + row);
    *e = __ldg(a.rowptr + row + 1);
    if (*e - *b > a.threshold) {
      a.y[row] = 0.f;
      want = dev::nchunks(*e - *b, a.chunk);
    } else {
      dl = *e - *b;
    }
  }
  float s = warp_light_rows(a, *b, dl);
  if (row < a.n && !want) a.y[row] = s;
  return want;
}

__device__ __forceinline__ unsigned clamp_count(const Args& a, unsigned base, unsigned total) {
  if (base >= a.pool.cap) return 0;
  return min(total, a.pool.cap - base);
}

__global__ void __launch_bounds__(256) warp_parent(Args a) {
  unsigned row = blockIdx.x * blockDim.x + threadIdx.x, b = 0, e = 0;
  unsigned want = parent_prework(a, row, &b, &e);
  unsigned bbase, btotal;
  unsigned at = dev::block_reserve(&a.hdr->count, want, &bbase, &btotal);
  if (want) {
    dev::write_chunks(a.pool, a.hdr, at, row, b, e, a.chunk);
    __threadfence();
  }
  // this warp's slice of the block slice: starts at lane 0's slot
  const unsigned wbase = __shfl_sync(kFull, at, 0), wtotal = dev::warp_sum(want);
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

// Allocator study (Fig. 5; memplan.hpp:45-58): the warp / block
// consolidation with each owner's buffer from the CUDA device heap (malloc in
// the parent, free in a tail-launched grid once the child is done) instead of
// a slice of the pre-allocated pool.  DPC_CFG_ALLOC_MALLOC.
__global__ void free_tail(void* p) { free(p); }

__global__ void __launch_bounds__(256) block_parent_malloc(Args a) {
  __shared__ Item* s_buf;
  unsigned row = blockIdx.x * blockDim.x + threadIdx.x, b = 0, e = 0;
  unsigned want = parent_prework(a, row, &b, &e);
  unsigned btotal;
  unsigned off = dev::block_excl_scan(want, &btotal);
  if (threadIdx.x == 0) {
    s_buf = btotal ? static_cast<Item*>(malloc(sizeof(Item) * btotal)) : nullptr;
    if (btotal && !s_buf) atomicOr(&a.hdr->overflow, 1u);
  }
  __syncthreads();
  if (want && s_buf) {
    dev::write_chunks(dev::Pool{s_buf, btotal}, a.hdr, off, row, b, e, a.chunk);
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_buf) {
    cons_child<<<dev::child_blocks(btotal, a.child_threads, a.child_blocks), a.child_threads, 0,
                 cudaStreamFireAndForget>>>(a, s_buf, btotal);
    dev::note_launch(a.hdr);
    free_tail<<<1, 1, 0, cudaStreamTailLaunch>>>(s_buf);
  }
}

__global__ void __launch_bounds__(256) warp_parent_malloc(Args a) {
  unsigned row = blockIdx.x * blockDim.x + threadIdx.x, b = 0, e = 0;
  unsigned want = parent_prework(a, row, &b, &e);
  const unsigned incl = dev::warp_incl_scan(want), wtotal = __shfl_sync(kFull, incl, 31);
  if (!wtotal) return;
  const unsigned leader = __ffs(__ballot_sync(kFull, want != 0)) - 1;
  unsigned long long p = 0;
  if (dev::lane_id() == leader) {
    p = reinterpret_cast<unsigned long long>(malloc(sizeof(Item) * wtotal));
    if (!p) atomicOr(&a.hdr->overflow, 1u);
  }
  Item* buf = reinterpret_cast<Item*>(__shfl_sync(kFull, p, leader));
  if (!buf) return;
  if (want) dev::write_chunks(dev::Pool{buf, wtotal}, a.hdr, incl - want, row, b, e, a.chunk);
  __threadfence();
  __syncwarp();
  if (dev::lane_id() == leader) {
    cons_child<<<dev::child_blocks(wtotal, a.child_threads, a.child_blocks), a.child_threads, 0,
                 cudaStreamFireAndForget>>>(a, buf, wtotal);
    dev::note_launch(a.hdr);
    free_tail<<<1, 1, 0, cudaStreamTailLaunch>>>(buf);
  }
}

__global__ void __launch_bounds__(256) grid_parent(Args a) {
  unsigned row = blockIdx.x * blockDim.x + threadIdx.x, b = 0, e = 0;
  unsigned want = parent_prework(a, row, &b, &e);
  unsigned bbase, btotal;
  unsigned at = dev::block_reserve(&a.hdr->count, want, &bbase, &btotal);
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

// Thread-serial prework (experiment switch: the light rows' inline work as
// the paper's per-thread loop instead of the warp-cooperative sweep).
__device__ __forceinline__ unsigned parent_prework_serial(const Args& a, unsigned row,
                                                          unsigned* b, unsigned* e) {
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

// Batched drain, one item at a time with U nonzeros per lane per step: all
// U col/val loads are in flight before the U x gathers (a 256-nonzero chunk
// is one step at U = 8).  Item descriptors are batch-loaded (one per lane).
template <int U>
__device__ __forceinline__ void drain_items_u(const Args& a, const Item* items, unsigned count,
                                              unsigned gwarp, unsigned nwarps) {
  const unsigned lane = dev::lane_id();
  const unsigned mine = count > gwarp ? (count - gwarp + nwarps - 1) / nwarps : 0;
  for (unsigned r0 = 0; r0 < mine; r0 += 32) {
    unsigned v = 0, b = 0, e = 0;
    if (r0 + lane < mine) {
      Item t = items[(r0 + lane) * nwarps + gwarp];
      v = t.v;
      b = t.begin;
      e = min(b + a.chunk, __ldg(a.rowptr + v + 1));
    }
    const unsigned nb = min(32u, mine - r0);
    for (unsigned p = 0; p < nb; p++) {
      const unsigned vp = __shfl_sync(kFull, v, p), bp = __shfl_sync(kFull, b, p);
      const unsigned n = __shfl_sync(kFull, e, p) - bp;
      float s = 0.f;
      for (unsigned o = lane; o < n; o += 32 * U) {
        int c[U];
        float w[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
          const bool ok = o + 32 * u < n;
          c[u] = ok ? ld_stream_i(a.col + bp + o + 32 * u) : 0;
          w[u] = ok ? ld_stream_f(a.val + bp + o + 32 * u) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; u++) s += w[u] * __ldg(a.x + c[u]);
      }
      s = dev::warp_sum(s);
      if (lane == 0) atomicAdd(a.y + vp, s);
    }
  }
}

// One warp per item (experiment switch: the unbatched drain).
__device__ __forceinline__ void drain_items_warp(const Args& a, const Item* items, unsigned count,
                                                 unsigned gwarp, unsigned nwarps) {
  for (unsigned i = gwarp; i < count; i += nwarps) {
    Item it = items[i];
    unsigned e = min(it.begin + a.chunk, __ldg(a.rowptr + it.v + 1));
    float s = warp_range_dot(a, it.begin, e);
    if (dev::lane_id() == 0) atomicAdd(a.y + it.v, s);
  }
}

// Grid-level consolidation as one persistent cooperative kernel: insert
// phase, device-wide barrier, drain phase.  Zero device launches.
// LM: 1 = warp-cooperative light rows, 0 = thread-serial; DM: 1 = batched
// drain, 0 = warp per item; MB: min resident blocks for ptxas.
// LM 3 / 4: timing probes only (wrong results): 3 = no light-row work,
// 4 = light rows only (no heavy-row insertion).
template <int LM, int DM, int MB>
__global__ void __launch_bounds__(256, MB) grid_persistent(Args a) {
  cg::grid_group grid = cg::this_grid();
  const unsigned stride = gridDim.x * blockDim.x;
  if (blockIdx.x == 0 && threadIdx.x == 0) a.hdr->t[0] = dev::global_ns();
  for (unsigned base = blockIdx.x * blockDim.x; base < a.n; base += stride) {
    unsigned row = base + threadIdx.x, b = 0, e = 0;
    unsigned want;
    if (LM == 3) {
      want = 0;
      if (row < a.n) {
        b = __ldg(a.rowptr + row);
        e = __ldg(a.rowptr + row + 1);
        if (e - b > a.threshold) want = dev::nchunks(e - b, a.chunk);
        a.y[row] = 0.f;
      }
    } else {
      want = LM == 2   ? parent_prework_stream(a, row, &b, &e)
             : LM == 1 || LM == 4 ? parent_prework(a, row, &b, &e)
                                  : parent_prework_serial(a, row, &b, &e);
      if (LM == 4) want = 0;
    }
    unsigned bbase, btotal;
    unsigned at = dev::block_reserve(&a.hdr->count, want, &bbase, &btotal);
    if (want) dev::write_chunks(a.pool, a.hdr, at, row, b, e, a.chunk);
  }
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) a.hdr->t[1] = dev::global_ns();
  unsigned cnt = min(*reinterpret_cast<volatile unsigned*>(&a.hdr->count), a.pool.cap);
  const unsigned gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = stride >> 5;
  if (DM == 4) drain_items_u<4>(a, a.pool.items, cnt, gw, nw);
  else if (DM == 3) drain_items_u<8>(a, a.pool.items, cnt, gw, nw);
  else if (DM == 2) drain_items_stream(a, a.pool.items, cnt, gw, nw);
  else if (DM == 1) drain_items(a, a.pool.items, cnt, gw, nw);
  else drain_items_warp(a, a.pool.items, cnt, gw, nw);
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&a.hdr->t[2], dev::global_ns());
}
// ------------------------------------------------------------------------
// Stream-balanced grid consolidation (the default grid variant).
//
// The consolidated child of the grid variant is the reference's MultiBlock
// drain (transform.hpp:564-598): every thread of the grid cooperates on the
// buffered items.  Here the buffered rows form ONE virtual stream of
// nonzeros and the drain cuts that stream into equal slices, one per warp,
// so every warp streams the same number of nonzeros and the grid finishes
// together (no per-item tail, whatever the degree distribution).
//
// dp_insert (transform.hpp:501-508; sim.hpp:1492-1528): a row with
// deg > threshold reserves its item slot AND its stream range with ONE
// 64-bit atomic per block (slot << 38 | positions), so slot order is stream
// order.  A row's stream range is its CSR range widened to 16-byte
// boundaries ([b & ~3, (e + 3) & ~3)), so every stream offset is a multiple
// of 4 and an aligned 4-position group of the stream lies inside ONE item
// and maps onto ONE aligned int4 of col / float4 of val; the widening
// elements are masked (their sectors are fetched by the neighbour rows
// anyway).
//
// Drain: a warp sweeps its slice in windows of 128 positions (4 per lane), V
// windows per step (2V vector loads + 4V x gathers in flight per lane).  The
// items of a window are located with one ballot and one OR-reduction (the
// lanes where an item starts), partial sums are combined per item with a
// 5-step segmented shuffle scan, and each item segment is written with a
// plain store when the item lies inside the window, else with atomicAdd.
constexpr int kPackShift = 38;  // packed reservation: items << 38 | positions
constexpr unsigned long long kNnzMask = (1ull << kPackShift) - 1;

struct Stream {
  uint2* seg;  // per item: {stream offset, CSR end}; Item {row, CSR begin} in the pool
  unsigned long long* sctr;
  const int* xhot_col;  // hot-column cache plan: column held by each slot (-1: none)
  float* xhot_val;      // x at those columns, gathered once per run
};

// Hot-column cache of x in shared memory.  R-MAT / power-law matrices reuse
// a few columns heavily (config 2: the 16K most popular columns take 59% of
// the nonzeros), and scattered 4-byte x gathers are bound by L1 tag
// throughput (~1 distinct line per SM clock), not by HBM.  A direct-mapped
// table of S = 2^SLOG {column, value} slots (multiplicative hash; per slot
// the most popular column, planned once per matrix on the device) serves the
// hits from shared memory; misses go to L1/L2 as before.
__device__ __forceinline__ unsigned xslot(unsigned c, int slog) { return (c * 2654435761u) >> (32 - slog); }

__device__ __forceinline__ unsigned long long warp_incl_scan64(unsigned long long v) {
  const unsigned lane = dev::lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long t = __shfl_up_sync(kFull, v, o);
    if (lane >= static_cast<unsigned>(o)) v += t;
  }
  return v;
}

// Stream length of CSR range [b, e) widened to G-element (4G-byte) boundaries.
template <int G>
__device__ __forceinline__ unsigned stream_len(unsigned b, unsigned e) {
  return ((e + (G - 1u)) & ~(G - 1u)) - (b & ~(G - 1u));
}

// One lane's aligned group of G stream positions: G/4 int4 of col, G/4
// float4 of val.
template <int G>
struct Grp {
  int4 c[G / 4];
  float4 w[G / 4];
};

template <int G>
__device__ __forceinline__ void grp_load(const Args& a, unsigned k, Grp<G>& g) {
#pragma unroll
  for (int i = 0; i < G / 4; i++) {
    if (kProbes && (a.xflags & 32u)) {  // probe: no col/val traffic (synthetic columns)
      const int cs = static_cast<int>(((k + 4 * i) * 2654435761u) & 0xfffffu);
      g.c[i] = make_int4(cs, cs ^ 1, cs ^ 2, cs ^ 3);
      g.w[i] = make_float4(1.f, 1.f, 1.f, 1.f);
    } else {
      g.c[i] = ldg_stream(reinterpret_cast<const int4*>(a.col + k + 4 * i));
      g.w[i] = ldg_stream(reinterpret_cast<const float4*>(a.val + k + 4 * i));
    }
  }
}

// Masked dot of a group with x: masked elements (the widening, invalid
// lanes) gather x[0] and weigh exactly 0.
template <int G, int SLOG>
__device__ __forceinline__ float grp_dot(const Args& a, const Grp<G>& g, unsigned m, const uint2* xc) {
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < G / 4; i++) {
    const int* cp = reinterpret_cast<const int*>(&g.c[i]);
    const float* wp = reinterpret_cast<const float*>(&g.w[i]);
    float part = 0.f;
#pragma unroll
    for (int e = 0; e < 4; e++) {
      const bool on = (m >> (4 * i + e)) & 1u;
      int idx = on ? cp[e] : 0;
      if (kProbes && (a.xflags & 64u)) idx &= 1023;      // probe: gathers confined to 4 KB of x
      if (kProbes && (a.xflags & 128u)) idx &= 0xffff;   // probe: gathers confined to 256 KB of x
      const float wt = on ? wp[e] : 0.f;
      float xv;
      if (SLOG > 0) {  // hot-column cache, misses to x (or the owner's x slice)
        const uint2 t = xc[xslot(static_cast<unsigned>(idx), SLOG)];
        xv = t.x == static_cast<unsigned>(idx) ? __uint_as_float(t.y)
             : a.xpeer && !a.xpull             ? peer_x(a, static_cast<unsigned>(idx))
                                               : __ldg(a.x + idx);
      } else if (a.xpeer && !a.xpull) {
        xv = peer_x(a, static_cast<unsigned>(idx));
      } else if (a.xpull) {
        // x was written by this kernel (the pull before the barrier): .nc
        // loads are only defined for data read-only for the whole kernel, so
        // a plain (weak, L1-cached) load, ordered by the barrier's acquire
        xv = ld_weak_f(a.x + idx);
      } else if (kProbes && (a.xflags & 16u)) {
        xv = 1.f;
      } else if (a.xflags & 256u) {
        xv = __ldcg(a.x + idx);  // probe: x gathers through L2 only
      } else if (a.xflags & 512u) {
        xv = ld_stream_f(a.x + idx);  // probe: x gathers without L1 allocation
      } else {
        xv = __ldg(a.x + idx);
      }
      part += wt * xv;
    }
    s += part;
  }
  return s;
}

// Bits of the aligned group at CSR index k that lie inside [b, e).
template <int G>
__device__ __forceinline__ unsigned grp_mask(unsigned k, unsigned b, unsigned e) {
  const int lo_e = max(static_cast<int>(b - k), 0);
  const int hi_e = min(max(static_cast<int>(e - k), 0), G);
  return ((((1u << G) - 1u) << lo_e) & ((1u << hi_e) - 1u)) & ((1u << G) - 1u);
}

// Insert of row `row` (CSR range [b, e)) at packed position `at`.
__device__ __forceinline__ void stream_insert(const Args& a, const Stream& st, unsigned long long at,
                                              unsigned row, unsigned b, unsigned e) {
  const unsigned slot = static_cast<unsigned>(at >> kPackShift);
  if (slot >= a.pool.cap) {
    atomicOr(&a.hdr->overflow, 1u);
    return;
  }
  if (!kProbes || !(a.xflags & 4u)) {
    a.pool.items[slot] = Item{row, b};
    st.seg[slot] = make_uint2(static_cast<unsigned>(at & kNnzMask), e);
  }
}

// Per-warp shared-memory window onto the item list: kBatch consecutive
// items {stream offset, CSR end, CSR begin, row}.
template <unsigned KB>
__device__ __forceinline__ void load_items(const Args& a, const Stream& st, unsigned ni, unsigned base,
                                           uint4* buf) {
  const unsigned lane = dev::lane_id();
#pragma unroll
  for (unsigned i = 0; i < KB / 32; i++) {
    const unsigned idx = base + lane + 32 * i;
    uint4 v = make_uint4(0xffffffffu, 0, 0, 0);
    if (idx < ni) {
      const uint2 sg = __ldcg(st.seg + idx);
      const Item it = a.pool.items[idx];
      v = make_uint4(sg.x, sg.y, it.begin, it.v);
    }
    buf[lane + 32 * i] = v;
  }
  __syncwarp();
}

// Drains this warp's slice [s0, s1) of the stream (s0 a multiple of the
// window 32G, s1 a multiple of it or the stream end).  All lanes call.
//   start: 32-ary search of the item covering s0 (log32(items) L2 rounds)
//   window: 32 groups of G positions (one per lane); its items are ja ..
//     ja+31 at most (items are >= G positions and start on G-aligned
//     positions); each lane reads item ja+lane from the shared-memory batch,
//     the lanes where an item starts form a bit mask (one OR-reduction), and
//     each lane's item is ja + popc(mask below it).  ja of the next window
//     follows from the mask; the batch is refilled from L2 when the window
//     could run past it.
//   fast step: V windows inside one long item need no lookup and no scan.
template <int G, int V, unsigned KB, int SLOG>
__device__ __forceinline__ void stream_drain(const Args& a, const Stream& st, unsigned ni,
                                             unsigned s0, unsigned s1, uint4* buf, const uint2* xc) {
  constexpr unsigned W = 32u * G;  // stream positions per window
  const unsigned lane = dev::lane_id();
  const unsigned lt_mask = (2u << lane) - 1u;  // lanes <= this one
  unsigned lo = 0, hi = ni;  // seg[lo].x <= s0 < seg[hi].x (hi = ni: end)
  while (hi - lo > 1) {
    const unsigned step = (hi - lo + 31) / 32;
    const unsigned probe = lo + lane * step;
    const unsigned v = probe < hi ? __ldcg(&st.seg[probe].x) : 0xffffffffu;
    const unsigned c = __popc(__ballot_sync(kFull, v <= s0));  // >= 1: lane 0 probes lo
    const unsigned nlo = lo + (c - 1) * step;
    hi = min(hi, nlo + step);
    lo = nlo;
  }
  unsigned ja = lo, bb = lo;
  load_items<KB>(a, st, ni, bb, buf);
  float carry = 0.f;  // this lane's partial sum for item ja from fast steps
  bool carrying = false;
  for (unsigned p0 = s0; p0 < s1; p0 += W * V) {
    {
      if (ja + 33 > bb + KB) {
        bb = ja;
        load_items<KB>(a, st, ni, bb, buf);
      }
      const uint4 it = buf[ja - bb];
      const unsigned iend = it.x + stream_len<G>(it.z, it.y);
      if (p0 + W * V <= min(iend, s1)) {
        const unsigned kb = (it.z & ~(G - 1u)) + (p0 - it.x) + G * lane;
        Grp<G> g[V];
#pragma unroll
        for (int v = 0; v < V; v++) grp_load<G>(a, kb + W * v, g[v]);
#pragma unroll
        for (int v = 0; v < V; v++)
          carry += grp_dot<G, SLOG>(a, g[v], grp_mask<G>(kb + W * v, it.z, it.y), xc);
        carrying = true;
        if (iend == p0 + W * V) {  // item ja ends exactly here: flush, move on
          const float t = dev::warp_sum(carry);
          if (lane == 0) atomicAdd(a.y + it.w, t);
          carry = 0.f;
          carrying = false;
          ja++;
        }
        continue;
      }
      if (carrying) {  // leaving item ja's fast steps: flush its partial sum
        const float t = dev::warp_sum(carry);
        if (lane == 0) atomicAdd(a.y + it.w, t);
        carry = 0.f;
        carrying = false;
      }
    }
    unsigned kk[V], info[V], rw[V];
#pragma unroll
    for (int v = 0; v < V; v++) {
      const unsigned pw = p0 + W * v;  // may lie past s1 on the last step: no lane is valid then
      if (ja + 33 > bb + KB) {
        bb = ja;
        load_items<KB>(a, st, ni, bb, buf);
      }
      const unsigned last = min(pw + W, s1) - 1;
      const unsigned off = buf[ja - bb + lane].x;
      // lanes where an item starts inside the window (lane 0 excluded)
      const unsigned bit = (off > pw && off <= last) ? 1u << ((off - pw) / G) : 0u;
      const unsigned smask = __reduce_or_sync(kFull, bit);
      const uint4 it = buf[ja - bb + __popc(smask & lt_mask)];  // {offset, end, begin, row}
      const unsigned q = pw + G * lane;
      const bool valid = q < s1;
      const unsigned k = valid ? (it.z & ~(G - 1u)) + (q - it.x) : 0u;
      const unsigned m = valid ? grp_mask<G>(k, it.z, it.y) : 0u;
      const unsigned ls = 31 - __clz((smask | 1u) & lt_mask);  // segment start lane
      const bool seg_end = valid && (lane == 31 || (((smask >> 1) >> lane) & 1u) || q + G >= s1);
      const bool whole = it.x >= pw && it.x + stream_len<G>(it.z, it.y) <= pw + W;
      kk[v] = k;
      rw[v] = it.w;
      info[v] = m | (ls << 16) | (seg_end ? 1u << 21 : 0u) | (whole ? 1u << 22 : 0u);
      // first item of the next window
      ja += __popc(smask);
      ja += buf[ja + 1 - bb].x == pw + W ? 1u : 0u;
    }
    Grp<G> g[V];
#pragma unroll
    for (int v = 0; v < V; v++) grp_load<G>(a, kk[v], g[v]);
    float s[V];
#pragma unroll
    for (int v = 0; v < V; v++) s[v] = grp_dot<G, SLOG>(a, g[v], info[v] & 0xffffu, xc);
#pragma unroll
    for (int v = 0; v < V; v++) {
      if (p0 + W * v >= s1) break;
      const unsigned ls = (info[v] >> 16) & 31u;
      float t = s[v];
#pragma unroll
      for (unsigned d = 1; d < 32; d <<= 1) {
        const float u = __shfl_up_sync(kFull, t, d);
        if (lane >= ls + d) t += u;
      }
      if (info[v] & (1u << 21)) {
        if (info[v] & (1u << 22)) a.y[rw[v]] = t;
        else atomicAdd(a.y + rw[v], t);
      }
    }
  }
  if (carrying) {
    const float t = dev::warp_sum(carry);
    if (lane == 0) atomicAdd(a.y + buf[ja - bb].w, t);
  }
}

// Window lookup of the general drain path (see stream_drain): fills the
// lane's CSR index, mask / segment bits and row for the window at pw, and
// advances ja to the first item of the next window.  All lanes call.
template <int G, unsigned KB>
__device__ __forceinline__ void window_lookup(const Args& a, const Stream& st, unsigned ni, unsigned s1,
                                              uint4* buf, unsigned pw, unsigned& ja, unsigned& bb,
                                              unsigned& kk, unsigned& info, unsigned& rw) {
  constexpr unsigned W = 32u * G;
  const unsigned lane = dev::lane_id();
  const unsigned lt_mask = (2u << lane) - 1u;
  if (ja + 33 > bb + KB) {
    bb = ja;
    load_items<KB>(a, st, ni, bb, buf);
  }
  const unsigned last = min(pw + W, s1) - 1;
  const unsigned off = buf[ja - bb + lane].x;
  const unsigned bit = (off > pw && off <= last) ? 1u << ((off - pw) / G) : 0u;
  const unsigned smask = __reduce_or_sync(kFull, bit);
  const uint4 it = buf[ja - bb + __popc(smask & lt_mask)];
  const unsigned q = pw + G * lane;
  const bool valid = q < s1;
  const unsigned k = valid ? (it.z & ~(G - 1u)) + (q - it.x) : 0u;
  const unsigned m = valid ? grp_mask<G>(k, it.z, it.y) : 0u;
  const unsigned ls = 31 - __clz((smask | 1u) & lt_mask);
  const bool seg_end = valid && (lane == 31 || (((smask >> 1) >> lane) & 1u) || q + G >= s1);
  const bool whole = it.x >= pw && it.x + stream_len<G>(it.z, it.y) <= pw + W;
  kk = k;
  rw = it.w;
  info = m | (ls << 16) | (seg_end ? 1u << 21 : 0u) | (whole ? 1u << 22 : 0u);
  ja += __popc(smask);
  ja += buf[ja + 1 - bb].x == pw + W ? 1u : 0u;
}

// Software-pipelined drain (shape bit 23): the window lookups of step s+1
// (shared-memory work) and an L2 prefetch of its col / val groups run while
// step s's loads are in flight.  General path only.
template <int G, int V, unsigned KB, int SLOG>
__device__ __forceinline__ void stream_drain_pipe(const Args& a, const Stream& st, unsigned ni,
                                                  unsigned s0, unsigned s1, uint4* buf, const uint2* xc) {
  constexpr unsigned W = 32u * G;
  const unsigned lane = dev::lane_id();
  unsigned lo = 0, hi = ni;
  while (hi - lo > 1) {
    const unsigned step = (hi - lo + 31) / 32;
    const unsigned probe = lo + lane * step;
    const unsigned v = probe < hi ? __ldcg(&st.seg[probe].x) : 0xffffffffu;
    const unsigned c = __popc(__ballot_sync(kFull, v <= s0));
    const unsigned nlo = lo + (c - 1) * step;
    hi = min(hi, nlo + step);
    lo = nlo;
  }
  unsigned ja = lo, bb = lo;
  load_items<KB>(a, st, ni, bb, buf);
  unsigned kk[V], info[V], rw[V];
#pragma unroll
  for (int v = 0; v < V; v++) window_lookup<G, KB>(a, st, ni, s1, buf, s0 + W * v, ja, bb, kk[v], info[v], rw[v]);
  for (unsigned p0 = s0; p0 < s1; p0 += W * V) {
    Grp<G> g[V];
#pragma unroll
    for (int v = 0; v < V; v++) grp_load<G>(a, kk[v], g[v]);
    // next step: lookups + L2 prefetch while this step's loads fly
    unsigned nk[V], ninfo[V], nrw[V];
    const unsigned pn = p0 + W * V;
#pragma unroll
    for (int v = 0; v < V; v++) {
      nk[v] = 0, ninfo[v] = 0, nrw[v] = 0;
      if (pn < s1) {
        window_lookup<G, KB>(a, st, ni, s1, buf, pn + W * v, ja, bb, nk[v], ninfo[v], nrw[v]);
        if (ninfo[v] & 0xffffu) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a.col + nk[v]));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a.val + nk[v]));
        }
      }
    }
    float sv[V];
#pragma unroll
    for (int v = 0; v < V; v++) sv[v] = grp_dot<G, SLOG>(a, g[v], info[v] & 0xffffu, xc);
#pragma unroll
    for (int v = 0; v < V; v++) {
      if (p0 + W * v < s1) {
        const unsigned ls = (info[v] >> 16) & 31u;
        float t = sv[v];
#pragma unroll
        for (unsigned d = 1; d < 32; d <<= 1) {
          const float u = __shfl_up_sync(kFull, t, d);
          if (lane >= ls + d) t += u;
        }
        if (info[v] & (1u << 21)) {
          if (info[v] & (1u << 22)) a.y[rw[v]] = t;
          else atomicAdd(a.y + rw[v], t);
        }
      }
    }
#pragma unroll
    for (int v = 0; v < V; v++) kk[v] = nk[v], info[v] = ninfo[v], rw[v] = nrw[v];
  }
}

// cp.async (LDGSTS) 16-byte global -> shared copies, L1 bypassed.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Asynchronously staged drain (shape bit pattern 0 = default when ASYNCCP):
// step s+1's col / val groups are copied to shared memory with cp.async
// while step s is gathered and reduced from shared memory, so the DRAM
// latency of the stream leaves the per-step chain (only the x gathers stay).
// Per warp: 2 stages x V windows x 32 lanes x G/4 (int4 + float4).
template <int G, int V, unsigned KB, int SLOG>
__device__ __forceinline__ void stream_drain_cp(const Args& a, const Stream& st, unsigned ni, unsigned s0,
                                                unsigned s1, uint4* buf, const uint2* xc, int4* stage) {
  constexpr unsigned W = 32u * G;
  constexpr int GQ = G / 4;                 // int4 per group
  constexpr int STAGE = V * 32 * GQ * 2;    // int4 per stage (col + val)
  const unsigned lane = dev::lane_id();
  unsigned lo = 0, hi = ni;
  while (hi - lo > 1) {
    const unsigned step = (hi - lo + 31) / 32;
    const unsigned probe = lo + lane * step;
    const unsigned v = probe < hi ? __ldcg(&st.seg[probe].x) : 0xffffffffu;
    const unsigned c = __popc(__ballot_sync(kFull, v <= s0));
    const unsigned nlo = lo + (c - 1) * step;
    hi = min(hi, nlo + step);
    lo = nlo;
  }
  unsigned ja = lo, bb = lo;
  load_items<KB>(a, st, ni, bb, buf);
  auto issue = [&](int stg, const unsigned* kk) {
#pragma unroll
    for (int v = 0; v < V; v++)
#pragma unroll
      for (int i = 0; i < GQ; i++) {
        int4* dst = stage + stg * STAGE + ((v * 32 + lane) * GQ + i) * 2;
        cp_async16(dst, a.col + kk[v] + 4 * i);
        cp_async16(dst + 1, a.val + kk[v] + 4 * i);
      }
    cp_async_commit();
  };
  unsigned kk[V], info[V], rw[V];
#pragma unroll
  for (int v = 0; v < V; v++) window_lookup<G, KB>(a, st, ni, s1, buf, s0 + W * v, ja, bb, kk[v], info[v], rw[v]);
  issue(0, kk);
  int cur = 0;
  for (unsigned p0 = s0; p0 < s1; p0 += W * V) {
    unsigned nk[V], ninfo[V], nrw[V];
    const unsigned pn = p0 + W * V;
#pragma unroll
    for (int v = 0; v < V; v++) {
      nk[v] = 0, ninfo[v] = 0, nrw[v] = 0;
      if (pn < s1) window_lookup<G, KB>(a, st, ni, s1, buf, pn + W * v, ja, bb, nk[v], ninfo[v], nrw[v]);
    }
    issue(cur ^ 1, nk);  // next step's groups (an empty group when past s1)
    cp_async_wait<1>();  // this step's groups have landed
    float sv[V];
#pragma unroll
    for (int v = 0; v < V; v++) {
      Grp<G> g;
#pragma unroll
      for (int i = 0; i < GQ; i++) {
        const int4* src = stage + cur * STAGE + ((v * 32 + lane) * GQ + i) * 2;
        g.c[i] = src[0];
        const int4 w = src[1];
        g.w[i] = make_float4(__int_as_float(w.x), __int_as_float(w.y), __int_as_float(w.z), __int_as_float(w.w));
      }
      sv[v] = grp_dot<G, SLOG>(a, g, info[v] & 0xffffu, xc);
    }
#pragma unroll
    for (int v = 0; v < V; v++) {
      if (p0 + W * v < s1) {
        const unsigned ls = (info[v] >> 16) & 31u;
        float t = sv[v];
#pragma unroll
        for (unsigned d = 1; d < 32; d <<= 1) {
          const float u = __shfl_up_sync(kFull, t, d);
          if (lane >= ls + d) t += u;
        }
        if (info[v] & (1u << 21)) {
          if (info[v] & (1u << 22)) a.y[rw[v]] = t;
          else atomicAdd(a.y + rw[v], t);
        }
      }
    }
#pragma unroll
    for (int v = 0; v < V; v++) kk[v] = nk[v], info[v] = ninfo[v], rw[v] = nrw[v];
    cur ^= 1;
  }
  cp_async_wait<0>();
}

// Persistent grid-consolidated SpMV.
//   insert: 256-row tiles are dealt to blocks round-robin (tile k*G + b of a
//     round goes to block b, row = lane), kRound tiles per thread per round.
//     The round's stream lengths of the rows with deg > threshold are
//     scanned per tile (slots in tile-major, then row order, so the item
//     stores of a warp are contiguous), ONE 64-bit atomic per block and
//     round reserves the slots and positions; lighter rows are done inline
//     (warp-cooperative).
//   one device-wide barrier (the paper's custom global barrier,
//     PAPER.md:244-250; legal because a cooperative launch co-schedules
//     the whole grid)
//   drain: stream-balanced, every warp the same number of positions.
template <bool INLINE, int G, int V, int NT, int MINB, int SLOG, unsigned KB, int PIPE = 0>
__global__ void __launch_bounds__(NT, MINB) grid_stream(Args a, Stream st) {
  constexpr unsigned kWin = 32u * G;
  constexpr int NW = NT / 32;
  constexpr int kRound = NT >= 1024 ? 4 : 8;  // tiles per thread per reservation round
  __shared__ unsigned long long s_w[kRound * NW];
  __shared__ unsigned long long s_base;
  extern __shared__ uint4 s_dyn[];  // [NW][KB] item windows, then 2^SLOG cache slots
  uint4* s_items = s_dyn;
  uint2* s_cache = reinterpret_cast<uint2*>(s_dyn + NW * KB);
  if (blockIdx.x == 0 && threadIdx.x == 0) a.hdr->t[0] = dev::global_ns();
  const unsigned lane = dev::lane_id(), wib = dev::warp_in_block();
  const unsigned lt_excl = (1u << lane) - 1u;
  const unsigned GB = gridDim.x, ntiles = (a.n + NT - 1) / NT;
  if (SLOG > 0)  // x at the planned hot columns, once per run
    for (unsigned i = blockIdx.x * NT + threadIdx.x; i < (1u << SLOG); i += GB * NT) {
      const int c = st.xhot_col[i];
      st.xhot_val[i] = c >= 0 ? (a.xpeer ? peer_x(a, static_cast<unsigned>(c)) : __ldg(a.x + c)) : 0.f;
    }
  for (unsigned t0 = blockIdx.x; t0 < ntiles; t0 += GB * kRound) {
    unsigned bb[kRound], ee[kRound], inc[kRound];
#pragma unroll
    for (int k = 0; k < kRound; k++) {
      const unsigned r = (t0 + k * GB) * NT + threadIdx.x;
      bb[k] = ee[k] = 0;
      if (t0 + k * GB < ntiles && r < a.n) bb[k] = __ldg(a.rowptr + r), ee[k] = __ldg(a.rowptr + r + 1);
    }
#pragma unroll
    for (int k = 0; k < kRound; k++) {
      const bool cons = ee[k] - bb[k] > a.threshold;
      const unsigned len = cons ? stream_len<G>(bb[k], ee[k]) : 0u;
      inc[k] = dev::warp_incl_scan(len);
      const unsigned cnt = __popc(__ballot_sync(kFull, cons));
      if (lane == 31) s_w[k * NW + wib] = (static_cast<unsigned long long>(cnt) << kPackShift) | inc[k];
    }
    __syncthreads();
    if (wib == 0) {  // tile-major scan of the kRound x NW warp totals, one reservation
      constexpr int PER = kRound * NW / 32;
      unsigned long long xs[PER], tsum = 0;
#pragma unroll
      for (int i = 0; i < PER; i++) xs[i] = s_w[PER * lane + i], tsum += xs[i];
      const unsigned long long pi = warp_incl_scan64(tsum);
      unsigned long long run = pi - tsum;
#pragma unroll
      for (int i = 0; i < PER; i++) s_w[PER * lane + i] = run, run += xs[i];
      if (lane == 31) s_base = pi ? atomicAdd(st.sctr, pi) : 0ull;
    }
    __syncthreads();
    const unsigned long long base = s_base;
#pragma unroll
    for (int k = 0; k < kRound; k++) {
      const unsigned r = (t0 + k * GB) * NT + threadIdx.x;
      const bool in = t0 + k * GB < ntiles && r < a.n;
      const unsigned b = bb[k], e = ee[k];
      const bool cons = e - b > a.threshold;
      const unsigned ball = __ballot_sync(kFull, cons);
      float sl = 0.f;
      if (INLINE) sl = warp_light_rows(a, b, in && !cons ? e - b : 0u);
      if (in && (!kProbes || !(a.xflags & 8u))) a.y[r] = cons ? 0.f : sl;
      if (cons) {
        const unsigned len = stream_len<G>(b, e);
        const unsigned long long at = base + s_w[k * NW + wib] +
                                      ((static_cast<unsigned long long>(__popc(ball & lt_excl)) << kPackShift) |
                                       (inc[k] - len));
        stream_insert(a, st, at, r, b, e);
      }
    }
    __syncthreads();  // s_w / s_base are reused by the next round
  }
  if (a.xpull) {
    // fused multi-GPU pull: every owner's x slice into the local x with
    // coalesced 16-byte peer reads (NVLink), overlapping the insert phase's
    // tail; the barrier below orders it before the drain's gathers, which
    // read the pulled x with plain weak loads (the barrier's acquire makes
    // them see it), not through the read-only (.nc) path.
    const unsigned nx = a.ncols, stride = GB * NT;
    if ((a.rows & 3u) == 0) {
      for (unsigned i = blockIdx.x * NT + threadIdx.x; 4 * i < nx; i += stride) {
        const unsigned c = 4 * i;
        const unsigned o = a.rshift != ~0u ? c >> a.rshift : c / a.rows;
        const unsigned l = c - o * a.rows;
        const float* src = a.xpeer[o] + l;
        if (c + 4 <= nx && !(reinterpret_cast<uintptr_t>(src) & 15u)) {
          reinterpret_cast<float4*>(a.xpull)[i] = __ldcg(reinterpret_cast<const float4*>(src));
        } else {
          for (unsigned j = c; j < min(c + 4, nx); j++) a.xpull[j] = __ldcg(src + (j - c));
        }
      }
    } else {
      for (unsigned c = blockIdx.x * NT + threadIdx.x; c < nx; c += stride) {
        const unsigned o = a.rshift != ~0u ? c >> a.rshift : c / a.rows;
        a.xpull[c] = __ldcg(a.xpeer[o] + (c - o * a.rows));
      }
    }
  }
  if (a.coop) cg::this_grid().sync();
  else dev::soft_grid_barrier(&a.hdr->ticket, &a.hdr->overflow);
  if (blockIdx.x == 0 && threadIdx.x == 0) a.hdr->t[1] = dev::global_ns();
  if (SLOG > 0) {
    for (unsigned i = threadIdx.x; i < (1u << SLOG); i += NT)
      s_cache[i] = make_uint2(static_cast<unsigned>(__ldcg(st.xhot_col + i)), __float_as_uint(__ldcg(st.xhot_val + i)));
    __syncthreads();
  }
  const unsigned long long tot = *reinterpret_cast<volatile unsigned long long*>(st.sctr);
  const unsigned ni = min(static_cast<unsigned>(tot >> kPackShift), a.pool.cap);
  const unsigned total = static_cast<unsigned>(tot & kNnzMask);
  const unsigned nw = (gridDim.x * NT) >> 5, gw = (blockIdx.x * NT + threadIdx.x) >> 5;
  const unsigned long long per = ((static_cast<unsigned long long>(total) + nw - 1) / nw + kWin - 1) /
                                 kWin * kWin;
  const unsigned long long s0 = static_cast<unsigned long long>(gw) * per;
  const bool drain_on = !kProbes || !(a.xflags & 1u);
  if (ni > 0 && s0 < total && drain_on && PIPE == 2)
    stream_drain_cp<G, V, KB, SLOG>(a, st, ni, static_cast<unsigned>(s0),
                                    static_cast<unsigned>(min(static_cast<unsigned long long>(total), s0 + per)),
                                    s_items + wib * KB, s_cache,
                                    reinterpret_cast<int4*>(s_dyn + NW * KB + (SLOG ? (1u << SLOG) / 2 : 0)) +
                                        wib * (2 * V * 32 * (G / 4) * 2));
  else if (ni > 0 && s0 < total && drain_on && PIPE == 1)
    stream_drain_pipe<G, V, KB, SLOG>(a, st, ni, static_cast<unsigned>(s0),
                                      static_cast<unsigned>(min(static_cast<unsigned long long>(total), s0 + per)),
                                      s_items + wib * KB, s_cache);
  else if (ni > 0 && s0 < total && drain_on)
    stream_drain<G, V, KB, SLOG>(a, st, ni, static_cast<unsigned>(s0),
                              static_cast<unsigned>(min(static_cast<unsigned long long>(total), s0 + per)),
                              s_items + wib * KB, s_cache);
  __syncthreads();
  if (threadIdx.x == 0) {
    // the last block out stamps the end and zeroes the counters of this run
    // (packed reservation, barrier count, exit ticket): the next run needs
    // no memset of the header
    __threadfence();
    if (atomicAdd(&a.hdr->aux0, 1u) == gridDim.x - 1) {
      a.hdr->t[2] = dev::global_ns();
      *st.sctr = 0;
      a.hdr->ticket = 0;
      a.hdr->aux0 = 0;
      __threadfence();
    }
  }
}

// Stream kernel shapes (dpc_launch_cfg.flags bits 20-22), measured on config 2
// (tools/prof_spmv.py --burst 10; the x gathers and the per-step latency
// chain, not HBM, bound all of them):
//   0: software-pipelined drain (step s+1's window lookups and an L2
//      prefetch of its col / val groups run under step s's loads), groups of
//      4 positions per lane, 2 windows per step, 1024 threads x 1 block/SM,
//      64-item batches per warp (32 KB shared: the rest of the 256 KB
//      unified L1 caches x; 128-item batches 82.0 us, 64 79.9, 32 84.0; a
//      max-shared carve-out doubles the drain time)
//      (default: 84.0 us vs 90.1 us for shape 6 on the same box, 128 items)
//   1: groups of 8, 2 windows per step, not pipelined
//   2: groups of 4, 4 windows, 256 threads x 4 blocks/SM
//   3: groups of 4, 4 windows, hot-column x cache of 2^14 slots
//   4: groups of 8, 2 windows, hot-column x cache
//   5: cp.async-staged drain (next step's col / val copied to shared memory
//      under this step's gathers), groups of 4, 2 windows: measured 2.9x
//      slower than shape 0 (196 vs 68 us drain)
//   6: groups of 4, 4 windows, not pipelined
//   7: pipelined, groups of 4, 3 windows
// Higher occupancy loses: shape 0 at 512 threads x 3 blocks/SM (40 regs,
// 216 B spills) 106.6 us, at 1024 x 2 (32 regs, 208 B spills, 32-item
// batches) 114.4 us, vs 78.1 us: spills and the smaller x share of L1 cost
// more than the extra warps hide.
// Register double-buffering (step s+1's col / val loaded into registers
// under step s's gathers, lookups two steps ahead) also loses: 768 threads
// x 80 regs 91.0 us, 512 x 96 regs 119.1 us, 1 window x 1024 threads 81.0 us
// (all parity-equal): with the L2 prefetch already in place, warps x
// gathers in flight is what the drain needs.
// On the vertex-permuted matrix (config 5 rows, tools/prof_spmv.py
// --permute --burst 10): shape 0 87.4 us, 3 90.0, 4 81.8, 6 93.5, 7 91.3 —
// the hot-column cache pays 6 % once permutation spreads the hubs; the
// fused peer-x path does not use it.
struct StreamShape {
  const void* fn;
  int threads;
  int slog;
  int group;
  size_t smem;  // dynamic shared memory bytes
};
constexpr int kHotLog = 14;
template <int G, int V, int NT, int MINB, int SLOG, unsigned KB, int PIPE = 0>
static StreamShape shape_of(bool inl) {
  const size_t cache = (SLOG ? sizeof(uint2) << SLOG : 0) +
                       (PIPE == 2 ? static_cast<size_t>(NT / 32) * 2 * V * 32 * (G / 4) * 2 * sizeof(int4) : 0);
  return {inl ? reinterpret_cast<const void*>(grid_stream<true, G, V, NT, MINB, SLOG, KB, PIPE>)
              : reinterpret_cast<const void*>(grid_stream<false, G, V, NT, MINB, SLOG, KB, PIPE>),
          NT, SLOG, G, (NT / 32) * KB * sizeof(uint4) + cache};
}
static StreamShape stream_shape(bool inl, unsigned flags) {
  switch ((flags >> 20) & 7u) {
    case 1: return shape_of<8, 2, 1024, 1, 0, 128>(inl);
    case 2: return shape_of<4, 4, 256, 4, 0, 128>(inl);
    case 3: return shape_of<4, 4, 1024, 1, kHotLog, 64>(inl);
    case 4: return shape_of<8, 2, 1024, 1, kHotLog, 64>(inl);
    case 5: return shape_of<4, 2, 1024, 1, 0, 64, 2>(inl);
    case 6: return shape_of<4, 4, 1024, 1, 0, 128>(inl);
    case 7: return shape_of<4, 3, 1024, 1, 0, 128, 1>(inl);
    default: return shape_of<4, 2, 1024, 1, 0, 64, 1>(inl);  // KB 64: 32 KB batch, more L1 for x (-2.6 %)
  }
}

using PersistentFn = void (*)(Args);
// [LM][DM][MB == 8]
static PersistentFn persistent_fn(unsigned flags) {
  const bool serial = flags & (1u << 8), warp_drain = flags & (1u << 9), low_occ = flags & (1u << 10);
#if DPC_TIMING_PROBES
  if (flags & (1u << 16)) return grid_persistent<3, 1, 8>;
  if (flags & (1u << 17)) return grid_persistent<4, 1, 8>;
#endif
  if (flags & (1u << 14)) return low_occ ? grid_persistent<1, 3, 4> : grid_persistent<1, 3, 8>;
  if (flags & (1u << 15)) return low_occ ? grid_persistent<1, 4, 4> : grid_persistent<1, 4, 8>;
  if (flags & (1u << 11)) return low_occ ? grid_persistent<2, 2, 4> : grid_persistent<2, 2, 8>;
  if (flags & (1u << 12)) return low_occ ? grid_persistent<2, 1, 4> : grid_persistent<2, 1, 8>;
  if (flags & (1u << 13)) return low_occ ? grid_persistent<1, 2, 4> : grid_persistent<1, 2, 8>;
  static const PersistentFn table[2][2][2] = {
      {{grid_persistent<0, 0, 4>, grid_persistent<0, 0, 8>}, {grid_persistent<0, 1, 4>, grid_persistent<0, 1, 8>}},
      {{grid_persistent<1, 0, 4>, grid_persistent<1, 0, 8>}, {grid_persistent<1, 1, 4>, grid_persistent<1, 1, 8>}}};
  return table[serial ? 0 : 1][warp_drain ? 0 : 1][low_occ ? 0 : 1];
}

}  // namespace spmv

static dpc_status ensure_stream(dpc_dgraph* g, uint64_t items) {
  if (items > g->soff_cap) {
    DPC_CUDA(cudaStreamSynchronize(g->ctx->stream));
    if (g->soff) cudaFree(g->soff);
    g->soff = nullptr;
    g->soff_cap = 0;
    DPC_CUDA(cudaMalloc(&g->soff, sizeof(uint2) * std::max<uint64_t>(items, 1)));
    g->soff_cap = items;
  }
  return DPC_OK;
}

// Hot-column cache plan (once per matrix): per slot, the most used column
// among those hashing to it (ties: the larger id).
namespace spmv {
__global__ void hot_count(const int* __restrict__ col, unsigned m, unsigned* cnt) {
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    atomicAdd(cnt + col[i], 1u);
}
__global__ void hot_pick(const unsigned* __restrict__ cnt, unsigned ncols, unsigned long long* best, int slog) {
  for (unsigned c = blockIdx.x * blockDim.x + threadIdx.x; c < ncols; c += gridDim.x * blockDim.x)
    if (cnt[c]) atomicMax(best + xslot(c, slog), (static_cast<unsigned long long>(cnt[c]) << 32) | c);
}
__global__ void hot_final(const unsigned long long* __restrict__ best, int* hot_col, unsigned slots) {
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < slots; i += gridDim.x * blockDim.x)
    hot_col[i] = best[i] ? static_cast<int>(best[i] & 0xffffffffu) : -1;
}
}  // namespace spmv

static dpc_status ensure_xhot(dpc_ctx* ctx, dpc_dgraph* g, int slog) {
  if (g->xhot_log == slog) return DPC_OK;
  cudaStream_t s = ctx->stream;
  DPC_CUDA(cudaStreamSynchronize(s));
  if (g->xhot_col) cudaFree(g->xhot_col);
  if (g->xhot_val) cudaFree(g->xhot_val);
  g->xhot_col = nullptr;
  g->xhot_val = nullptr;
  g->xhot_log = 0;
  const size_t slots = size_t{1} << slog, nc = static_cast<size_t>(std::max<int64_t>(g->ncols, 1));
  unsigned* cnt = nullptr;
  unsigned long long* best = nullptr;
  DPC_CUDA(cudaMalloc(&g->xhot_col, sizeof(int) * slots));
  DPC_CUDA(cudaMalloc(&g->xhot_val, sizeof(float) * slots));
  DPC_CUDA(cudaMalloc(&cnt, sizeof(unsigned) * nc));
  cudaError_t e = cudaMalloc(&best, sizeof(unsigned long long) * slots);
  if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, sizeof(unsigned) * nc, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(best, 0, sizeof(unsigned long long) * slots, s);
  if (e == cudaSuccess) {
    const unsigned grid = 4u * static_cast<unsigned>(ctx->sms);
    if (g->m > 0) spmv::hot_count<<<grid, 256, 0, s>>>(g->col, static_cast<unsigned>(g->m), cnt);
    spmv::hot_pick<<<grid, 256, 0, s>>>(cnt, static_cast<unsigned>(nc), best, slog);
    spmv::hot_final<<<grid, 256, 0, s>>>(best, g->xhot_col, static_cast<unsigned>(slots));
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(cnt);
  if (best) cudaFree(best);
  if (e != cudaSuccess) return cuda_fail(e, "SpMV hot-column plan");
  g->xhot_log = slog;
  return DPC_OK;
}

// Resident blocks of a stream kernel shape (dynamic shared memory attribute
// set and occupancy queried once per function and device, then cached: both
// are host API calls on the per-step path otherwise).
static int stream_blocks(dpc_ctx* ctx, const spmv::StreamShape& sh) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_pair(sh.fn, ctx->device);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (cudaFuncSetAttribute(sh.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sh.smem)) !=
      cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  // unified L1 / shared memory: as little carve-out as the batch needs, the
  // rest stays L1 for the x gathers (DPC_SPMV_CARVEOUT overrides, percent)
  static const int carve = std::getenv("DPC_SPMV_CARVEOUT") ? std::atoi(std::getenv("DPC_SPMV_CARVEOUT")) : -2;
  if (carve != -2 &&
      cudaFuncSetAttribute(sh.fn, cudaFuncAttributePreferredSharedMemoryCarveout, carve) != cudaSuccess)
    cudaGetLastError();
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sh.fn, sh.threads, sh.smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  const int nb = per_sm * ctx->sms;
  cache[key] = nb;
  return nb;
}

static int coop_blocks(dpc_ctx* ctx, const void* fn, int threads, size_t smem = 0) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    per_sm = 1;
  }
  return std::max(1, per_sm) * ctx->sms;
}

}  // namespace dpc

using namespace dpc;

namespace dpc {
dpc_status spmv_run(dpc_ctx* ctx, dpc_dgraph* g, const float* d_x, float* d_y, const dpc_launch_cfg* cfg,
                    dpc_metrics* met, const float* const* xpeer, uint64_t rows);
}

extern "C" dpc_status dpc_spmv_device(dpc_ctx* ctx, dpc_dgraph* g, const float* d_x, float* d_y,
                                      const dpc_launch_cfg* cfg, dpc_metrics* met) {
  clear_error();
  return dpc::spmv_run(ctx, g, d_x, d_y, cfg, met, nullptr, 0);
}

dpc_status dpc::spmv_run(dpc_ctx* ctx, dpc_dgraph* g, const float* d_x, float* d_y, const dpc_launch_cfg* cfg,
                         dpc_metrics* met, const float* const* xpeer, uint64_t rows) {
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
  a.xflags = c.flags >> 24;
  a.xpeer = xpeer;
  a.xpull = nullptr;
  a.ncols = static_cast<unsigned>(g->ncols);
  if (xpeer && !(c.flags & DPC_CFG_X_PEER_GATHER)) {
    if (!g->x) return fail(DPC_E_INVALID, "fused SpMV pull mode needs the graph's x buffer");
    a.xpull = g->x;
    a.x = g->x;
  }
  a.rows = static_cast<unsigned>(rows);
  a.rshift = ~0u;
  if (rows && (rows & (rows - 1)) == 0) a.rshift = static_cast<unsigned>(__builtin_ctzll(rows));
  a.coop = 1;
  // grid variant with the cached per-matrix window plan (spmv_plan.cu)
  if (c.variant == DPC_GRID && c.grid_persistent && !xpeer &&
      !(c.flags & (DPC_CFG_SPMV_STREAM | DPC_CFG_GRID_CHUNKED | DPC_CFG_COOP_LAUNCH))) {
    if (!g->hdr_clean || met) {
      st = flush_check(ctx, g);
      if (st != DPC_OK) return st;
      st = begin_run(ctx, g->hdr);
      if (st != DPC_OK) return st;
    }
    int launches = 0;
    if (g->m > 0 || g->n > 0) {
      st = spmv_plan_run(ctx, g, d_x, d_y, c.flags, &launches);
      if (st != DPC_OK) return st;
      DPC_CUDA(cudaGetLastError());
    }
    g->hdr_clean = true;  // the plan kernel writes only fault bits into the header
    if (met) {
      met->host_launches += launches;
      met->edges_processed += g->m;
      met->iterations += 1;
      return finish_metrics(ctx, g->hdr, g->hdr_host, met);
    }
    defer_check(g);
    return DPC_OK;
  }
  // stream-balanced grid drain (grid_stream)
  const bool use_stream = c.variant == DPC_GRID && c.grid_persistent && !(c.flags & DPC_CFG_GRID_CHUNKED);
  if (xpeer && !(use_stream && c.threshold == 0))
    return fail(DPC_E_INVALID, "fused multi-GPU SpMV runs on the grid stream kernel (threshold 0)");
  spmv::Stream sa{};
  if (use_stream) {
    const uint64_t heavy = pool_need(g, c.threshold, 1u << 30);
    st = ensure_pool(g, heavy);
    if (st != DPC_OK) return st;
    // stream positions <= m + 6 per item (16-byte widening)
    st = ensure_stream(g, heavy);
    if (st != DPC_OK) return st;
    sa = spmv::Stream{reinterpret_cast<uint2*>(g->soff), &g->hdr->work, nullptr, nullptr};
  } else if (c.variant != DPC_FLAT && c.variant != DPC_BASIC) {
    st = ensure_pool(g, pool_need(g, c.threshold, c.chunk));
    if (st != DPC_OK) return st;
  }
  a.pool = dev::Pool{g->items, use_stream ? static_cast<unsigned>(std::min<uint64_t>(g->cap, g->soff_cap))
                                          : g->cap};
  st = ensure_pending_for(ctx, g, c.variant, c.threshold, c.parent_threads);
  if (st != DPC_OK) return st;
  if ((c.flags & DPC_CFG_ALLOC_MALLOC) && (c.variant == DPC_WARP || c.variant == DPC_BLOCK)) {
    // device heap for the per-owner buffers (+ one tail launch per owner)
    st = ensure_pending_limit(ctx, 2 * static_cast<size_t>(std::max<int64_t>(g->n / 32, 1)) + 1024);
    if (st != DPC_OK) return st;
    // the device heap is sized once at context creation (kDeviceHeap); a
    // malloc that does not fit raises the overflow fault
  }
  // the stream kernel zeroes its header counters on exit (its last block),
  // so back-to-back stream runs need no per-run memset; their fault bits
  // are sticky until a check reads them (flush_check)
  if (!(use_stream && g->hdr_clean && !met)) {
    st = flush_check(ctx, g);  // the memset below would erase a pending fault
    if (st != DPC_OK) return st;
    st = begin_run(ctx, g->hdr);
    if (st != DPC_OK) return st;
  }
  g->hdr_clean = false;
  const unsigned blocks = std::max(1u, dev::ceil_div(a.n, 256u));
  cudaStream_t s = ctx->stream;
  if (a.n > 0) {
    switch (c.variant) {
      case DPC_FLAT: spmv::flat_kernel<<<blocks, 256, 0, s>>>(a); break;
      case DPC_BASIC: spmv::basic_parent<<<blocks, 256, 0, s>>>(a); break;
      case DPC_WARP:
        if (c.flags & DPC_CFG_ALLOC_MALLOC) spmv::warp_parent_malloc<<<blocks, 256, 0, s>>>(a);
        else spmv::warp_parent<<<blocks, 256, 0, s>>>(a);
        break;
      case DPC_BLOCK:
        if (c.flags & DPC_CFG_ALLOC_MALLOC) spmv::block_parent_malloc<<<blocks, 256, 0, s>>>(a);
        else spmv::block_parent<<<blocks, 256, 0, s>>>(a);
        break;
      case DPC_GRID:
        if (use_stream) {
          const spmv::StreamShape sh = spmv::stream_shape(c.threshold > 0, c.flags);
          const int nb = stream_blocks(ctx, sh);
          if (nb <= 0) return fail(DPC_E_CUDA, "stream kernel does not fit on the device");
          if (sh.slog > 0) {
            st = ensure_xhot(ctx, g, sh.slog);
            if (st != DPC_OK) return st;
          }
          sa.xhot_col = g->xhot_col;
          sa.xhot_val = g->xhot_val;
          // one block per resident slot; all co-resident, so a normal launch
          // with the software grid barrier is safe (cooperative on request)
          a.coop = (c.flags & DPC_CFG_COOP_LAUNCH) ? 1u : 0u;
          void* args[] = {&a, &sa};
          if (a.coop) {
            DPC_CUDA(cudaLaunchCooperativeKernel(sh.fn, dim3(nb), dim3(sh.threads), args, sh.smem, s));
          } else {
            DPC_CUDA(cudaLaunchKernel(sh.fn, dim3(nb), dim3(sh.threads), args, sh.smem, s));
          }
          g->hdr_clean = true;
        } else if (c.grid_persistent) {
          const void* fn = reinterpret_cast<const void*>(spmv::persistent_fn(c.flags));
          int nb = coop_blocks(ctx, fn, 256);
          void* args[] = {&a};
          DPC_CUDA(cudaLaunchCooperativeKernel(fn, dim3(nb), dim3(256), args, 0, s));
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
  defer_check(g);  // fault bits stay in the header until the next check
  return DPC_OK;
}
