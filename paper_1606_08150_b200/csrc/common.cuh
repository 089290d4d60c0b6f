// Device-side consolidation runtime primitives (sm_100a).
//
// These are the B200 realisation of the dp_* builtins the reference's
// transform emits (transform.hpp:478-632) and the simulator executes
// (sim.hpp:1409-1541, 1665-1717):
//   dp_buffers / own_buffer  -> one pre-allocated pool per graph (Pool), owner
//                               slices reserved by a bump pointer (a3, a6)
//   dp_insert                -> warp_reserve / block_reserve: ballot-free warp
//                               scan + one atomicAdd per warp / block (a5)
//   dp_grid_last             -> grid_last_block(): fence + ticket (a10)
//   device launch            -> CDP2 fire-and-forget launch by an elected
//                               live lane, counted in RunHeader.launches (a7)
//   dp_buf_count/get         -> the child kernel's (items, count) arguments
#pragma once

#include <cooperative_groups.h>
#include <cstdint>

namespace dpc {
namespace dev {

constexpr unsigned kFull = 0xffffffffu;

// Per-run device counters; zeroed by one cudaMemsetAsync per run.
struct RunHeader {
  unsigned count;      // items reserved in the pool (grid-level worklist size)
  unsigned overflow;   // bit0: pool overflow, bit1: device launch failed
  unsigned launches;   // device-side child launches
  unsigned ticket;     // grid-level last-block ticket (sim.hpp:1708-1717)
  unsigned next_count; // next frontier size (SSSP / GC)
  unsigned iter;       // iteration counter (device-driven loops)
  unsigned aux0;       // app-specific
  unsigned aux1;
  unsigned long long work; // edges processed (diagnostic)
  unsigned long long t[3]; // %globaltimer stamps (ns): start, barrier, end (persistent kernels)
  unsigned long long bar;  // grid_sync64 arrivals of this run (monotonic; zeroed with the header)
};
static_assert(sizeof(RunHeader) == 72, "RunHeader must be 72 bytes");

// A consolidation work item: vertex/row id and the first edge of its chunk.
// The chunk covers [begin, min(begin + chunk, rowptr[v + 1])).
struct Item {
  unsigned v;
  unsigned begin;
};

// Pre-allocated pool (Fig. 5 "pre-alloc" allocator): no device
// malloc on the hot path; owners get contiguous slices by bump allocation.
struct Pool {
  Item* items;
  unsigned cap;
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned warp_in_block() { return threadIdx.x >> 5; }

// Inclusive warp scan (all 32 lanes must call).
__device__ __forceinline__ unsigned warp_incl_scan(unsigned v) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned t = __shfl_up_sync(kFull, v, o);
    if (lane >= static_cast<unsigned>(o)) v += t;
  }
  return v;
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Warp-aggregated reservation (dp_insert at warp granularity): each lane asks
// for `want` slots; one atomicAdd per warp.  Returns this lane's first slot
// and writes the warp's base / total to *wbase / *wtotal.  All 32 lanes call.
__device__ __forceinline__ unsigned warp_reserve(unsigned* counter, unsigned want,
                                                 unsigned* wbase, unsigned* wtotal) {
  unsigned incl = warp_incl_scan(want);
  unsigned total = __shfl_sync(kFull, incl, 31);
  unsigned base = 0;
  if (lane_id() == 31 && total) base = atomicAdd(counter, total);
  base = __shfl_sync(kFull, base, 31);
  *wbase = base;
  *wtotal = total;
  return base + incl - want;
}

// Block-wide exclusive scan of `want` through shared memory (blockDim.x is a
// multiple of 32, <= 1024).  Returns this thread's offset inside the block and
// the block total in *btotal.  All threads call.
__device__ __forceinline__ unsigned block_excl_scan(unsigned want, unsigned* btotal) {
  __shared__ unsigned s_warp[33];  // 32 warp offsets + the block total (a 1024-thread block has 32 warps)
  unsigned incl = warp_incl_scan(want);
  const unsigned w = warp_in_block(), nw = blockDim.x >> 5;
  if (lane_id() == 31) s_warp[w] = incl;
  __syncthreads();
  if (w == 0) {
    unsigned x = lane_id() < nw ? s_warp[lane_id()] : 0;
    unsigned xi = warp_incl_scan(x);
    if (lane_id() < nw) s_warp[lane_id()] = xi - x;  // exclusive warp offsets
    if (lane_id() == 31) s_warp[32] = xi;             // lane 31 holds the total
  }
  __syncthreads();
  unsigned off = s_warp[w] + incl - want;
  *btotal = s_warp[32];
  __syncthreads();  // s_warp is reused by the next call
  return off;
}

// Block-aggregated reservation (dp_insert with one global atomic per block):
// same-address global atomics serialise at ~0.7 ns each on B200
// (tools/probes/atomics_sync), so a per-warp atomic on one counter costs
// ~20 us per 30K warps.  Returns this thread's first slot; *bbase / *btotal
// receive the block's slice.  All threads call; ends with a barrier.
__device__ __forceinline__ unsigned block_reserve(unsigned* counter, unsigned want,
                                                  unsigned* bbase, unsigned* btotal) {
  __shared__ unsigned s_base;
  unsigned off = block_excl_scan(want, btotal);
  if (threadIdx.x == 0) s_base = *btotal ? atomicAdd(counter, *btotal) : 0u;
  __syncthreads();
  *bbase = s_base;
  unsigned at = s_base + off;
  __syncthreads();  // s_base is reused by the next call
  return at;
}

// Two block-aggregated reservations at once (one scan pass, both global
// atomics issued back to back by one thread): *at_a / *at_b receive this
// thread's first slots on counters ca / cb.  All threads call; ends with a
// barrier.
__device__ __forceinline__ void block_reserve2(unsigned* ca, unsigned wa, unsigned* cb, unsigned wb,
                                               unsigned* at_a, unsigned* at_b, unsigned* base_b = nullptr,
                                               unsigned* tot_b = nullptr) {
  __shared__ unsigned s_a[32], s_b[32], s_base[2], s_totb;
  const unsigned ia = warp_incl_scan(wa), ib = warp_incl_scan(wb);
  const unsigned w = warp_in_block(), nw = blockDim.x >> 5;
  if (lane_id() == 31) s_a[w] = ia, s_b[w] = ib;
  __syncthreads();
  if (w == 0) {
    const unsigned x = lane_id() < nw ? s_a[lane_id()] : 0, y = lane_id() < nw ? s_b[lane_id()] : 0;
    const unsigned xi = warp_incl_scan(x), yi = warp_incl_scan(y);
    if (lane_id() < nw) s_a[lane_id()] = xi - x, s_b[lane_id()] = yi - y;
    if (lane_id() == 31) {
      const unsigned ba = xi ? atomicAdd(ca, xi) : 0u;
      const unsigned bb = yi ? atomicAdd(cb, yi) : 0u;
      s_base[0] = ba, s_base[1] = bb, s_totb = yi;
    }
  }
  __syncthreads();
  *at_a = s_base[0] + s_a[w] + ia - wa;
  *at_b = s_base[1] + s_b[w] + ib - wb;
  if (base_b) *base_b = s_base[1];
  if (tot_b) *tot_b = s_totb;
  __syncthreads();  // the shared slots are reused by the next call
}

// Block-local append queue in shared memory: pushes are shared-memory
// atomics; flush() publishes the block's items with ONE global atomic.  A
// push that finds the queue full spills straight to global memory.
template <unsigned CAP>
struct BlockQueue {
  unsigned n;
  unsigned base;
  unsigned items[CAP];

  __device__ __forceinline__ void init() {
    if (threadIdx.x == 0) n = 0;
  }
  __device__ __forceinline__ void push(unsigned v, unsigned* gcount, unsigned* gdst) {
    cooperative_groups::coalesced_group g = cooperative_groups::coalesced_threads();
    unsigned s = 0;
    if (g.thread_rank() == 0) s = atomicAdd(&n, g.size());
    s = g.shfl(s, 0) + g.thread_rank();
    if (s < CAP) {
      items[s] = v;
    } else {
      unsigned gs = atomicAdd(gcount, 1u);
      gdst[gs] = v;
    }
  }
  // Appends v unless the queue is full (then the caller places it itself).
  __device__ __forceinline__ bool try_push(unsigned v) {
    cooperative_groups::coalesced_group g = cooperative_groups::coalesced_threads();
    unsigned s = 0;
    if (g.thread_rank() == 0) s = atomicAdd(&n, g.size());
    s = g.shfl(s, 0) + g.thread_rank();
    if (s < CAP) items[s] = v;
    return s < CAP;
  }
  // All threads of the block call (uniform control flow).
  __device__ __forceinline__ void flush(unsigned* gcount, unsigned* gdst) {
    __syncthreads();
    const unsigned cnt = n < CAP ? n : CAP;
    if (threadIdx.x == 0) base = cnt ? atomicAdd(gcount, cnt) : 0u;
    __syncthreads();
    for (unsigned i = threadIdx.x; i < cnt; i += blockDim.x) gdst[base + i] = items[i];
    __syncthreads();
    if (threadIdx.x == 0) n = 0;
    __syncthreads();
  }
};

// Block-level sum / max accumulators flushed with one global atomic.
__device__ __forceinline__ void block_add_u64(unsigned long long* smem_acc, unsigned v) {
  unsigned s = warp_sum(v);
  if (lane_id() == 0 && s) atomicAdd(smem_acc, static_cast<unsigned long long>(s));
}

// Writes the chunk items of vertex v (edges [b, e)) starting at slot `at`.
// Slots past the pool capacity set the overflow flag (sim.hpp:1512-1517
// turns overflow into a fault; we report it as DPC_E_OVERFLOW).
__device__ __forceinline__ void write_chunks(const Pool& pool, RunHeader* hdr, unsigned at,
                                             unsigned v, unsigned b, unsigned e, unsigned chunk) {
  for (unsigned s = b; s < e; s += chunk, at++) {
    if (at < pool.cap) pool.items[at] = Item{v, s};
    else atomicOr(&hdr->overflow, 1u);
  }
}

__device__ __forceinline__ unsigned nchunks(unsigned deg, unsigned chunk) {
  return (deg + chunk - 1) / chunk;
}

// Grid-level last-block election (the paper's global barrier counter,
// PAPER.md:248; sim.hpp:1708-1717).  Every block calls once after its
// insertions; returns true in all threads of exactly one block — the last to
// arrive — with all other blocks' pool writes visible.  The ticket is reset by
// the last block so the next parent grid can reuse it.
__device__ __forceinline__ bool grid_last_block(unsigned* ticket) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();  // release this block's items before taking a ticket
    unsigned t = atomicAdd(ticket, 1u);
    s_last = (t == gridDim.x - 1);
    if (s_last) {
      __threadfence();  // acquire: all other blocks' items are now visible
      *ticket = 0;
    }
  }
  __syncthreads();
  return s_last;
}

// Fault bit of a device-wide barrier that timed out (RunHeader.overflow):
// reported as DPC_E_DEADLOCK, the reference's deadlock fault (sim.hpp:946-955).
constexpr unsigned kFaultBarrier = 16u;

// Device-wide barrier for a grid whose blocks are all co-resident (checked
// by the host with the occupancy calculator before a normal launch): the
// paper's custom global barrier without the cooperative
// launch's extra setup cost.  `count` is zero at kernel start and used once.
// If the grid is not co-resident after all (another context on the GPU, MPS)
// the watchdog fires after 2 s: the block proceeds so the device never hangs,
// and the run is marked failed (kFaultBarrier in *fault) -- its result is
// never reported as valid.
__device__ __forceinline__ void soft_grid_barrier(unsigned* count, unsigned* fault) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(count, 1u);
    unsigned seen;
    const unsigned long long t0 = global_ns();
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(count) : "memory");
      if (seen < gridDim.x) __nanosleep(20);
      if (global_ns() - t0 > 2000000000ull) {  // watchdog: never hang the device
        atomicOr(fault, kFaultBarrier);
        break;
      }
    } while (seen < gridDim.x);
  }
  __syncthreads();
}

// Reusable device-wide barrier (generation counting): `count` and `gen` are
// zero at kernel start; the last block to arrive resets the count and bumps
// the generation the others wait on.
__device__ __forceinline__ void soft_grid_sync(unsigned* count, unsigned* gen, unsigned* watchdog) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g0;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g0) : "l"(gen) : "memory");
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      *reinterpret_cast<volatile unsigned*>(count) = 0;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      unsigned g;
      const unsigned long long t0 = global_ns();
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
        if (g == g0) __nanosleep(20);
        if (global_ns() - t0 > 2000000000ull) {  // watchdog: a block never arrived
          atomicOr(watchdog, 4u);
          break;
        }
      } while (g == g0);
    }
  }
  __syncthreads();
}

// Device-wide barrier on a monotonic 64-bit arrival count (zero when the
// kernel starts, every block arrives once per round): thread 0 arrives with
// one release atomic, derives its round's target from the count it saw, and
// polls (acquire) until all blocks of the round are in -- one atomic round
// trip plus the poll, no reset and no second counter.  B200, 2000 rounds:
// 1.20 us vs 1.95 us for soft_grid_sync at 296 x 512, 2.09 vs 2.77 us at
// 1184 x 256, 1.24 vs 1.91 us at 148 x 1024; cooperative groups' grid.sync
// 1.21 / 2.41 / 1.22 us (tools/probes/lab_r02/barrier_probe.cu).  Same
// watchdog as soft_grid_sync.
__device__ __forceinline__ void grid_sync64(unsigned long long* count, unsigned* watchdog) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long old, seen;
    asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(count) : "memory");
    const unsigned long long target = (old / gridDim.x + 1) * gridDim.x;
    const unsigned long long t0 = global_ns();
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(seen) : "l"(count) : "memory");
      if (seen >= target) break;
      __nanosleep(20);
      if (global_ns() - t0 > 2000000000ull) {  // watchdog: a block never arrived
        atomicOr(watchdog, 4u);
        break;
      }
    }
  }
  __syncthreads();
}

// Records a device-side launch, flags a failed one (first error code kept in
// aux0 so the host can name it).
__device__ __forceinline__ void note_launch(RunHeader* hdr) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    atomicOr(&hdr->overflow, 2u);
    atomicCAS(&hdr->aux0, 0u, static_cast<unsigned>(e));
  } else {
    atomicAdd(&hdr->launches, 1u);
  }
}


__host__ __device__ __forceinline__ unsigned ceil_div(unsigned a, unsigned b) { return (a + b - 1) / b; }

// Child geometry for `items` chunk items, one warp per item: "1-1" sizing
// capped at `max_blocks` (KC_X cap from the measured table).
__device__ __forceinline__ unsigned child_blocks(unsigned items, unsigned threads,
                                                 unsigned max_blocks) {
  unsigned b = ceil_div(items, threads / 32u);
  if (max_blocks && b > max_blocks) b = max_blocks;
  return b ? b : 1u;
}

}  // namespace dev
}  // namespace dpc
