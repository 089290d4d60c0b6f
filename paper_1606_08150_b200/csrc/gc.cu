// Graph coloring (GC) in five variants: greedy first-fit in descending
// priority order -- SPEC.md:454's canonical node order (default: "greedy
// first-fit coloring under canonical node order"; :468 determinism), a
// seeded hash order or largest-log-degree-first (see prio()).
//
// Parallel form: data-driven Jones-Plassmann.  cnt[v] = number of
// higher-priority neighbours not yet colored.  A vertex is ready when
// cnt[v] == 0; it takes color mex{color[u] : u higher neighbour} — exactly the
// color sequential greedy gives it, because in sequential order the colored
// neighbours of v are precisely its higher neighbours — and decrements cnt[]
// of its lower neighbours, appending those that reach 0 to the next round's
// frontier.  Output is therefore bit-identical to the sequential oracle for
// every variant and schedule.
//
// Two irregular loops per vertex, both consolidated:
//   init pass  : count higher neighbours (chunk items, warp per chunk, sum)
//   color pass : mex + decrements.  Heavy vertices are split into chunk
//                items too: a warp ORs its chunk's neighbour colors into a
//                shared-memory bitmap and then into the vertex's global
//                bitmap; the warp that finishes the vertex's LAST chunk
//                (per-vertex countdown — the paper's last-block protocol at
//                item granularity) computes the mex and writes the color.
//                basic-dp keeps the paper's per-vertex child (<<<1, T>>>,
//                SoloBlock, shared-memory bitmap).
// Frontier appends and the color-count maximum are block-aggregated.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#ifndef BW_CFG
#define BW_CFG 4
#endif

#include "common.cuh"
#include "ctx.h"

namespace cg = cooperative_groups;

namespace dpc {
namespace gc {

using dev::Item;
using dev::kFull;
using dev::Pool;
using dev::RunHeader;

constexpr unsigned kBitmapWords = 1024;  // SoloBlock window: 32768 colors
constexpr unsigned kVW = 32;             // chunked heavy vertex: 1024-color window
constexpr unsigned kStateWords = 36;     // per heavy vertex: 32 bitmap + remaining + overflow + pad
constexpr unsigned kQueue = 2048;
using Queue = dev::BlockQueue<kQueue>;

struct Ctr {
  unsigned fsize[3];
  unsigned pool[3];
  unsigned iters;
  int maxcolor;
  unsigned pad[8];
};

struct Args {
  const unsigned* __restrict__ rowptr;
  const int* __restrict__ col;
  int* color;
  unsigned* cnt;
  unsigned* front0;
  unsigned* front1;
  unsigned* state;  // kStateWords per pool slot (heavy-vertex bitmaps)
  Ctr* ctr;
  Pool pool;
  RunHeader* hdr;
  unsigned long long seed;
  unsigned n;
  unsigned threshold;
  unsigned chunk;
  unsigned child_threads;
  unsigned child_blocks;
  unsigned it;
  unsigned fsize;
  unsigned long long* trace;  // optional: per-vertex %globaltimer at color write (DPC_TRACE=1)
  unsigned order;             // 0 hash, 1 canonical node order, 2 largest-log-degree-first
  const unsigned long long* __restrict__ parr;  // order 2: per-vertex priority (llf_prio_kernel)
};

struct Block {
  Queue q;
  int maxc;
  unsigned wbm[8][kVW];  // per-warp chunk bitmaps
};

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Greedy order (descending priority, ties: larger id first), one of
//   canonical ~v: nodes 0, 1, ..., n-1 -- SPEC.md:454's GC oracle  default
//   hash      (mix64(v ^ seed), v)                                 DPC_CFG_GC_HASH
//   LLF       (bits(deg v) << 58 | mix64(v ^ seed) >> 6, v): largest-log-degree-first
//             (Hasenplaugh et al., SPAA 2014); precomputed per run   DPC_CFG_GC_LLF
// oracle/oracle.c orc_color_greedy_order restates all three.
__device__ __forceinline__ unsigned long long prio(const Args& a, unsigned v) {
  if (a.order == 1) return ~static_cast<unsigned long long>(v);
  if (a.order == 2) return __ldg(a.parr + v);
  return mix64(static_cast<unsigned long long>(v) ^ a.seed);
}

__global__ void __launch_bounds__(256) llf_prio_kernel(const unsigned* __restrict__ rowptr, unsigned n,
                                                       unsigned long long seed, unsigned long long* parr) {
  for (unsigned v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const unsigned d = __ldg(rowptr + v + 1) - __ldg(rowptr + v);
    const unsigned long long bits = d ? 32u - __clz(d) : 0u;
    parr[v] = (bits << 58) | (mix64(static_cast<unsigned long long>(v) ^ seed) >> 6);
  }
}

// u precedes v in the greedy order
__device__ __forceinline__ bool higher(unsigned u, unsigned long long pu, unsigned v,
                                       unsigned long long pv) {
  return pu > pv || (pu == pv && u > v);
}

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
  if (threadIdx.x == 0) s.maxc = -1;
  __syncthreads();
}

__device__ __forceinline__ void block_end(const Args& a, unsigned it, Block& s) {
  s.q.flush(next_count(a, it), next_front(a, it));
  if (threadIdx.x == 0 && s.maxc >= 0) {
    atomicMax(&a.ctr->maxcolor, s.maxc);
    s.maxc = -1;
  }
  __syncthreads();
}

__device__ __forceinline__ void set_color(const Args& a, Block& s, unsigned v, int c) {
  a.color[v] = c;
  atomicMax(&s.maxc, c);
}

// A count-down past zero: u was released by more higher neighbours than it
// counted -- the adjacency is not symmetric (fault bit 8: DPC_E_INVALID).
__device__ __noinline__ void asymmetric(const Args& a) { atomicOr(&a.hdr->overflow, 8u); }

// Lower neighbour u of a vertex being colored: count down, append when ready.
__device__ __forceinline__ void release(const Args& a, unsigned it, Block& s, unsigned u) {
  const unsigned old = atomicSub(a.cnt + u, 1u);
  if (old == 1u) s.q.push(u, next_count(a, it), next_front(a, it));
  else if (old == 0u) asymmetric(a);
}

// --------------------------------------------------------------- init pass
__device__ __forceinline__ unsigned count_higher(const Args& a, unsigned v, unsigned b, unsigned e,
                                                 unsigned step, unsigned start) {
  const unsigned long long pv = prio(a, v);
  unsigned c = 0;
  for (unsigned k = b + start; k < e; k += step) {
    unsigned u = static_cast<unsigned>(__ldg(a.col + k));
    if (u != v && higher(u, prio(a, u), v, pv)) c++;
  }
  return c;
}

__device__ __forceinline__ void init_drain(const Args& a, const Item* items, unsigned count,
                                           unsigned gwarp, unsigned nwarps) {
  for (unsigned i = gwarp; i < count; i += nwarps) {
    Item t = items[i];
    unsigned e = min(t.begin + a.chunk, __ldg(a.rowptr + t.v + 1));
    unsigned c = dev::warp_sum(count_higher(a, t.v, t.begin, e, 32, dev::lane_id()));
    if (dev::lane_id() == 0 && c) atomicAdd(a.cnt + t.v, c);
  }
}

__global__ void __launch_bounds__(256) init_child(Args a, const Item* items, unsigned count) {
  init_drain(a, items, count, (blockIdx.x * blockDim.x + threadIdx.x) >> 5,
             (gridDim.x * blockDim.x) >> 5);
}

// basic-dp init child: <<<ceil(deg/T), T>>>, one arc per thread
__global__ void __launch_bounds__(256) init_basic_child(Args a, unsigned v, unsigned b, unsigned e) {
  unsigned k = b + blockIdx.x * blockDim.x + threadIdx.x;
  unsigned c = 0;
  if (k < e) {
    unsigned u = static_cast<unsigned>(__ldg(a.col + k));
    c = (u != v && higher(u, prio(a, u), v, prio(a, v))) ? 1u : 0u;
  }
  c = dev::warp_sum(c);
  if (dev::lane_id() == 0 && c) atomicAdd(a.cnt + v, c);
}

// variant: 0 flat, 1 basic, 2 warp, 3 block, 4 grid(CDP) — the init pass
template <int V>
__global__ void __launch_bounds__(256) init_parent(Args a) {
  unsigned v = blockIdx.x * blockDim.x + threadIdx.x, b = 0, e = 0, want = 0;
  if (v < a.n) {
    b = __ldg(a.rowptr + v);
    e = __ldg(a.rowptr + v + 1);
    if (V == 0 || e - b <= a.threshold) {
      a.cnt[v] = count_higher(a, v, b, e, 1, 0);
    } else if (V == 1) {
      init_basic_child<<<dev::ceil_div(e - b, a.child_threads), a.child_threads, 0,
                         cudaStreamFireAndForget>>>(a, v, b, e);
      dev::note_launch(a.hdr);
    } else {
      want = dev::nchunks(e - b, a.chunk);
    }
  }
  if (V == 0 || V == 1) return;
  unsigned bbase, bt;
  unsigned at = dev::block_reserve(&a.ctr->pool[0], want, &bbase, &bt);
  if (want) {
    dev::write_chunks(a.pool, a.hdr, at, v, b, e, a.chunk);
    __threadfence();
  }
  if (V == 3) {
    __syncthreads();
    if (threadIdx.x == 0 && bt && bbase < a.pool.cap) {
      unsigned c = min(bt, a.pool.cap - bbase);
      init_child<<<dev::child_blocks(c, a.child_threads, a.child_blocks), a.child_threads, 0,
                   cudaStreamFireAndForget>>>(a, a.pool.items + bbase, c);
      dev::note_launch(a.hdr);
    }
  } else if (V == 2) {
    const unsigned wb = __shfl_sync(kFull, at, 0), wt = dev::warp_sum(want);
    if (wt) {
      unsigned leader = __ffs(__ballot_sync(kFull, want != 0)) - 1;
      __syncwarp();
      if (dev::lane_id() == leader && wb < a.pool.cap) {
        unsigned c = min(wt, a.pool.cap - wb);
        init_child<<<dev::child_blocks(c, a.child_threads, a.child_blocks), a.child_threads, 0,
                     cudaStreamFireAndForget>>>(a, a.pool.items + wb, c);
        dev::note_launch(a.hdr);
      }
    }
  } else if (dev::grid_last_block(&a.hdr->ticket) && threadIdx.x == 0) {
    unsigned c = min(*reinterpret_cast<volatile unsigned*>(&a.ctr->pool[0]), a.pool.cap);
    if (c) {
      init_child<<<dev::child_blocks(c, a.child_threads, a.child_blocks), a.child_threads, 0,
                   cudaStreamFireAndForget>>>(a, a.pool.items, c);
      dev::note_launch(a.hdr);
    }
  }
}

// frontier 0 = vertices with no higher neighbour
__global__ void __launch_bounds__(256) seed_kernel(Args a) {
  __shared__ Block s;
  block_begin(s);
  for (unsigned v = blockIdx.x * blockDim.x + threadIdx.x; v < a.n; v += gridDim.x * blockDim.x)
    if (a.cnt[v] == 0) s.q.push(v, next_count(a, 0xffffffffu), next_front(a, 0xffffffffu));
  block_end(a, 0xffffffffu, s);
}

// --------------------------------------------------------------- color pass
// Thread-serial color of v (light vertices; the flat variant for all).
__device__ __forceinline__ void color_serial(const Args& a, unsigned it, Block& s, unsigned v,
                                             unsigned b, unsigned e) {
  const unsigned long long pv = prio(a, v);
  unsigned long long used = 0;
  for (unsigned k = b; k < e; k++) {
    unsigned u = static_cast<unsigned>(__ldg(a.col + k));
    if (u == v) continue;
    if (higher(u, prio(a, u), v, pv)) {
      int c = __ldcg(a.color + u);
      if (c < 64) used |= 1ull << c;
    } else {
      release(a, it, s, u);
    }
  }
  int mex;
  if (~used) {
    mex = __ffsll(static_cast<long long>(~used)) - 1;
  } else {  // windowed mex: colors >= 64 (only for high-degree vertices)
    mex = -1;
    for (int base = 64; mex < 0; base += 64) {
      unsigned long long w = 0;
      for (unsigned k = b; k < e; k++) {
        unsigned u = static_cast<unsigned>(__ldg(a.col + k));
        if (u != v && higher(u, prio(a, u), v, pv)) {
          int c = __ldcg(a.color + u) - base;
          if (c >= 0 && c < 64) w |= 1ull << c;
        }
      }
      if (~w) mex = base + __ffsll(static_cast<long long>(~w)) - 1;
    }
  }
  set_color(a, s, v, mex);
}

// Block-cooperative color of v (basic-dp SoloBlock child).  All threads call.
__device__ void color_block(const Args& a, unsigned it, Block& s, unsigned v, unsigned* bm,
                            int* s_mex) {
  const unsigned b = __ldg(a.rowptr + v), e = __ldg(a.rowptr + v + 1);
  const unsigned long long pv = prio(a, v);
  int mex = -1;
  for (int base = 0; mex < 0; base += kBitmapWords * 32) {
    for (unsigned i = threadIdx.x; i < kBitmapWords; i += blockDim.x) bm[i] = 0;
    if (threadIdx.x == 0) *s_mex = 0x7fffffff;
    __syncthreads();
    for (unsigned k = b + threadIdx.x; k < e; k += blockDim.x) {
      unsigned u = static_cast<unsigned>(__ldg(a.col + k));
      if (u == v) continue;
      if (higher(u, prio(a, u), v, pv)) {
        int c = __ldcg(a.color + u) - base;
        if (c >= 0 && c < static_cast<int>(kBitmapWords * 32)) atomicOr(bm + (c >> 5), 1u << (c & 31));
      } else if (base == 0) {
        release(a, it, s, u);
      }
    }
    __syncthreads();
    for (unsigned i = threadIdx.x; i < kBitmapWords; i += blockDim.x) {
      unsigned free_bits = ~bm[i];
      if (free_bits) atomicMin(s_mex, static_cast<int>(i * 32 + __ffs(free_bits) - 1));
    }
    __syncthreads();
    if (*s_mex != 0x7fffffff) mex = base + *s_mex;
    __syncthreads();
  }
  if (threadIdx.x == 0) set_color(a, s, v, mex);
}

__global__ void __launch_bounds__(256) color_basic_child(Args a, unsigned v) {
  __shared__ Block s;
  __shared__ unsigned bm[kBitmapWords];
  __shared__ int s_mex;
  block_begin(s);
  color_block(a, a.it, s, v, bm, &s_mex);
  block_end(a, a.it, s);
}

// Per-vertex state of a chunked heavy vertex: 32-word color bitmap (colors
// < 1024), chunks remaining, overflow flag.  Initialised by the inserting
// thread, owned by the vertex's first chunk slot.
__device__ __forceinline__ void state_init(const Args& a, unsigned slot, unsigned nch) {
  if (slot >= a.pool.cap) return;
  unsigned* st = a.state + static_cast<size_t>(slot) * kStateWords;
  for (unsigned i = 0; i < kVW; i++) st[i] = 0;
  st[kVW] = nch;
  st[kVW + 1] = 0;
}

// Finishes a heavy vertex whose chunks have all been scanned (one warp):
// mex over the global bitmap, or a windowed warp scan when every color
// below 1024 is taken.
__device__ void finish_vertex(const Args& a, Block& s, unsigned v, unsigned* st) {
  const unsigned lane = dev::lane_id();
  unsigned word = __ldcg(st + lane);
  unsigned freeb = ~word;
  unsigned ball = __ballot_sync(kFull, freeb != 0);
  int mex = -1;
  if (ball) {
    unsigned l = __ffs(ball) - 1;
    unsigned fw = __shfl_sync(kFull, freeb, l);
    mex = static_cast<int>(l * 32 + __ffs(fw) - 1);
  } else {
    const unsigned b = __ldg(a.rowptr + v), e = __ldg(a.rowptr + v + 1);
    const unsigned long long pv = prio(a, v);
    for (int base = kVW * 32; mex < 0; base += 32) {
      unsigned w = 0;
      for (unsigned k = b + lane; k < e; k += 32) {
        unsigned u = static_cast<unsigned>(__ldg(a.col + k));
        if (u != v && higher(u, prio(a, u), v, pv)) {
          int c = __ldcg(a.color + u) - base;
          if (c >= 0 && c < 32) w |= 1u << c;
        }
      }
      for (int o = 16; o > 0; o >>= 1) w |= __shfl_xor_sync(kFull, w, o);
      if (~w) mex = base + __ffs(~w) - 1;
    }
  }
  if (lane == 0) set_color(a, s, v, mex);
}

// Chunked color drain: warp per chunk item; the last chunk of a vertex
// finishes it.  Uses the block's per-warp shared bitmaps.
__device__ __forceinline__ void color_chunks(const Args& a, unsigned it, Block& s, const Item* items,
                                             unsigned count, unsigned gwarp, unsigned nwarps) {
  const unsigned lane = dev::lane_id(), wib = dev::warp_in_block();
  unsigned* wbm = s.wbm[wib & 7];
  for (unsigned i = gwarp; i < count; i += nwarps) {
    const Item t = items[i];
    const unsigned b0 = __ldg(a.rowptr + t.v), e0 = __ldg(a.rowptr + t.v + 1);
    const unsigned e = min(t.begin + a.chunk, e0);
    // the vertex's first chunk (absolute pool slot: `items` may be a slice)
    const unsigned slot = static_cast<unsigned>(items - a.pool.items) + i - (t.begin - b0) / a.chunk;
    unsigned* st = a.state + static_cast<size_t>(slot) * kStateWords;
    wbm[lane] = 0;
    __syncwarp();
    const unsigned long long pv = prio(a, t.v);
    bool over = false;
    for (unsigned k = t.begin + lane; k < e; k += 32) {
      unsigned u = static_cast<unsigned>(__ldg(a.col + k));
      if (u == t.v) continue;
      if (higher(u, prio(a, u), t.v, pv)) {
        int c = __ldcg(a.color + u);
        if (c < static_cast<int>(kVW * 32)) atomicOr(wbm + (c >> 5), 1u << (c & 31));
        else over = true;
      } else {
        release(a, it, s, u);
      }
    }
    __syncwarp();
    unsigned wv = wbm[lane];
    if (wv) atomicOr(st + lane, wv);
    if (__any_sync(kFull, over) && lane == 0) atomicOr(st + kVW + 1, 1u);
    __threadfence();
    unsigned last = 0;
    if (lane == 0) last = atomicSub(st + kVW, 1u) == 1u;
    last = __shfl_sync(kFull, last, 0);
    if (last) {
      __threadfence();
      finish_vertex(a, s, t.v, st);
    }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(256) color_child(Args a, const Item* items, unsigned count) {
  __shared__ Block s;
  block_begin(s);
  color_chunks(a, a.it, s, items, count, (blockIdx.x * blockDim.x + threadIdx.x) >> 5,
               (gridDim.x * blockDim.x) >> 5);
  block_end(a, a.it, s);
}

// Parent of one color round.  Heavy vertices -> chunk items + vertex state.
template <int V>
__global__ void __launch_bounds__(256) color_parent(Args a) {
  __shared__ Block s;
  block_begin(s);
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x, v = 0, want = 0, b = 0, e = 0;
  if (i < a.fsize) {
    v = cur_front(a, a.it)[i];
    b = __ldg(a.rowptr + v);
    e = __ldg(a.rowptr + v + 1);
    if (V == 0 || e - b <= a.threshold) {
      color_serial(a, a.it, s, v, b, e);
    } else if (V == 1) {
      color_basic_child<<<1, a.child_threads, 0, cudaStreamFireAndForget>>>(a, v);
      dev::note_launch(a.hdr);
    } else {
      want = dev::nchunks(e - b, a.chunk);
    }
  }
  if (V >= 2) {
    const unsigned slot = a.it % 3;
    unsigned bbase, bt;
    unsigned at = dev::block_reserve(&a.ctr->pool[slot], want, &bbase, &bt);
    if (want) {
      state_init(a, at, want);
      dev::write_chunks(a.pool, a.hdr, at, v, b, e, a.chunk);
      __threadfence();
    }
    if (V == 3) {
      __syncthreads();
      if (threadIdx.x == 0 && bt && bbase < a.pool.cap) {
        unsigned c = min(bt, a.pool.cap - bbase);
        color_child<<<dev::child_blocks(c, a.child_threads, a.child_blocks), a.child_threads, 0,
                      cudaStreamFireAndForget>>>(a, a.pool.items + bbase, c);
        dev::note_launch(a.hdr);
      }
    } else if (V == 2) {
      const unsigned wb = __shfl_sync(kFull, at, 0), wt = dev::warp_sum(want);
      if (wt) {
        unsigned leader = __ffs(__ballot_sync(kFull, want != 0)) - 1;
        __syncwarp();
        if (dev::lane_id() == leader && wb < a.pool.cap) {
          unsigned c = min(wt, a.pool.cap - wb);
          color_child<<<dev::child_blocks(c, a.child_threads, a.child_blocks), a.child_threads, 0,
                        cudaStreamFireAndForget>>>(a, a.pool.items + wb, c);
          dev::note_launch(a.hdr);
        }
      }
    }
  }
  block_end(a, a.it, s);
  if (V == 4 && dev::grid_last_block(&a.hdr->ticket) && threadIdx.x == 0) {
    unsigned c = min(*reinterpret_cast<volatile unsigned*>(&a.ctr->pool[a.it % 3]), a.pool.cap);
    if (c) {
      color_child<<<dev::child_blocks(c, a.child_threads, a.child_blocks), a.child_threads, 0,
                    cudaStreamFireAndForget>>>(a, a.pool.items, c);
      dev::note_launch(a.hdr);
    }
  }
}

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
  // init pass: light vertices inline, heavy -> chunk items in pool[0]
  for (unsigned base = blockIdx.x * blockDim.x; base < a.n; base += stride) {
    unsigned v = base + threadIdx.x, b = 0, e = 0, want = 0;
    if (v < a.n) {
      b = __ldg(a.rowptr + v);
      e = __ldg(a.rowptr + v + 1);
      if (e - b <= a.threshold) a.cnt[v] = count_higher(a, v, b, e, 1, 0);
      else want = dev::nchunks(e - b, a.chunk);
    }
    unsigned bbase, bt;
    unsigned at = dev::block_reserve(&a.ctr->pool[0], want, &bbase, &bt);
    if (want) dev::write_chunks(a.pool, a.hdr, at, v, b, e, a.chunk);
  }
  grid.sync();
  init_drain(a, a.pool.items, min(*reinterpret_cast<volatile unsigned*>(&a.ctr->pool[0]), a.pool.cap),
             gtid >> 5, stride >> 5);
  grid.sync();
  if (gtid == 0) {
    atomicAdd(&a.hdr->aux1, a.ctr->pool[0]);
    a.ctr->pool[0] = 0;
  }
  for (unsigned v = gtid; v < a.n; v += stride)
    if (a.cnt[v] == 0) s.q.push(v, next_count(a, 0xffffffffu), next_front(a, 0xffffffffu));
  block_end(a, 0xffffffffu, s);
  grid.sync();
  unsigned it = 0;
  for (; it < max_iters; it++) {
    const unsigned fs = *reinterpret_cast<volatile unsigned*>(&a.ctr->fsize[it % 3]);
    if (fs == 0) break;
    for (unsigned base = blockIdx.x * blockDim.x; base < fs; base += stride) {
      unsigned i = base + threadIdx.x, v = 0, want = 0, b = 0, e = 0;
      if (i < fs) {
        v = cur_front(a, it)[i];
        b = __ldg(a.rowptr + v);
        e = __ldg(a.rowptr + v + 1);
        if (e - b <= a.threshold) color_serial(a, it, s, v, b, e);
        else want = dev::nchunks(e - b, a.chunk);
      }
      unsigned bbase, bt;
      unsigned at = dev::block_reserve(&a.ctr->pool[it % 3], want, &bbase, &bt);
      if (want) {
        state_init(a, at, want);
        dev::write_chunks(a.pool, a.hdr, at, v, b, e, a.chunk);
      }
    }
    grid.sync();
    unsigned c = min(*reinterpret_cast<volatile unsigned*>(&a.ctr->pool[it % 3]), a.pool.cap);
    color_chunks(a, it, s, a.pool.items, c, gtid >> 5, stride >> 5);
    block_end(a, it, s);
    if (gtid == 0) rotate(a, it);
    grid.sync();
  }
  if (gtid == 0) a.ctr->iters = it;
}

// ---------------------------------------------------------------------------
// Asynchronous grid consolidation (the default grid form).
//
// The round-synchronous forms pay one or two device-wide barriers per JP
// round, and config 3 has ~1700 rounds of a few hundred vertices each: the
// barriers, not the arcs, bound them.  Here the grid-level buffer is a
// device-wide FIFO of ready vertices drained by a persistent grid with no
// barrier between rounds (position p served by warp p mod W): a vertex is colored as soon as its last
// higher-priority neighbour is, so the run time is the longest dependency
// chain times the per-link latency instead of rounds times barrier cost.
//   task queue Q: u64 slots, written once, EMPTY = ~0; one tail counter
//   light vertex (deg <= kAsyncHeavy): one warp: mex of the higher
//     neighbours' colors (shared-memory bitmap), write the color, release
//     the lower neighbours (the one taking a count to 0 enqueues it)
//   heavy vertex: split into chunk tasks -- phase A chunks OR the higher
//     colors into a per-vertex bitmap, the last one computes the mex and
//     writes the color, then enqueues phase B chunks that release the lower
//     neighbours (releases must follow the color write)
// Same coloring as sequential greedy in priority order (see top of file).
// Widths measured on config 3: wider steps (16 edges per lane, 512-edge
// warp tasks) cost registers (72 -> 3 blocks/SM) and ran 35 ms vs 22 ms.
constexpr int kAsyncW = 4;               // edges per lane per step, light vertices
constexpr int kAsyncWide = 4;            // edges per lane per step, medium / chunk tasks
constexpr unsigned kAsyncLight = 128;    // light: one 128-edge step
constexpr unsigned kAsyncHeavy = 128;    // medium (<= this): one warp
constexpr unsigned kAsyncChunk = 128;    // edges per heavy chunk task
constexpr unsigned long long kEmpty = ~0ull;

// Queue counters, one per 128-byte line: thousands of warps poll / bump
// them, and sharing a line would serialise all of them on one L2 slice.
constexpr unsigned kTail = 32, kSlots = 64, kColored = 96, kDeadlock = 128, kDone = 160, kBTail = 192,
                   kBDone = 224;
constexpr unsigned kBlockMax = 4096;  // medium vertices (kAsyncHeavy, kBlockMax] go to a block server
constexpr int kBW = BW_CFG;           // edges per thread per block-server step
// Idle servers sleep between polls.  ncu counts 9.4G instructions (50 % SM
// throughput) for the 18 ms config-3 run, mostly polling, yet longer sleeps
// measured slower (100 ns: 18.2 ms, 400: 18.6, 1500: 19.6): the detection
// delay on the dependency chain costs more than the issue slots.
// Round 2, config 3 canonical / hash (min of 5, two passes): 64 ns 11.41 /
// 16.17 ms, 16 ns 11.35 / 15.96, 4 ns 11.34 / 15.97, 0 ns 11.34 / 15.97.
#ifndef POLL_NS
#define POLL_NS 16
#endif
constexpr unsigned kPollNs = POLL_NS;

struct Async {
  const int* hcol;         // adjacency split per vertex: [b, b + h) higher-priority neighbours, [b + h, e) the rest
  const unsigned* hsplit;  // h per vertex (= the initial pending count)
  unsigned long long* q;   // warp queue: light vertices and chunk tasks
  unsigned* qctr;          // counters, one per 128-byte line (see k* offsets)
  unsigned qcap;
  unsigned* hstate;        // kStateWords per heavy vertex in flight
  unsigned hcap;
  unsigned long long* bq;  // block queue: medium vertices, served by a whole block
  unsigned bqcap;
  unsigned char* vclass;   // per vertex: 0 light, 1 medium (block), 2 heavy (chunked)
  unsigned nbs;            // block servers: blocks [0, nbs)
  unsigned bmax;           // medium vertices have (kAsyncHeavy, bmax] edges
};

// Release / acquire primitives (PTX memory model, gpu scope): a color
// written before a release is visible to whoever acquires the queue slot
// (cumulative through the acq_rel count-down chain), so no full fences sit
// on the critical path.
__device__ __forceinline__ unsigned atom_sub_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(0u - v) : "memory");
  return old;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Task word: vertex (32) | chunk (12) | heavy-state slot + 1 (19) | phase (1).
constexpr unsigned kChunkBits = 12, kSlotBits = 19;
__device__ __forceinline__ unsigned long long task(unsigned v, unsigned chunk, unsigned slot, unsigned phase) {
  return static_cast<unsigned long long>(v) | (static_cast<unsigned long long>(chunk) << 32) |
         (static_cast<unsigned long long>(slot) << (32 + kChunkBits)) | (static_cast<unsigned long long>(phase) << 63);
}

// Warp-aggregated append of the lanes' tasks (want = true) to one queue.
// All lanes call.
__device__ __forceinline__ void append(const Args& a, const Async& q, unsigned long long* qq, unsigned cap,
                                       unsigned tail_off, bool want, unsigned long long t) {
  const unsigned ball = __ballot_sync(kFull, want);
  if (!ball) return;
  const unsigned lane = dev::lane_id();
  unsigned base = 0;
  if (lane == __ffs(ball) - 1) base = atomicAdd(q.qctr + tail_off, __popc(ball));
  base = __shfl_sync(kFull, base, __ffs(ball) - 1);
  if (want) {
    const unsigned at = base + __popc(ball & ((1u << lane) - 1u));
    if (at < cap) {
      // the slot store depends on the count-down's returned value, which
      // follows the (fenced) color stores of every higher neighbour
      *reinterpret_cast<volatile unsigned long long*>(qq + at) = t;
      if (a.trace && (t >> 32) == 0) a.trace[a.n + static_cast<unsigned>(t)] = dev::global_ns();
    } else {
      atomicOr(&a.hdr->overflow, 1u);
      atomicExch(q.qctr + kDeadlock, 1u);
    }
  }
}

// Enqueue of tasks: medium vertex tasks go to the block queue, everything
// else (light vertices, heavy vertices, chunk tasks) to the warp queue.
__device__ __forceinline__ void enqueue(const Args& a, const Async& q, bool want, unsigned long long t,
                                        unsigned cls = 0) {
  const bool blk = want && cls == 1 && (t >> 32) == 0;
  append(a, q, q.q, q.qcap, kTail, want && !blk, t);
  append(a, q, q.bq, q.bqcap, kBTail, blk, t);
}

// Lower neighbours of a colored vertex v among edges [b, e): release each
// (relaxed count-down: the color store was fenced once before), and keep ONE
// vertex that became ready as this warp's next task -- work-first: the
// releaser serves it itself, without a queue round trip -- enqueueing the
// rest.  Four edges per lane per step.  Returns the kept task or kEmpty.
// All lanes call.
// KEEPX: the class this server may not keep (1 for warps: medium vertices
// belong to block servers; 0 for block servers: light ones to warps).
template <int W, unsigned KEEPX = 1>
__device__ __forceinline__ unsigned long long release_range(const Args& a, const Async& q, unsigned v,
                                                            unsigned b, unsigned e, unsigned long long keep) {
  // [b, e) lies in v's lower part of the split adjacency: no priority tests
  for (unsigned k0 = b; k0 < e; k0 += 32 * W) {
    unsigned u[W];
    bool low[W], ready[W];
#pragma unroll
    for (int j = 0; j < W; j++) {
      const unsigned k = k0 + 32 * j + dev::lane_id();
      u[j] = k < e ? static_cast<unsigned>(__ldg(q.hcol + k)) : v;
      low[j] = u[j] != v;
    }
    unsigned cls[W];
#pragma unroll
    for (int j = 0; j < W; j++) cls[j] = low[j] ? q.vclass[u[j]] : 0u;  // issued beside the count-downs
#pragma unroll
    for (int j = 0; j < W; j++) {
      const unsigned old = low[j] ? atomicSub(a.cnt + u[j], 1u) : 2u;
      ready[j] = old == 1u;
      if (old == 0u) asymmetric(a);
    }
#pragma unroll
    for (int j = 0; j < W; j++) {
      if (keep == kEmpty) {  // work-first: keep one this server can take
        const unsigned ball = __ballot_sync(kFull, ready[j] && cls[j] != KEEPX);
        if (ball) {
          const unsigned l = __ffs(ball) - 1;
          keep = task(__shfl_sync(kFull, u[j], l), 0, 0, 0);
          if (dev::lane_id() == l) ready[j] = false;
        }
      }
      enqueue(a, q, ready[j], task(u[j], 0, 0, 0), cls[j]);
    }
  }
  return keep;
}

// ORs the colors of the higher neighbours in [b, e) (a slice of the split
// adjacency's higher part) into the warp bitmap (colors < 32 * kVW); returns
// true (warp-uniform) if a larger color was seen.
template <int W>
__device__ __forceinline__ bool gather_colors(const Args& a, const Async& q, unsigned b, unsigned e,
                                              unsigned* wbm) {
  bool over = false;
  for (unsigned k0 = b; k0 < e; k0 += 32 * W) {
    int c[W];
#pragma unroll
    for (int j = 0; j < W; j++) {
      const unsigned k = k0 + 32 * j + dev::lane_id();
      c[j] = k < e ? static_cast<int>(__ldg(q.hcol + k)) : -1;
    }
#pragma unroll
    for (int j = 0; j < W; j++) c[j] = c[j] >= 0 ? __ldcg(a.color + c[j]) : -1;
#pragma unroll
    for (int j = 0; j < W; j++) {
      if (c[j] >= static_cast<int>(kVW * 32)) over = true;
      else if (c[j] >= 0) atomicOr(wbm + (c[j] >> 5), 1u << (c[j] & 31));
    }
  }
  return __any_sync(kFull, over);
}

// mex of a 32-word bitmap held one word per lane; -1 if all set.
__device__ __forceinline__ int bitmap_mex(unsigned word) {
  const unsigned freeb = ~word;
  const unsigned ball = __ballot_sync(kFull, freeb != 0);
  if (!ball) return -1;
  const unsigned l = __ffs(ball) - 1;
  return static_cast<int>(l * 32 + __ffs(__shfl_sync(kFull, freeb, l)) - 1);
}

// Colors >= 32 * kVW: windowed warp scan over all of v's higher neighbours.
__device__ int mex_windowed(const Args& a, const Async& q, unsigned v) {
  const unsigned b = __ldg(a.rowptr + v), e = b + __ldg(q.hsplit + v);
  for (int base = kVW * 32;; base += 32) {
    unsigned w = 0;
    for (unsigned k = b + dev::lane_id(); k < e; k += 32) {
      const int c = __ldcg(a.color + __ldg(q.hcol + k)) - base;
      if (c >= 0 && c < 32) w |= 1u << c;
    }
    for (int o = 16; o > 0; o >>= 1) w |= __shfl_xor_sync(kFull, w, o);
    if (~w) return base + __ffs(~w) - 1;
  }
}

__device__ __forceinline__ void set_color_async(const Args& a, const Async& q, Block& s, unsigned v, int c) {
  if (dev::lane_id() == 0) {
    __stcg(a.color + v, c);
    if (a.trace) a.trace[v] = dev::global_ns();
    atomicMax(&s.maxc, c);
    __threadfence();  // the color is visible before any count-down it enables
    atomicAdd(q.qctr + kColored, 1u);
  }
  __syncwarp();
}

// Serves one task with the whole warp.  Gathers read v's higher part
// [b, b + h) of the split adjacency, releases its lower part [b + h, e).
__device__ unsigned long long serve(const Args& a, const Async& q, Block& s, unsigned long long t) {
  const unsigned lane = dev::lane_id();
  unsigned* wbm = s.wbm[dev::warp_in_block() & 7];
  const unsigned v = static_cast<unsigned>(t);
  const unsigned chunk = static_cast<unsigned>(t >> 32) & ((1u << kChunkBits) - 1u);
  const unsigned slot = static_cast<unsigned>(t >> (32 + kChunkBits)) & ((1u << kSlotBits) - 1u);
  const bool phase_b = t >> 63;
  const unsigned b = __ldg(a.rowptr + v), e = __ldg(a.rowptr + v + 1);
  const unsigned m = b + __ldg(q.hsplit + v);  // end of the higher part
  if (e - b <= kAsyncHeavy && !phase_b && chunk == 0 && slot == 0) {
    wbm[lane] = 0;
    __syncwarp();
    const bool over = e - b <= kAsyncLight ? gather_colors<kAsyncW>(a, q, b, m, wbm)
                                           : gather_colors<kAsyncWide>(a, q, b, m, wbm);
    __syncwarp();
    int c = bitmap_mex(wbm[lane]);
    if (c < 0 || over) c = c < 0 ? mex_windowed(a, q, v) : c;
    __syncwarp();
    set_color_async(a, q, s, v, c);
    return e - b <= kAsyncLight ? release_range<kAsyncW>(a, q, v, m, e, kEmpty)
                                : release_range<kAsyncWide>(a, q, v, m, e, kEmpty);
  }
  const unsigned ncha = (m - b + kAsyncChunk - 1) / kAsyncChunk;   // gather chunks
  const unsigned nchb = (e - m + kAsyncChunk - 1) / kAsyncChunk;   // release chunks
  if (!phase_b && chunk == 0 && slot == 0) {
    if (ncha == 0) {  // no higher neighbour: color 0, then the release chunks
      set_color_async(a, q, s, v, 0);
      for (unsigned c0 = 0; c0 < nchb; c0 += 32)
        enqueue(a, q, c0 + lane < nchb && c0 + lane > 0, task(v, c0 + lane, 1, 1));
      return release_range<kAsyncWide>(a, q, v, m, min(e, m + kAsyncChunk), kEmpty);
    }
    // heavy vertex: take a state slot, fan out phase A chunks
    unsigned sl = 0;
    if (lane == 0) sl = atomicAdd(q.qctr + kSlots, 1u);
    sl = __shfl_sync(kFull, sl, 0);
    if (sl >= q.hcap) {
      if (lane == 0) atomicOr(&a.hdr->overflow, 1u), atomicExch(q.qctr + kDeadlock, 1u);
      return kEmpty;
    }
    unsigned* st = q.hstate + static_cast<size_t>(sl) * kStateWords;
    if (lane < kVW) st[lane] = 0;
    if (lane == 0) st[kVW] = ncha, st[kVW + 1] = 0;
    __threadfence();
    for (unsigned c0 = 0; c0 < ncha; c0 += 32)
      enqueue(a, q, c0 + lane < ncha, task(v, c0 + lane, sl + 1, 0));
    return kEmpty;
  }
  if (!phase_b) {
    const unsigned cb = b + chunk * kAsyncChunk, ce = min(m, cb + kAsyncChunk);
    unsigned* st = q.hstate + static_cast<size_t>(slot - 1) * kStateWords;
    wbm[lane] = 0;
    __syncwarp();
    const bool over = gather_colors<kAsyncWide>(a, q, cb, ce, wbm);
    __syncwarp();
    const unsigned wv = wbm[lane];
    if (wv) atomicOr(st + lane, wv);
    if (over && lane == 0) atomicOr(st + kVW + 1, 1u);
    __threadfence();
    unsigned last = 0;
    if (lane == 0) last = atomicSub(st + kVW, 1u) == 1u;
    if (!__shfl_sync(kFull, last, 0)) return kEmpty;
    __threadfence();
    int c = bitmap_mex(__ldcg(st + lane));
    if (c < 0 || __ldcg(st + kVW + 1)) c = c < 0 ? mex_windowed(a, q, v) : c;
    set_color_async(a, q, s, v, c);
    // phase B: release chunk 0 by this warp right away, the rest queued
    for (unsigned c0 = 0; c0 < nchb; c0 += 32)
      enqueue(a, q, c0 + lane < nchb && c0 + lane > 0, task(v, c0 + lane, slot, 1));
    return release_range<kAsyncWide>(a, q, v, m, min(e, m + kAsyncChunk), kEmpty);
  }
  const unsigned rb = m + chunk * kAsyncChunk;
  return release_range<kAsyncWide>(a, q, v, rb, min(e, rb + kAsyncChunk), kEmpty);
}

// Whether the asynchronous drain is over (thread-level; call from one lane):
// every vertex colored, a fault raised, or both queues drained with
// vertices left uncolored (asymmetric input).  done counters are read
// before the tails: equal pairs mean nothing was in flight in between.
__device__ bool async_over(const Args& a, const Async& q, unsigned long long* since) {
  volatile unsigned* vq = q.qctr;
  if (vq[kColored] >= a.n || vq[kDeadlock]) return true;
  const unsigned long long now = dev::global_ns();
  if (!*since) *since = now;
  if (now - *since > 2000000000ull) {  // watchdog: the reference's deadlock fault (sim.hpp:946-955)
    atomicOr(&a.hdr->overflow, 4u);
    atomicExch(q.qctr + kDeadlock, 1u);
    return true;
  }
  const unsigned dl = vq[kDone], db = vq[kBDone];
  if (dl == vq[kTail] && db == vq[kBTail] && vq[kColored] < a.n) {
    atomicOr(&a.hdr->overflow, 8u);
    atomicExch(q.qctr + kDeadlock, 1u);
    return true;
  }
  return false;
}

// A medium vertex served by a whole block (block-level consolidation of its
// edge loop): 256 threads gather the higher neighbours' colors (the split
// adjacency's higher part) into a shared bitmap, warp 0 takes the mex and
// writes the color, then every warp releases its share of the lower part.
// All threads call.
__device__ void block_serve(const Args& a, const Async& q, Block& s, unsigned v, unsigned* sbm, unsigned* sflag,
                            unsigned long long* skeep) {
  const unsigned tid = threadIdx.x;
  const unsigned b = __ldg(a.rowptr + v), e = __ldg(a.rowptr + v + 1);
  const unsigned m = b + __ldg(q.hsplit + v);
  // the first release batch's neighbours and classes do not depend on the
  // color: load them before the gather of the higher neighbours' colors,
  // off the dependency chain
  unsigned u[kBW], cls[kBW];
#pragma unroll
  for (int j = 0; j < kBW; j++) {
    const unsigned k = m + j * blockDim.x + tid;
    u[j] = k < e ? static_cast<unsigned>(__ldg(q.hcol + k)) : v;
  }
#pragma unroll
  for (int j = 0; j < kBW; j++) cls[j] = u[j] != v ? q.vclass[u[j]] : 0u;
  if (tid < kVW) sbm[tid] = 0;
  if (tid == 0) *sflag = 0;
  __syncthreads();
  bool over = false;
  for (unsigned k0 = b; k0 < m; k0 += kBW * blockDim.x) {
    int c[kBW];
#pragma unroll
    for (int j = 0; j < kBW; j++) {
      const unsigned k = k0 + j * blockDim.x + tid;
      c[j] = k < m ? static_cast<int>(__ldg(q.hcol + k)) : -1;
    }
#pragma unroll
    for (int j = 0; j < kBW; j++) c[j] = c[j] >= 0 ? __ldcg(a.color + c[j]) : -1;
#pragma unroll
    for (int j = 0; j < kBW; j++) {
      if (c[j] >= static_cast<int>(kVW * 32)) over = true;
      else if (c[j] >= 0) atomicOr(sbm + (c[j] >> 5), 1u << (c[j] & 31));
    }
  }
  if (over) atomicOr(sflag, 1u);
  __syncthreads();
  if (tid < 32) {
    int c = bitmap_mex(sbm[tid]);
    if (c < 0) c = mex_windowed(a, q, v);
    set_color_async(a, q, s, v, c);
  }
  __syncthreads();
  // Only the first kBW * blockDim.x lower edges are released by this block:
  // the rest go out as phase-B release chunks to the warp servers, so the
  // block moves on to the medium vertex it keeps (work-first) without
  // waiting for the whole lower part.
  const unsigned rend = min(e, m + kBW * blockDim.x);
  if (e > rend) {
    const unsigned nchb = (e - m + kAsyncChunk - 1) / kAsyncChunk;
    for (unsigned c0 = (rend - m) / kAsyncChunk; c0 < nchb; c0 += blockDim.x)
      enqueue(a, q, c0 + tid < nchb, task(v, c0 + tid, 1, 1));
  }
  for (unsigned k0 = m; k0 < rend; k0 += kBW * blockDim.x) {
    bool low[kBW], ready[kBW];
    if (k0 != m) {
#pragma unroll
      for (int j = 0; j < kBW; j++) {
        const unsigned k = k0 + j * blockDim.x + tid;
        u[j] = k < rend ? static_cast<unsigned>(__ldg(q.hcol + k)) : v;
        cls[j] = u[j] != v ? q.vclass[u[j]] : 0u;
      }
    }
#pragma unroll
    for (int j = 0; j < kBW; j++) low[j] = u[j] != v;
#pragma unroll
    for (int j = 0; j < kBW; j++) {
      const unsigned old = low[j] ? atomicSub(a.cnt + u[j], 1u) : 2u;
      ready[j] = old == 1u;
      if (old == 0u) asymmetric(a);
    }
#pragma unroll
    for (int j = 0; j < kBW; j++) {
      // work-first: the block keeps one medium vertex it made ready and
      // serves it next, without the block-queue round trip
      if (ready[j] && cls[j] == 1 && *skeep == kEmpty &&
          atomicCAS(skeep, kEmpty, task(u[j], 0, 0, 0)) == kEmpty)
        ready[j] = false;
      enqueue(a, q, ready[j], task(u[j], 0, 0, 0), cls[j]);
    }
  }
}

// Adjacency split by JP priority (init of the asynchronous form): v's
// higher-priority neighbours go to the front of its slice of hcol, the rest
// (lower, self loops) to the back; positions inside each part are free.
// Light vertices: one thread, serial (independent loads, no atomics).
__device__ __forceinline__ unsigned split_serial(const Args& a, const Async& q, unsigned v, unsigned b,
                                                 unsigned e) {
  const unsigned long long pv = prio(a, v);
  int* hcol = const_cast<int*>(q.hcol);
  unsigned h = 0, l = 0;
  for (unsigned k = b; k < e; k++) {
    const unsigned u = static_cast<unsigned>(__ldg(a.col + k));
    if (u != v && higher(u, prio(a, u), v, pv)) hcol[b + h++] = static_cast<int>(u);
    else hcol[e - 1 - l++] = static_cast<int>(u);
  }
  return h;
}

// Heavy vertices: one warp per chunk item of a.chunk edges; the parts'
// fill counters (hpos = hsplit, lpos) are claimed once per chunk.
__device__ __forceinline__ void split_chunk(const Args& a, const Async& q, unsigned* lpos, const Item& t) {
  const unsigned lane = dev::lane_id();
  const unsigned v = t.v, b = __ldg(a.rowptr + v), e = __ldg(a.rowptr + v + 1);
  const unsigned ce = min(t.begin + a.chunk, e);
  const unsigned long long pv = prio(a, v);
  int* hcol = const_cast<int*>(q.hcol);
  unsigned* hpos = const_cast<unsigned*>(q.hsplit);
  for (unsigned k0 = t.begin; k0 < ce; k0 += 32) {
    const unsigned k = k0 + lane;
    const unsigned u = k < ce ? static_cast<unsigned>(__ldg(a.col + k)) : v;
    const bool hi = k < ce && u != v && higher(u, prio(a, u), v, pv);
    const bool lo = k < ce && !hi;
    const unsigned hb = __ballot_sync(kFull, hi), lb = __ballot_sync(kFull, lo);
    unsigned hbase = 0, lbase = 0;
    if (lane == 0) {
      if (hb) hbase = atomicAdd(hpos + v, __popc(hb));
      if (lb) lbase = atomicAdd(lpos + v, __popc(lb));
    }
    hbase = __shfl_sync(kFull, hbase, 0);
    lbase = __shfl_sync(kFull, lbase, 0);
    const unsigned lt = (1u << lane) - 1u;
    if (hi) hcol[b + hbase + __popc(hb & lt)] = static_cast<int>(u);
    if (lo) hcol[e - 1 - (lbase + __popc(lb & lt))] = static_cast<int>(u);
  }
}

__global__ void __launch_bounds__(256) async_persistent(Args a, Async q) {
  __shared__ Block s;
  cg::grid_group grid = cg::this_grid();
  const unsigned stride = gridDim.x * blockDim.x;
  const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned lane = dev::lane_id();
  block_begin(s);
  // init pass: split every adjacency by priority and count the higher
  // neighbours (= pending count): light vertices inline, heavy ones as chunk
  // items drained by warps; vertex classes
  unsigned* lpos = const_cast<unsigned*>(q.hsplit) + a.n;
  for (unsigned base = blockIdx.x * blockDim.x; base < a.n; base += stride) {
    unsigned v = base + threadIdx.x, b = 0, e = 0, want = 0;
    if (v < a.n) {
      b = __ldg(a.rowptr + v);
      e = __ldg(a.rowptr + v + 1);
      if (e - b <= a.threshold) {
        const unsigned h = split_serial(a, q, v, b, e);
        const_cast<unsigned*>(q.hsplit)[v] = h;
        a.cnt[v] = h;
      } else {
        want = dev::nchunks(e - b, a.chunk);
      }
      q.vclass[v] = e - b <= kAsyncHeavy ? 0 : (e - b <= q.bmax && q.nbs ? 1 : 2);
    }
    unsigned bbase, bt;
    unsigned at = dev::block_reserve(&a.ctr->pool[0], want, &bbase, &bt);
    if (want) dev::write_chunks(a.pool, a.hdr, at, v, b, e, a.chunk);
  }
  grid.sync();
  {
    const unsigned cnt = min(*reinterpret_cast<volatile unsigned*>(&a.ctr->pool[0]), a.pool.cap);
    for (unsigned i = gtid >> 5; i < cnt; i += stride >> 5) split_chunk(a, q, lpos, a.pool.items[i]);
  }
  grid.sync();
  for (unsigned v = gtid; v < a.n; v += stride) {
    const unsigned deg = __ldg(a.rowptr + v + 1) - __ldg(a.rowptr + v);
    if (deg > a.threshold) a.cnt[v] = __ldcg(q.hsplit + v);
  }
  grid.sync();
  // seed: every vertex without a higher neighbour is ready
  for (unsigned base = blockIdx.x * blockDim.x; base < a.n; base += stride) {
    const unsigned v = base + threadIdx.x;
    const bool ready = v < a.n && __ldcg(a.cnt + v) == 0;
    enqueue(a, q, ready, task(v, 0, 0, 0), ready ? q.vclass[v] : 0u);
  }
  grid.sync();
  if (blockIdx.x < q.nbs) {
    // block servers: block-queue position p is served by block p mod nbs
    __shared__ unsigned long long s_task, s_keep;
    __shared__ unsigned s_bm[kVW], s_flag;
    if (threadIdx.x == 0) s_keep = kEmpty;
    for (unsigned p = blockIdx.x; p < q.bqcap; p += q.nbs) {
      if (threadIdx.x == 0) {
        unsigned long long t = kEmpty, since = 0;
        unsigned spins = 0;
        while (true) {
          t = *reinterpret_cast<volatile unsigned long long*>(q.bq + p);
          if (t != kEmpty) break;
          if ((++spins & 15) == 0 && async_over(a, q, &since)) break;
          if (spins > 32) __nanosleep(kPollNs);
        }
        s_task = t;
      }
      __syncthreads();
      const unsigned long long t = s_task;
      __syncthreads();
      if (t == kEmpty) break;
      if (a.trace && threadIdx.x == 0) a.trace[2ull * a.n + static_cast<unsigned>(t)] = dev::global_ns();
      block_serve(a, q, s, static_cast<unsigned>(t), s_bm, &s_flag, &s_keep);
      __syncthreads();
      while (true) {  // the work-first chain of kept medium vertices
        const unsigned long long k = s_keep;
        __syncthreads();
        if (k == kEmpty) break;
        if (threadIdx.x == 0) s_keep = kEmpty;
        __syncthreads();
        if (a.trace && threadIdx.x == 0) a.trace[2ull * a.n + static_cast<unsigned>(k)] = dev::global_ns();
        block_serve(a, q, s, static_cast<unsigned>(k), s_bm, &s_flag, &s_keep);
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(q.qctr + kBDone, 1u);
      }
    }
    block_end(a, 0, s);
    return;
  }
  // drain: queue position p is served by warp p mod W, in order (no claim
  // atomics; consecutive tasks land on different warps).  A position is
  // filled by the p-th enqueue, whose producer serves an earlier position,
  // so in-order waiting cannot deadlock.  Stop once every vertex is colored
  // (positions past the last task never fill).
  const unsigned nwarps = (stride - q.nbs * blockDim.x) >> 5, gw = (gtid - q.nbs * blockDim.x) >> 5;
  for (unsigned p = gw; p < q.qcap; p += nwarps) {
    unsigned long long t = kEmpty;
    unsigned spins = 0;
    unsigned long long since = 0;
    while (true) {
      if (lane == 0) t = *reinterpret_cast<volatile unsigned long long*>(q.q + p);
      t = __shfl_sync(kFull, t, 0);
      if (t != kEmpty) break;
      unsigned fin = 0;
      if (lane == 0 && (++spins & 15) == 0) fin = async_over(a, q, &since);
      if (__shfl_sync(kFull, fin, 0)) break;
      if (spins > 32) __nanosleep(kPollNs);
    }
    if (t == kEmpty) break;
    // serve it, then the vertices it makes ready first (work-first chain)
    while (t != kEmpty) {
      if (a.trace && lane == 0 && (t >> 32) == 0) a.trace[2ull * a.n + static_cast<unsigned>(t)] = dev::global_ns();
      t = serve(a, q, s, t);
    }
    if (lane == 0) {
      __threadfence();
      atomicAdd(q.qctr + kDone, 1u);
    }
  }
  block_end(a, 0, s);
}

}  // namespace gc
}  // namespace dpc

using namespace dpc;

extern "C" dpc_status dpc_color_device(dpc_ctx* ctx, dpc_dgraph* g, uint64_t seed,
                                       const dpc_launch_cfg* cfg, dpc_metrics* met) {
  clear_error();
  if (!ctx || !g) return fail(DPC_E_INVALID, "NULL argument");
  if (g->ncols != g->n) return fail(DPC_E_INVALID, "coloring needs a square graph (not a row slice)");
  dpc_status st = flush_check(ctx, g);
  if (st != DPC_OK) return st;
  Cfg c;
  st = resolve_cfg(ctx, DPC_APP_COLOR, cfg, &c);
  if (st != DPC_OK) return st;
  if (c.parent_threads != 256 || c.child_threads != 256)
    return fail(DPC_E_INVALID, "GC kernels are built for parent_threads = child_threads = 256");
  if (!g->ctr) {
    DPC_CUDA(cudaMalloc(&g->ctr, 64));
    DPC_CUDA(cudaMallocHost(&g->ctr_host, 64));
  }
  static_assert(sizeof(gc::Ctr) == 64, "Ctr must fit the 64-byte counter block");
  gc::Args a;
  a.rowptr = g->rowptr;
  a.col = g->col;
  a.color = g->color;
  a.cnt = g->stamp;
  a.front0 = g->front[0];
  a.front1 = g->front[1];
  a.ctr = reinterpret_cast<gc::Ctr*>(g->ctr);
  a.hdr = g->hdr;
  a.seed = seed;
  a.n = static_cast<unsigned>(g->n);
  a.threshold = c.threshold;
  a.chunk = c.chunk;
  a.child_threads = c.child_threads;
  a.child_blocks = c.child_blocks;
  a.it = 0;
  a.fsize = 0;
  a.state = nullptr;
  a.trace = nullptr;
  a.order = (c.flags & DPC_CFG_GC_HASH) ? 0u : (c.flags & DPC_CFG_GC_LLF) ? 2u : 1u;
  a.parr = nullptr;
  if ((c.flags & DPC_CFG_GC_HASH) && (c.flags & DPC_CFG_GC_LLF))
    return fail(DPC_E_INVALID, "DPC_CFG_GC_HASH and DPC_CFG_GC_LLF are exclusive");
  if (const char* tr = getenv("DPC_TRACE")) {
    if (tr[0] == '1') {
      if (!g->trace) DPC_CUDA(cudaMalloc(&g->trace, 3 * sizeof(unsigned long long) * std::max<int64_t>(g->n, 1)));
      a.trace = static_cast<unsigned long long*>(g->trace);
    }
  }
  if (c.variant != DPC_FLAT && c.variant != DPC_BASIC) {
    st = ensure_pool(g, pool_need(g, c.threshold, c.chunk));
    if (st != DPC_OK) return st;
    if (g->gc_state_slots < g->cap) {
      DPC_CUDA(cudaStreamSynchronize(ctx->stream));
      if (g->gc_state) cudaFree(g->gc_state);
      g->gc_state = nullptr;
      g->gc_state_slots = 0;
      DPC_CUDA(cudaMalloc(&g->gc_state, sizeof(unsigned) * gc::kStateWords * g->cap));
      g->gc_state_slots = g->cap;
    }
    a.state = g->gc_state;
  }
  a.pool = dev::Pool{g->items, g->cap};
  st = ensure_pending_for(ctx, g, c.variant, c.threshold, c.parent_threads);
  if (st != DPC_OK) return st;
  g->hdr_clean = false;
  st = begin_run(ctx, g->hdr);
  if (st != DPC_OK) return st;
  cudaStream_t s = ctx->stream;
  const size_t nv = static_cast<size_t>(std::max<int64_t>(g->n, 1));
  DPC_CUDA(cudaMemsetAsync(g->ctr, 0, 64, s));
  DPC_CUDA(cudaMemsetAsync(g->stamp, 0, sizeof(unsigned) * nv, s));
  DPC_CUDA(cudaMemsetAsync(g->color, 0xff, sizeof(int) * nv, s));
  if (a.order == 2 && a.n) {
    if (!g->gc_prio) DPC_CUDA(cudaMalloc(&g->gc_prio, sizeof(unsigned long long) * nv));
    gc::llf_prio_kernel<<<std::min(dev::ceil_div(a.n, 256u), 8u * static_cast<unsigned>(ctx->sms)), 256, 0, s>>>(
        a.rowptr, a.n, a.seed, static_cast<unsigned long long*>(g->gc_prio));
    DPC_CUDA(cudaGetLastError());
    a.parr = static_cast<const unsigned long long*>(g->gc_prio);
  }
  auto* ctr_host = reinterpret_cast<gc::Ctr*>(g->ctr_host);
  int64_t host_launches = 0, iters = 0;
  const unsigned nb = std::max(1u, dev::ceil_div(a.n, 256u));
  if (a.n == 0) {
    ctr_host->maxcolor = -1;
  } else if (c.variant == DPC_GRID && c.grid_persistent && (c.flags & DPC_CFG_GRID_ASYNC)) {
    // asynchronous worklist form: task queue, heavy-vertex states
    const uint64_t heavy = pool_need(g, gc::kAsyncHeavy, 1u << 30);
    if (heavy + 1 >= (1ull << gc::kSlotBits) || static_cast<uint64_t>(g->max_deg) >= (uint64_t{gc::kAsyncChunk} << gc::kChunkBits))
      return fail(DPC_E_OVERFLOW, "asynchronous GC task encoding exceeded (clear DPC_CFG_GRID_ASYNC)");
    const uint64_t qcap = static_cast<uint64_t>(g->n) + 2 * pool_need(g, gc::kAsyncHeavy, gc::kAsyncChunk) + 32;
    const uint64_t bqcap = static_cast<uint64_t>(g->n) + 32;
    // one buffer: [warp queue][1 KB counters][block queue][vertex classes]
    const uint64_t words = qcap + 128 + bqcap + (static_cast<uint64_t>(g->n) + 7) / 8;
    if (g->gc_q_cap < words) {
      DPC_CUDA(cudaStreamSynchronize(s));
      if (g->gc_q) cudaFree(g->gc_q);
      g->gc_q = nullptr;
      g->gc_q_cap = 0;
      DPC_CUDA(cudaMalloc(&g->gc_q, sizeof(unsigned long long) * words));
      g->gc_q_cap = words;
    }
    if (g->gc_hstate_cap < heavy + 1) {
      DPC_CUDA(cudaStreamSynchronize(s));
      if (g->gc_hstate) cudaFree(g->gc_hstate);
      g->gc_hstate = nullptr;
      g->gc_hstate_cap = 0;
      DPC_CUDA(cudaMalloc(&g->gc_hstate, sizeof(unsigned) * gc::kStateWords * (heavy + 1)));
      g->gc_hstate_cap = heavy + 1;
    }
    int per_sm = 0;
    DPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(gc::async_persistent),
                                                  256, 0));
    int blocks = std::max(1, per_sm) * ctx->sms;
    gc::Async q;
    q.q = reinterpret_cast<unsigned long long*>(g->gc_q);
    q.qctr = reinterpret_cast<unsigned*>(q.q + qcap);
    q.qcap = static_cast<unsigned>(qcap);
    q.bq = q.q + qcap + 128;
    q.bqcap = static_cast<unsigned>(bqcap);
    q.vclass = reinterpret_cast<unsigned char*>(q.bq + bqcap);
    q.hstate = g->gc_hstate;
    q.hcap = static_cast<unsigned>(g->gc_hstate_cap);
    // one block server per SM when there are more blocks per SM to host the
    // warp servers (flag bit 19 off); flag bit 19: warp servers only
    q.nbs = (per_sm > 1 && !(c.flags & (1u << 19))) ? static_cast<unsigned>(ctx->sms) : 0u;
    // experiment switch (flag bits 24-27): medium bound = 256 << k, default kBlockMax
    // the block-server bound, measured per order on config 3: canonical /
    // LLF orders put the hubs on the dependency chain, where a whole block
    // (up to 32K edges) beats the chunk-task fan-out (11.88 -> 11.46 ms,
    // 15.2 -> 14.4 ms); the hash order keeps 4096 (16.1 vs 16.5 ms)
    q.bmax = (c.flags >> 24) & 15u ? (256u << ((c.flags >> 24) & 15u))
                                   : (a.order == 0 ? gc::kBlockMax : 8u * gc::kBlockMax);
    DPC_CUDA(cudaMemsetAsync(q.q, 0xff, sizeof(unsigned long long) * (qcap + 128 + bqcap), s));
    DPC_CUDA(cudaMemsetAsync(q.qctr, 0, 1024, s));
    // the adjacency split by this run's priorities (built by the kernel's
    // init pass): hcol (m), hsplit + lpos fill counters (2n, zeroed)
    if (!g->gc_hcol) {
      DPC_CUDA(cudaStreamSynchronize(s));
      DPC_CUDA(cudaMalloc(&g->gc_hcol, sizeof(int) * static_cast<size_t>(std::max<int64_t>(g->m, 1))));
      DPC_CUDA(cudaMalloc(&g->gc_hsplit, sizeof(unsigned) * 2 * nv));
    }
    DPC_CUDA(cudaMemsetAsync(g->gc_hsplit, 0, sizeof(unsigned) * 2 * nv, s));
    q.hcol = g->gc_hcol;
    q.hsplit = g->gc_hsplit;
    void* args[] = {&a, &q};
    DPC_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(gc::async_persistent), dim3(blocks),
                                         dim3(256), args, 0, s));
    host_launches = 1;
    DPC_CUDA(cudaMemcpyAsync(ctr_host, a.ctr, sizeof(gc::Ctr), cudaMemcpyDeviceToHost, s));
    DPC_CUDA(cudaStreamSynchronize(s));
    iters = 1;
  } else if (c.variant == DPC_GRID && c.grid_persistent) {
    int per_sm = 0;
    DPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(gc::grid_persistent),
                                                  256, 0));
    int blocks = std::max(1, per_sm) * ctx->sms;
    unsigned max_iters = a.n + 1;
    void* args[] = {&a, &max_iters};
    DPC_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(gc::grid_persistent),
                                         dim3(blocks), dim3(256), args, 0, s));
    host_launches = 1;
    DPC_CUDA(cudaMemcpyAsync(ctr_host, a.ctr, sizeof(gc::Ctr), cudaMemcpyDeviceToHost, s));
    DPC_CUDA(cudaStreamSynchronize(s));
    iters = ctr_host->iters;
  } else {
    switch (c.variant) {
      case DPC_FLAT: gc::init_parent<0><<<nb, 256, 0, s>>>(a); break;
      case DPC_BASIC: gc::init_parent<1><<<nb, 256, 0, s>>>(a); break;
      case DPC_WARP: gc::init_parent<2><<<nb, 256, 0, s>>>(a); break;
      case DPC_BLOCK: gc::init_parent<3><<<nb, 256, 0, s>>>(a); break;
      default: gc::init_parent<4><<<nb, 256, 0, s>>>(a); break;
    }
    DPC_CUDA(cudaGetLastError());
    // pool slot 0 is reused by round 0: clear it after the init children ran
    DPC_CUDA(cudaMemsetAsync(&a.ctr->pool[0], 0, sizeof(unsigned), s));
    gc::seed_kernel<<<std::min(nb, 4u * static_cast<unsigned>(ctx->sms)), 256, 0, s>>>(a);
    host_launches += 2;
    DPC_CUDA(cudaGetLastError());
    DPC_CUDA(cudaMemcpyAsync(&ctr_host->fsize[0], &a.ctr->fsize[0], sizeof(unsigned),
                             cudaMemcpyDeviceToHost, s));
    DPC_CUDA(cudaStreamSynchronize(s));
    unsigned fsize = ctr_host->fsize[0];
    for (unsigned it = 0; fsize > 0 && it <= a.n; it++) {
      a.it = it;
      a.fsize = fsize;
      const unsigned pb = std::max(1u, dev::ceil_div(fsize, 256u));
      switch (c.variant) {
        case DPC_FLAT: gc::color_parent<0><<<pb, 256, 0, s>>>(a); break;
        case DPC_BASIC: gc::color_parent<1><<<pb, 256, 0, s>>>(a); break;
        case DPC_WARP: gc::color_parent<2><<<pb, 256, 0, s>>>(a); break;
        case DPC_BLOCK: gc::color_parent<3><<<pb, 256, 0, s>>>(a); break;
        default: gc::color_parent<4><<<pb, 256, 0, s>>>(a); break;
      }
      gc::rotate_kernel<<<1, 32, 0, s>>>(a);
      host_launches += 2;
      DPC_CUDA(cudaGetLastError());
      DPC_CUDA(cudaMemcpyAsync(&ctr_host->fsize[(it + 1) % 3], &a.ctr->fsize[(it + 1) % 3],
                               sizeof(unsigned), cudaMemcpyDeviceToHost, s));
      DPC_CUDA(cudaStreamSynchronize(s));
      fsize = ctr_host->fsize[(it + 1) % 3];
      iters = it + 1;
    }
    DPC_CUDA(cudaMemcpyAsync(ctr_host, a.ctr, sizeof(gc::Ctr), cudaMemcpyDeviceToHost, s));
    DPC_CUDA(cudaStreamSynchronize(s));
  }
  DPC_CUDA(cudaMemcpyAsync(g->hdr_host, g->hdr, sizeof(dev::RunHeader), cudaMemcpyDeviceToHost, s));
  DPC_CUDA(cudaStreamSynchronize(s));
  st = check_header(g->hdr_host);
  if (st != DPC_OK) return st;
  if (met) {
    met->child_launch_count += g->hdr_host->launches;
    met->host_launches += host_launches;
    met->iterations += iters;
    met->edges_processed += 2 * g->m;
    met->buffer_items_inserted += g->hdr_host->aux1;
    met->pool_peak = std::max<int64_t>(met->pool_peak, g->hdr_host->count);
    met->result_count = ctr_host->maxcolor + 1;
  }
  return DPC_OK;
}

