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
#include <cstdio>
#include <cstdlib>
#include <vector>

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
  // vertex partition (multi-GPU): this rank owns global
  // vertices [r0, r0 + n); single GPU: r0 = 0 and nothing is remote.
  unsigned r0;
  unsigned rows_per_rank;  // owner(v) = v / rows_per_rank
  unsigned* rdist;         // best distance sent so far per global vertex (remote filter)
  uint2* sendbuf;          // [world][sendcap] {global vertex, distance}
  unsigned* sendcnt;       // [world]
  unsigned sendcap;
  unsigned coop;           // grid_persistent1: cooperative launch (grid.sync) vs soft barrier
  unsigned classify;       // grid_persistent1: next-level vertices are classified at push time
  unsigned long long* ptrace;  // optional phase timeline (DPC_SSSP_PHASES=1): per level, max over blocks
  const struct Peer* peers;    // fused multi-GPU relaxation: every rank's buffers (nullptr = send buffers)
  uint2* fbe0;                 // classify form: {row start, row end} of each light-list entry (front0 / front1)
  uint2* fbe1;
  unsigned m;                  // edges (bound of the drain's speculative col / w loads)
};

// One rank's SSSP buffers as seen from this process (own or IPC-mapped):
// the fused form relaxes remote vertices straight into their owner's
// distance / stamp / next-frontier arrays (NVLink peer atomics).
struct Peer {
  unsigned* dist;
  unsigned* stamp;
  unsigned* front0;
  unsigned* front1;
  Ctr* ctr;
};

__device__ void spill_classify(const Args& a, unsigned it, unsigned v);

// Edge weight; BFS (a.w == nullptr) is SSSP with unit weights: its levels are
// the unit-weight distances (the reference's BFS-Rec benchmark).
__device__ __forceinline__ unsigned edge_w(const Args& a, unsigned k) {
  return a.w ? static_cast<unsigned>(__ldg(a.w + k)) : 1u;
}

// Per-block state every relaxing kernel carries in shared memory.
constexpr unsigned kCoopW = 256;  // cooperative chunk writing in the flush (blocks up to this size)

struct Block {
  Queue q;
  unsigned long long work;
  unsigned coff[kCoopW], cv[kCoopW], cb[kCoopW];  // flush: per-thread chunk offsets, vertices, row starts
};

__device__ __forceinline__ unsigned* cur_front(const Args& a, unsigned it) {
  return (it & 1) ? a.front1 : a.front0;
}
__device__ __forceinline__ unsigned* next_front(const Args& a, unsigned it) {
  return (it & 1) ? a.front0 : a.front1;
}
__device__ __forceinline__ uint2* cur_fbe(const Args& a, unsigned it) {
  return (it & 1) ? a.fbe1 : a.fbe0;
}
__device__ __forceinline__ uint2* next_fbe(const Args& a, unsigned it) {
  return (it & 1) ? a.fbe0 : a.fbe1;
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

// Remote relaxation (multi-GPU): the candidate distance of a vertex another
// rank owns is min-filtered against the best one already sent and appended
// to that rank's send buffer; the owner applies it after the exchange.
__device__ __noinline__ void relax_remote(const Args& a, unsigned v, unsigned nd) {
  if (nd >= __ldcg(a.rdist + v) || nd >= atomicMin(a.rdist + v, nd)) return;
  const unsigned d = v / a.rows_per_rank;
  const unsigned slot = atomicAdd(a.sendcnt + d, 1u);
  if (slot < a.sendcap) a.sendbuf[static_cast<size_t>(d) * a.sendcap + slot] = make_uint2(v, nd);
  else atomicOr(&a.hdr->overflow, 1u);
}

// Fused remote relaxation: atomicMin on the owner's distance, the owner's
// stamp for dedup, and an append to the owner's next frontier (system-scope
// atomics on peer memory; the level's peer barrier publishes them).
__device__ __noinline__ void relax_peer(const Args& a, unsigned it, unsigned gv, unsigned nd) {
  const unsigned o = gv / a.rows_per_rank, l = gv - o * a.rows_per_rank;
  const Peer& p = a.peers[o];
  if (nd >= __ldcv(p.dist + l)) return;
  const unsigned old = atomicMin_system(p.dist + l, nd);
  if (nd < old && atomicExch_system(p.stamp + l, it + 1) != it + 1) {
    const unsigned slot = atomicAdd_system(&p.ctr->fsize[(it + 1) % 3], 1u);
    ((it & 1) ? p.front0 : p.front1)[slot] = l;
  }
}

__device__ __forceinline__ void relax(const Args& a, unsigned it, Block& s, unsigned gv,
                                      unsigned nd) {
  const unsigned v = gv - a.r0;  // local index (wraps for vertices below r0)
  if (v >= a.n) {
    if (a.peers) relax_peer(a, it, gv, nd);
    else relax_remote(a, gv, nd);
    return;
  }
  if (nd < __ldcg(a.dist + v)) {
    unsigned old = atomicMin(a.dist + v, nd);
    if (nd < old && atomicExch(a.stamp + v, it + 1) != it + 1) {
      if (!a.classify) s.q.push(v, next_count(a, it), next_front(a, it));
      else if (!s.q.try_push(v)) spill_classify(a, it, v);
    }
  }
}

// One-barrier form, shared queue full: classify v for level it+1 right here
// (heavy -> chunk items in pool half (it+1) % 2, light -> next list).
__device__ __noinline__ void spill_classify(const Args& a, unsigned it, unsigned v) {
  const unsigned b = __ldg(a.rowptr + v), e = __ldg(a.rowptr + v + 1);
  const unsigned nxt = (it + 1) % 3;
  if (e - b > a.threshold) {
    const unsigned nch = dev::nchunks(e - b, a.chunk);
    const unsigned at = atomicAdd(&a.ctr->pool[nxt], nch);
    const dev::Pool p{a.pool.items + ((it + 1) % 2) * a.pool.cap, a.pool.cap};
    dev::write_chunks(p, a.hdr, at, v, b, e, a.chunk);
  } else {
    const unsigned at = atomicAdd(&a.ctr->fsize[nxt], 1u);
    next_front(a, it)[at] = v;
    next_fbe(a, it)[at] = make_uint2(b, e);
  }
}

__device__ __forceinline__ void relax_edge(const Args& a, unsigned it, Block& s, unsigned du,
                                           unsigned k) {
  unsigned long long nd = static_cast<unsigned long long>(du) + edge_w(a, k);
  if (nd < kInf) relax(a, it, s, static_cast<unsigned>(__ldg(a.col + k)), static_cast<unsigned>(nd));
}

__device__ __forceinline__ void relax_serial(const Args& a, unsigned it, Block& s, unsigned du,
                                             unsigned b, unsigned e) {
  for (unsigned k = b; k < e; k++) relax_edge(a, it, s, du, k);
}

// Warp-cooperative relaxation of edges [b, e) of a vertex at distance du.
// The part of relax() after the distance load (cur = dist[v] already read).
__device__ __forceinline__ void relax_loaded(const Args& a, unsigned it, Block& s, unsigned gv, unsigned nd,
                                             unsigned cur) {
  const unsigned v = gv - a.r0;
  if (v >= a.n) {
    if (a.peers) relax_peer(a, it, gv, nd);
    else relax_remote(a, gv, nd);
    return;
  }
  if (nd < cur) {
    const unsigned old = atomicMin(a.dist + v, nd);
    if (nd < old && atomicExch(a.stamp + v, it + 1) != it + 1) {
      if (!a.classify) s.q.push(v, next_count(a, it), next_front(a, it));
      else if (!s.q.try_push(v)) spill_classify(a, it, v);
    }
  }
}

// Relaxes K candidate edges held by this lane with the dependent atomics of
// all K in flight together: every atomicMin, then every stamp exchange of
// the improved ones, then the frontier pushes (two atomic round trips for K
// edges instead of 2K).  g = target (global id), nd = candidate distance
// (>= kInf: none), c = the target's distance read earlier.
template <int K>
__device__ __forceinline__ void relax_k(const Args& a, unsigned it, Block& s, const unsigned (&g)[K],
                                        const unsigned long long (&nd)[K], const unsigned (&c)[K]) {
  unsigned old[K];
#pragma unroll
  for (int k = 0; k < K; k++) {
    old[k] = 0u;
    const unsigned v = g[k] - a.r0;
    if (nd[k] < kInf && v >= a.n) relax_loaded(a, it, s, g[k], static_cast<unsigned>(nd[k]), c[k]);  // remote
    else if (nd[k] < c[k]) old[k] = atomicMin(a.dist + v, static_cast<unsigned>(nd[k]));
  }
  unsigned st[K];
#pragma unroll
  for (int k = 0; k < K; k++) {
    const unsigned v = g[k] - a.r0;
    st[k] = it + 1;
    if (v < a.n && nd[k] < old[k]) st[k] = atomicExch(a.stamp + v, it + 1);
  }
#pragma unroll
  for (int k = 0; k < K; k++) {
    if (st[k] != it + 1) {
      const unsigned v = g[k] - a.r0;
      if (!a.classify) s.q.push(v, next_count(a, it), next_front(a, it));
      else if (!s.q.try_push(v)) spill_classify(a, it, v);
    }
  }
}

// Two edges per lane per step: both edges' col / w loads, then both dist
// loads, are in flight before either compare (a level's drain is a few such
// dependent rounds per warp).
__device__ __forceinline__ void relax_warp(const Args& a, unsigned it, Block& s, unsigned du,
                                           unsigned b, unsigned e) {
  for (unsigned k = b + dev::lane_id(); k < e; k += 64) {
    const unsigned k2 = k + 32;
    const bool ok2 = k2 < e;
    const unsigned g1 = static_cast<unsigned>(__ldg(a.col + k));
    const unsigned g2 = ok2 ? static_cast<unsigned>(__ldg(a.col + k2)) : a.r0;
    const unsigned long long t1 = static_cast<unsigned long long>(du) + edge_w(a, k);
    const unsigned long long t2 = ok2 ? static_cast<unsigned long long>(du) + edge_w(a, k2) : kInf;
    const unsigned v1 = g1 - a.r0, v2 = g2 - a.r0;
    const unsigned c1 = (t1 < kInf && v1 < a.n) ? __ldcg(a.dist + v1) : 0u;
    const unsigned c2 = (t2 < kInf && v2 < a.n) ? __ldcg(a.dist + v2) : 0u;
    const unsigned g[2] = {g1, g2}, c[2] = {c1, c2};
    const unsigned long long nd[2] = {t1, t2};
    relax_k<2>(a, it, s, g, nd, c);
  }
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

// `source` is a global vertex id; only its owner seeds the frontier.
__global__ void __launch_bounds__(256) init_kernel(Args a, unsigned source) {
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned ls = source - a.r0;
  const bool mine = ls < a.n;
  if (i < a.n) {
    a.dist[i] = i == ls ? 0u : kInf;
    a.stamp[i] = 0;
  }
  if (i == 0) {
    a.front0[0] = ls;
    a.ctr->fsize[0] = mine ? 1u : 0u;
    a.ctr->fsize[1] = a.ctr->fsize[2] = 0;
    a.ctr->pool[0] = a.ctr->pool[1] = a.ctr->pool[2] = 0;
    a.ctr->iters = 0;
    if (mine && a.classify) {  // one-barrier form: a heavy source starts as chunk items
      const unsigned b = a.rowptr[ls], e = a.rowptr[ls + 1];
      a.fbe0[0] = make_uint2(b, e);
      if (e - b > a.threshold) {
        a.ctr->pool[0] = dev::nchunks(e - b, a.chunk);
        a.ctr->fsize[0] = 0;
      }
    }
  }
  if (mine && a.classify) {  // the source's chunk items, one per thread (not a serial loop)
    const unsigned b = __ldg(a.rowptr + ls), e = __ldg(a.rowptr + ls + 1);
    if (e - b > a.threshold && i < dev::nchunks(e - b, a.chunk)) {
      if (i < a.pool.cap) a.pool.items[i] = Item{ls, b + i * a.chunk};
      else atomicOr(&a.hdr->overflow, 1u);
    }
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

// Applies the {global vertex, distance} pairs other ranks sent for the
// vertices this rank owns (the exchange step of iteration a.it): improved
// vertices join F_{it+1} like local relaxations do.
__global__ void __launch_bounds__(256) apply_kernel(Args a, const uint2* __restrict__ recv, unsigned count) {
  __shared__ Block s;
  block_begin(s);
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    const uint2 p = recv[i];
    relax(a, a.it, s, p.x, p.y);
  }
  block_end(a, a.it, s);
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

// Level-synchronous persistent form with ONE device-wide barrier per level:
// the consolidation of level it+1 happens while level it is flushed.  A
// block's queued next-frontier vertices are classified at flush time: heavy
// ones become chunk items of the next level right away (pool half
// (it+1) % 2), light ones go to the next frontier list.  So after the
// barrier a level needs no insert phase: every warp relaxes its share of the
// light list (warp-cooperative) and drains its share of the chunk items in
// the same pass.  (Vertices spilled past the shared queue land in the list
// and are relaxed warp-cooperatively whatever their degree.)
// Level form (grid_persistent1) light pass: like warp_light_relax, two edges
// per lane, with each list entry's row bounds read beside it (fbe) and the
// col / w loads issued before the owner's distance is needed -- the entry's
// distance load, the edge loads and the bounds are one round trip.
__device__ __forceinline__ void light_relax1(const Args& a, unsigned it, Block& s, unsigned b, unsigned du,
                                             unsigned dl) {
  const unsigned lane = dev::lane_id();
  const unsigned incl = dev::warp_incl_scan(dl);
  const unsigned total = __shfl_sync(kFull, incl, 31);
  const unsigned lo = incl - dl;
  for (unsigned base = 0; base < total; base += 64) {  // warp-uniform
    unsigned l[2], g[2], wk[2];
    bool ok[2];
#pragma unroll
    for (int j = 0; j < 2; j++) {
      const unsigned jj = base + 32 * j + lane;
      unsigned q = 0;
#pragma unroll
      for (unsigned st = 16; st > 0; st >>= 1) {
        const unsigned c = q + st;
        if (__shfl_sync(kFull, lo, c) <= jj) q = c;
      }
      l[j] = q;
      ok[j] = jj < total;
      const unsigned k = __shfl_sync(kFull, b, q) + (jj - __shfl_sync(kFull, lo, q));
      g[j] = ok[j] ? static_cast<unsigned>(__ldg(a.col + k)) : a.r0;
      wk[j] = ok[j] ? edge_w(a, k) : 0u;
    }
    unsigned long long nd[2];
    unsigned c[2];
#pragma unroll
    for (int j = 0; j < 2; j++) {
      const unsigned dul = __shfl_sync(kFull, du, l[j]);
      nd[j] = ok[j] ? static_cast<unsigned long long>(dul) + wk[j] : kInf;
      const unsigned v = g[j] - a.r0;
      c[j] = (nd[j] < kInf && v < a.n) ? __ldcg(a.dist + v) : 0u;
    }
    relax_k<2>(a, it, s, g, nd, c);
  }
}

// Level form drain: item t (prefetched one item ahead) relaxes its first 64
// edges with the col / w loads issued speculatively up to begin + chunk
// (bounded by m) beside the row-end and distance loads of its vertex, one
// round trip instead of two.
__device__ __forceinline__ void drain_items1(const Args& a, unsigned it, Block& s, const Item* items,
                                             unsigned count, unsigned gwarp, unsigned nwarps, Item t) {
  const unsigned lane = dev::lane_id();
  for (unsigned i = gwarp; i < count; i += nwarps) {
    Item tn{0u, 0u};
    if (i + nwarps < count) tn = items[i + nwarps];
    const unsigned lim = min(t.begin + a.chunk, a.m);
    const unsigned k1 = t.begin + lane, k2 = k1 + 32;
    unsigned g[2], wk[2];
    g[0] = k1 < lim ? static_cast<unsigned>(__ldg(a.col + k1)) : a.r0;
    g[1] = k2 < lim ? static_cast<unsigned>(__ldg(a.col + k2)) : a.r0;
    wk[0] = k1 < lim ? edge_w(a, k1) : 0u;
    wk[1] = k2 < lim ? edge_w(a, k2) : 0u;
    const unsigned e = min(t.begin + a.chunk, __ldg(a.rowptr + t.v + 1));
    const unsigned du = __ldcg(a.dist + t.v);
    unsigned long long nd[2];
    unsigned c[2];
#pragma unroll
    for (int j = 0; j < 2; j++) {
      const bool ok = (j ? k2 : k1) < e;
      if (!ok) g[j] = a.r0;
      nd[j] = ok ? static_cast<unsigned long long>(du) + wk[j] : kInf;
      const unsigned v = g[j] - a.r0;
      c[j] = (nd[j] < kInf && v < a.n) ? __ldcg(a.dist + v) : 0u;
    }
    relax_k<2>(a, it, s, g, nd, c);
    if (t.begin + 64 < e) relax_warp(a, it, s, du, t.begin + 64, e);  // chunks above 64 edges
    t = tn;
  }
}

__device__ __forceinline__ void flush_classify(const Args& a, unsigned it, Block& s, unsigned half) {
  __syncthreads();
  const unsigned n = min(s.q.n, kQueue);
  const unsigned nxt = (it + 1) % 3;
  for (unsigned base = 0; base < n; base += blockDim.x) {  // uniform trip count
    const unsigned i = base + threadIdx.x;
    unsigned v = 0, b = 0, e = 0, want = 0, light = 0;
    if (i < n) {
      v = s.q.items[i];
      b = __ldg(a.rowptr + v);
      e = __ldg(a.rowptr + v + 1);
      if (e - b > a.threshold) want = dev::nchunks(e - b, a.chunk);
      else light = 1;
    }
    dev::block_add_u64(&s.work, want ? e - b : 0u);  // heavy edges are relaxed next level (all lanes)
    unsigned lat, cat, cbase, ctot;
    dev::block_reserve2(&a.ctr->fsize[nxt], light, &a.ctr->pool[nxt], want, &lat, &cat, &cbase, &ctot);
    if (light) {
      next_front(a, it)[lat] = v;
      next_fbe(a, it)[lat] = make_uint2(b, e);  // the next level's light pass needs no rowptr round trip
    }
    const dev::Pool p{a.pool.items + half * a.pool.cap, a.pool.cap};
    if (blockDim.x <= kCoopW) {
      // the block's chunk items written cooperatively: slot t belongs to the
      // last thread whose exclusive offset is <= t (a hub's hundreds of
      // chunks no longer serialise on one thread)
      s.coff[threadIdx.x] = cat - cbase;
      s.cv[threadIdx.x] = v;
      s.cb[threadIdx.x] = b;
      __syncthreads();
      for (unsigned t = threadIdx.x; t < ctot; t += blockDim.x) {
        unsigned lo = 0, hi = blockDim.x;  // upper_bound(t) over s.coff[0, blockDim)
        while (lo < hi) {
          const unsigned mid = (lo + hi) >> 1;
          if (s.coff[mid] <= t) lo = mid + 1;
          else hi = mid;
        }
        const unsigned o = lo - 1, at = cbase + t;
        if (at < p.cap) p.items[at] = Item{s.cv[o], s.cb[o] + (t - s.coff[o]) * a.chunk};
        else atomicOr(&a.hdr->overflow, 1u);
      }
      __syncthreads();
    } else if (want) {
      dev::write_chunks(p, a.hdr, cat, v, b, e, a.chunk);
    }
  }
  if (threadIdx.x == 0) s.q.n = 0;  // (s.work is published once, at kernel end)
  __syncthreads();
}

__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// a.pool.cap = capacity of ONE half of the pool (the host allocates two).
__global__ void __launch_bounds__(256) grid_persistent1(Args a, unsigned max_iters) {
  __shared__ Block s;
  const unsigned stride = gridDim.x * blockDim.x;
  const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x;
  block_begin(s);
  unsigned it = 0;
  for (; it < max_iters; it++) {
    // level sizes (written before the barrier; relaxed gpu-scope loads, the
    // barrier orders them -- volatile would be system-scope)
    const unsigned fs = ld_relaxed_gpu(&a.ctr->fsize[it % 3]);
    const unsigned pc = min(ld_relaxed_gpu(&a.ctr->pool[it % 3]), a.pool.cap);
    if (fs == 0 && pc == 0) break;
    if (gtid == 0) {  // the counters level it+1 produces into were last read at level it-1
      atomicAdd(&a.hdr->aux1, pc);
      atomicMax(&a.hdr->count, pc);
      a.ctr->fsize[(it + 2) % 3] = 0;
      a.ctr->pool[(it + 2) % 3] = 0;
    }
    auto mark = [&](int k) {
      if (a.ptrace && threadIdx.x == 0 && it < 64) {
        if (k == 0) atomicMin(a.ptrace + it * 8, dev::global_ns());
        else atomicMax(a.ptrace + it * 8 + k, dev::global_ns());
        if (k == 0 && blockIdx.x == 0) {
          a.ptrace[it * 8 + 5] = fs;
          a.ptrace[it * 8 + 6] = pc;
        }
      }
    };
    mark(0);
    // the level's chunk items (inserted while the previous level flushed);
    // warp rank block-interleaved: consecutive items land in different
    // blocks, so a short item list (e.g. the source's chunks) spreads its
    // pushes over every block's queue instead of a few.  The warp's first
    // item is loaded now, under the light pass.
    const Item* items = a.pool.items + (it % 2) * a.pool.cap;
    const unsigned iw = dev::warp_in_block() * gridDim.x + blockIdx.x;
    Item t0{0u, 0u};
    if (iw < pc) t0 = items[iw];
    // the level's light list, warp-cooperatively (any degree), spread over
    // ALL warps: each takes a contiguous slice of ceil(fs / warps) vertices
    // (a level's relax rounds per warp, not the first fs / 256 blocks, set
    // its latency)
    {
      const unsigned nw = stride >> 5, gw = gtid >> 5;
      const unsigned per = max(1u, (fs + nw - 1) / nw);
      const unsigned v0 = min(fs, gw * per), v1 = min(fs, v0 + per);
      for (unsigned base = v0; base < v1; base += 32) {  // warp-uniform
        const unsigned i = base + dev::lane_id();
        unsigned b = 0, du = 0, deg = 0;
        if (i < v1) {
          const unsigned u = __ldcg(cur_front(a, it) + i);
          const uint2 be = __ldcg(cur_fbe(a, it) + i);
          b = be.x;
          deg = be.y - be.x;
          du = __ldcg(a.dist + u);
        }
        dev::block_add_u64(&s.work, deg);
        light_relax1(a, it, s, b, du, deg);
      }
    }
    mark(1);
    drain_items1(a, it, s, items, pc, iw, stride >> 5, t0);
    mark(2);
    flush_classify(a, it, s, (it + 1) % 2);
    mark(3);
    if (a.coop) cg::this_grid().sync();
    else dev::grid_sync64(&a.hdr->bar, &a.hdr->overflow);
    mark(4);
  }
  if (gtid == 0) a.ctr->iters = it;
  // the block's edge count (a metric): one atomic per block per run, not per
  // level -- per-level adds queued on the header line beside the barrier's
  if (threadIdx.x == 0 && s.work) atomicAdd(&a.hdr->work, s.work);
}

// ---------------------------------------------------------------------------
// Asynchronous grid consolidation (DPC_CFG_GRID_ASYNC; single GPU).  Measured
// slower than the level-synchronous persistent form on R-MAT SSSP (the
// relaxations, not the barriers, dominate), so it is not the default here.
//
// Level-synchronous Bellman-Ford pays a device-wide barrier (or a host round
// trip) per level; here the grid-level buffer is a device-wide FIFO of
// {vertex, distance} tasks drained by a persistent grid without barriers
// (chaotic relaxation: same unique fixpoint = Dijkstra's distances).  Every
// distance drop queues a task carrying the new distance; a task whose
// vertex has since dropped further is stale and skipped (the drop queued its
// own), so no dedup flags and no store-buffering fences are needed.  Queue
// position p is served by warp p mod W in order; the warp that makes a
// distance drop serves one such task itself next (work-first); heavy
// vertices fan out into chunk tasks.  The run ends when the FIFO is drained
// (every queued task served, none in flight).
constexpr int kAW = 4;                      // edges per lane per step
constexpr unsigned kAsyncHeavy = 128;       // edges one warp task takes
constexpr unsigned kAsyncChunk = 128;       // edges per chunk task
constexpr unsigned long long kEmpty = ~0ull;
constexpr unsigned long long kChunkTask = 1ull << 63;
constexpr unsigned kTail = 0, kDone = 32, kStop = 64;

struct Async {
  unsigned long long* q;  // vertex | dist << 32, or vertex | chunk << 32 | kChunkTask
  unsigned* qctr;         // [kTail], [kDone], [kStop], one line each
  unsigned qcap;
};

__device__ __forceinline__ unsigned long long vtask(unsigned v, unsigned d) {
  return static_cast<unsigned long long>(v) | (static_cast<unsigned long long>(d) << 32);
}

__device__ __forceinline__ void a_enqueue(const Args& a, const Async& q, bool want, unsigned long long t) {
  const unsigned ball = __ballot_sync(kFull, want);
  if (!ball) return;
  const unsigned lane = dev::lane_id(), lead = __ffs(ball) - 1;
  unsigned base = 0;
  if (lane == lead) base = atomicAdd(q.qctr + kTail, __popc(ball));
  base = __shfl_sync(kFull, base, lead);
  if (want) {
    const unsigned at = base + __popc(ball & ((1u << lane) - 1u));
    if (at < q.qcap) {
      *reinterpret_cast<volatile unsigned long long*>(q.q + at) = t;
    } else {
      atomicOr(&a.hdr->overflow, 1u);
      atomicExch(q.qctr + kStop, 1u);
    }
  }
}

// Relaxes edges [b, e) from distance du; each drop queues a task, one kept
// as this warp's continuation.
__device__ __forceinline__ unsigned long long a_relax(const Args& a, const Async& q, unsigned b, unsigned e,
                                                      unsigned du, unsigned long long* work) {
  unsigned long long keep = kEmpty;
  for (unsigned k0 = b; k0 < e; k0 += 32 * kAW) {
    unsigned v[kAW], nd[kAW];
    bool drop[kAW];
#pragma unroll
    for (int j = 0; j < kAW; j++) {
      const unsigned k = k0 + 32 * j + dev::lane_id();
      nd[j] = kInf;
      v[j] = 0;
      if (k < e) {
        v[j] = static_cast<unsigned>(__ldg(a.col + k));
        const unsigned long long d = static_cast<unsigned long long>(du) + edge_w(a, k);
        nd[j] = d < 0x7fffffffull ? static_cast<unsigned>(d) : kInf;  // task words hold 31-bit distances
      }
    }
#pragma unroll
    for (int j = 0; j < kAW; j++)
      drop[j] = nd[j] < kInf && nd[j] < __ldcg(a.dist + v[j]) && nd[j] < atomicMin(a.dist + v[j], nd[j]);
#pragma unroll
    for (int j = 0; j < kAW; j++) {
      if (keep == kEmpty) {
        const unsigned ball = __ballot_sync(kFull, drop[j]);
        if (ball) {
          const unsigned l = __ffs(ball) - 1;
          keep = vtask(__shfl_sync(kFull, v[j], l), __shfl_sync(kFull, nd[j], l));
          if (dev::lane_id() == l) drop[j] = false;
        }
      }
      a_enqueue(a, q, drop[j], vtask(v[j], nd[j]));
    }
  }
  if (dev::lane_id() == 0) *work += e - b;
  return keep;
}

__device__ unsigned long long a_serve(const Args& a, const Async& q, unsigned long long t,
                                      unsigned long long* work) {
  const unsigned u = static_cast<unsigned>(t);
  const unsigned b = __ldg(a.rowptr + u), e = __ldg(a.rowptr + u + 1);
  const unsigned du = __ldcg(a.dist + u);
  if (!(t & kChunkTask)) {
    if (du != static_cast<unsigned>(t >> 32)) return kEmpty;  // stale: a later drop queued u again
    if (e - b <= kAsyncHeavy) return a_relax(a, q, b, e, du, work);
    const unsigned nch = (e - b + kAsyncChunk - 1) / kAsyncChunk;
    for (unsigned c0 = 1; c0 < nch; c0 += 32)
      a_enqueue(a, q, c0 + dev::lane_id() < nch,
                u | (static_cast<unsigned long long>(c0 + dev::lane_id()) << 32) | kChunkTask);
    return a_relax(a, q, b, b + kAsyncChunk, du, work);
  }
  const unsigned chunk = static_cast<unsigned>(t >> 32) & 0x7fffffffu;
  const unsigned cb = b + chunk * kAsyncChunk, ce = min(e, cb + kAsyncChunk);
  return a_relax(a, q, cb, ce, du, work);  // the freshest distance of u is as good
}

__global__ void __launch_bounds__(256) async_persistent(Args a, Async q, unsigned source) {
  const unsigned stride = gridDim.x * blockDim.x;
  const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x, lane = dev::lane_id();
  const unsigned nwarps = stride >> 5, gw = gtid >> 5;
  volatile unsigned* vq = q.qctr;
  unsigned long long work = 0;
  if (gtid == 0) {
    atomicAdd(q.qctr + kTail, 1u);
    *reinterpret_cast<volatile unsigned long long*>(q.q) = vtask(source, 0);
  }
  for (unsigned p = gw; p < q.qcap; p += nwarps) {
    unsigned long long t = kEmpty;
    unsigned spins = 0;
    unsigned long long since = 0;
    while (true) {
      if (lane == 0) t = *reinterpret_cast<volatile unsigned long long*>(q.q + p);
      t = __shfl_sync(kFull, t, 0);
      if (t != kEmpty) break;
      unsigned fin = 0;
      if (lane == 0 && (++spins & 15) == 0) {
        const unsigned d = vq[kDone];  // read before tail: equal means nothing in flight
        fin = (d > 0 && d == vq[kTail]) || vq[kStop];
        const unsigned long long now = dev::global_ns();
        if (!since) since = now;
        if (now - since > 2000000000ull) {
          atomicOr(&a.hdr->overflow, 4u);
          atomicExch(q.qctr + kStop, 1u);
          fin = 1;
        }
      }
      if (__shfl_sync(kFull, fin, 0)) break;
      if (spins > 32) __nanosleep(64);
    }
    if (t == kEmpty) break;
    while (t != kEmpty) t = a_serve(a, q, t, &work);
    if (lane == 0) {
      __threadfence();
      atomicAdd(q.qctr + kDone, 1u);
    }
  }
  if (lane == 0 && work) atomicAdd(&a.hdr->work, work);
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

// Builds the kernel arguments of one SSSP run on `g` (a square graph, or the
// row block [r0, r0 + g->n) of an n_global-vertex graph).
static dpc_status sssp_setup(dpc_ctx* ctx, dpc_dgraph* g, const dpc_launch_cfg* cfg, sssp::Args* a,
                             Cfg* c, bool unit = false) {
  if (!unit && g->m > 0 && !g->w) return fail(DPC_E_INVALID, "graph was uploaded without weights (w)");
  dpc_status st = resolve_cfg(ctx, DPC_APP_SSSP, cfg, c);
  if (st != DPC_OK) return st;
  if (c->parent_threads != 256 || c->child_threads > 256)
    return fail(DPC_E_INVALID, "SSSP kernels are built for parent_threads = 256, child_threads <= 256");
  if (!g->ctr) {
    DPC_CUDA(cudaMalloc(&g->ctr, sizeof(sssp::Ctr)));
    DPC_CUDA(cudaMallocHost(&g->ctr_host, sizeof(sssp::Ctr)));
  }
  *a = sssp::Args{};
  a->rowptr = g->rowptr;
  a->col = g->col;
  a->w = unit ? nullptr : g->w;
  a->dist = g->dist;
  a->stamp = g->stamp;
  a->front0 = g->front[0];
  a->front1 = g->front[1];
  a->ctr = reinterpret_cast<sssp::Ctr*>(g->ctr);
  a->hdr = g->hdr;
  a->n = static_cast<unsigned>(g->n);
  a->m = static_cast<unsigned>(g->m);
  a->threshold = c->threshold;
  a->chunk = c->chunk;
  a->child_threads = c->child_threads;
  a->child_blocks = c->child_blocks;
  a->it = 0;
  a->fsize = 1;
  a->r0 = 0;
  a->rows_per_rank = 0xffffffffu;
  a->classify = 0;
  a->coop = 1;
  if (c->variant != DPC_FLAT && c->variant != DPC_BASIC) {
    st = ensure_pool(g, pool_need(g, c->threshold, c->chunk));
    if (st != DPC_OK) return st;
  }
  a->pool = dev::Pool{g->items, g->cap};
  st = ensure_pending_for(ctx, g, c->variant, c->threshold, c->parent_threads);
  if (st != DPC_OK) return st;
  g->hdr_clean = false;
  return begin_run(ctx, g->hdr);
}

// One host-loop iteration: relax F_it (the variant's parent grid + its
// consolidated children) and rotate the per-iteration counters.
static dpc_status sssp_iterate(dpc_ctx* ctx, const Cfg& c, sssp::Args& a, unsigned it, unsigned fsize) {
  cudaStream_t s = ctx->stream;
  a.it = it;
  a.fsize = fsize;
  const unsigned pb = std::max(1u, dev::ceil_div(fsize, 256u));
  if (fsize > 0) {
    switch (c.variant) {
      case DPC_FLAT: sssp::flat_kernel<<<pb, 256, 0, s>>>(a); break;
      case DPC_BASIC: sssp::basic_parent<<<pb, 256, 0, s>>>(a); break;
      case DPC_WARP: sssp::warp_parent<<<pb, 256, 0, s>>>(a); break;
      case DPC_BLOCK: sssp::block_parent<<<pb, 256, 0, s>>>(a); break;
      default: sssp::grid_parent<<<pb, 256, 0, s>>>(a); break;
    }
  }
  DPC_CUDA(cudaGetLastError());
  return DPC_OK;
}

// A run without metrics returns as soon as its work is enqueued (like the
// SpMV path): its header is copied back asynchronously and checked for
// faults at the next call on this graph (or dpc_dgraph_check).
extern "C" dpc_status dpc_dgraph_check(dpc_ctx* ctx, dpc_dgraph* g) {
  clear_error();
  if (!ctx || !g) return fail(DPC_E_INVALID, "NULL argument");
  return flush_check(ctx, g);
}

static dpc_status sssp_finish(dpc_ctx* ctx, dpc_dgraph* g, int64_t host_launches, int64_t iters,
                              dpc_metrics* met) {
  cudaStream_t s = ctx->stream;
  if (met) {
    met->host_launches += host_launches;
    met->iterations += iters;
    dpc_status st = finish_metrics(ctx, g->hdr, g->hdr_host, met);
    if (st != DPC_OK) return st;
    met->edges_processed += static_cast<int64_t>(g->hdr_host->work);
    met->buffer_items_inserted = g->hdr_host->aux1;
    return DPC_OK;
  }
  DPC_CUDA(cudaMemcpyAsync(g->hdr_host, g->hdr, sizeof(dev::RunHeader), cudaMemcpyDeviceToHost, s));
  g->check_pending = true;
  g->hdr_copied = true;
  return DPC_OK;
}

static dpc_status sssp_run(dpc_ctx* ctx, dpc_dgraph* g, int32_t source, const dpc_launch_cfg* cfg,
                           dpc_metrics* met, bool unit) {
  clear_error();
  if (!ctx || !g) return fail(DPC_E_INVALID, "NULL argument");
  if (g->ncols != g->n) return fail(DPC_E_INVALID, "SSSP needs a square graph (not a row slice)");
  if (source < 0 || source >= g->n) return fail(DPC_E_INVALID, "source out of range");
  Cfg c;
  sssp::Args a;
  dpc_status st = flush_check(ctx, g);
  if (st != DPC_OK) return st;
  st = sssp_setup(ctx, g, cfg, &a, &c, unit);
  if (st != DPC_OK) return st;
  cudaStream_t s = ctx->stream;
  const bool one_barrier = c.variant == DPC_GRID && c.grid_persistent &&
                           !(c.flags & (DPC_CFG_GRID_ASYNC | DPC_CFG_GRID_CHUNKED));
  if (one_barrier) {
    // two pool halves: level it drains one while its flush fills the other
    const uint64_t half = pool_need(g, c.threshold, c.chunk) + 1;
    st = ensure_pool(g, 2 * half);
    if (st != DPC_OK) return st;
    a.pool = dev::Pool{g->items, static_cast<unsigned>(half)};
    a.classify = 1;
    if (!g->sssp_fbe) DPC_CUDA(cudaMalloc(&g->sssp_fbe, sizeof(uint2) * 2 * static_cast<size_t>(std::max<int64_t>(g->n, 1))));
    a.fbe0 = g->sssp_fbe;
    a.fbe1 = g->sssp_fbe + std::max<int64_t>(g->n, 1);
    a.coop = (c.flags & DPC_CFG_COOP_LAUNCH) ? 1u : 0u;
  }
  // frontier stream form: forced by DPC_CFG_GRID_STREAM, default from 2^24
  // edges (tools/probes/sssp_forms.py: equal at scale 20, 1.6x at scale 22,
  // 4.4x at scale 24 where dist and the level form's stamps outgrow L2)
  const bool stream_form = c.variant == DPC_GRID && c.grid_persistent &&
                           !(c.flags & (DPC_CFG_GRID_ASYNC | DPC_CFG_GRID_CHUNKED | DPC_CFG_GRID_LEVEL)) &&
                           ((c.flags & DPC_CFG_GRID_STREAM) || g->m >= (int64_t{1} << 24));
  if (stream_form) {
    int64_t host_launches = 0, levels = 0;
    st = sssp_stream_run(ctx, g, source, unit, (c.flags & DPC_CFG_COOP_LAUNCH) != 0, &host_launches, &levels,
                         met);
    if (st != DPC_OK) return st;
    if (met) {  // edges_processed was filled by the stream form's own counters
      met->host_launches += host_launches;
      met->iterations += levels;
      return finish_metrics(ctx, g->hdr, g->hdr_host, met);
    }
    return sssp_finish(ctx, g, host_launches, levels, nullptr);
  }
  const unsigned nb = std::max(1u, dev::ceil_div(a.n, 256u));
  sssp::init_kernel<<<nb, 256, 0, s>>>(a, static_cast<unsigned>(source));
  DPC_CUDA(cudaGetLastError());
  int64_t host_launches = 1, iters = 0;
  auto* ctr_host = reinterpret_cast<sssp::Ctr*>(g->ctr_host);
  if (c.variant == DPC_GRID && c.grid_persistent && (c.flags & DPC_CFG_GRID_ASYNC)) {
    const uint64_t qcap = 8 * (static_cast<uint64_t>(g->n) + static_cast<uint64_t>(g->m)) + 64;
    if (g->gc_q_cap < qcap) {
      DPC_CUDA(cudaStreamSynchronize(s));
      if (g->gc_q) cudaFree(g->gc_q);
      g->gc_q = nullptr;
      g->gc_q_cap = 0;
      DPC_CUDA(cudaMalloc(&g->gc_q, sizeof(unsigned long long) * qcap + 1024));
      g->gc_q_cap = qcap;
    }
    sssp::Async q;
    q.q = reinterpret_cast<unsigned long long*>(g->gc_q);
    q.qcap = static_cast<unsigned>(std::min<uint64_t>(g->gc_q_cap, 0xffffffffull));
    q.qctr = reinterpret_cast<unsigned*>(q.q + g->gc_q_cap);
    DPC_CUDA(cudaMemsetAsync(q.q, 0xff, sizeof(unsigned long long) * g->gc_q_cap, s));
    DPC_CUDA(cudaMemsetAsync(q.qctr, 0, 1024, s));
    int blocks = coop_blocks_sssp(ctx, reinterpret_cast<const void*>(sssp::async_persistent), 256);
    unsigned src = static_cast<unsigned>(source);
    void* args[] = {&a, &q, &src};
    DPC_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(sssp::async_persistent),
                                         dim3(blocks), dim3(256), args, 0, s));
    host_launches += 1;
    iters = 1;
  } else if (one_barrier) {
    const void* fn = reinterpret_cast<const void*>(sssp::grid_persistent1);
    int blocks = coop_blocks_sssp(ctx, fn, 256);
    unsigned max_iters = a.n + 1;
    // DPC_SSSP_PHASES=1: per-level phase timeline to stderr (diagnostics)
    static const bool phases = std::getenv("DPC_SSSP_PHASES") != nullptr;
    std::vector<unsigned long long> ph(64 * 8, 0);
    if (phases) {
      for (int i = 0; i < 64; i++) ph[i * 8] = ~0ull;
      DPC_CUDA(cudaMalloc(&a.ptrace, sizeof(unsigned long long) * ph.size()));
      DPC_CUDA(cudaMemcpyAsync(a.ptrace, ph.data(), sizeof(unsigned long long) * ph.size(),
                               cudaMemcpyHostToDevice, s));
    }
    void* args[] = {&a, &max_iters};
    if (a.coop) DPC_CUDA(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(256), args, 0, s));
    else DPC_CUDA(cudaLaunchKernel(fn, dim3(blocks), dim3(256), args, 0, s));
    host_launches += 1;
    if (met || phases) {  // the level count is a metric; no host round trip without it
      DPC_CUDA(cudaMemcpyAsync(ctr_host, a.ctr, sizeof(sssp::Ctr), cudaMemcpyDeviceToHost, s));
      DPC_CUDA(cudaStreamSynchronize(s));
      iters = ctr_host->iters;
    }
    if (phases) {
      DPC_CUDA(cudaMemcpy(ph.data(), a.ptrace, sizeof(unsigned long long) * ph.size(), cudaMemcpyDeviceToHost));
      cudaFree(a.ptrace);
      a.ptrace = nullptr;
      const unsigned long long t0 = ph[0];
      for (int64_t i = 0; i < std::min<int64_t>(iters, 64); i++) {
        const unsigned long long* r = &ph[i * 8];
        std::fprintf(stderr, "sssp level %2lld fs %7llu pc %6llu | start %7.2f light %6.2f drain %6.2f flush %6.2f "
                     "barrier %6.2f us\n", static_cast<long long>(i), r[5], r[6], (r[0] - t0) / 1e3,
                     (r[1] - r[0]) / 1e3, (r[2] - r[1]) / 1e3, (r[3] - r[2]) / 1e3, (r[4] - r[3]) / 1e3);
      }
    }
  } else if (c.variant == DPC_GRID && c.grid_persistent) {
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
      st = sssp_iterate(ctx, c, a, it, fsize);
      if (st != DPC_OK) return st;
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
  return sssp_finish(ctx, g, host_launches, iters, met);
}

extern "C" dpc_status dpc_sssp_device(dpc_ctx* ctx, dpc_dgraph* g, int32_t source,
                                      const dpc_launch_cfg* cfg, dpc_metrics* met) {
  return sssp_run(ctx, g, source, cfg, met, false);
}

extern "C" dpc_status dpc_bfs_device(dpc_ctx* ctx, dpc_dgraph* g, int32_t source,
                                     const dpc_launch_cfg* cfg, dpc_metrics* met) {
  return sssp_run(ctx, g, source, cfg, met, true);
}

// ---------------------------------------------------------------------------
// Vertex-partitioned SSSP (BASELINE config 5).  Rank p owns
// the global vertices [p*R, p*R + n_p) and their out-edges (a row block from
// dpc_gen_rmat_rows); columns are global ids.  Each iteration:
//   relax   : the local consolidated relaxation of F_it; targets this rank
//             owns are atomicMin'd in place, others are min-filtered
//             (rdist) into per-owner send buffers {vertex, distance}
//   exchange: the send buffers go to their owners (NCCL send/recv over
//             NVLink in dpc_multi_sssp; any transport through the step API)
//   apply   : received pairs are atomicMin'd; improved vertices join F_it+1
//   stop    : when the global |F_it+1| (sum over ranks) is 0
// The step API (dpc_msssp_*) exposes relax / apply so the exchange can be
// driven by any transport; dpc_multi_sssp composes them with NCCL.
struct MsState {
  sssp::Args a;
  Cfg c;
  int world = 1;
  unsigned it = 0;
  unsigned fsize = 0;
  int64_t host_launches = 0;
  int64_t remote_sent = 0;
};

static MsState* ms_state(dpc_dgraph* g) { return reinterpret_cast<MsState*>(g->ms_state); }

namespace dpc {
void sssp_state_free(void* state) { delete reinterpret_cast<MsState*>(state); }
}  // namespace dpc

extern "C" dpc_status dpc_msssp_begin(dpc_ctx* ctx, dpc_dgraph* g, int64_t r0, int64_t rows_per_rank,
                                      int64_t n_global, int32_t world, int64_t source,
                                      const dpc_launch_cfg* cfg) {
  clear_error();
  if (!ctx || !g) return fail(DPC_E_INVALID, "NULL argument");
  if (world < 1 || rows_per_rank < 1 || r0 < 0 || r0 + g->n > n_global || g->ncols != n_global ||
      n_global >= (int64_t{1} << 32) || (n_global + rows_per_rank - 1) / rows_per_rank > world ||
      r0 % rows_per_rank != 0)
    return fail(DPC_E_INVALID, "bad partition: need r0 = rank * rows_per_rank, ncols = n_global");
  if (source < 0 || source >= n_global) return fail(DPC_E_INVALID, "source out of range");
  {
    const dpc_status pst = flush_check(ctx, g);
    if (pst != DPC_OK) return pst;
  }
  if (!g->ms_state) g->ms_state = new (std::nothrow) MsState();
  MsState* m = ms_state(g);
  if (!m) return fail(DPC_E_OOM, "state allocation failed");
  dpc_status st = sssp_setup(ctx, g, cfg, &m->a, &m->c);
  if (st != DPC_OK) return st;
  if (m->c.variant == DPC_GRID) m->c.grid_persistent = 0;  // one exchange per iteration
  // buffers: rdist over all global vertices, one send segment per owner
  // (a segment holds at most every local edge), one receive area
  const size_t cap = static_cast<size_t>(std::max<int64_t>(g->m, 1));
  const size_t need_send = cap * static_cast<size_t>(world);
  if (g->ms_n < static_cast<size_t>(n_global) || g->ms_cap < need_send) {
    DPC_CUDA(cudaStreamSynchronize(ctx->stream));
    for (void* p : {static_cast<void*>(g->ms_rdist), static_cast<void*>(g->ms_send),
                    static_cast<void*>(g->ms_recv), static_cast<void*>(g->ms_cnt)})
      if (p) cudaFree(p);
    g->ms_rdist = nullptr, g->ms_send = nullptr, g->ms_recv = nullptr, g->ms_cnt = nullptr;
    g->ms_n = g->ms_cap = 0;
    DPC_CUDA(cudaMalloc(&g->ms_rdist, sizeof(unsigned) * static_cast<size_t>(n_global)));
    DPC_CUDA(cudaMalloc(&g->ms_send, sizeof(uint2) * need_send));
    DPC_CUDA(cudaMalloc(&g->ms_recv, sizeof(uint2) * need_send));
    DPC_CUDA(cudaMalloc(&g->ms_cnt, sizeof(unsigned) * 2 * 64));
    g->ms_n = static_cast<size_t>(n_global);
    g->ms_cap = need_send;
    g->ms_rcap = need_send;
  }
  if (world > 64) return fail(DPC_E_INVALID, "world > 64");
  m->world = world;
  m->a.r0 = static_cast<unsigned>(r0);
  m->a.rows_per_rank = static_cast<unsigned>(rows_per_rank);
  m->a.rdist = g->ms_rdist;
  m->a.sendbuf = reinterpret_cast<uint2*>(g->ms_send);
  m->a.sendcnt = g->ms_cnt;
  m->a.sendcap = static_cast<unsigned>(cap);
  m->a.peers = nullptr;
  m->it = 0;
  m->host_launches = 0;
  m->remote_sent = 0;
  cudaStream_t s = ctx->stream;
  DPC_CUDA(cudaMemsetAsync(g->ms_rdist, 0xff, sizeof(unsigned) * static_cast<size_t>(n_global), s));
  DPC_CUDA(cudaMemsetAsync(g->ms_cnt, 0, sizeof(unsigned) * 64, s));
  const unsigned nb = std::max(1u, dev::ceil_div(m->a.n, 256u));
  sssp::init_kernel<<<nb, 256, 0, s>>>(m->a, static_cast<unsigned>(source));
  DPC_CUDA(cudaGetLastError());
  m->host_launches = 1;
  m->fsize = (source >= r0 && source < r0 + g->n) ? 1u : 0u;
  DPC_CUDA(cudaStreamSynchronize(s));
  return DPC_OK;
}

extern "C" dpc_status dpc_msssp_relax(dpc_ctx* ctx, dpc_dgraph* g, uint32_t* send_counts) {
  clear_error();
  if (!ctx || !g || !send_counts) return fail(DPC_E_INVALID, "NULL argument");
  MsState* m = ms_state(g);
  if (!m) return fail(DPC_E_INVALID, "dpc_msssp_begin was not called");
  cudaStream_t s = ctx->stream;
  DPC_CUDA(cudaMemsetAsync(m->a.sendcnt, 0, sizeof(unsigned) * static_cast<size_t>(m->world), s));
  dpc_status st = sssp_iterate(ctx, m->c, m->a, m->it, m->fsize);
  if (st != DPC_OK) return st;
  m->host_launches += 1;
  DPC_CUDA(cudaMemcpyAsync(send_counts, m->a.sendcnt, sizeof(unsigned) * static_cast<size_t>(m->world),
                           cudaMemcpyDeviceToHost, s));
  DPC_CUDA(cudaStreamSynchronize(s));
  for (int p = 0; p < m->world; p++) {
    if (send_counts[p] > m->a.sendcap) return fail(DPC_E_OVERFLOW, "send buffer overflow");
    m->remote_sent += send_counts[p];
  }
  return DPC_OK;
}

// Fused form: the device pointers this rank exports (dist, stamp, front0,
// front1, counters) and the table of every rank's (own + IPC-mapped).
extern "C" dpc_status dpc_msssp_buffers(dpc_dgraph* g, void* out[5]) {
  clear_error();
  if (!g || !out) return fail(DPC_E_INVALID, "NULL argument");
  if (!g->ctr) return fail(DPC_E_INVALID, "dpc_msssp_begin was not called");
  out[0] = g->dist;
  out[1] = g->stamp;
  out[2] = g->front[0];
  out[3] = g->front[1];
  out[4] = g->ctr;
  return DPC_OK;
}

extern "C" dpc_status dpc_msssp_set_peers(dpc_dgraph* g, const void* d_peer_table) {
  clear_error();
  MsState* m = g ? ms_state(g) : nullptr;
  if (!m) return fail(DPC_E_INVALID, "dpc_msssp_begin was not called");
  m->a.peers = static_cast<const sssp::Peer*>(d_peer_table);
  return DPC_OK;
}

extern "C" const void* dpc_msssp_send_buffer(dpc_dgraph* g, int32_t owner) {
  MsState* m = g ? ms_state(g) : nullptr;
  if (!m || owner < 0 || owner >= m->world) return nullptr;
  return m->a.sendbuf + static_cast<size_t>(owner) * m->a.sendcap;
}

extern "C" void* dpc_msssp_recv_buffer(dpc_dgraph* g) { return g ? g->ms_recv : nullptr; }

extern "C" uint64_t dpc_msssp_recv_capacity(dpc_dgraph* g) { return g ? g->ms_rcap : 0; }

// A rank receives at most what its peers queued for it, which is bounded by
// the PEERS' local edge counts, not by its own: the receive area grows to
// the count the caller learned from the exchange of send counts.
extern "C" dpc_status dpc_msssp_recv_reserve(dpc_ctx* ctx, dpc_dgraph* g, uint64_t pairs, void** out) {
  clear_error();
  if (!ctx || !g || !out) return fail(DPC_E_INVALID, "NULL argument");
  if (!ms_state(g)) return fail(DPC_E_INVALID, "dpc_msssp_begin was not called");
  if (pairs > g->ms_rcap) {
    DPC_CUDA(cudaStreamSynchronize(ctx->stream));
    if (g->ms_recv) cudaFree(g->ms_recv);
    g->ms_recv = nullptr;
    g->ms_rcap = 0;
    DPC_CUDA(cudaMalloc(&g->ms_recv, sizeof(uint2) * static_cast<size_t>(pairs)));
    g->ms_rcap = static_cast<size_t>(pairs);
  }
  *out = g->ms_recv;
  return DPC_OK;
}

extern "C" const uint32_t* dpc_msssp_send_counts(dpc_dgraph* g) {
  MsState* m = g ? ms_state(g) : nullptr;
  return m ? m->a.sendcnt : nullptr;
}

extern "C" dpc_status dpc_msssp_apply(dpc_ctx* ctx, dpc_dgraph* g, const void* d_pairs, uint64_t count,
                                      uint32_t* next_fsize) {
  clear_error();
  if (!ctx || !g || !next_fsize || (count && !d_pairs)) return fail(DPC_E_INVALID, "NULL argument");
  MsState* m = ms_state(g);
  if (!m) return fail(DPC_E_INVALID, "dpc_msssp_begin was not called");
  cudaStream_t s = ctx->stream;
  m->a.it = m->it;
  if (count) {
    const unsigned nb = std::min(4u * static_cast<unsigned>(ctx->sms),
                                 std::max(1u, dev::ceil_div(static_cast<unsigned>(count), 256u)));
    sssp::apply_kernel<<<nb, 256, 0, s>>>(m->a, static_cast<const uint2*>(d_pairs), static_cast<unsigned>(count));
    m->host_launches += 1;
  }
  sssp::rotate_kernel<<<1, 32, 0, s>>>(m->a);
  m->host_launches += 1;
  DPC_CUDA(cudaGetLastError());
  auto* ctr_host = reinterpret_cast<sssp::Ctr*>(g->ctr_host);
  DPC_CUDA(cudaMemcpyAsync(&ctr_host->fsize[(m->it + 1) % 3], &m->a.ctr->fsize[(m->it + 1) % 3],
                           sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  DPC_CUDA(cudaStreamSynchronize(s));
  m->fsize = ctr_host->fsize[(m->it + 1) % 3];
  m->it++;
  *next_fsize = m->fsize;
  return DPC_OK;
}

extern "C" dpc_status dpc_msssp_end(dpc_ctx* ctx, dpc_dgraph* g, dpc_metrics* met) {
  clear_error();
  if (!ctx || !g) return fail(DPC_E_INVALID, "NULL argument");
  MsState* m = ms_state(g);
  if (!m) return fail(DPC_E_INVALID, "dpc_msssp_begin was not called");
  dpc_status st = sssp_finish(ctx, g, m->host_launches, m->it, met);
  if (st == DPC_OK && met) met->result_count = m->remote_sent;
  return st;
}
