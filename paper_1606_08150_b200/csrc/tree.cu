// Tree descendants (TD) and tree heights (TH) — the paper's parallel-recursion
// apps (Fig. 1(c)): tree_traversal(node) <<<1, nc(node)>>>
// gives each thread one child; a child with children recurses, a leaf does
// leaf work; postwork folds the children's results into the node:
//     TD: desc[v]   = sum_c (desc[c] + 1)
//     TH: height[v] = max_c (height[c] + 1)
//
// CDP1's parent-side cudaDeviceSynchronize is gone on sm_100,
// so postwork runs in TAIL-launched grids: a tail launch starts only after
// the launching grid and all its descendant work have completed
// (tools/probes/cdp2_probe Q1), which is exactly "after the subtree is done".
//
//   flat   : host loop over levels; thread per node, serial child loops;
//            then a reverse level loop gathers results (no device launches)
//   basic  : Fig. 1(c) literally: one <<<ceil(nc/T), T>>> grid per internal
//            node (CDP2 fire-and-forget) + one tail-launched postwork grid
//   warp / block / grid : recursive consolidation (transform.hpp:874-964):
//            <k>_cons drains a buffer of internal nodes, inserts their
//            internal children into owner buffers (warp / block / grid), the
//            owner launches one <k>_cons per buffer, and every <k>_cons grid
//            tail-launches one <k>_post over its own items
//   grid (persistent) : one cooperative kernel: top-down levels with a
//            device-wide barrier between them, then the bottom-up levels in
//            reverse (PAPER.md:244-250 global barrier), zero launches.
//
// Work items are internal nodes; a group of g lanes (g = power of two <= 32
// sized to the mean fan-out) handles one item's children.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <new>

#include "common.cuh"
#include "ctx.h"

namespace cg = cooperative_groups;

namespace dpc {
namespace tree {

using dev::RunHeader;

struct Args {
  const unsigned* __restrict__ cstart;
  const int* __restrict__ clist;
  int* res;
  unsigned* nodes;  // pool / level lists of internal nodes
  unsigned* cnt;    // [0] bump pointer of `nodes`, [1..] level offsets (persistent/flat)
  unsigned cap;
  RunHeader* hdr;
  unsigned n;
  unsigned group;  // lanes per item (1, 2, 4, ..., 32)
  unsigned child_threads;
  unsigned child_blocks;
  int is_max;      // TH (max) vs TD (sum)
  const int* parent;  // persistent grid: parent[v] (-1 at the root)
  unsigned* pend;     // persistent grid: internal children not yet folded
  unsigned root;
  unsigned root_internal;
};

__device__ __forceinline__ unsigned nkids(const Args& a, unsigned v) {
  return __ldg(a.cstart + v + 1) - __ldg(a.cstart + v);
}

// Postwork for one node over a g-lane group: gather children's results.
__device__ __forceinline__ void fold_node(const Args& a, unsigned v, unsigned sub, unsigned g,
                                          bool active) {
  int acc = 0;
  if (active) {
    unsigned b = __ldg(a.cstart + v), e = __ldg(a.cstart + v + 1);
    for (unsigned k = b + sub; k < e; k += g) {
      int r = __ldcg(a.res + __ldg(a.clist + k)) + 1;
      acc = a.is_max ? max(acc, r) : acc + r;
    }
  }
  for (unsigned o = g >> 1; o > 0; o >>= 1) {
    int t = __shfl_xor_sync(dev::kFull, acc, o);
    acc = a.is_max ? max(acc, t) : acc + t;
  }
  if (active && sub == 0) a.res[v] = acc;
}

// Top-down expansion of one node: returns (per lane) how many internal
// children this lane owns; they are written by write_kids once slots exist.
__device__ __forceinline__ unsigned count_kids(const Args& a, unsigned v, unsigned sub, unsigned g,
                                               bool active) {
  unsigned c = 0;
  if (active) {
    unsigned b = __ldg(a.cstart + v), e = __ldg(a.cstart + v + 1);
    for (unsigned k = b + sub; k < e; k += g) c += nkids(a, static_cast<unsigned>(__ldg(a.clist + k))) > 0;
  }
  return c;
}

__device__ __forceinline__ void write_kids(const Args& a, unsigned v, unsigned sub, unsigned g,
                                           bool active, unsigned at) {
  if (!active) return;
  unsigned b = __ldg(a.cstart + v), e = __ldg(a.cstart + v + 1);
  for (unsigned k = b + sub; k < e; k += g) {
    unsigned c = static_cast<unsigned>(__ldg(a.clist + k));
    if (nkids(a, c) > 0) {
      if (at < a.cap) a.nodes[at] = c;
      else atomicOr(&a.hdr->overflow, 1u);
      at++;
    }
  }
}

// ---------------------------------------------------------------- flat
__global__ void __launch_bounds__(256) flat_down(Args a, unsigned lo, unsigned hi) {
  unsigned i = lo + blockIdx.x * blockDim.x + threadIdx.x;
  bool active = i < hi;
  unsigned v = active ? a.nodes[i] : 0;
  unsigned want = count_kids(a, v, 0, 1, active);
  unsigned bb, bt;
  unsigned at = dev::block_reserve(&a.cnt[0], want, &bb, &bt);
  write_kids(a, v, 0, 1, active && want, at);
}

__global__ void __launch_bounds__(256) flat_up(Args a, unsigned lo, unsigned hi) {
  unsigned i = lo + blockIdx.x * blockDim.x + threadIdx.x;
  bool active = i < hi;
  fold_node(a, active ? a.nodes[i] : 0, 0, 1, active);
}

// ---------------------------------------------------------------- basic
// Fig. 1(c) with CDP2: tree_traversal(node) <<<ceil(nc/T), T>>>, thread per
// child; an internal child launches its own traversal (fire-and-forget).
// Postwork runs by COUNT-DOWN on the child side instead of a tail-launched
// grid per node (those stay pending until their whole subtree is done: ~1.7M
// outstanding launches on the 4.2M-node config-4 tree, past the device
// runtime's ~599K pending-launch pool, profiles/r01_pending_limit.txt):
// pend[v] starts at nc(v); a block folds its leaf children into res[v] and
// subtracts their count; a finished internal child folds itself into its
// parent and subtracts one.  The thread that brings pend[v] to zero owns v's
// final result and carries it upward (the postwork of PAPER.md:96-105,
// executed once per node, after all of its children).
__device__ __forceinline__ void fold_into(const Args& a, unsigned p, int r) {
  if (a.is_max) atomicMax(a.res + p, r);
  else atomicAdd(a.res + p, r);
}

// v's result is final: fold it into its ancestors while this thread
// completes them.
__device__ void basic_finish(const Args& a, unsigned v) {
  while (v != a.root) {
    const unsigned p = static_cast<unsigned>(__ldg(a.parent + v));
    fold_into(a, p, __ldcg(a.res + v) + 1);
    __threadfence();  // release: the fold before the count-down
    if (atomicSub(a.pend + p, 1u) != 1u) return;
    __threadfence();  // acquire: every child's fold into p is visible
    v = p;
  }
}

// The device runtime's pending-launch pool is full (cudaLimitDevRuntime-
// PendingLaunchCount caps at ~599K on B200): the launching thread computes
// the child's subtree itself -- a stackless post-order walk (parent pointers,
// sibling position by search) folding each finished node into its parent with
// plain stores (the subtree is this thread's alone).  Same results; counted
// in RunHeader.next_count (metrics.result_count of a basic tree run).
__device__ void subtree_inline(const Args& a, unsigned c) {
  unsigned x = c;
  while (nkids(a, x) > 0) x = static_cast<unsigned>(__ldg(a.clist + __ldg(a.cstart + x)));
  while (x != c) {
    const unsigned p = static_cast<unsigned>(__ldg(a.parent + x));
    const int r = a.res[x] + 1;
    a.res[p] = a.is_max ? max(a.res[p], r) : a.res[p] + r;
    unsigned pos = __ldg(a.cstart + p);
    while (static_cast<unsigned>(__ldg(a.clist + pos)) != x) pos++;
    if (pos + 1 < __ldg(a.cstart + p + 1)) {
      x = static_cast<unsigned>(__ldg(a.clist + pos + 1));
      while (nkids(a, x) > 0) x = static_cast<unsigned>(__ldg(a.clist + __ldg(a.cstart + x)));
    } else {
      x = p;  // p's last child is folded: p is final
    }
  }
}

__global__ void __launch_bounds__(256) basic_pend_init(Args a) {
  const unsigned v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < a.n) a.pend[v] = nkids(a, v);
}

// tree_traversal(node) <<<ceil(nc/T), T>>>: thread per child.
__global__ void __launch_bounds__(256) basic_traverse(Args a, unsigned v) {
  __shared__ int s_r;
  __shared__ unsigned s_c;
  if (threadIdx.x == 0) {
    s_r = 0;
    s_c = 0;
  }
  __syncthreads();
  const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned b = __ldg(a.cstart + v), e = __ldg(a.cstart + v + 1);
  if (b + k < e) {
    const unsigned c = static_cast<unsigned>(__ldg(a.clist + b + k));
    const unsigned nc = nkids(a, c);
    int r = 1;  // leaf child: desc 0 + 1, height 0 + 1
    bool folded = true;
    if (nc > 0) {
      basic_traverse<<<dev::ceil_div(nc, a.child_threads), a.child_threads, 0,
                       cudaStreamFireAndForget>>>(a, c);
      const cudaError_t err = cudaGetLastError();
      if (err == cudaSuccess) {
        atomicAdd(&a.hdr->launches, 1u);
        folded = false;  // the child's subtree folds itself into v (count-down)
      } else if (err == cudaErrorLaunchPendingCountExceeded) {
        subtree_inline(a, c);
        atomicAdd(&a.hdr->next_count, 1u);
        r = a.res[c] + 1;
      } else {
        atomicOr(&a.hdr->overflow, 2u);
        atomicCAS(&a.hdr->aux0, 0u, static_cast<unsigned>(err));
        folded = false;
      }
    }
    if (folded) {
      if (a.is_max) atomicMax(&s_r, r);
      else atomicAdd(&s_r, r);
      atomicAdd(&s_c, 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_c) {
    fold_into(a, v, s_r);
    __threadfence();
    if (atomicSub(a.pend + v, s_c) == s_c) {
      __threadfence();
      basic_finish(a, v);
    }
  }
}

// ---------------------------------------------------------------- consolidated
enum Gran { kWarp = 2, kBlock = 3, kGrid = 4 };

__global__ void __launch_bounds__(256) cons_post(Args a, const unsigned* items, unsigned count) {
  const unsigned g = a.group;
  const unsigned gid = (blockIdx.x * blockDim.x + threadIdx.x) / g, sub = threadIdx.x & (g - 1);
  const unsigned ngroups = (gridDim.x * blockDim.x) / g;
  // uniform trip count across the warp so the group shuffles stay converged
  const unsigned base = gid - (threadIdx.x & 31u) / g;
  for (unsigned i0 = base; i0 < count; i0 += ngroups) {
    unsigned i = i0 + (threadIdx.x & 31u) / g;
    bool active = i < count;
    fold_node(a, active ? items[i] : 0, sub, g, active);
  }
}

__device__ __forceinline__ unsigned cons_blocks(const Args& a, unsigned count) {
  unsigned per_block = a.child_threads / a.group;
  unsigned b = dev::ceil_div(count, per_block);
  if (a.child_blocks && b > a.child_blocks) b = a.child_blocks;
  return b ? b : 1u;
}

template <int G>
__global__ void __launch_bounds__(256) cons_kernel(Args a, const unsigned* items, unsigned count) {
  __shared__ unsigned s_base;
  const unsigned g = a.group;
  const unsigned lane = threadIdx.x & 31u, sub = threadIdx.x & (g - 1);
  const unsigned gpw = 32 / g;  // groups per warp
  const unsigned warp_g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned nwarps = (gridDim.x * blockDim.x) >> 5;
  // Block-level and grid-level owners need every block to take part in the
  // insert; a single pass over the items keeps the barrier count uniform.
  unsigned rounds = dev::ceil_div(count, nwarps * gpw);
  for (unsigned r = 0; r < rounds; r++) {
    unsigned i = (r * nwarps + warp_g) * gpw + lane / g;
    bool active = i < count;
    unsigned v = active ? items[i] : 0;
    unsigned want = count_kids(a, v, sub, g, active);
    if (G == kWarp || G == kGrid) {
      unsigned bb, bt;
      unsigned at = dev::block_reserve(&a.cnt[0], want, &bb, &bt);
      write_kids(a, v, sub, g, active && want, at);
      const unsigned wb = __shfl_sync(dev::kFull, at, 0), wt = dev::warp_sum(want);
      if (G == kWarp && wt) {
        __threadfence();
        unsigned leader = __ffs(__ballot_sync(dev::kFull, want != 0)) - 1;
        __syncwarp();
        if (lane == leader && wb < a.cap) {
          unsigned cnt = min(wt, a.cap - wb);
          cons_kernel<kWarp><<<cons_blocks(a, cnt), a.child_threads, 0, cudaStreamFireAndForget>>>(
              a, a.nodes + wb, cnt);
          dev::note_launch(a.hdr);
        }
      }
    } else {  // block owner
      unsigned bt;
      unsigned off = dev::block_excl_scan(want, &bt);
      if (threadIdx.x == 0 && bt) s_base = atomicAdd(&a.cnt[0], bt);
      __syncthreads();
      write_kids(a, v, sub, g, active && want, s_base + off);
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0 && bt && s_base < a.cap) {
        unsigned cnt = min(bt, a.cap - s_base);
        cons_kernel<kBlock><<<cons_blocks(a, cnt), a.child_threads, 0, cudaStreamFireAndForget>>>(
            a, a.nodes + s_base, cnt);
        dev::note_launch(a.hdr);
      }
      __syncthreads();
    }
  }
  if (G == kGrid) {
    // next level = every item inserted by this grid: [level_end, cnt[0])
    __threadfence();
    if (dev::grid_last_block(&a.hdr->ticket) && threadIdx.x == 0) {
      unsigned lo = static_cast<unsigned>(items - a.nodes) + count;
      unsigned hi = min(*reinterpret_cast<volatile unsigned*>(&a.cnt[0]), a.cap);
      if (hi > lo) {
        cons_kernel<kGrid><<<cons_blocks(a, hi - lo), a.child_threads, 0, cudaStreamFireAndForget>>>(
            a, a.nodes + lo, hi - lo);
        dev::note_launch(a.hdr);
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // consolidated postwork over this grid's items, after all descendants
    cons_post<<<cons_blocks(a, count), a.child_threads, 0, cudaStreamTailLaunch>>>(a, items, count);
    dev::note_launch(a.hdr);
  }
}

// Run init: level counters / offsets and the root item.
__global__ void __launch_bounds__(32) init_run(unsigned* off, unsigned* nodes, unsigned c0, unsigned r,
                                               unsigned root, bool root_internal) {
  if (threadIdx.x == 0) {
    off[0] = c0;
    off[1] = off[2] = off[3] = 0;
    off[4] = r;
    if (root_internal) nodes[0] = root;
  }
}

// ---------------------------------------------------------------- persistent
// Top-down: the recursion's levels, consolidated per level with a
// device-wide barrier; each internal node also records
// its leaf children's share of the postwork (TD: one per leaf child, TH: 1
// if it has one) in res[v] and its internal-children count in pend[v].
// Bottom-up: the postwork of a node runs once all its children's postwork
// has (the tail-launch semantics) by count-down instead of a barrier per
// level: a finished node pushes res + 1 into its parent and the child that
// brings the parent's count to zero carries on with the parent, so the
// chains climb the tree concurrently (<= depth dependent steps, no barrier).
constexpr unsigned kNoInternal = 0x80000000u;  // pend mark: no internal child
constexpr unsigned kSmallLevel = 3;            // levels of <= 3 block passes run in block 0 alone
constexpr unsigned kPullMin = 65536;           // bottom-up levels this wide fold by gathering

__global__ void __launch_bounds__(256) grid_persistent(Args a, unsigned max_levels) {
  cg::grid_group grid = cg::this_grid();
  const unsigned g = a.group, lane = threadIdx.x & 31u, sub = threadIdx.x & (g - 1);
  const unsigned gpw = 32 / g;
  const unsigned nwarps = (gridDim.x * blockDim.x) >> 5;
  // cnt[0..2]: per-level append counters, triple-buffered so that the
  // counter read after a level's barrier is never reset or appended to by a
  // block that already raced ahead (same rotation as sssp::rotate).
  // off[L] (= cnt + 3) = start of level L in nodes[].
  unsigned* ctr = a.cnt;
  unsigned* off = a.cnt + 3;
  if (blockIdx.x == 0 && threadIdx.x == 0) a.hdr->t[0] = dev::global_ns();
  // run init inside the kernel (no memset / init launches before it): zero
  // the results, set the level counters and the root item
  for (unsigned v = blockIdx.x * blockDim.x + threadIdx.x; v < a.n; v += gridDim.x * blockDim.x) a.res[v] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned r = a.root_internal ? 1u : 0u;
    ctr[0] = ctr[1] = ctr[2] = 0;
    off[0] = 0;
    off[1] = r;
    if (r) a.nodes[0] = a.root;
  }
  grid.sync();
  unsigned lo = 0, hi = *reinterpret_cast<volatile unsigned*>(off + 1), levels = 0;
  // one pass over the level's items [lo, hi): every block-uniform loop
  // iteration takes per_block items (block_reserve synchronises the block)
  const unsigned per_block = (blockDim.x >> 5) * gpw;
  auto expand = [&](unsigned base0, unsigned stride, unsigned* app) {
    for (unsigned base = base0; base < hi; base += stride) {
      unsigned i = base + dev::warp_in_block() * gpw + lane / g;
      bool active = i < hi;
      unsigned v = active ? a.nodes[i] : 0;
      // the lane's first kKeep internal children stay in registers for the
      // write below (no second dependent clist / cstart round trip)
      constexpr unsigned kKeep = 4;
      unsigned want = 0, leaves = 0, kid[kKeep];
      if (active) {
        const unsigned b = __ldg(a.cstart + v), e = __ldg(a.cstart + v + 1);
        for (unsigned k = b + sub; k < e; k += g) {
          const unsigned c = static_cast<unsigned>(__ldg(a.clist + k));
          if (nkids(a, c) > 0) {
#pragma unroll
            for (unsigned j = 0; j < kKeep; j++)
              if (j == want) kid[j] = c;
            want++;
          } else {
            leaves++;
          }
        }
      }
      unsigned wi = want, wl = leaves;
      for (unsigned o = g >> 1; o > 0; o >>= 1) {
        wi += __shfl_xor_sync(dev::kFull, wi, o);
        wl += __shfl_xor_sync(dev::kFull, wl, o);
      }
      if (active && sub == 0) {
        a.res[v] = a.is_max ? (wl ? 1 : 0) : static_cast<int>(wl);
        a.pend[v] = wi ? wi : kNoInternal;
      }
      unsigned bb, bt;
      unsigned at = hi + dev::block_reserve(app, want, &bb, &bt);
      if (active && want) {
#pragma unroll
        for (unsigned j = 0; j < kKeep; j++) {
          if (j < want) {
            if (at + j < a.cap) a.nodes[at + j] = kid[j];
            else atomicOr(&a.hdr->overflow, 1u);
          }
        }
        if (want > kKeep) {  // rare: more internal children than kept
          const unsigned b = __ldg(a.cstart + v), e = __ldg(a.cstart + v + 1);
          unsigned seen = 0, pos = at + kKeep;
          for (unsigned k = b + sub; k < e; k += g) {
            const unsigned c = static_cast<unsigned>(__ldg(a.clist + k));
            if (nkids(a, c) > 0 && seen++ >= kKeep) {
              if (pos < a.cap) a.nodes[pos] = c;
              else atomicOr(&a.hdr->overflow, 1u);
              pos++;
            }
          }
        }
      }
    }
  };
  // top-down, small levels: block 0 alone with block barriers (a device-wide
  // barrier costs more than the few passes such a level needs)
  __shared__ unsigned s_state[3];
  if (blockIdx.x == 0) {
    while (hi > lo && levels < max_levels && hi - lo <= kSmallLevel * per_block) {
      unsigned* app = ctr + levels % 3;
      if (threadIdx.x == 0) ctr[(levels + 1) % 3] = 0;
      __syncthreads();
      expand(lo, per_block, app);
      __syncthreads();
      levels++;
      lo = hi;
      hi = min(hi + *reinterpret_cast<volatile unsigned*>(app), a.cap);
      if (threadIdx.x == 0) off[levels + 1] = hi;
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      unsigned* st = off + max_levels + 2;  // scratch past the level offsets: hand the state to every block
      st[0] = lo;
      st[1] = hi;
      st[2] = levels;
    }
  }
  grid.sync();
  if (threadIdx.x == 0) {
    const volatile unsigned* st = off + max_levels + 2;
    s_state[0] = st[0];
    s_state[1] = st[1];
    s_state[2] = st[2];
  }
  __syncthreads();
  lo = s_state[0];
  hi = s_state[1];
  levels = s_state[2];
  // top-down, the rest: every block, one device-wide barrier per level
  while (hi > lo && levels < max_levels) {
    unsigned* app = ctr + levels % 3;
    if (blockIdx.x == 0 && threadIdx.x == 0) ctr[(levels + 1) % 3] = 0;
    expand(lo + blockIdx.x * per_block, nwarps * gpw, app);
    grid.sync();
    levels++;
    lo = hi;
    hi = min(hi + *reinterpret_cast<volatile unsigned*>(app), a.cap);
    if (blockIdx.x == 0 && threadIdx.x == 0) off[levels + 1] = hi;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) a.hdr->t[1] = dev::global_ns();
  // bottom-up.  The deep, wide levels (>= kPullMin internal nodes, a suffix
  // of the levels) and the one above them fold by gathering their
  // children's results, one device-wide barrier per level (no atomics);
  // everything above by count-down chains started from that level and from
  // the leaf-only nodes higher up.
  const unsigned stride = gridDim.x * blockDim.x;
  const unsigned gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  unsigned P = levels;
  while (P > 0 && off[P] - off[P - 1] >= kPullMin) P--;
  const unsigned pull_top = P > 0 ? P - 1 : 0;  // levels [pull_top, levels) gather
  if (P < levels) {
    // the deepest level's nodes have only leaf children: the top-down
    // already left their final result (the leaf share) in res
    for (int L = static_cast<int>(levels) - 2; L >= static_cast<int>(pull_top); L--) {
      const unsigned l0 = off[L], l1 = off[L + 1];
      for (unsigned base = l0 + gwarp * gpw; base < l1; base += nwarps * gpw) {
        const unsigned i = base + lane / g;
        const bool active = i < l1;
        fold_node(a, active ? a.nodes[i] : 0, sub, g, active);
      }
      grid.sync();
    }
  }
  const unsigned chain_end = P < levels ? off[pull_top + 1] : lo;   // nodes of the chain levels
  const unsigned folded0 = P < levels ? off[pull_top] : lo;         // [folded0, chain_end): folded, start
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < chain_end; i += stride) {
    unsigned u = a.nodes[i];
    if (i < folded0 && __ldcg(a.pend + u) != kNoInternal) continue;
    while (true) {
      const int r = atomicAdd(a.res + u, 0);  // every child's share is in
      const int p = __ldg(a.parent + u);
      if (p < 0) break;
      if (a.is_max) atomicMax(a.res + p, r + 1);
      else atomicAdd(a.res + p, r + 1);
      // acq_rel count-down: releases this share, and the child that takes
      // the count to zero acquires every sibling's (no full fences)
      unsigned old;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;"
                   : "=r"(old) : "l"(a.pend + p), "r"(0xffffffffu) : "memory");
      if (old != 1u) break;
      u = static_cast<unsigned>(p);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) a.hdr->iter = levels;
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&a.hdr->t[2], dev::global_ns());  // phase timeline: end
}

}  // namespace tree
}  // namespace dpc

using namespace dpc;

extern "C" {

// Phase timeline of the last persistent-grid tree run (ns): kernel start,
// end of the top-down levels, end of the bottom-up postwork.
dpc_status dpc_dtree_phase_ns(dpc_dtree* d, uint64_t out[3]) {
  if (!d || !out || !d->hdr_host) return fail(DPC_E_INVALID, "bad arguments");
  for (int i = 0; i < 3; i++) out[i] = d->hdr_host->t[i];
  return DPC_OK;
}

dpc_status dpc_dtree_upload(dpc_ctx* c, const dpc_tree* t, dpc_dtree** out) {
  clear_error();
  if (!c || !t || !out) return fail(DPC_E_INVALID, "NULL argument");
  if (t->n < 1 || !t->cstart || !t->clist || t->root < 0 || t->root >= t->n)
    return fail(DPC_E_INVALID, "invalid tree");
  auto* d = new (std::nothrow) dpc_dtree();
  if (!d) return fail(DPC_E_OOM, "dtree allocation failed");
  d->ctx = c;
  d->n = t->n;
  d->root = t->root;
  d->depth = t->depth;
  const size_t n = static_cast<size_t>(t->n);
  std::vector<unsigned> cs(n + 1);
  int64_t internal = 0;
  for (size_t v = 0; v <= n; v++) cs[v] = static_cast<unsigned>(t->cstart[v]);
  for (size_t v = 0; v < n; v++) {
    int64_t k = t->cstart[v + 1] - t->cstart[v];
    d->max_children = std::max(d->max_children, k);
    internal += k > 0;
  }
  d->internal = internal;
  d->root_children = t->cstart[t->root + 1] - t->cstart[t->root];
  double mean = internal ? static_cast<double>(n - 1) / static_cast<double>(internal) : 1.0;
  unsigned g = 1;
  while (g < 32 && g < mean) g <<= 1;
  d->group = g;
  cudaError_t e = cudaSuccess;
  auto chk = [&](cudaError_t x) {
    if (e == cudaSuccess) e = x;
  };
  chk(cudaMalloc(&d->parent, sizeof(int) * n));
  chk(cudaMalloc(&d->cstart, sizeof(unsigned) * (n + 1)));
  chk(cudaMalloc(&d->clist, sizeof(int) * n));
  chk(cudaMalloc(&d->result, sizeof(int) * n));
  chk(cudaMalloc(&d->level_nodes, sizeof(unsigned) * std::max<size_t>(1, static_cast<size_t>(internal))));
  chk(cudaMalloc(&d->level_off, sizeof(unsigned) * (static_cast<size_t>(t->depth) + 16)));
  chk(cudaMalloc(&d->hdr, sizeof(dev::RunHeader)));
  chk(cudaMallocHost(&d->hdr_host, sizeof(dev::RunHeader)));
  chk(cudaMallocHost(&d->off_host, sizeof(unsigned) * (static_cast<size_t>(t->depth) + 8)));
  if (e == cudaSuccess) {
    cudaStream_t s = c->stream;
    chk(cudaMemcpyAsync(d->parent, t->parent, sizeof(int) * n, cudaMemcpyHostToDevice, s));
    chk(cudaMemcpyAsync(d->cstart, cs.data(), sizeof(unsigned) * (n + 1), cudaMemcpyHostToDevice, s));
    chk(cudaMemcpyAsync(d->clist, t->clist, sizeof(int) * n, cudaMemcpyHostToDevice, s));
    chk(cudaStreamSynchronize(s));
  }
  if (e != cudaSuccess) {
    dpc_dtree_free(d);
    return cuda_fail(e, "dpc_dtree_upload");
  }
  d->cap = static_cast<unsigned>(std::max<int64_t>(1, internal));
  *out = d;
  return DPC_OK;
}

void dpc_dtree_free(dpc_dtree* d) {
  if (!d) return;
  if (d->ctx) cudaStreamSynchronize(d->ctx->stream);
  void* bufs[] = {d->parent, d->cstart, d->clist, d->result, d->level_nodes, d->level_off, d->hdr, d->pend};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (d->hdr_host) cudaFreeHost(d->hdr_host);
  if (d->off_host) cudaFreeHost(d->off_host);
  delete d;
}

int32_t* dpc_dtree_result(dpc_dtree* d) { return d ? d->result : nullptr; }

dpc_status dpc_dtree_check(dpc_ctx* c, dpc_dtree* d) {
  clear_error();
  if (!c || !d) return fail(DPC_E_INVALID, "NULL argument");
  if (!d->check_pending) return DPC_OK;
  d->check_pending = false;
  DPC_CUDA(cudaStreamSynchronize(c->stream));
  return check_header(d->hdr_host);
}

dpc_status dpc_tree_device(dpc_ctx* c, dpc_dtree* d, int32_t which, const dpc_launch_cfg* cfg,
                           dpc_metrics* met) {
  clear_error();
  if (!c || !d) return fail(DPC_E_INVALID, "NULL argument");
  {
    dpc_status pst = dpc_dtree_check(c, d);
    if (pst != DPC_OK) return pst;
  }
  if (which != DPC_APP_TREE_DESC && which != DPC_APP_TREE_HEIGHT)
    return fail(DPC_E_INVALID, "which must be DPC_APP_TREE_DESC or DPC_APP_TREE_HEIGHT");
  Cfg k;
  dpc_status st = resolve_cfg(c, which, cfg, &k);
  if (st != DPC_OK) return st;
  if (k.child_threads > 256 || k.parent_threads != 256)
    return fail(DPC_E_INVALID, "tree kernels are built for parent_threads = 256, child_threads <= 256");
  tree::Args a;
  a.cstart = d->cstart;
  a.clist = d->clist;
  a.res = d->result;
  a.nodes = d->level_nodes;
  a.cnt = d->level_off;
  a.cap = d->cap;
  a.hdr = d->hdr;
  a.n = static_cast<unsigned>(d->n);
  a.group = d->group;
  a.child_threads = k.child_threads;
  a.child_blocks = k.child_blocks;
  a.is_max = which == DPC_APP_TREE_HEIGHT;
  a.parent = d->parent;
  a.pend = nullptr;
  cudaStream_t s = c->stream;
  size_t need = 2048;
  if (k.variant == DPC_BASIC) need = static_cast<size_t>(d->internal) + 1024;  // capped by the runtime (~599K)
  else if (k.variant == DPC_WARP || k.variant == DPC_BLOCK) need = 2 * static_cast<size_t>(d->internal) + 1024;
  else if (k.variant == DPC_GRID) need = 4 * static_cast<size_t>(d->depth) + 1024;
  st = ensure_pending_limit(c, need);
  if (st != DPC_OK) return st;
  const bool persistent_grid = k.variant == DPC_GRID && k.grid_persistent;
  DPC_CUDA(cudaMemsetAsync(d->hdr, 0, sizeof(dev::RunHeader), s));
  if (!persistent_grid)  // the persistent kernel zeroes the results itself
    DPC_CUDA(cudaMemsetAsync(d->result, 0, sizeof(int) * static_cast<size_t>(d->n), s));
  const unsigned root = static_cast<unsigned>(d->root);
  const bool root_internal = d->internal > 0;
  // level_off[0] = bump pointer, level_off[1 + L] = start of level L
  // CDP / flat variants: cnt[0] = bump pointer of nodes[] (root at slot 0).
  // persistent grid: cnt[0..2] = per-level append counters, cnt[3 + L] =
  // start of level L.
  const unsigned r = root_internal ? 1u : 0u;
  const bool persistent = k.variant == DPC_GRID && k.grid_persistent;
  // (a kernel, not pageable host copies: those cost a host round trip each)
  a.root = root;
  a.root_internal = root_internal ? 1u : 0u;
  if (!persistent) {
    tree::init_run<<<1, 32, 0, s>>>(d->level_off, d->level_nodes, 0u + r, r, root, root_internal);
    DPC_CUDA(cudaGetLastError());
  }
  int64_t host_launches = 0, levels = 0;
  if (root_internal) {
    switch (k.variant) {
      case DPC_FLAT: {
        // host loop: level ranges come back through a pinned counter
        std::vector<unsigned> off{0, 1};
        unsigned lo = 0, hi = 1;
        while (hi > lo) {
          unsigned nb = std::max(1u, dev::ceil_div(hi - lo, 256u));
          tree::flat_down<<<nb, 256, 0, s>>>(a, lo, hi);
          host_launches++;
          DPC_CUDA(cudaGetLastError());
          DPC_CUDA(cudaMemcpyAsync(d->off_host, d->level_off, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
          DPC_CUDA(cudaStreamSynchronize(s));
          lo = hi;
          hi = std::min(d->off_host[0], d->cap);
          off.push_back(hi);
          levels++;
        }
        for (int64_t L = levels - 1; L >= 0; L--) {
          unsigned l0 = off[L], l1 = off[L + 1];
          unsigned nb = std::max(1u, dev::ceil_div(l1 - l0, 256u));
          tree::flat_up<<<nb, 256, 0, s>>>(a, l0, l1);
          host_launches++;
        }
        DPC_CUDA(cudaGetLastError());
        break;
      }
      case DPC_BASIC: {
        if (!d->pend) DPC_CUDA(cudaMalloc(&d->pend, sizeof(unsigned) * static_cast<size_t>(d->n)));
        a.pend = d->pend;
        tree::basic_pend_init<<<std::max(1u, dev::ceil_div(a.n, 256u)), 256, 0, s>>>(a);
        const unsigned nc = static_cast<unsigned>(d->root_children);
        tree::basic_traverse<<<dev::ceil_div(nc, k.child_threads), k.child_threads, 0, s>>>(a, root);
        host_launches += 2;
        DPC_CUDA(cudaGetLastError());
        break;
      }
      case DPC_WARP:
        tree::cons_kernel<tree::kWarp><<<1, k.child_threads, 0, s>>>(a, d->level_nodes, 1);
        host_launches++;
        break;
      case DPC_BLOCK:
        tree::cons_kernel<tree::kBlock><<<1, k.child_threads, 0, s>>>(a, d->level_nodes, 1);
        host_launches++;
        break;
      case DPC_GRID:
        if (k.grid_persistent) {
          if (!d->pend) DPC_CUDA(cudaMalloc(&d->pend, sizeof(unsigned) * static_cast<size_t>(d->n)));
          a.pend = d->pend;
          static int per_sm_cached[64] = {};
          int& per_sm = per_sm_cached[c->device & 63];
          if (!per_sm)
            DPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &per_sm, reinterpret_cast<const void*>(tree::grid_persistent), 256, 0));
          int blocks = std::max(1, per_sm) * c->sms;
          unsigned max_levels = static_cast<unsigned>(d->depth) + 1;
          void* args[] = {&a, &max_levels};
          DPC_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(tree::grid_persistent),
                                               dim3(blocks), dim3(256), args, 0, s));
        } else {
          tree::cons_kernel<tree::kGrid><<<1, k.child_threads, 0, s>>>(a, d->level_nodes, 1);
        }
        host_launches++;
        break;
    }
    DPC_CUDA(cudaGetLastError());
  }
  DPC_CUDA(cudaMemcpyAsync(d->hdr_host, d->hdr, sizeof(dev::RunHeader), cudaMemcpyDeviceToHost, s));
  if (!met) {  // asynchronous: the fault check happens at the next call (dpc_dtree_check)
    d->check_pending = true;
    return DPC_OK;
  }
  DPC_CUDA(cudaStreamSynchronize(s));
  st = check_header(d->hdr_host);
  if (st != DPC_OK) return st;
  if (met) {
    met->child_launch_count += d->hdr_host->launches;
    met->host_launches += host_launches;
    met->iterations += levels ? levels : d->hdr_host->iter;
    met->edges_processed += d->n - 1;
    met->buffer_items_inserted += d->internal;
    if (k.variant == DPC_BASIC) met->result_count += static_cast<int32_t>(d->hdr_host->next_count);
  }
  return DPC_OK;
}

}  // extern "C"
