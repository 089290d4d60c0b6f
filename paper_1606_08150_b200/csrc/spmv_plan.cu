// SpMV grid consolidation with a cached per-matrix plan (the default grid
// form on one GPU; DPC_CFG_SPMV_STREAM selects the round-1 stream kernel).
//
// The grid variant consolidates every non-empty row into one stream of
// nonzeros drained in equal slices (the reference's MultiBlock drain,
// transform.hpp:564-598).  spmv.cu's grid_stream redoes that consolidation
// -- an insert phase reserving each row's slot and stream range -- on every
// call and looks each window's rows up in an item table: ~280 warp
// instructions per 128 nonzeros, issue-bound (profiles/r01_spmv_grid_stream.txt).
//
// The matrix structure is immutable once uploaded, so the consolidation is
// too: a plan built once per matrix (host, from the CSR row offsets) holds,
// for every window of W nonzeros in CSR order, which positions start a row,
// the row segment open when the window starts, and prefix counts of the
// start bits; seg_row[s] = the row of the s-th non-empty row.  The drain
// needs no item lookup: lane l takes W/32 consecutive nonzeros straight from
// the CSR arrays (aligned int4 / float4 loads), sums its products per row
// segment from its start bits, and one 5-step segmented shuffle scan (segment
// heads from one ballot) closes the segments that span lanes.  Chunks of C
// windows are dealt round-robin to the warps; a warp carries the open
// segment from window to window in registers, so only segments cut by a
// chunk boundary are added atomically (y is zeroed first, one device-wide
// barrier).
//   default  W = 256 (8 nonzeros per lane): plan 64 B per window; the
//            per-window work (plan entry, scan, carry) is paid once per 256
//            nonzeros -- 17M warp instructions on config 2 (grid_stream:
//            36M).  It also keeps the 32K most used columns' x in shared
//            memory (slot-encoded col, per-call hot_gather + bulk-copy
//            fill; the remaining gathers read L2 only) and splits the
//            device-wide barrier (arrive after y = 0, wait before the
//            first y write).  Shape bit 13 drops the x cache.
//   bit 9    W = 128, register-staged loads (24M instructions)
//   bit 12   W = 128, col / val / plan staged in a per-warp shared-memory
//            ring by bulk copies (cp.async.bulk + mbarrier): the smem ring
//            shrinks L1, whose hits the x gathers need (measured slower)
// What bounds the default: the latency of the remaining (cold) x gathers
// and of the HBM stream on 32 warps per SM (profiles/r02_spmv_hot_lab.md).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "ctx.h"
#include "dpc_internal.h"

#ifndef DPC_TIMING_PROBES
#define DPC_TIMING_PROBES 0
#endif

namespace dpc {
namespace spmvp {

using dev::kFull;
constexpr unsigned W = 128;  // nonzeros per window (32 lanes x 4)
constexpr unsigned kNone = 0xffffffffu;

struct Args {
  const int* __restrict__ col;
  const float* __restrict__ val;
  const float* __restrict__ x;
  float* y;
  const uint4* __restrict__ plan;     // [2 * nwin]: per window {row-start bits}, {s_in, 0, 0, 0}
  const unsigned* __restrict__ seg_row;  // [nseg]
  unsigned n, m, nwin;
  unsigned* bar;  // [2]: persistent barrier count / generation (self-resetting)
  dev::RunHeader* hdr;
  unsigned probe;  // timing-probe builds only: 1 = x gathers confined to 4 KB, 2 = no x gathers
};

// x gather (timing-probe builds can confine or drop it: wrong results)
__device__ __forceinline__ float xg(const Args& a, int c) {
  if (DPC_TIMING_PROBES && a.probe == 1) return __ldg(a.x + (c & 1023));
  if (DPC_TIMING_PROBES && a.probe == 2) return 1.f;
  return __ldg(a.x + c);
}

__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

// One window's loads: the plan entry and this lane's 4 nonzeros.
struct Win {
  uint4 mk;
  unsigned sin;
  int4 c;
  float4 v;
};

__device__ __forceinline__ void win_load(const Args& a, unsigned w, Win& d) {
  const unsigned lane = dev::lane_id();
  d.mk = __ldg(a.plan + 2 * w);
  d.sin = __ldg(a.plan + 2 * w + 1).x;
  const unsigned base = w * W + 4 * lane;
  if (base + 4 <= a.m) {
    d.c = ld_stream(reinterpret_cast<const int4*>(a.col + base));
    d.v = ld_stream(reinterpret_cast<const float4*>(a.val + base));
  } else {  // the ragged last window
    int cc[4] = {0, 0, 0, 0};
    float vv[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int e = 0; e < 4; e++)
      if (base + e < a.m) cc[e] = __ldg(a.col + base + e), vv[e] = __ldg(a.val + base + e);
    d.c = make_int4(cc[0], cc[1], cc[2], cc[3]);
    d.v = make_float4(vv[0], vv[1], vv[2], vv[3]);
  }
}

__device__ __forceinline__ void row_add(const Args& a, unsigned seg, float s, bool atomic) {
  const unsigned r = __ldg(a.seg_row + seg);
  if (atomic) atomicAdd(a.y + r, s);
  else a.y[r] = s;
}

// Drains one window given its loads and the products p[4]; carry / open
// flags thread the warp's open segment through consecutive windows.
//   carry   : the open segment's sum so far (all lanes hold it)
//   partial : the open segment began before this warp's chunk (atomic close)
//   skip    : the open segment belongs wholly to the previous warp (the
//             chunk starts exactly on a row start): close without writing
__device__ __forceinline__ void win_drain(const Args& a, const Win& d, const float p[4], float& carry,
                                          bool& partial, bool& skip) {
  const unsigned lane = dev::lane_id();
  const unsigned wsel = lane >> 3;
  const unsigned word = wsel == 0 ? d.mk.x : wsel == 1 ? d.mk.y : wsel == 2 ? d.mk.z : d.mk.w;
  const unsigned sh = (lane & 7u) * 4u;
  const unsigned my4 = (word >> sh) & 0xfu;
  const unsigned before = (wsel > 0 ? __popc(d.mk.x) : 0u) + (wsel > 1 ? __popc(d.mk.y) : 0u) +
                          (wsel > 2 ? __popc(d.mk.z) : 0u) + __popc(word & ((1u << sh) - 1u));
  // per-lane segmentation: head (before the first start), inner segments, tail
  float head = 0.f, run = 0.f;
  unsigned k = 0;  // starts seen in this lane
#pragma unroll
  for (int e = 0; e < 4; e++) {
    if ((my4 >> e) & 1u) {
      if (k == 0) head = run;
      else row_add(a, d.sin + before + k, run, false);  // inner segment: whole inside this lane
      run = 0.f;
      k++;
    }
    run += p[e];
  }
  if (k == 0) head = run;
  const float tail = k ? run : 0.f;
  // lanes' recurrence carry_l = (k_l == 0) ? carry_{l-1} + head_l : tail_l:
  // a segmented inclusive scan whose segments start at the lanes holding a
  // row start (known to every lane from one ballot)
  const unsigned starts = __ballot_sync(kFull, k != 0);
  const unsigned upto = starts & (lane == 31 ? kFull : (2u << lane) - 1u);
  const unsigned sfirst = upto ? 31u - __clz(upto) : 0u;
  float val = k ? tail : head;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float t = __shfl_up_sync(kFull, val, o);
    if (lane >= sfirst + static_cast<unsigned>(o)) val += t;
  }
  // entering lane l: the lanes before it (+ the carry from earlier windows
  // when none of them starts a row)
  float ex = __shfl_up_sync(kFull, val, 1);
  if (k != 0) {
    const bool none_before = (starts & ((1u << lane) - 1u)) == 0u;
    if (lane == 0) ex = 0.f;
    if (none_before) ex += carry;
    const float total = ex + head;
    const unsigned seg = d.sin + before;
    if (none_before) {  // closes the segment that entered the window
      if (!skip && seg != kNone) row_add(a, seg, total, partial);
    } else {
      row_add(a, seg, total, false);
    }
  }
  const float v31 = __shfl_sync(kFull, val, 31);
  carry = starts ? v31 : carry + v31;
  if (starts) {
    partial = false;
    skip = false;
  }
}


template <int V, int NT, unsigned C>
__global__ void __launch_bounds__(NT, 1024 / NT) plan_drain(Args a) {
  const unsigned stride = gridDim.x * NT;
  const unsigned gtid = blockIdx.x * NT + threadIdx.x;
  // phase 0: y = 0 (rows closed by plain stores overwrite it; cut rows and
  // empty rows rely on it), then one device-wide barrier
  if ((reinterpret_cast<uintptr_t>(a.y) & 15u) == 0) {
    float4* y4 = reinterpret_cast<float4*>(a.y);
    for (unsigned i = gtid; i < a.n / 4; i += stride) y4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (unsigned i = (a.n & ~3u) + gtid; i < a.n; i += stride) a.y[i] = 0.f;
  } else {
    for (unsigned i = gtid; i < a.n; i += stride) a.y[i] = 0.f;
  }
  dev::soft_grid_sync(a.bar, a.bar + 1, &a.hdr->overflow);
  // phase 1: chunks of C windows dealt round-robin to the warps (warp rank
  // block-interleaved): statistically even work per warp, whatever the
  // row-length mix of a region; each chunk's open segments at its two ends
  // are the only ones added atomically
  const unsigned nw = stride >> 5;
  const unsigned gw = dev::warp_in_block() * gridDim.x + blockIdx.x;
  const unsigned nchunks = (a.nwin + C - 1) / C;
  for (unsigned ch = gw; ch < nchunks; ch += nw) {
    const unsigned w0 = ch * C, w1 = min(a.nwin, w0 + C);
    float carry = 0.f;
    bool partial = true;
    // the chunk starts on a row start: the open segment is the previous chunk's alone
    bool skip = (__ldg(a.plan + 2 * w0).x & 1u) != 0u;
    for (unsigned w = w0; w < w1; w += V) {
      Win d[V];
#pragma unroll
      for (int v = 0; v < V; v++)
        if (w + v < w1) win_load(a, w + v, d[v]);
      float p[V][4];
#pragma unroll
      for (int v = 0; v < V; v++) {
        if (w + v < w1) {
          p[v][0] = d[v].v.x * xg(a, d[v].c.x);
          p[v][1] = d[v].v.y * xg(a, d[v].c.y);
          p[v][2] = d[v].v.z * xg(a, d[v].c.z);
          p[v][3] = d[v].v.w * xg(a, d[v].c.w);
        }
      }
#pragma unroll
      for (int v = 0; v < V; v++)
        if (w + v < w1) win_drain(a, d[v], p[v], carry, partial, skip);
    }
    // the segment still open at the chunk end continues into the next chunk
    const uint4 mk = __ldg(a.plan + 2 * (w1 - 1));
    const unsigned seg = __ldg(a.plan + 2 * (w1 - 1) + 1).x + __popc(mk.x) + __popc(mk.y) + __popc(mk.z) + __popc(mk.w);
    if (dev::lane_id() == 0 && !skip && seg != kNone && carry != 0.f) row_add(a, seg, carry, true);
  }
}

// ---- TMA-staged drain: the col / val / plan bytes of each chunk arrive in a
// per-warp shared-memory ring by bulk copies (cp.async.bulk, the TMA unit)
// issued S-1 chunks ahead by one lane, completion tracked by an mbarrier per
// stage; the lanes read their nonzeros from shared memory.  HBM latency
// leaves the per-chunk dependent chain and no registers hold loads in flight.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile("{\n .reg .pred p;\n W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}" ::"r"(
                   smem_u32(bar)), "r"(parity)
               : "memory");
}

template <int V>
struct Stage {
  int col[V * W];
  float val[V * W];
  uint4 plan[2 * V];
};

template <int V, int NT, int S>
__global__ void __launch_bounds__(NT, 1024 / NT) plan_drain_tma(Args a) {
  extern __shared__ __align__(128) unsigned char smem[];
  auto* ring = reinterpret_cast<Stage<V>*>(smem) + dev::warp_in_block() * S;
  auto* bars = reinterpret_cast<unsigned long long*>(reinterpret_cast<Stage<V>*>(smem) + (NT / 32) * S) +
               dev::warp_in_block() * S;
  const unsigned lane = dev::lane_id();
  const unsigned stride = gridDim.x * NT;
  const unsigned gtid = blockIdx.x * NT + threadIdx.x;
  const unsigned nw = stride >> 5;
  const unsigned gw = dev::warp_in_block() * gridDim.x + blockIdx.x;
  const unsigned nchunks = (a.nwin + V - 1) / V;
  if (lane == 0) {
    for (int i = 0; i < S; i++) mbar_init(bars + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  // chunk it of this warp (= V windows) into stage it % S
  auto issue = [&](unsigned it) {
    const unsigned ch = gw + it * nw;
    if (ch >= nchunks) return;
    const unsigned w0 = ch * V, nwv = min(static_cast<unsigned>(V), a.nwin - w0);
    const unsigned p0 = w0 * W, np = min(a.m, p0 + nwv * W) - p0;
    const unsigned bytes = (np * 4u + 15u) & ~15u;  // <= 12 B past m: the CSR arrays carry 16 B of padding
    Stage<V>& st = ring[it % S];
    mbar_expect_tx(bars + it % S, 2u * bytes + nwv * 32u);
    bulk_g2s(st.col, a.col + p0, bytes, bars + it % S);
    bulk_g2s(st.val, a.val + p0, bytes, bars + it % S);
    bulk_g2s(st.plan, a.plan + 2 * w0, nwv * 32u, bars + it % S);
  };
  // the first S-1 chunks' bytes start flowing before the y = 0 phase
  if (lane == 0)
    for (unsigned it = 0; it + 1 < S; it++) issue(it);
  if ((reinterpret_cast<uintptr_t>(a.y) & 15u) == 0) {
    float4* y4 = reinterpret_cast<float4*>(a.y);
    for (unsigned i = gtid; i < a.n / 4; i += stride) y4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (unsigned i = (a.n & ~3u) + gtid; i < a.n; i += stride) a.y[i] = 0.f;
  } else {
    for (unsigned i = gtid; i < a.n; i += stride) a.y[i] = 0.f;
  }
  dev::soft_grid_sync(a.bar, a.bar + 1, &a.hdr->overflow);
  for (unsigned it = 0;; it++) {
    const unsigned ch = gw + it * nw;
    if (ch >= nchunks) break;
    if (lane == 0) issue(it + S - 1);  // its stage was drained at iteration it-1
    mbar_wait(bars + it % S, (it / S) & 1u);
    const Stage<V>& st = ring[it % S];
    const unsigned w0 = ch * V, nwv = min(static_cast<unsigned>(V), a.nwin - w0);
    Win d[V];
    float p[V][4];
#pragma unroll
    for (int v = 0; v < V; v++) {
      d[v].mk = st.plan[2 * v];
      d[v].sin = st.plan[2 * v + 1].x;
      const unsigned q = (w0 + v) * W + 4 * lane;  // global position of this lane's first nonzero
      if (v < nwv && q + 4 <= a.m) {
        d[v].c = *reinterpret_cast<const int4*>(st.col + v * W + 4 * lane);
        d[v].v = *reinterpret_cast<const float4*>(st.val + v * W + 4 * lane);
      } else {
        int cc[4] = {0, 0, 0, 0};
        float vv[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int e = 0; e < 4; e++)
          if (v < nwv && q + e < a.m) cc[e] = st.col[v * W + 4 * lane + e], vv[e] = st.val[v * W + 4 * lane + e];
        d[v].c = make_int4(cc[0], cc[1], cc[2], cc[3]);
        d[v].v = make_float4(vv[0], vv[1], vv[2], vv[3]);
      }
    }
#pragma unroll
    for (int v = 0; v < V; v++) {
      p[v][0] = d[v].v.x * xg(a, d[v].c.x);
      p[v][1] = d[v].v.y * xg(a, d[v].c.y);
      p[v][2] = d[v].v.z * xg(a, d[v].c.z);
      p[v][3] = d[v].v.w * xg(a, d[v].c.w);
    }
    __syncwarp();
    if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // reads before the stage's refill
    float carry = 0.f;
    bool partial = true;
    bool skip = (d[0].mk.x & 1u) != 0u;  // the chunk starts on a row start
#pragma unroll
    for (int v = 0; v < V; v++)
      if (v < nwv) win_drain(a, d[v], p[v], carry, partial, skip);
    uint4 lm = d[0].mk;
    unsigned ls = d[0].sin;
#pragma unroll
    for (int v = 1; v < V; v++)
      if (v < nwv) lm = d[v].mk, ls = d[v].sin;  // the chunk's last window (no dynamic indexing: registers)
    const unsigned seg = ls + __popc(lm.x) + __popc(lm.y) + __popc(lm.z) + __popc(lm.w);
    if (lane == 0 && !skip && seg != kNone && carry != 0.f) row_add(a, seg, carry, true);
  }
}

// ---- G = 8 form (default): 256-nonzero windows, 8 per lane (two int4 /
// float4 loads each of col and val), so the per-window work (plan entry,
// lane scan, carry) is paid once per 256 nonzeros.  Plan entry per window
// (64 B): row-start bits 0..255 (8 words), s_in, and the 8 per-word prefix
// counts of the start bits (bytes).
//
// Hot-column x cache: R-MAT / power-law matrices reuse few columns heavily
// (config 2: the 32K most used columns take 71 % of the nonzeros).  A
// per-matrix analysis (spmv_plan8_hot_build) picks them and re-encodes col
// with those columns replaced by slot | 0x80000000; per call a small kernel
// gathers x at the slots (hot_gather), and every block bulk-copies the slot
// table into shared memory (cp.async.bulk, one mbarrier).  A hot gather is
// then a 4-byte shared-memory access instead of a 128-byte L1TEX line per
// lane (the bound of the plain form: L1TEX 82 %, profiles/r02_spmv_hot_lab.md).
constexpr unsigned W8 = 256;

struct Args8 {
  const int* __restrict__ col;  // hot columns re-encoded (HOT)
  const float* __restrict__ val;
  const float* __restrict__ x;
  float* y;
  const unsigned* __restrict__ plan;  // [16 * nwin]
  const unsigned* __restrict__ seg_row;
  unsigned n, m, nwin;
  unsigned* bar;  // [2]: split-phase barrier count / generation (self-resetting)
  dev::RunHeader* hdr;
  const float* xh;  // HOT: [nhot4] x at the hot columns (this call's, from hot_gather)
  unsigned nhot4;   // slots, a multiple of 4
  unsigned probe;   // timing-probe builds only (wrong results): 1 prologue only, 2 no x gathers,
                    // 3 no segmentation / y stores, 4 = 2 + 3, 5 return at entry
};

// x gather through the hot-column cache: slot-encoded columns read shared memory.
// With the cache the remaining (cold) gathers are read L2-only (ld.global.cg):
// measured 52.5 vs 54.3 us on config 2 (L1-allocating) and 55.8 us
// (L1::no_allocate); without it, L1 is the only cache x has.
template <bool HOT>
__device__ __forceinline__ float xget(const float* __restrict__ x, const float* sx, int c) {
  if (HOT && c < 0) return sx[c & 0x7fffffff];
  if (HOT) return __ldcg(x + c);
  return __ldg(x + c);
}

struct WinPlan {
  unsigned word, sin, pre;  // this lane's start-bit word, the open segment, the word's prefix count
};
struct WinData {
  int cc[8];
  float vv[8];
};
__device__ __forceinline__ WinPlan load_plan(const Args8& a, unsigned w, unsigned j) {
  const unsigned* pe = a.plan + 16 * w;
  WinPlan P;
  P.word = __ldg(pe + j);
  P.sin = __ldg(pe + 8);
  P.pre = (__ldg(pe + 9 + (j >> 2)) >> (8 * (j & 3))) & 0xffu;
  return P;
}
__device__ __forceinline__ WinData load_data(const Args8& a, unsigned w, unsigned lane) {
  WinData D;
  const unsigned q = w * W8 + 8 * lane;
  if (q + 8 <= a.m) {
    const int4 c0 = ld_stream(reinterpret_cast<const int4*>(a.col + q));
    const int4 c1 = ld_stream(reinterpret_cast<const int4*>(a.col + q + 4));
    const float4 v0 = ld_stream(reinterpret_cast<const float4*>(a.val + q));
    const float4 v1 = ld_stream(reinterpret_cast<const float4*>(a.val + q + 4));
    D.cc[0] = c0.x, D.cc[1] = c0.y, D.cc[2] = c0.z, D.cc[3] = c0.w;
    D.cc[4] = c1.x, D.cc[5] = c1.y, D.cc[6] = c1.z, D.cc[7] = c1.w;
    D.vv[0] = v0.x, D.vv[1] = v0.y, D.vv[2] = v0.z, D.vv[3] = v0.w;
    D.vv[4] = v1.x, D.vv[5] = v1.y, D.vv[6] = v1.z, D.vv[7] = v1.w;
  } else {
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const bool in = q + e < a.m;
      D.cc[e] = in ? __ldg(a.col + q + e) : 0;
      D.vv[e] = in ? __ldg(a.val + q + e) : 0.f;
    }
  }
  return D;
}

// x at the hot columns, once per call.  The drain is launched as its
// programmatic dependent and waits for it (griddepcontrol.wait) only before
// the shared-memory fill.
__global__ void hot_gather(const float* __restrict__ x, const int* __restrict__ hot, float* xh, unsigned n4) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x)
    xh[i] = __ldg(x + __ldg(hot + i));
}

// Chunks of kChunk windows are dealt round-robin to the warps (warp rank
// block-interleaved), so at any moment the grid streams one contiguous
// region of col / val (HBM page locality; per-warp contiguous ranges measured
// 17 % slower).  The device-wide barrier that orders y = 0 before the
// atomics of cut rows is split-phase: a block arrives once its zeros are
// written, and each warp waits just before its first y write, after its first
// window's loads and gathers.
constexpr unsigned kChunk = 2;

template <int NT, bool HOT>
__global__ void __launch_bounds__(NT, 1024 / NT) plan8_drain(Args8 a) {
  extern __shared__ __align__(128) float sx[];  // HOT: x at the hot columns
  __shared__ unsigned long long s_bar;
  __shared__ unsigned s_gen0;
  const unsigned stride = gridDim.x * NT;
  const unsigned gtid = blockIdx.x * NT + threadIdx.x;
  const unsigned lane = dev::lane_id();
  const unsigned nw = stride >> 5;
  const unsigned gw = dev::warp_in_block() * gridDim.x + blockIdx.x;
  const unsigned nchunks = (a.nwin + kChunk - 1) / kChunk;
  const unsigned j = lane >> 2, sh = (lane & 3u) * 8u;
  if (DPC_TIMING_PROBES && a.probe == 5) return;
  // the warp's first window's loads go out first: their HBM latency overlaps
  // the y = 0 pass, the barrier arrival and the hot-column fill
  WinPlan P{};
  WinData D{};
  if (gw < nchunks) {
    P = load_plan(a, gw * kChunk, j);
    D = load_data(a, gw * kChunk, lane);
  }
  if (threadIdx.x == 0) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(s_gen0) : "l"(a.bar + 1) : "memory");
    if (HOT) {
      mbar_init(&s_bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  if ((reinterpret_cast<uintptr_t>(a.y) & 15u) == 0) {
    float4* y4 = reinterpret_cast<float4*>(a.y);
    for (unsigned i = gtid; i < a.n / 4; i += stride) y4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (unsigned i = (a.n & ~3u) + gtid; i < a.n; i += stride) a.y[i] = 0.f;
  } else {
    for (unsigned i = gtid; i < a.n; i += stride) a.y[i] = 0.f;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // barrier arrival (the last block opens the next generation)
    __threadfence();
    if (atomicAdd(a.bar, 1u) == gridDim.x - 1) {
      *reinterpret_cast<volatile unsigned*>(a.bar) = 0;
      __threadfence();
      atomicAdd(a.bar + 1, 1u);
    }
    if (HOT) {  // the slot table: one bulk copy per 32 KB (TMA unit)
      asm volatile("griddepcontrol.wait;" ::: "memory");
      asm volatile("fence.proxy.async.global;" ::: "memory");
      const unsigned bytes = a.nhot4 * 4u;
      mbar_expect_tx(&s_bar, bytes);
      for (unsigned off = 0; off < bytes; off += 32768u)
        bulk_g2s(reinterpret_cast<unsigned char*>(sx) + off, reinterpret_cast<const unsigned char*>(a.xh) + off,
                 min(32768u, bytes - off), &s_bar);
    }
  }
  if (HOT) mbar_wait(&s_bar, 0);
  if (DPC_TIMING_PROBES && a.probe == 1) return;
  const bool no_gather = DPC_TIMING_PROBES && (a.probe == 2 || a.probe == 4);
  const bool no_scan = DPC_TIMING_PROBES && (a.probe == 3 || a.probe == 4);
  float probe_acc = 0.f;
  bool wait_bar = true;  // this warp has not yet seen the barrier complete
  unsigned ch = gw;
  if (ch >= nchunks) return;
  unsigned w = ch * kChunk;
  bool first = true;
  float carry = 0.f;
  bool partial = true, skip = false;
  for (;;) {
    const unsigned w1 = min(a.nwin, ch * kChunk + kChunk);
    if (!first) {
      P = load_plan(a, w, j);
      D = load_data(a, w, lane);
    }
    first = false;
    const unsigned word = P.word, sin = P.sin, pre = P.pre;
    // this lane's row starts, and the rows of the first two segments it
    // closes, loaded while the gathers are in flight
    const unsigned my8 = (word >> sh) & 0xffu;
    const unsigned before = pre + __popc(word & ((1u << sh) - 1u));
    const unsigned kl = __popc(my8);
    const unsigned seg0 = sin + before;
    const unsigned r0 = (kl && seg0 != kNone) ? __ldg(a.seg_row + seg0) : 0u;
    const unsigned r1 = kl > 1 ? __ldg(a.seg_row + (seg0 + 1u)) : 0u;
    if (w == ch * kChunk) {  // chunk start: the open segment is the previous chunk's alone when it starts a row
      carry = 0.f;
      partial = true;
      skip = (__shfl_sync(kFull, word, 0) & 1u) != 0u;
    }
    float p[8];
#pragma unroll
    for (int e = 0; e < 8; e++)
      p[e] = no_gather ? D.vv[e] + __int_as_float(D.cc[e]) : D.vv[e] * xget<HOT>(a.x, sx, D.cc[e]);
    if (no_scan) {
#pragma unroll
      for (int e = 0; e < 8; e++) probe_acc += p[e] + __uint_as_float(word + sin + pre + r0 + r1);
    } else {
      if (wait_bar) {  // the device-wide barrier: every block's y = 0 is written
        if (lane == 0) {
          const unsigned long long t0 = dev::global_ns();
          for (;;) {
            unsigned gnow;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(gnow) : "l"(a.bar + 1) : "memory");
            if (gnow != s_gen0) break;
            if (dev::global_ns() - t0 > 2000000000ull) {  // watchdog: a block never arrived
              atomicOr(&a.hdr->overflow, 4u);
              break;
            }
            __nanosleep(32);
          }
        }
        __syncwarp();
        wait_bar = false;
      }
      float head = 0.f, run = 0.f;
      unsigned k = 0;
#pragma unroll
      for (int e = 0; e < 8; e++) {
        const bool st = (my8 >> e) & 1u;
        if (st && k) a.y[k == 1 ? r1 : __ldg(a.seg_row + (seg0 + k))] = run;  // segment whole inside this lane
        if (st && !k) head = run;
        run = st ? p[e] : run + p[e];
        k += st;
      }
      if (!k) head = run;
      const float tail = k ? run : 0.f;
      // lanes' recurrence carry_l = (k_l == 0) ? carry_{l-1} + head_l : tail_l:
      // a segmented inclusive scan whose segments start at the lanes holding a
      // row start (known to every lane from one ballot)
      const unsigned starts = __ballot_sync(kFull, k != 0);
      const unsigned upto = starts & (lane == 31 ? kFull : (2u << lane) - 1u);
      const unsigned sfirst = upto ? 31u - __clz(upto) : 0u;
      float v = k ? tail : head;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float t = __shfl_up_sync(kFull, v, o);
        if (lane >= sfirst + static_cast<unsigned>(o)) v += t;
      }
      float ex = __shfl_up_sync(kFull, v, 1);
      if (k) {
        const bool none_before = (starts & ((1u << lane) - 1u)) == 0u;
        if (lane == 0) ex = 0.f;
        if (none_before) ex += carry;
        if (none_before) {  // closes the segment that entered the window
          if (!skip && seg0 != kNone) {
            if (partial) atomicAdd(a.y + r0, ex + head);
            else a.y[r0] = ex + head;
          }
        } else {
          a.y[r0] = ex + head;
        }
      }
      const float v31 = __shfl_sync(kFull, v, 31);
      carry = starts ? v31 : carry + v31;
      if (starts) partial = false, skip = false;
      if (w + 1 == w1) {  // chunk end: the segment still open continues into the next chunk
        const unsigned seg_end = sin + __shfl_sync(kFull, before + k, 31);
        if (lane == 0 && !skip && seg_end != kNone && carry != 0.f)
          atomicAdd(a.y + __ldg(a.seg_row + seg_end), carry);
      }
    }
    unsigned nxt = w + 1;
    if (nxt >= w1) ch += nw, nxt = ch * kChunk;
    if (ch >= nchunks) break;
    w = nxt;
  }
  if (no_scan && probe_acc == 1.2345f) a.y[0] = probe_acc;  // keeps the probe's loads alive
}

}  // namespace spmvp

// Builds (once per matrix) the window plan from the host row offsets.
dpc_status spmv_plan_build(dpc_ctx* ctx, dpc_dgraph* g) {
  if (g->plan_mask) return DPC_OK;
  const int64_t n = g->n, m = g->m;
  if (m >= (int64_t{1} << 32) - 256) return fail(DPC_E_INVALID, "SpMV plan: too many nonzeros");
  const uint64_t nwin = static_cast<uint64_t>((m + spmvp::W - 1) / spmvp::W);
  std::vector<uint32_t> mask(4 * std::max<uint64_t>(nwin, 1), 0u), s_in(std::max<uint64_t>(nwin, 1), 0u);
  std::vector<uint32_t> seg_row;
  seg_row.reserve(static_cast<size_t>(std::min<int64_t>(n, m)) + 1);
  const auto& rp = g->host_rowptr;
  uint64_t w = 0;
  for (int64_t r = 0; r < n; r++) {
    const int64_t b = rp[r], e = rp[r + 1];
    if (e == b) continue;
    const uint32_t s = static_cast<uint32_t>(seg_row.size());
    seg_row.push_back(static_cast<uint32_t>(r));
    mask[4 * (b >> 7) + ((b & 127) >> 5)] |= 1u << (b & 31);
    // the non-empty rows tile [0, m): windows whose position -1 lies in
    // [b, e) open inside this row (window 0 opens on nothing)
    for (; w < nwin && static_cast<int64_t>(w * spmvp::W) - 1 < e; w++) s_in[w] = w == 0 ? spmvp::kNone : s;
  }
  const size_t nseg = std::max<size_t>(seg_row.size(), 1);
  std::vector<uint32_t> plan(8 * std::max<uint64_t>(nwin, 1), 0u);  // 32 B per window
  for (uint64_t i = 0; i < nwin; i++) {
    for (int j = 0; j < 4; j++) plan[8 * i + j] = mask[4 * i + j];
    plan[8 * i + 4] = s_in[i];
  }
  cudaStream_t s = ctx->stream;
  uint32_t* d_plan = nullptr;
  uint32_t* d_seg = nullptr;
  cudaError_t e = cudaMalloc(&d_plan, sizeof(uint32_t) * plan.size());
  if (e == cudaSuccess) e = cudaMalloc(&d_seg, sizeof(uint32_t) * nseg);
  if (e == cudaSuccess && !g->plan_bar) {
    e = cudaMalloc(&g->plan_bar, 2 * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemsetAsync(g->plan_bar, 0, 2 * sizeof(unsigned), s);
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_plan, plan.data(), sizeof(uint32_t) * plan.size(), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && !seg_row.empty())
    e = cudaMemcpyAsync(d_seg, seg_row.data(), sizeof(uint32_t) * seg_row.size(), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // the host vectors go out of scope
  if (e != cudaSuccess) {  // nothing half-built is published
    cudaFree(d_plan);
    cudaFree(d_seg);
    return cuda_fail(e, "SpMV plan (upload)");
  }
  g->plan_mask = d_plan;
  g->plan_segrow = d_seg;
  g->plan_nwin = static_cast<unsigned>(nwin);
  return DPC_OK;
}

// G = 8 window plan: 64 B per 256 nonzeros (+ the shared seg_row).
dpc_status spmv_plan8_build(dpc_ctx* ctx, dpc_dgraph* g) {
  if (g->plan8) return DPC_OK;
  const int64_t n = g->n, m = g->m;
  if (m >= (int64_t{1} << 32) - 512) return fail(DPC_E_INVALID, "SpMV plan: too many nonzeros");
  const uint64_t nwin = static_cast<uint64_t>((m + spmvp::W8 - 1) / spmvp::W8);
  std::vector<uint32_t> plan(16 * std::max<uint64_t>(nwin, 1), 0u);
  std::vector<uint32_t> seg_row;
  seg_row.reserve(static_cast<size_t>(std::min<int64_t>(n, m)) + 1);
  const auto& rp = g->host_rowptr;
  uint64_t w = 0;
  for (int64_t r = 0; r < n; r++) {
    const int64_t b = rp[r], e = rp[r + 1];
    if (e == b) continue;
    const uint32_t s = static_cast<uint32_t>(seg_row.size());
    seg_row.push_back(static_cast<uint32_t>(r));
    plan[16 * (b >> 8) + ((b & 255) >> 5)] |= 1u << (b & 31);
    for (; w < nwin && static_cast<int64_t>(w * spmvp::W8) - 1 < e; w++) plan[16 * w + 8] = w == 0 ? spmvp::kNone : s;
  }
  for (uint64_t i = 0; i < nwin; i++) {
    uint32_t acc = 0;
    for (int jj = 0; jj < 8; jj++) {
      plan[16 * i + 9 + jj / 4] |= acc << (8 * (jj % 4));
      acc += static_cast<uint32_t>(__builtin_popcount(plan[16 * i + jj]));
    }
  }
  // built into locals and published only when complete: a failed build
  // leaves no half-filled plan behind for the next call to trust
  cudaStream_t s = ctx->stream;
  uint32_t* d_plan = nullptr;
  uint32_t* d_seg = nullptr;
  cudaError_t e = cudaMalloc(&d_plan, sizeof(uint32_t) * plan.size());
  if (e == cudaSuccess) e = cudaMalloc(&d_seg, sizeof(uint32_t) * std::max<size_t>(seg_row.size(), 1));
  if (e == cudaSuccess && !g->plan_bar) {
    e = cudaMalloc(&g->plan_bar, 2 * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemsetAsync(g->plan_bar, 0, 2 * sizeof(unsigned), s);
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_plan, plan.data(), sizeof(uint32_t) * plan.size(), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && !seg_row.empty())
    e = cudaMemcpyAsync(d_seg, seg_row.data(), sizeof(uint32_t) * seg_row.size(), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // the host vectors go out of scope
  if (e != cudaSuccess) {
    cudaFree(d_plan);
    cudaFree(d_seg);
    return cuda_fail(e, "SpMV plan (upload)");
  }
  g->plan8 = d_plan;
  g->plan8_segrow = d_seg;
  g->plan8_nwin = static_cast<unsigned>(nwin);
  return DPC_OK;
}

namespace spmvp {
__global__ void col_degree(const int* __restrict__ col, unsigned m, unsigned* cnt) {
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    atomicAdd(cnt + __ldg(col + i), 1u);
}
__global__ void col_encode(const int* __restrict__ col, unsigned m, const int* __restrict__ slot_of, int* colh) {
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int c = __ldg(col + i), sl = __ldg(slot_of + c);
    colh[i] = sl >= 0 ? static_cast<int>(static_cast<unsigned>(sl) | 0x80000000u) : c;
  }
}
}  // namespace spmvp

// Hot-column plan (once per matrix and slot capacity): the `cap` most used
// columns (at least kHotMin uses; ties: the smaller column), slots in column
// order, and a copy of col with those columns replaced by their slot.
static dpc_status spmv_plan8_hot_build(dpc_ctx* ctx, dpc_dgraph* g, unsigned cap) {
  constexpr unsigned kHotMin = 2;
  if (g->plan8h_cap == cap) return DPC_OK;
  cudaStream_t s = ctx->stream;
  DPC_CUDA(cudaStreamSynchronize(s));
  for (void* b : {static_cast<void*>(g->plan8h_col), static_cast<void*>(g->plan8h_hot), static_cast<void*>(g->plan8h_xh)})
    if (b) cudaFree(b);
  g->plan8h_col = g->plan8h_hot = nullptr;
  g->plan8h_xh = nullptr;
  g->plan8h_cap = 0;
  const size_t nc = static_cast<size_t>(std::max<int64_t>(g->ncols, 1));
  if (g->ncols >= (int64_t{1} << 31)) return fail(DPC_E_INVALID, "SpMV hot plan: too many columns");
  const unsigned m = static_cast<unsigned>(g->m);
  std::vector<unsigned> cnt(nc, 0u);
  unsigned* d_cnt = nullptr;
  int* d_slot = nullptr;
  DPC_CUDA(cudaMalloc(&d_cnt, sizeof(unsigned) * nc));
  cudaError_t e = cudaMemsetAsync(d_cnt, 0, sizeof(unsigned) * nc, s);
  const unsigned grid = 4u * static_cast<unsigned>(ctx->sms);
  if (e == cudaSuccess && m) spmvp::col_degree<<<grid, 256, 0, s>>>(g->col, m, d_cnt);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(unsigned) * nc, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(d_cnt);
  if (e != cudaSuccess) return cuda_fail(e, "SpMV hot plan (degrees)");
  std::vector<unsigned> cand;
  for (size_t c = 0; c < nc; c++)
    if (cnt[c] >= kHotMin) cand.push_back(static_cast<unsigned>(c));
  auto hotter = [&](unsigned a, unsigned b) { return cnt[a] != cnt[b] ? cnt[a] > cnt[b] : a < b; };
  if (cand.size() > cap) {
    std::nth_element(cand.begin(), cand.begin() + cap, cand.end(), hotter);
    cand.resize(cap);
  }
  std::sort(cand.begin(), cand.end());
  const unsigned nhot4 = static_cast<unsigned>((cand.size() + 3) & ~size_t{3});
  std::vector<int> hot(std::max(nhot4, 4u), 0), slot_of(nc, -1);
  for (size_t i = 0; i < cand.size(); i++) hot[i] = static_cast<int>(cand[i]), slot_of[cand[i]] = static_cast<int>(i);
  DPC_CUDA(cudaMalloc(&g->plan8h_col, sizeof(int) * (static_cast<size_t>(m) + 16)));
  DPC_CUDA(cudaMalloc(&g->plan8h_hot, sizeof(int) * hot.size()));
  DPC_CUDA(cudaMalloc(&g->plan8h_xh, sizeof(float) * hot.size()));
  DPC_CUDA(cudaMalloc(&d_slot, sizeof(int) * nc));
  e = cudaMemcpyAsync(g->plan8h_hot, hot.data(), sizeof(int) * hot.size(), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_slot, slot_of.data(), sizeof(int) * nc, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(g->plan8h_col + m, 0, sizeof(int) * 16, s);  // the CSR arrays' padding
  if (e == cudaSuccess && m) spmvp::col_encode<<<grid, 256, 0, s>>>(g->col, m, d_slot, g->plan8h_col);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(d_slot);
  if (e != cudaSuccess) return cuda_fail(e, "SpMV hot plan (encode)");
  g->plan8h_nhot4 = nhot4;
  g->plan8h_cap = cap;
  return DPC_OK;
}

// Hot-column slot capacity: DPC_SPMV_HOT_CAP (slots; 0 disables; labs) or the
// measured default, 32K slots = 128 KB of shared memory per block
// (profiles/r02_spmv_hot_lab.md: 16K 61 us, 32K 54 us, 40K 56 us, 53K 85 us
// on config 2 -- past ~160 KB the L1 left for the streaming loads in flight
// is too small).
static unsigned spmv_hot_cap() {
  const char* e = getenv("DPC_SPMV_HOT_CAP");
  return e ? static_cast<unsigned>(atoi(e)) : 32768u;
}

template <int NT, bool HOT>
static dpc_status plan8_launch(dpc_ctx* ctx, const spmvp::Args8& a0, size_t smem) {
  const void* fn = reinterpret_cast<const void*>(spmvp::plan8_drain<NT, HOT>);
  static std::mutex mu;
  static std::map<std::pair<int, size_t>, int> cache;  // (device, smem) -> blocks per SM
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({ctx->device, smem});
    if (it != cache.end()) {
      per_sm = it->second;
    } else {
      if (smem > 48 * 1024)
        DPC_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      DPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, smem));
      cache[{ctx->device, smem}] = per_sm;
    }
  }
  if (per_sm < 1) return fail(DPC_E_CUDA, "SpMV plan kernel does not fit on an SM");
  spmvp::Args8 a = a0;
  void* args[] = {&a};
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(static_cast<unsigned>(per_sm * ctx->sms));  // all blocks co-resident (the barrier)
  lc.blockDim = dim3(NT);
  lc.dynamicSmemBytes = smem;
  lc.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = HOT ? 1 : 0;  // the hot-column gather kernel precedes it
  DPC_CUDA(cudaLaunchKernelExC(&lc, fn, args));
  return DPC_OK;
}

// y = A x with the G = 8 plan: one hot_gather launch + one persistent drain
// launch (all blocks co-resident); nohot (shape bit 13) drops the x cache.
static dpc_status spmv_plan8_run(dpc_ctx* ctx, dpc_dgraph* g, const float* d_x, float* d_y, bool nohot,
                                 unsigned probe, int* launches) {
  dpc_status st = spmv_plan8_build(ctx, g);
  if (st != DPC_OK) return st;
  spmvp::Args8 a{};
  a.col = g->col;
  a.val = g->val;
  a.x = d_x;
  a.y = d_y;
  a.plan = g->plan8;
  a.seg_row = g->plan8_segrow;
  a.n = static_cast<unsigned>(g->n);
  a.m = static_cast<unsigned>(g->m);
  a.nwin = g->plan8_nwin;
  a.bar = g->plan_bar;
  a.hdr = g->hdr;
  a.probe = probe;
  const unsigned cap = nohot ? 0u : spmv_hot_cap();
  if (cap == 0 || g->m == 0) return plan8_launch<512, false>(ctx, a, 0);
  st = spmv_plan8_hot_build(ctx, g, cap);
  if (st != DPC_OK) return st;
  a.col = g->plan8h_col;
  a.xh = g->plan8h_xh;
  a.nhot4 = g->plan8h_nhot4;
  spmvp::hot_gather<<<static_cast<unsigned>(ctx->sms), 256, 0, ctx->stream>>>(d_x, g->plan8h_hot, g->plan8h_xh,
                                                                            a.nhot4);
  DPC_CUDA(cudaGetLastError());
  *launches += 1;
  const size_t smem = sizeof(float) * std::max(a.nhot4, 4u);
  // two 512-thread blocks per SM while both copies fit, else one of 1024
  if (2 * (smem + 1024) <= static_cast<size_t>(ctx->smem_per_sm)) return plan8_launch<512, true>(ctx, a, smem);
  return plan8_launch<1024, true>(ctx, a, smem);
}

// flags: DPC_CFG_* shape bits: default = the G = 8 window form; bit 9 = the
// G = 4 form with register-staged loads, bit 12 = the G = 4 form with the
// TMA ring (both measured slower on BASELINE config 2).
dpc_status spmv_plan_run(dpc_ctx* ctx, dpc_dgraph* g, const float* d_x, float* d_y, int flags, int* launches) {
  *launches += 1;
  if (!(flags & ((1 << 9) | (1 << 12))))
    return spmv_plan8_run(ctx, g, d_x, d_y, (flags & (1 << 13)) != 0,
                          DPC_TIMING_PROBES ? static_cast<unsigned>((flags >> 16) & 7) : 0u, launches);
  dpc_status st = spmv_plan_build(ctx, g);
  if (st != DPC_OK) return st;
  spmvp::Args a{};
  a.col = g->col;
  a.val = g->val;
  a.x = d_x;
  a.y = d_y;
  a.plan = reinterpret_cast<const uint4*>(g->plan_mask);
  a.seg_row = g->plan_segrow;
  a.n = static_cast<unsigned>(g->n);
  a.m = static_cast<unsigned>(g->m);
  a.nwin = g->plan_nwin;
  a.bar = g->plan_bar;
  a.hdr = g->hdr;
  a.probe = DPC_TIMING_PROBES ? static_cast<unsigned>((flags >> 10) & 3) : 0u;
  constexpr int NT = 512, V = 2, S = 2;
  constexpr unsigned C = 4;  // windows per chunk (register form)
  const bool tma = (flags & (1 << 12)) != 0;
  const void* fn = tma ? reinterpret_cast<const void*>(spmvp::plan_drain_tma<V, NT, S>)
                       : reinterpret_cast<const void*>(spmvp::plan_drain<V, NT, C>);
  const size_t smem = tma ? (NT / 32) * S * (sizeof(spmvp::Stage<V>) + sizeof(unsigned long long)) : 0;
  static int per_sm_cached[64][2] = {};
  int& per_sm = per_sm_cached[ctx->device & 63][tma];
  if (!per_sm) {
    if (smem > 48 * 1024)
      DPC_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    DPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, smem));
  }
  if (per_sm < 1) return fail(DPC_E_CUDA, "SpMV plan kernel does not fit on an SM");
  void* args[] = {&a};
  DPC_CUDA(cudaLaunchKernel(fn, dim3(per_sm * ctx->sms), dim3(NT), args, smem, ctx->stream));
  return DPC_OK;
}

}  // namespace dpc
