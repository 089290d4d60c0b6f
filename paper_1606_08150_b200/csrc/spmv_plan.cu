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
//            nonzeros -- 17M warp instructions on config 2 (grid_stream: 36M)
//   bit 9    W = 128, register-staged loads (24M instructions)
//   bit 12   W = 128, col / val / plan staged in a per-warp shared-memory
//            ring by bulk copies (cp.async.bulk + mbarrier): the smem ring
//            shrinks L1, whose hits the x gathers need (measured slower)
// What bounds the default form: L1TEX at 82 % of peak, serving the 16.8M
// scattered x gathers (one 128-byte line per lane per gather instruction).
#include <cuda_runtime.h>

#include <algorithm>
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

// L2 prefetch of a contiguous range with one bulk-copy instruction (TMA unit).
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
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

// ---- G = 8 form: 256-nonzero windows, 8 per lane (two int4 / float4 loads),
// so the per-window work (plan entry, lane scan, carry) is paid once per 256
// nonzeros.  Plan entry per window (64 B): row-start bits 0..255 (8 words),
// s_in, and the 8 per-word prefix counts of the start bits (bytes).
constexpr unsigned W8 = 256;

struct Args8 {
  const int* __restrict__ col;
  const float* __restrict__ val;
  const float* __restrict__ x;
  float* y;
  const unsigned* __restrict__ plan;  // [16 * nwin]
  const unsigned* __restrict__ seg_row;
  unsigned n, m, nwin;
  unsigned* bar;
  dev::RunHeader* hdr;
};

__device__ __forceinline__ void row_put8(const Args8& a, unsigned seg, float s, bool atomic) {
  const unsigned r = __ldg(a.seg_row + seg);
  if (atomic) atomicAdd(a.y + r, s);
  else a.y[r] = s;
}

template <int NT, unsigned C>
__global__ void __launch_bounds__(NT, 1024 / NT) plan8_drain(Args8 a) {
  const unsigned stride = gridDim.x * NT;
  const unsigned gtid = blockIdx.x * NT + threadIdx.x;
  const unsigned lane = dev::lane_id();
  if ((reinterpret_cast<uintptr_t>(a.y) & 15u) == 0) {
    float4* y4 = reinterpret_cast<float4*>(a.y);
    for (unsigned i = gtid; i < a.n / 4; i += stride) y4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (unsigned i = (a.n & ~3u) + gtid; i < a.n; i += stride) a.y[i] = 0.f;
  } else {
    for (unsigned i = gtid; i < a.n; i += stride) a.y[i] = 0.f;
  }
  dev::soft_grid_sync(a.bar, a.bar + 1, &a.hdr->overflow);
  const unsigned nw = stride >> 5;
  const unsigned gw = dev::warp_in_block() * gridDim.x + blockIdx.x;
  const unsigned nchunks = (a.nwin + C - 1) / C;
  const unsigned j = lane >> 2, sh = (lane & 3u) * 8u;
  for (unsigned ch = gw; ch < nchunks; ch += nw) {
    const unsigned w0 = ch * C, w1 = min(a.nwin, w0 + C);
    float carry = 0.f;
    bool partial = true;
    bool skip = (__ldg(a.plan + 16 * w0) & 1u) != 0u;  // the chunk starts on a row start
    unsigned seg_end = kNone;
    for (unsigned w = w0; w < w1; w++) {
      const unsigned* pe = a.plan + 16 * w;
      const unsigned word = __ldg(pe + j);
      const unsigned sin = __ldg(pe + 8);
      const unsigned pre = (__ldg(pe + 9 + (j >> 2)) >> (8 * (j & 3))) & 0xffu;
      const unsigned q = w * W8 + 8 * lane;
      int cc[8];
      float vv[8];
      if (q + 8 <= a.m) {
        const int4 c0 = ld_stream(reinterpret_cast<const int4*>(a.col + q));
        const int4 c1 = ld_stream(reinterpret_cast<const int4*>(a.col + q + 4));
        const float4 v0 = ld_stream(reinterpret_cast<const float4*>(a.val + q));
        const float4 v1 = ld_stream(reinterpret_cast<const float4*>(a.val + q + 4));
        cc[0] = c0.x, cc[1] = c0.y, cc[2] = c0.z, cc[3] = c0.w, cc[4] = c1.x, cc[5] = c1.y, cc[6] = c1.z, cc[7] = c1.w;
        vv[0] = v0.x, vv[1] = v0.y, vv[2] = v0.z, vv[3] = v0.w, vv[4] = v1.x, vv[5] = v1.y, vv[6] = v1.z, vv[7] = v1.w;
      } else {
#pragma unroll
        for (int e = 0; e < 8; e++) {
          const bool in = q + e < a.m;
          cc[e] = in ? __ldg(a.col + q + e) : 0;
          vv[e] = in ? __ldg(a.val + q + e) : 0.f;
        }
      }
      float p[8];
#pragma unroll
      for (int e = 0; e < 8; e++) p[e] = vv[e] * __ldg(a.x + cc[e]);
      const unsigned my8 = (word >> sh) & 0xffu;
      const unsigned before = pre + __popc(word & ((1u << sh) - 1u));
      float head = 0.f, run = 0.f;
      unsigned k = 0;
#pragma unroll
      for (int e = 0; e < 8; e++) {
        const bool st = (my8 >> e) & 1u;
        if (st && k) row_put8(a, sin + before + k, run, false);  // segment whole inside this lane
        if (st && !k) head = run;
        run = st ? p[e] : run + p[e];
        k += st;
      }
      if (!k) head = run;
      const float tail = k ? run : 0.f;
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
        const unsigned seg = sin + before;
        if (none_before) {
          if (!skip && seg != kNone) row_put8(a, seg, ex + head, partial);
        } else {
          row_put8(a, seg, ex + head, false);
        }
      }
      const float v31 = __shfl_sync(kFull, v, 31);
      carry = starts ? v31 : carry + v31;
      if (starts) partial = false, skip = false;
      // segment open at this window's end
      seg_end = sin + __shfl_sync(kFull, before + k, 31);
    }
    if (lane == 0 && !skip && seg_end != kNone && carry != 0.f) row_put8(a, seg_end, carry, true);
  }
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
  DPC_CUDA(cudaMalloc(&g->plan_mask, sizeof(uint32_t) * plan.size()));
  DPC_CUDA(cudaMalloc(&g->plan_segrow, sizeof(uint32_t) * nseg));
  DPC_CUDA(cudaMalloc(&g->plan_bar, 2 * sizeof(unsigned)));
  DPC_CUDA(cudaMemcpyAsync(g->plan_mask, plan.data(), sizeof(uint32_t) * plan.size(), cudaMemcpyHostToDevice, s));
  if (!seg_row.empty())
    DPC_CUDA(cudaMemcpyAsync(g->plan_segrow, seg_row.data(), sizeof(uint32_t) * seg_row.size(),
                             cudaMemcpyHostToDevice, s));
  DPC_CUDA(cudaMemsetAsync(g->plan_bar, 0, 2 * sizeof(unsigned), s));
  DPC_CUDA(cudaStreamSynchronize(s));  // the host vectors go out of scope
  g->plan_nwin = static_cast<unsigned>(nwin);
  return DPC_OK;
}

// y = A x with the cached plan: one persistent launch (all blocks co-resident).
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
  cudaStream_t s = ctx->stream;
  DPC_CUDA(cudaMalloc(&g->plan8, sizeof(uint32_t) * plan.size()));
  DPC_CUDA(cudaMalloc(&g->plan8_segrow, sizeof(uint32_t) * std::max<size_t>(seg_row.size(), 1)));
  if (!g->plan_bar) {
    DPC_CUDA(cudaMalloc(&g->plan_bar, 2 * sizeof(unsigned)));
    DPC_CUDA(cudaMemsetAsync(g->plan_bar, 0, 2 * sizeof(unsigned), s));
  }
  DPC_CUDA(cudaMemcpyAsync(g->plan8, plan.data(), sizeof(uint32_t) * plan.size(), cudaMemcpyHostToDevice, s));
  if (!seg_row.empty())
    DPC_CUDA(cudaMemcpyAsync(g->plan8_segrow, seg_row.data(), sizeof(uint32_t) * seg_row.size(),
                             cudaMemcpyHostToDevice, s));
  DPC_CUDA(cudaStreamSynchronize(s));
  g->plan8_nwin = static_cast<unsigned>(nwin);
  return DPC_OK;
}

static dpc_status spmv_plan8_run(dpc_ctx* ctx, dpc_dgraph* g, const float* d_x, float* d_y) {
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
  constexpr int NT = 512;
  constexpr unsigned C = 2;
  const void* fn = reinterpret_cast<const void*>(spmvp::plan8_drain<NT, C>);
  static int per_sm_cached[64] = {};
  int& per_sm = per_sm_cached[ctx->device & 63];
  if (!per_sm) DPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, 0));
  if (per_sm < 1) return fail(DPC_E_CUDA, "SpMV plan kernel does not fit on an SM");
  void* args[] = {&a};
  DPC_CUDA(cudaLaunchKernel(fn, dim3(per_sm * ctx->sms), dim3(NT), args, 0, ctx->stream));
  return DPC_OK;
}

// flags: DPC_CFG_* shape bits: default = the G = 8 window form; bit 9 = the
// G = 4 form with register-staged loads, bit 12 = the G = 4 form with the
// TMA ring (both measured slower on BASELINE config 2).
dpc_status spmv_plan_run(dpc_ctx* ctx, dpc_dgraph* g, const float* d_x, float* d_y, int flags) {
  if (!(flags & ((1 << 9) | (1 << 12)))) return spmv_plan8_run(ctx, g, d_x, d_y);
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
