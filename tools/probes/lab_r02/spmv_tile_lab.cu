// LAB RECORD (round 2), not built: the TMA-producer tile form and the warp-range
// form of the SpMV grid drain, both correct and both measured slower than the
// plan8 hot-cache form (profiles/r02_spmv_hot_lab.md).  Kept as a record only.
// SpMV grid consolidation, tile-pipelined form: the default grid drain on one
// GPU (DPC_CFG_SPMV_STREAM selects the round-1 stream kernel; shape bit 14
// the plan8 register form of spmv_plan.cu).
//
// Same consolidation as spmv_plan.cu -- every non-empty row is one segment of
// the CSR nonzero stream, cut into 256-nonzero windows described by the
// cached per-matrix plan (row-start bits, open segment, prefix counts; the
// reference's MultiBlock drain, transform.hpp:564-598) -- laid out for B200:
//
//  * one block per SM, each owning a contiguous range of windows;
//  * warp 0 is a TMA producer: one lane streams the range's col / val / plan
//    bytes into an S-stage shared-memory ring with cp.async.bulk (complete_tx
//    on a per-stage mbarrier), so HBM streaming holds no registers and no L1
//    and never waits on the consumers' gathers;
//  * warps 1..31 are consumers: window l of the range goes to consumer l % 31,
//    which reads its 8 nonzeros per lane from shared memory, gathers x (hot
//    columns from a shared-memory copy of x, the rest through L1 / L2), sums
//    per row segment (lane-local runs + one segmented shuffle scan) and
//    stores y;
//  * no device-wide barrier and no y = 0 pass: rows inside one window are
//    stored once; a row cut by window boundaries ("cut row", at most one per
//    boundary) adds its per-window pieces into a self-resetting accumulator,
//    and the piece that completes the count (release / acquire atomics)
//    stores y and resets the slot; empty rows are stored as 0 from the plan's
//    list;
//  * the hot-column x values are gathered by a small kernel launched just
//    before (hot_gather), with programmatic dependent launch: the drain
//    starts streaming immediately and waits for the gather
//    (griddepcontrol.wait) only before its first x read.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>

#include "common.cuh"
#include "ctx.h"
#include "dpc_internal.h"

#ifndef DPC_TIMING_PROBES
#define DPC_TIMING_PROBES 0
#endif

namespace dpc {
namespace spmvt {

using dev::kFull;
constexpr unsigned W = 256;  // nonzeros per window (8 per lane)
constexpr unsigned kNone = 0xffffffffu;
constexpr int kConsumers = 31;

struct Args {
  const int* __restrict__ col;        // hot columns re-encoded as slot | 0x80000000 (HOT)
  const float* __restrict__ val;
  const float* __restrict__ x;
  float* y;
  const unsigned* __restrict__ plan;  // [16 * nwin]: bits 0-7, s_in 8, prefix bytes 9-10, ent 11, ext 12,
                                      // 13 = cut rows created before the window
  const unsigned* __restrict__ seg_row;
  const unsigned* __restrict__ cut_row;     // [ncut]
  const unsigned* __restrict__ cut_ctas;    // [ncut] blocks whose window ranges the cut row touches
  float* cut_acc;                           // [ncut], zero between runs
  unsigned* cut_cnt;                        // [ncut], zero between runs
  const unsigned* __restrict__ empty_rows;  // [nempty]
  const float* xh;                          // [nhot4] x at the hot columns (HOT)
  unsigned nempty, nhot4, m, nwin, ncut;
  dev::RunHeader* hdr;
  unsigned probe;  // timing-probe builds only
};

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
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Waits for the phase with the given parity; a 2 s watchdog raises fault bit
// 4 (DPC_E_DEADLOCK) and gives up instead of hanging the device.
__device__ __forceinline__ bool mbar_wait(unsigned long long* bar, unsigned parity, unsigned* fault) {
  if (mbar_try(bar, parity)) return true;
  const unsigned long long t0 = dev::global_ns();
  for (;;) {
    if (mbar_try(bar, parity)) return true;
    if (dev::global_ns() - t0 > 2000000000ull) {
      atomicOr(fault, 4u);
      return false;
    }
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int T>
struct Stage {
  int col[T * W];
  float val[T * W];
  unsigned plan[T * 16];
};

// One piece of a cut row (fire-and-forget reduction; finalised per block).
__device__ __forceinline__ void cut_piece(const Args& a, unsigned c, float v) { atomicAdd(a.cut_acc + c, v); }

// Block epilogue: the cut rows this block's windows touch.  A row inside the
// block is complete once the block's consumers are (named barrier); a row
// spanning blocks is complete when its last block arrives (acq_rel count).
__device__ __forceinline__ void cut_finish(const Args& a, unsigned c) {
  const unsigned nb = __ldg(a.cut_ctas + c);
  if (nb > 1) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(a.cut_cnt + c) : "memory");
    if (old + 1u != nb) return;
    a.cut_cnt[c] = 0u;
  }
  a.y[__ldg(a.cut_row + c)] = atomicExch(a.cut_acc + c, 0.f);
}

template <bool HOT>
__device__ __forceinline__ float xget(const float* __restrict__ x, const float* sx, int c) {
  if (HOT && c < 0) return sx[c & 0x7fffffff];
  return __ldg(x + c);
}

// x at the hot columns, once per call; lets the dependent drain launch at once.
__global__ void hot_gather(const float* __restrict__ x, const int* __restrict__ hot, float* xh, unsigned n4) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x)
    xh[i] = __ldg(x + __ldg(hot + i));
}

template <int T, int S, bool HOT>
__global__ void __launch_bounds__(32 * (kConsumers + 1), 1) tile_drain(Args a) {
  extern __shared__ __align__(128) unsigned char smem[];
  auto* ring = reinterpret_cast<Stage<T>*>(smem);
  float* sx = reinterpret_cast<float*>(ring + S);  // HOT: x at the hot columns
  __shared__ unsigned long long full[S], empty[S], hotbar;
  const unsigned lane = dev::lane_id(), wib = dev::warp_in_block();
  unsigned* fault = &a.hdr->overflow;
  // this block's windows: a contiguous range, equal in nonzeros
  const unsigned G = gridDim.x;
  const unsigned wb = static_cast<unsigned>((static_cast<unsigned long long>(a.nwin) * blockIdx.x) / G);
  const unsigned we = static_cast<unsigned>((static_cast<unsigned long long>(a.nwin) * (blockIdx.x + 1)) / G);
  const unsigned nloc = we - wb, nst = (nloc + T - 1) / T;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) mbar_init(full + s, 1), mbar_init(empty + s, T);
    mbar_init(&hotbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (wib == 0) {  // ---- producer: one lane streams the range into the ring
    if (lane == 0) {
      for (unsigned i = 0; i < nst; i++) {
        const unsigned s = i % S;
        if (i >= S && !mbar_wait(empty + s, ((i / S) - 1) & 1u, fault)) break;
        const unsigned w0 = wb + i * T, nwv = min(static_cast<unsigned>(T), we - w0);
        const unsigned p0 = w0 * W, np = min(a.m - p0, nwv * W);
        const unsigned bytes = (np * 4u + 15u) & ~15u;  // the CSR arrays carry 16 B of padding
        mbar_expect_tx(full + s, 2u * bytes + nwv * 64u);
        bulk_g2s(ring[s].col, a.col + p0, bytes, full + s);
        bulk_g2s(ring[s].val, a.val + p0, bytes, full + s);
        bulk_g2s(ring[s].plan, a.plan + 16 * w0, nwv * 64u, full + s);
      }
    }
    return;
  }
  // ---- consumers
  const unsigned cw = wib - 1;
  {
    // empty rows of the matrix are y = 0 (no other write reaches them)
    const unsigned ct = blockIdx.x * (kConsumers * 32) + cw * 32 + lane;
    for (unsigned i = ct; i < a.nempty; i += G * kConsumers * 32) a.y[__ldg(a.empty_rows + i)] = 0.f;
  }
  if (HOT) {
    if (cw == 0 && lane == 0) {  // the hot-column values (the preceding gather kernel)
      asm volatile("griddepcontrol.wait;" ::: "memory");
      asm volatile("fence.proxy.async.global;" ::: "memory");
      const unsigned bytes = a.nhot4 * 4u;
      mbar_expect_tx(&hotbar, bytes);
      for (unsigned off = 0; off < bytes; off += 32768u)
        bulk_g2s(reinterpret_cast<unsigned char*>(sx) + off, reinterpret_cast<const unsigned char*>(a.xh) + off,
                 min(32768u, bytes - off), &hotbar);
    }
  }
  // (a failed wait -- watchdog fault raised -- skips the drain but still
  // reaches the consumers' named barrier below)
  bool ok = !HOT || mbar_wait(&hotbar, 0, fault);
  const unsigned j = lane >> 2, sh = (lane & 3u) * 8u;
  for (unsigned l = cw; ok && l < nloc; l += kConsumers) {
    const unsigned i = l / T, s = i % S, t = l % T;
    if (!mbar_wait(full + s, (i / S) & 1u, fault)) {
      ok = false;
      break;
    }
    const Stage<T>& st = ring[s];
    const unsigned* pe = st.plan + 16 * t;
    const unsigned word = pe[j], sin = pe[8];
    const unsigned pre = (pe[9 + (j >> 2)] >> (8 * (j & 3))) & 0xffu;
    const unsigned ent = pe[11], ext = pe[12];
    const unsigned q = (wb + l) * W + 8 * lane;
    int cc[8];
    float vv[8];
    {
      const int4 c0 = *reinterpret_cast<const int4*>(st.col + t * W + 8 * lane);
      const int4 c1 = *reinterpret_cast<const int4*>(st.col + t * W + 8 * lane + 4);
      const float4 v0 = *reinterpret_cast<const float4*>(st.val + t * W + 8 * lane);
      const float4 v1 = *reinterpret_cast<const float4*>(st.val + t * W + 8 * lane + 4);
      cc[0] = c0.x, cc[1] = c0.y, cc[2] = c0.z, cc[3] = c0.w, cc[4] = c1.x, cc[5] = c1.y, cc[6] = c1.z, cc[7] = c1.w;
      vv[0] = v0.x, vv[1] = v0.y, vv[2] = v0.z, vv[3] = v0.w, vv[4] = v1.x, vv[5] = v1.y, vv[6] = v1.z, vv[7] = v1.w;
#pragma unroll
      for (int e = 0; e < 8; e++)
        if (q + e >= a.m) cc[e] = 0, vv[e] = 0.f;  // the ragged last window (bytes past m are padding)
    }
    __syncwarp();
    if (lane == 0) {  // the window's shared-memory bytes are in registers: release them for the refill
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(empty + s);
    }
    // this lane's row starts and the rows of the first two segments it closes
    const unsigned my8 = (word >> sh) & 0xffu;
    const unsigned before = pre + __popc(word & ((1u << sh) - 1u));
    const unsigned kl = __popc(my8);
    const unsigned seg0 = sin + before;
    const unsigned r0 = (kl && seg0 != kNone) ? __ldg(a.seg_row + seg0) : 0u;
    const unsigned r1 = kl > 1 ? __ldg(a.seg_row + (seg0 + 1u)) : 0u;
    // the last row start's segment runs to the window end: its row, unless cut
    const unsigned sb = __ballot_sync(kFull, kl != 0);
    const bool last = sb && lane == 31u - __clz(sb);
    const unsigned rt = (last && ext == kNone) ? __ldg(a.seg_row + (seg0 + kl)) : 0u;
    float p[8];
#pragma unroll
    for (int e = 0; e < 8; e++) p[e] = vv[e] * xget<HOT>(a.x, sx, cc[e]);
    float head = 0.f, run = 0.f;
    unsigned k = 0;
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const bool stt = (my8 >> e) & 1u;
      if (stt && k) a.y[k == 1 ? r1 : __ldg(a.seg_row + (seg0 + k))] = run;  // segment whole inside this lane
      if (stt && !k) head = run;
      run = stt ? p[e] : run + p[e];
      k += stt;
    }
    if (!k) head = run;
    const float tail = k ? run : 0.f;
    const unsigned starts = __ballot_sync(kFull, k != 0);
    const unsigned upto = starts & (lane == 31 ? kFull : (2u << lane) - 1u);
    const unsigned sfirst = upto ? 31u - __clz(upto) : 0u;
    float v = k ? tail : head;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const float tt = __shfl_up_sync(kFull, v, o);
      if (lane >= sfirst + static_cast<unsigned>(o)) v += tt;
    }
    float ex = __shfl_up_sync(kFull, v, 1);
    if (lane == 0) ex = 0.f;
    const float v31 = __shfl_sync(kFull, v, 31);
    if (k) {
      const bool none_before = (starts & ((1u << lane) - 1u)) == 0u;
      if (!none_before) {
        a.y[r0] = ex + head;
      } else if (ent != kNone) {  // the row entering the window is cut: its piece here
        cut_piece(a, ent, ex + head);
      }
      // the last start's segment runs to the window end
      if (lane == 31u - __clz(starts)) {
        if (ext != kNone) cut_piece(a, ext, v31);
        else a.y[rt] = v31;
      }
    } else if (starts == 0u && lane == 0) {  // no row starts here: the whole window is one piece
      cut_piece(a, ent, v31);
    }
  }
  // epilogue: every consumer's pieces are in (fence + named barrier of the
  // consumer warps), then the block's cut rows are finalised
  __threadfence();
  asm volatile("bar.sync 1, %0;" ::"r"(kConsumers * 32) : "memory");
  if (nloc == 0) return;
  const unsigned e0 = __ldg(a.plan + 16 * wb + 11);
  const unsigned lo = e0 != kNone ? e0 : __ldg(a.plan + 16 * wb + 13);
  const unsigned hi = we < a.nwin ? __ldg(a.plan + 16 * we + 13) : a.ncut;
  for (unsigned c = lo + cw * 32 + lane; c < hi; c += kConsumers * 32) cut_finish(a, c);
}


// ---- warp-range form: every warp streams, gathers and sums a contiguous
// range of windows (register loads, the next window's plan and col / val
// loaded ahead when PF), carrying the open row segment from window to window
// in registers.  Only rows crossing a warp-range boundary ("cut rows", at most
// one per boundary) are summed across warps: each touching warp adds its
// piece and the piece completing the count stores y.  No device-wide barrier,
// no y = 0 pass.
struct WArgs {
  const int* __restrict__ col;
  const float* __restrict__ val;
  const float* __restrict__ x;
  float* y;
  const unsigned* __restrict__ plan;  // [16 * nwin] (G = 8 plan)
  const unsigned* __restrict__ seg_row;
  const unsigned* __restrict__ wcut;    // [2 * nwarps]: cut row entering / leaving each warp's range
  const unsigned* __restrict__ cut_row;
  const unsigned* __restrict__ cut_pieces;
  float* cut_acc;
  unsigned* cut_cnt;
  const unsigned* __restrict__ empty_rows;
  const float* xh;
  unsigned nempty, nhot4, m, nwin;
  dev::RunHeader* hdr;
};

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

struct WPlan {
  unsigned word, sin, pre;
};
struct WData {
  int cc[8];
  float vv[8];
};
__device__ __forceinline__ WPlan wload_plan(const WArgs& a, unsigned w, unsigned j) {
  const unsigned* pe = a.plan + 16 * w;
  WPlan P;
  P.word = __ldg(pe + j);
  P.sin = __ldg(pe + 8);
  P.pre = (__ldg(pe + 9 + (j >> 2)) >> (8 * (j & 3))) & 0xffu;
  return P;
}
__device__ __forceinline__ WData wload_data(const WArgs& a, unsigned w, unsigned lane) {
  WData D;
  const unsigned q = w * W + 8 * lane;
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

// A warp's piece of a cut row; the piece completing the count stores y and
// resets the slot for the next call.
__device__ __forceinline__ void wr_piece(const WArgs& a, unsigned c, float v) {
  atomicAdd(a.cut_acc + c, v);
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(a.cut_cnt + c) : "memory");
  if (old + 1u == __ldg(a.cut_pieces + c)) {
    a.y[__ldg(a.cut_row + c)] = atomicExch(a.cut_acc + c, 0.f);
    a.cut_cnt[c] = 0u;
  }
}

template <int NT, bool HOT, int PF, int MINB>
__global__ void __launch_bounds__(NT, MINB) wrange_drain(WArgs a) {
  extern __shared__ __align__(128) float sx[];  // HOT: x at the hot columns
  __shared__ unsigned long long hotbar;
  const unsigned lane = dev::lane_id();
  const unsigned nwarps = gridDim.x * (NT / 32);
  const unsigned k = blockIdx.x * (NT / 32) + dev::warp_in_block();
  const unsigned wb = static_cast<unsigned>((static_cast<unsigned long long>(a.nwin) * k) / nwarps);
  const unsigned we = static_cast<unsigned>((static_cast<unsigned long long>(a.nwin) * (k + 1)) / nwarps);
  const unsigned j = lane >> 2, sh = (lane & 3u) * 8u;
  unsigned* fault = &a.hdr->overflow;
  // the first window's loads go out before anything else
  WPlan P{};
  WData D{};
  if (wb < we) {
    P = wload_plan(a, wb, j);
    if (PF == 2) D = wload_data(a, wb, lane);
  }
  if (HOT && threadIdx.x == 0) {
    mbar_init(&hotbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {  // empty rows are y = 0 (no other write reaches them)
    const unsigned stride = gridDim.x * NT;
    unsigned i = blockIdx.x * NT + threadIdx.x;
    for (; i + 3 * stride < a.nempty; i += 4 * stride) {
      const unsigned r0 = __ldg(a.empty_rows + i), r1 = __ldg(a.empty_rows + i + stride);
      const unsigned r2 = __ldg(a.empty_rows + i + 2 * stride), r3 = __ldg(a.empty_rows + i + 3 * stride);
      a.y[r0] = 0.f, a.y[r1] = 0.f, a.y[r2] = 0.f, a.y[r3] = 0.f;
    }
    for (; i < a.nempty; i += stride) a.y[__ldg(a.empty_rows + i)] = 0.f;
  }
  bool ok = true;
  if (HOT) {
    __syncthreads();  // the mbarrier's initialisation
    if (threadIdx.x == 0) {  // the hot-column values from the preceding gather kernel
      asm volatile("griddepcontrol.wait;" ::: "memory");
      asm volatile("fence.proxy.async.global;" ::: "memory");
      const unsigned bytes = a.nhot4 * 4u;
      mbar_expect_tx(&hotbar, bytes);
      for (unsigned off = 0; off < bytes; off += 32768u)
        bulk_g2s(reinterpret_cast<unsigned char*>(sx) + off, reinterpret_cast<const unsigned char*>(a.xh) + off,
                 min(32768u, bytes - off), &hotbar);
    }
    ok = mbar_wait(&hotbar, 0, fault);
  }
  if (!ok || wb >= we) return;
  const unsigned ent_cut = __ldg(a.wcut + 2 * k), ext_cut = __ldg(a.wcut + 2 * k + 1);
  float carry = 0.f;
  bool partial = true;  // the open segment entered the range (a cut row's piece)
  bool skip = (__shfl_sync(kFull, P.word, 0) & 1u) != 0u;  // the range starts on a row start
  for (unsigned w = wb; w < we; w++) {
    const bool more = w + 1 < we;
    WPlan Pn{};
    WData Dn{};
    if (more) Pn = wload_plan(a, w + 1, j);
    if (PF == 2 && more) Dn = wload_data(a, w + 1, lane);
    if (PF != 2) D = wload_data(a, w, lane);
    const unsigned word = P.word, sin = P.sin, pre = P.pre;
    const unsigned my8 = (word >> sh) & 0xffu;
    const unsigned before = pre + __popc(word & ((1u << sh) - 1u));
    const unsigned kl = __popc(my8);
    const unsigned seg0 = sin + before;
    const unsigned r0 = (kl && seg0 != kNone) ? __ldg(a.seg_row + seg0) : 0u;
    const unsigned r1 = kl > 1 ? __ldg(a.seg_row + (seg0 + 1u)) : 0u;
    float p[8];
#pragma unroll
    for (int e = 0; e < 8; e++) p[e] = D.vv[e] * xget<HOT>(a.x, sx, D.cc[e]);
    float head = 0.f, run = 0.f;
    unsigned kk = 0;
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const bool st = (my8 >> e) & 1u;
      if (st && kk) a.y[kk == 1 ? r1 : __ldg(a.seg_row + (seg0 + kk))] = run;  // segment whole inside this lane
      if (st && !kk) head = run;
      run = st ? p[e] : run + p[e];
      kk += st;
    }
    if (!kk) head = run;
    const float tail = kk ? run : 0.f;
    const unsigned starts = __ballot_sync(kFull, kk != 0);
    const unsigned upto = starts & (lane == 31 ? kFull : (2u << lane) - 1u);
    const unsigned sfirst = upto ? 31u - __clz(upto) : 0u;
    float v = kk ? tail : head;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const float t = __shfl_up_sync(kFull, v, o);
      if (lane >= sfirst + static_cast<unsigned>(o)) v += t;
    }
    float ex = __shfl_up_sync(kFull, v, 1);
    if (kk) {
      const bool none_before = (starts & ((1u << lane) - 1u)) == 0u;
      if (lane == 0) ex = 0.f;
      if (none_before) {
        ex += carry;
        if (!skip && seg0 != kNone) {
          if (partial) wr_piece(a, ent_cut, ex + head);
          else a.y[r0] = ex + head;
        }
      } else {
        a.y[r0] = ex + head;
      }
    }
    const float v31 = __shfl_sync(kFull, v, 31);
    carry = starts ? v31 : carry + v31;
    if (starts) partial = false, skip = false;
    if (!more) {  // range end: the open segment
      const unsigned seg_end = sin + __shfl_sync(kFull, before + kk, 31);
      if (lane == 0) {
        if (ext_cut != kNone) wr_piece(a, ext_cut, carry);  // runs on into the next range
        else if (partial) wr_piece(a, ent_cut, carry);       // entered, no row start, ends here
        else if (seg_end != kNone) a.y[__ldg(a.seg_row + seg_end)] = carry;
      }
      break;
    }
    P = Pn;
    if (PF == 2) D = Dn;
  }
}

}  // namespace spmvt

// ---- host side -----------------------------------------------------------

dpc_status spmv_plan8_build(dpc_ctx* ctx, dpc_dgraph* g);
dpc_status spmv_plan8_hot_build(dpc_ctx* ctx, dpc_dgraph* g, unsigned cap);
dpc_status spmv_tile_cuts(dpc_ctx* ctx, dpc_dgraph* g, unsigned grid);
unsigned spmv_hot_cap(unsigned dflt);
unsigned spmv_hot_cap(unsigned dflt);

template <int T, int S, bool HOT>
static dpc_status tile_launch(dpc_ctx* ctx, const spmvt::Args& a0, size_t hot_bytes) {
  const void* fn = reinterpret_cast<const void*>(spmvt::tile_drain<T, S, HOT>);
  const size_t smem = sizeof(spmvt::Stage<T>) * S + hot_bytes;
  static std::mutex mu;
  static std::map<std::pair<int, size_t>, bool> ok;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!ok.count({ctx->device, smem})) {
      DPC_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      int per_sm = 0;
      DPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * (spmvt::kConsumers + 1), smem));
      if (per_sm < 1) return fail(DPC_E_CUDA, "SpMV tile kernel does not fit on an SM");
      ok[{ctx->device, smem}] = true;
    }
  }
  spmvt::Args a = a0;
  void* args[] = {&a};
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(static_cast<unsigned>(ctx->sms));
  lc.blockDim = dim3(32 * (spmvt::kConsumers + 1));
  lc.dynamicSmemBytes = smem;
  lc.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = HOT ? 1 : 0;
  DPC_CUDA(cudaLaunchKernelExC(&lc, fn, args));
  return DPC_OK;
}


// x at the hot columns into xh (a small kernel; the drain that follows is
// launched as its programmatic dependent and waits for it only before the
// hot-column fill).
dpc_status spmv_hot_gather(dpc_ctx* ctx, const float* d_x, const int* hot, float* xh, unsigned n4) {
  spmvt::hot_gather<<<static_cast<unsigned>(ctx->sms), 256, 0, ctx->stream>>>(d_x, hot, xh, n4);
  DPC_CUDA(cudaGetLastError());
  return DPC_OK;
}

// Per-warp cut tables of the warp-range form for `nwarps` warps (warp k owns
// windows [nwin * k / nwarps, nwin * (k + 1) / nwarps)).
static dpc_status wrange_tables(dpc_ctx* ctx, dpc_dgraph* g, unsigned nwarps) {
  if (g->wr_nwarps == nwarps) return DPC_OK;
  const uint64_t nwin = g->plan8_nwin;
  const auto& pl = g->host_plan8;
  std::vector<uint32_t> wcut(2 * static_cast<size_t>(nwarps), spmvt::kNone), row, pieces;
  std::vector<uint32_t> nst(nwin + 1, 0);  // start counts, prefix
  for (uint64_t w = 0; w < nwin; w++) {
    uint32_t c = 0;
    for (int q = 0; q < 8; q++) c += static_cast<uint32_t>(__builtin_popcount(pl[16 * w + q]));
    nst[w + 1] = nst[w] + c;
  }
  uint32_t open = spmvt::kNone;
  for (unsigned k = 0; k < nwarps; k++) {
    const uint64_t wb = nwin * k / nwarps, we = nwin * (k + 1) / nwarps;
    if (wb == we) continue;
    const uint32_t ent = (pl[16 * wb] & 1u) ? spmvt::kNone : open;
    if (ent != spmvt::kNone) pieces[ent]++;
    uint32_t ext = spmvt::kNone;
    if (we < nwin && !(pl[16 * we] & 1u)) {
      if (nst[we] == nst[wb]) {
        ext = ent;  // no row starts in the range: the same row runs through
      } else {
        ext = static_cast<uint32_t>(row.size());
        row.push_back(g->host_segrow8[pl[16 * we + 8]]);
        pieces.push_back(1u);
      }
    }
    wcut[2 * k] = ent;
    wcut[2 * k + 1] = ext;
    open = ext;
  }
  for (void* b : {static_cast<void*>(g->wr_cut), static_cast<void*>(g->wr_row), static_cast<void*>(g->wr_pieces),
                  static_cast<void*>(g->wr_acc), static_cast<void*>(g->wr_cnt)})
    if (b) cudaFree(b);
  g->wr_cut = g->wr_row = g->wr_pieces = g->wr_cnt = nullptr;
  g->wr_acc = nullptr;
  g->wr_nwarps = 0;
  const size_t nc = std::max<size_t>(row.size(), 1);
  cudaStream_t s = ctx->stream;
  DPC_CUDA(cudaMalloc(&g->wr_cut, sizeof(uint32_t) * wcut.size()));
  DPC_CUDA(cudaMalloc(&g->wr_row, sizeof(uint32_t) * nc));
  DPC_CUDA(cudaMalloc(&g->wr_pieces, sizeof(uint32_t) * nc));
  DPC_CUDA(cudaMalloc(&g->wr_acc, sizeof(float) * nc));
  DPC_CUDA(cudaMalloc(&g->wr_cnt, sizeof(uint32_t) * nc));
  DPC_CUDA(cudaMemcpyAsync(g->wr_cut, wcut.data(), sizeof(uint32_t) * wcut.size(), cudaMemcpyHostToDevice, s));
  if (!row.empty()) {
    DPC_CUDA(cudaMemcpyAsync(g->wr_row, row.data(), sizeof(uint32_t) * row.size(), cudaMemcpyHostToDevice, s));
    DPC_CUDA(cudaMemcpyAsync(g->wr_pieces, pieces.data(), sizeof(uint32_t) * row.size(), cudaMemcpyHostToDevice, s));
  }
  DPC_CUDA(cudaMemsetAsync(g->wr_acc, 0, sizeof(float) * nc, s));
  DPC_CUDA(cudaMemsetAsync(g->wr_cnt, 0, sizeof(uint32_t) * nc, s));
  DPC_CUDA(cudaStreamSynchronize(s));
  g->wr_nwarps = nwarps;
  return DPC_OK;
}

template <int NT, bool HOT, int PF, int MINB>
static dpc_status wrange_launch(dpc_ctx* ctx, dpc_dgraph* g, spmvt::WArgs a, size_t smem) {
  const void* fn = reinterpret_cast<const void*>(spmvt::wrange_drain<NT, HOT, PF, MINB>);
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
  if (per_sm < 1) return fail(DPC_E_CUDA, "SpMV warp-range kernel does not fit on an SM");
  const unsigned grid = static_cast<unsigned>(per_sm * ctx->sms);
  dpc_status st = wrange_tables(ctx, g, grid * (NT / 32));
  if (st != DPC_OK) return st;
  a.wcut = g->wr_cut;
  a.cut_row = g->wr_row;
  a.cut_pieces = g->wr_pieces;
  a.cut_acc = g->wr_acc;
  a.cut_cnt = g->wr_cnt;
  void* args[] = {&a};
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(NT);
  lc.dynamicSmemBytes = smem;
  lc.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = HOT ? 1 : 0;
  DPC_CUDA(cudaLaunchKernelExC(&lc, fn, args));
  return DPC_OK;
}

static dpc_status spmv_wrange_run(dpc_ctx* ctx, dpc_dgraph* g, const float* d_x, float* d_y, int flags, int form) {
  spmvt::WArgs a{};
  a.col = g->col;
  a.val = g->val;
  a.x = d_x;
  a.y = d_y;
  a.plan = g->plan8;
  a.seg_row = g->plan8_segrow;
  a.empty_rows = g->tile_empty;
  a.nempty = g->tile_nempty;
  a.m = static_cast<unsigned>(g->m);
  a.nwin = g->plan8_nwin;
  a.hdr = g->hdr;
  const unsigned cap = (flags & (1 << 13)) ? 0u : spmv_hot_cap(32768u);
  size_t smem = 0;
  if (cap > 0 && g->m > 0) {
    dpc_status st = spmv_plan8_hot_build(ctx, g, cap);
    if (st != DPC_OK) return st;
    a.col = g->plan8h_col;
    a.xh = g->plan8h_xh;
    a.nhot4 = g->plan8h_nhot4;
    smem = sizeof(float) * std::max(a.nhot4, 4u);
    spmvt::hot_gather<<<static_cast<unsigned>(ctx->sms), 256, 0, ctx->stream>>>(d_x, g->plan8h_hot, g->plan8h_xh,
                                                                              a.nhot4);
    DPC_CUDA(cudaGetLastError());
  }
  const bool two = 2 * (smem + 1024) <= static_cast<size_t>(ctx->smem_per_sm);  // two block copies fit
  if (smem == 0) {
    if (form == 12) return wrange_launch<512, false, 2, 1>(ctx, g, a, 0);
    return wrange_launch<512, false, 1, 2>(ctx, g, a, 0);
  }
  if (form == 12) return wrange_launch<512, true, 2, 1>(ctx, g, a, smem);
  return two ? wrange_launch<512, true, 1, 2>(ctx, g, a, smem) : wrange_launch<1024, true, 1, 1>(ctx, g, a, smem);
}

// y = A x, tile-pipelined drain with the cached plan (one gather launch + one drain launch).
dpc_status spmv_tile_run(dpc_ctx* ctx, dpc_dgraph* g, const float* d_x, float* d_y, int flags) {
  dpc_status st = spmv_plan8_build(ctx, g);
  if (st != DPC_OK) return st;
  const char* fe = getenv("DPC_SPMV_TILE");
  const int form = fe ? atoi(fe) : 11;
  if (form >= 10) return spmv_wrange_run(ctx, g, d_x, d_y, flags, form);
  st = spmv_tile_cuts(ctx, g, static_cast<unsigned>(ctx->sms));
  if (st != DPC_OK) return st;
  spmvt::Args a{};
  a.col = g->col;
  a.val = g->val;
  a.x = d_x;
  a.y = d_y;
  a.plan = g->plan8;
  a.seg_row = g->plan8_segrow;
  a.cut_row = g->tile_cut_row;
  a.cut_ctas = g->tile_cut_ctas;
  a.ncut = g->tile_ncut;
  a.cut_acc = g->tile_cut_acc;
  a.cut_cnt = g->tile_cut_cnt;
  a.empty_rows = g->tile_empty;
  a.nempty = g->tile_nempty;
  a.m = static_cast<unsigned>(g->m);
  a.nwin = g->plan8_nwin;
  a.hdr = g->hdr;
  const unsigned cap = (flags & (1 << 13)) ? 0u : spmv_hot_cap(24576u);
  size_t hot_bytes = 0;
  if (cap > 0 && g->m > 0) {
    st = spmv_plan8_hot_build(ctx, g, cap);
    if (st != DPC_OK) return st;
    a.col = g->plan8h_col;
    a.xh = g->plan8h_xh;
    a.nhot4 = g->plan8h_nhot4;
    hot_bytes = sizeof(float) * std::max(a.nhot4, 4u);
    spmvt::hot_gather<<<static_cast<unsigned>(ctx->sms), 256, 0, ctx->stream>>>(d_x, g->plan8h_hot, g->plan8h_xh,
                                                                              a.nhot4);
    DPC_CUDA(cudaGetLastError());
  }
  if (hot_bytes) {
    switch (form) {
      case 1: return tile_launch<8, 8, true>(ctx, a, hot_bytes);
      case 2: return tile_launch<4, 12, true>(ctx, a, hot_bytes);
      case 3: return tile_launch<16, 4, true>(ctx, a, hot_bytes);
      default: return tile_launch<8, 6, true>(ctx, a, hot_bytes);
    }
  }
  switch (form) {
    case 1: return tile_launch<8, 8, false>(ctx, a, 0);
    case 2: return tile_launch<4, 12, false>(ctx, a, 0);
    case 3: return tile_launch<16, 4, false>(ctx, a, 0);
    default: return tile_launch<8, 6, false>(ctx, a, 0);
  }
}

}  // namespace dpc
