// SSSP / BFS grid consolidation for graphs that outgrow L2: the frontier
// stream form (DPC_CFG_GRID_STREAM).
//
// The grid variant's consolidated child is the reference's MultiBlock drain
// (transform.hpp:564-598): all grid threads work through the buffered items.
// Here, as in the SpMV grid form (spmv.cu, grid_stream), the buffered items
// of one level -- the frontier vertices -- form ONE virtual stream of
// out-edges, cut into equal slices, one per warp, so every warp relaxes the
// same number of edges whatever the degree distribution (the paper's
// Fig. 1(b) loop, with the per-vertex child launches
// replaced by stream slices).
//
// Level L of data-driven Bellman-Ford inside ONE persistent kernel:
//   drain  each warp relaxes its slice of F_L's edge stream: aligned int4
//          loads of col / w (streamed past L1, evict-first in L2), dist[v]
//          gathers through L2, atomicMin on improvement;
//   mark   an improved vertex sets its bit in the level-parity bitmap
//          (n/8 bytes: L2-resident even at scale 24, where the 64 MB stamp
//          array of the level form is not); the lane that sets the bit
//          queues the vertex in the block's shared-memory queue;
//   flush  a block reserves its queued vertices' item slots AND their edge
//          stream range with ONE packed 64-bit atomic (slot << 36 | edges),
//          so slot order is stream order; vertices without out-edges are
//          dropped;
//   clear  the bitmap that marked F_L is zeroed (grid-stride) for level L+1;
//   one device-wide barrier.
// Distances reach the unique fixpoint (Dijkstra's), so the result is
// bit-exact whatever the schedule (oracle: orc_sssp_dijkstra).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "ctx.h"
#include "dpc_internal.h"

namespace dpc {
namespace ssst {

using dev::kFull;
constexpr unsigned kInf = 0xffffffffu;
constexpr int kShift = 36;  // packed reservation: items << 36 | stream positions
constexpr unsigned long long kPosMask = (1ull << kShift) - 1;
constexpr int G = 4;           // stream positions per lane group (one int4 of col / w)
constexpr unsigned W = 32u * G;  // positions per warp window
constexpr unsigned KB = 64;    // items per warp window buffer
constexpr unsigned QW = 256;    // per-warp queue of next-frontier vertices

// Counters (64 B, in the graph's ctr buffer): res[L % 3] = level L's packed
// reservation; relaxed = sum of the levels' exact edge counts; fverts = sum of
// the frontier sizes; levels.
struct Ctr {
  unsigned long long res[3];
  unsigned long long relaxed;
  unsigned long long fverts;
  unsigned levels;
  unsigned pad[5];
};
static_assert(sizeof(Ctr) == 64, "Ctr must be 64 bytes");

struct Args {
  const unsigned* __restrict__ rowptr;
  const int* __restrict__ col;
  const int* __restrict__ w;  // nullptr: unit weights (BFS levels)
  unsigned* dist;
  unsigned* bits;  // [2][nwords] level-parity membership bitmaps
  uint4* items;    // [2][cap] {stream offset, CSR begin, CSR end, vertex}
  Ctr* ctr;
  dev::RunHeader* hdr;
  unsigned n, nwords, cap;
  unsigned coop;
};

// One warp's drain state: its window onto the item list and its queue of
// next-frontier vertices (flushed with one 64-bit reservation per 32).
struct Warp {
  uint4* buf;   // KB items
  unsigned* dub;  // their sources' distances
  unsigned* q;  // QW queued vertices
  unsigned qn;  // warp-uniform
  unsigned edges;  // this lane's share of the flushed items' edges
};

// Streamed CSR data: past L1, evict-first in L2 (keeps dist and the bitmaps
// L2-resident while the edge stream flows through).
__device__ __forceinline__ unsigned long long evict_first_policy() {
  unsigned long long pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ int4 ld_stream4(const int* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(evict_first_policy()));
  return r;
}

__device__ __forceinline__ unsigned stream_len(unsigned b, unsigned e) {
  return ((e + (G - 1u)) & ~(G - 1u)) - (b & ~(G - 1u));
}

// Bits of the aligned group at CSR index k that lie inside [b, e).
__device__ __forceinline__ unsigned grp_mask(unsigned k, unsigned b, unsigned e) {
  const int lo_e = max(static_cast<int>(b - k), 0);
  const int hi_e = min(max(static_cast<int>(e - k), 0), G);
  return ((((1u << G) - 1u) << lo_e) & ((1u << hi_e) - 1u)) & ((1u << G) - 1u);
}

__device__ __forceinline__ unsigned long long warp_incl_scan64(unsigned long long v) {
  const unsigned lane = dev::lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(kFull, v, o);
    if (lane >= static_cast<unsigned>(o)) v += t;
  }
  return v;
}

// Block-wide exclusive scan of a 64-bit value; *total = block sum.
__device__ __forceinline__ unsigned long long block_excl_scan64(unsigned long long v, unsigned long long* total) {
  __shared__ unsigned long long s_w[33];
  const unsigned long long incl = warp_incl_scan64(v);
  const unsigned w = dev::warp_in_block(), nw = blockDim.x >> 5;
  if (dev::lane_id() == 31) s_w[w] = incl;
  __syncthreads();
  if (w == 0) {
    const unsigned long long x = dev::lane_id() < nw ? s_w[dev::lane_id()] : 0ull;
    const unsigned long long xi = warp_incl_scan64(x);
    if (dev::lane_id() < nw) s_w[dev::lane_id()] = xi - x;
    if (dev::lane_id() == 31) s_w[32] = xi;
  }
  __syncthreads();
  const unsigned long long off = s_w[w] + incl - v;
  *total = s_w[32];
  __syncthreads();
  return off;
}

// Writes vertex v's item at packed position `at` (slot, stream offset).
__device__ __forceinline__ void put_item(const Args& a, uint4* dst, unsigned long long at, unsigned b, unsigned e,
                                         unsigned v) {
  const unsigned long long slot = at >> kShift;
  if (slot < a.cap) dst[slot] = make_uint4(static_cast<unsigned>(at & kPosMask), b, e, v);
  else atomicOr(&a.hdr->overflow, 1u);
}

// dist[] stays L2-resident: gathers and atomics carry an evict-last hint
// (the streamed col / w carry evict-first).
__device__ __forceinline__ unsigned long long evict_last_policy() {
  unsigned long long pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ unsigned ld_dist(const unsigned* p) {
  unsigned r;
  asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(evict_last_policy()));
  return r;
}
__device__ __forceinline__ unsigned atomic_min_dist(unsigned* p, unsigned v) {
  unsigned r;
  asm volatile("atom.relaxed.gpu.global.min.L2::cache_hint.u32 %0, [%1], %2, %3;"
               : "=r"(r) : "l"(p), "r"(v), "l"(evict_last_policy()) : "memory");
  return r;
}

// Publishes the warp's queued vertices as items of level lvl+1: per 32
// vertices one packed 64-bit reservation (slot << 36 | edge positions), so
// slot order is stream order; vertices without out-edges are dropped.
__device__ __forceinline__ void warp_flush(const Args& a, Warp& wp, unsigned lvl) {
  __syncwarp();
  const unsigned lane = dev::lane_id();
  uint4* dst = a.items + static_cast<size_t>((lvl + 1) & 1) * a.cap;
  for (unsigned base = 0; base < wp.qn; base += 32) {
    const unsigned i = base + lane;
    unsigned v = 0, b = 0, e = 0;
    if (i < wp.qn) {
      v = wp.q[i];
      b = __ldg(a.rowptr + v);
      e = __ldg(a.rowptr + v + 1);
    }
    const unsigned long long want = e > b ? (1ull << kShift) | stream_len(b, e) : 0ull;
    const unsigned long long incl = warp_incl_scan64(want);
    const unsigned long long tot = __shfl_sync(kFull, incl, 31);
    unsigned long long at = 0;
    if (lane == 31 && tot) at = atomicAdd(&a.ctr->res[(lvl + 1) % 3], tot);
    at = __shfl_sync(kFull, at, 31);
    if (want) put_item(a, dst, at + incl - want, b, e, v);
    wp.edges += e - b;
  }
  wp.qn = 0;
  __syncwarp();
}

// Relaxes the masked elements of V groups (cols c[v], weights wv[v], from
// source distances du[v]); a vertex whose distance drops joins F_{lvl+1}
// once (bitmap dedup) through the warp's queue.  The 4V elements' distance
// loads, then their atomicMins, then the improved ones' bitmap marks go out
// together: three round trips per call, not up to 2 per element.  All lanes
// call.
template <bool UNIT, int V>
__device__ __forceinline__ void relax_grps(const Args& a, Warp& wp, unsigned* nbits, unsigned lvl,
                                           const unsigned (&du)[V], const int4 (&c)[V], const int4 (&wv)[V],
                                           const unsigned (&m)[V]) {
  unsigned cc[4 * V], nd[4 * V], old[4 * V];
#pragma unroll
  for (int v = 0; v < V; v++) {
    const int cv[4] = {c[v].x, c[v].y, c[v].z, c[v].w};
    const int wvv[4] = {wv[v].x, wv[v].y, wv[v].z, wv[v].w};
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const unsigned long long t = static_cast<unsigned long long>(du[v]) + (UNIT ? 1u : static_cast<unsigned>(wvv[i]));
      cc[4 * v + i] = static_cast<unsigned>(cv[i]);
      nd[4 * v + i] = ((m[v] >> i) & 1u) && t < kInf ? static_cast<unsigned>(t) : kInf;
    }
  }
#pragma unroll
  for (int k = 0; k < 4 * V; k++) old[k] = nd[k] != kInf ? ld_dist(a.dist + cc[k]) : 0u;
#pragma unroll
  for (int k = 0; k < 4 * V; k++) old[k] = nd[k] < old[k] ? atomic_min_dist(a.dist + cc[k], nd[k]) : 0u;
  unsigned ins = 0;
#pragma unroll
  for (int k = 0; k < 4 * V; k++) {
    if (nd[k] < old[k]) {
      const unsigned bit = 1u << (cc[k] & 31u);
      if (!(atomicOr(nbits + (cc[k] >> 5), bit) & bit)) ins |= 1u << k;
    }
  }
  const unsigned lane = dev::lane_id();
#pragma unroll
  for (int k = 0; k < 4 * V; k++) {
    const bool in = (ins >> k) & 1u;
    const unsigned ball = __ballot_sync(kFull, in);
    if (in) wp.q[wp.qn + __popc(ball & ((1u << lane) - 1u))] = cc[k];
    wp.qn += __popc(ball);
    if (k % 4 == 3 && wp.qn > QW - 128) warp_flush(a, wp, lvl);
  }
}

// Per-warp window onto the level's item list: KB items + their sources'
// distances (read once per refill: any current dist[u] is a real path
// length no larger than the one that queued u, so relaxing from it is exact).
__device__ __forceinline__ void load_items(const Args& a, const uint4* items, unsigned ni, unsigned base, uint4* buf,
                                           unsigned* dub) {
  const unsigned lane = dev::lane_id();
#pragma unroll
  for (unsigned i = 0; i < KB / 32; i++) {
    const unsigned idx = base + lane + 32 * i;
    uint4 v = make_uint4(0xffffffffu, 0, 0, 0);
    unsigned du = 0;
    if (idx < ni) {
      v = __ldcg(items + idx);
      du = ld_dist(a.dist + v.w);
    }
    buf[lane + 32 * i] = v;
    dub[lane + 32 * i] = du;
  }
  __syncwarp();
}

// Relaxes this warp's slice [s0, s1) of the level's edge stream (s0 a
// multiple of W).  Same window mechanics as the SpMV stream drain (spmv.cu,
// stream_drain): a 32-ary search finds the item covering s0; per window of
// W positions the lanes where an item starts form a mask (one OR reduction)
// and each lane's item is the popcount below it; V windows inside one long
// item take a lookup-free fast path.
template <bool UNIT, int V>
__device__ __forceinline__ void drain(const Args& a, Warp& wp, const uint4* items, unsigned ni, unsigned s0,
                                      unsigned s1, unsigned* nbits, unsigned lvl) {
  uint4* buf = wp.buf;
  unsigned* dub = wp.dub;
  const unsigned lane = dev::lane_id();
  const unsigned lt_mask = (2u << lane) - 1u;
  unsigned lo = 0, hi = ni;
  while (hi - lo > 1) {
    const unsigned step = (hi - lo + 31) / 32;
    const unsigned probe = lo + lane * step;
    const unsigned v = probe < hi ? __ldcg(&items[probe].x) : 0xffffffffu;
    const unsigned c = __popc(__ballot_sync(kFull, v <= s0));
    const unsigned nlo = lo + (c - 1) * step;
    hi = min(hi, nlo + step);
    lo = nlo;
  }
  unsigned ja = lo, bb = lo;
  load_items(a, items, ni, bb, buf, dub);
  for (unsigned p0 = s0; p0 < s1; p0 += W * V) {
    if (ja + 33 > bb + KB) {
      bb = ja;
      load_items(a, items, ni, bb, buf, dub);
    }
    {
      const uint4 it = buf[ja - bb];
      const unsigned iend = it.x + stream_len(it.y, it.z);
      if (p0 + W * V <= min(iend, s1)) {  // fast path: V windows inside item ja
        const unsigned du = dub[ja - bb];
        const unsigned kb = (it.y & ~(G - 1u)) + (p0 - it.x) + G * lane;
        int4 c[V], wv[V];
#pragma unroll
        for (int v = 0; v < V; v++) {
          c[v] = ld_stream4(a.col + kb + W * v);
          wv[v] = UNIT ? make_int4(1, 1, 1, 1) : ld_stream4(a.w + kb + W * v);
        }
        unsigned dus[V], ms[V];
#pragma unroll
        for (int v = 0; v < V; v++) dus[v] = du, ms[v] = grp_mask(kb + W * v, it.y, it.z);
        relax_grps<UNIT, V>(a, wp, nbits, lvl, dus, c, wv, ms);
        if (iend == p0 + W * V) ja++;
        continue;
      }
    }
    unsigned kk[V], mm[V], dd[V];
#pragma unroll
    for (int v = 0; v < V; v++) {
      const unsigned pw = p0 + W * v;
      if (ja + 33 > bb + KB) {
        bb = ja;
        load_items(a, items, ni, bb, buf, dub);
      }
      const unsigned last = min(pw + W, s1) - 1;
      const unsigned off = buf[ja - bb + lane].x;
      const unsigned bit = (off > pw && off <= last) ? 1u << ((off - pw) / G) : 0u;
      const unsigned smask = __reduce_or_sync(kFull, bit);
      const unsigned j = ja - bb + __popc(smask & lt_mask);
      const uint4 it = buf[j];
      const unsigned q = pw + G * lane;
      const bool valid = q < s1 && pw < s1;
      kk[v] = valid ? (it.y & ~(G - 1u)) + (q - it.x) : 0u;
      mm[v] = valid ? grp_mask(kk[v], it.y, it.z) : 0u;
      dd[v] = dub[j];
      ja += __popc(smask);
      ja += buf[ja + 1 - bb].x == pw + W ? 1u : 0u;
    }
    int4 c[V], wv[V];
#pragma unroll
    for (int v = 0; v < V; v++) {
      c[v] = mm[v] ? ld_stream4(a.col + kk[v]) : make_int4(0, 0, 0, 0);
      wv[v] = UNIT || !mm[v] ? make_int4(1, 1, 1, 1) : ld_stream4(a.w + kk[v]);
    }
    relax_grps<UNIT, V>(a, wp, nbits, lvl, dd, c, wv, mm);
  }
}

template <bool UNIT, int NT, int V>
__global__ void __launch_bounds__(NT, 1024 / NT) stream_persistent(Args a) {
  __shared__ uint4 s_buf[NT / 32][KB];
  __shared__ unsigned s_du[NT / 32][KB];
  __shared__ unsigned s_q[NT / 32][QW];
  __shared__ unsigned long long s_edges;
  const unsigned stride = gridDim.x * NT;
  const unsigned gtid = blockIdx.x * NT + threadIdx.x;
  const unsigned nw = stride >> 5;
  // warp rank block-interleaved: a short stream spreads over every block
  const unsigned gw = dev::warp_in_block() * gridDim.x + blockIdx.x;
  Warp wp{s_buf[dev::warp_in_block()], s_du[dev::warp_in_block()], s_q[dev::warp_in_block()], 0u, 0u};
  if (threadIdx.x == 0) s_edges = 0;
  __syncthreads();
  unsigned lvl = 0;
  for (;; lvl++) {
    const unsigned long long r = *reinterpret_cast<volatile unsigned long long*>(&a.ctr->res[lvl % 3]);
    const unsigned ni = static_cast<unsigned>(r >> kShift);
    const unsigned np = static_cast<unsigned>(r & kPosMask);
    if (ni == 0) break;
    if (gtid == 0) {
      a.ctr->res[(lvl + 2) % 3] = 0;  // last read at level lvl-1, before the barrier
      a.ctr->fverts += ni;
    }
    unsigned* cb = a.bits + static_cast<size_t>(lvl & 1) * a.nwords;  // marked F_lvl: no longer needed
    for (unsigned i = gtid; i < a.nwords; i += stride) cb[i] = 0u;
    unsigned* nbits = a.bits + static_cast<size_t>((lvl + 1) & 1) * a.nwords;
    const unsigned per = ((np + nw - 1) / nw + W - 1) / W * W;
    const unsigned s0 = min(np, gw * per), s1 = min(np, s0 + per);
    if (s0 < s1) drain<UNIT, V>(a, wp, a.items + static_cast<size_t>(lvl & 1) * a.cap, ni, s0, s1, nbits, lvl);
    warp_flush(a, wp, lvl);
    const unsigned we = dev::warp_sum(wp.edges);
    wp.edges = 0;
    if (dev::lane_id() == 0 && we) atomicAdd(&s_edges, static_cast<unsigned long long>(we));
    __syncthreads();
    if (a.coop) cooperative_groups::this_grid().sync();
    else dev::grid_sync64(&a.hdr->bar, &a.hdr->overflow);
  }
  if (gtid == 0) a.ctr->levels = lvl;
  // the block's edge count: one atomic per block per run, not per level (the
  // counters' line also carries the levels' reservations)
  __syncthreads();
  if (threadIdx.x == 0 && s_edges) atomicAdd(&a.ctr->relaxed, s_edges);
}

// Seeds F_0 = {source}.
__global__ void init_kernel(Args a, unsigned source) {
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < a.n) a.dist[i] = i == source ? 0u : kInf;
  if (i < 2 * a.nwords) a.bits[i] = 0u;
  if (i == 0) {
    const unsigned b = a.rowptr[source], e = a.rowptr[source + 1];
    a.ctr->res[1] = a.ctr->res[2] = 0;
    a.ctr->fverts = 0;
    a.ctr->levels = 0;
    a.ctr->relaxed = e - b;
    a.ctr->res[0] = e > b ? (1ull << kShift) | stream_len(b, e) : 0ull;
    if (e > b) a.items[0] = make_uint4(0u, b, e, source);
  }
}

}  // namespace ssst

// The frontier stream form of the grid variant (sssp.cu dispatches here).
dpc_status sssp_stream_run(dpc_ctx* ctx, dpc_dgraph* g, int32_t source, bool unit, bool coop,
                           int64_t* host_launches, int64_t* levels, dpc_metrics* met) {
  cudaStream_t s = ctx->stream;
  if (g->n >= (int64_t{1} << (64 - ssst::kShift)))
    return fail(DPC_E_INVALID, "frontier stream form: too many vertices for the packed reservation");
  const size_t cap = static_cast<size_t>(g->n) + 1;
  if (g->sst_cap < cap) {
    DPC_CUDA(cudaStreamSynchronize(s));
    if (g->sst_items) cudaFree(g->sst_items);
    g->sst_items = nullptr;
    g->sst_cap = 0;
    DPC_CUDA(cudaMalloc(&g->sst_items, 2 * cap * sizeof(uint4)));
    g->sst_cap = cap;
  }
  ssst::Args a{};
  a.rowptr = g->rowptr;
  a.col = g->col;
  a.w = unit ? nullptr : g->w;
  a.dist = g->dist;
  a.bits = g->stamp;  // n words >= 2 * ceil(n / 32) for n >= 2; stamp is SSSP scratch
  a.items = reinterpret_cast<uint4*>(g->sst_items);
  a.ctr = reinterpret_cast<ssst::Ctr*>(g->ctr);
  a.hdr = g->hdr;
  a.n = static_cast<unsigned>(g->n);
  a.nwords = static_cast<unsigned>((g->n + 31) / 32);
  a.cap = static_cast<unsigned>(cap);
  a.coop = coop ? 1u : 0u;
  if (2 * static_cast<int64_t>(a.nwords) > std::max<int64_t>(g->n, 2))
    return fail(DPC_E_INVALID, "frontier stream form needs n >= 64");
  const unsigned nb = std::max(1u, dev::ceil_div(std::max(a.n, 2 * a.nwords), 256u));
  ssst::init_kernel<<<nb, 256, 0, s>>>(a, static_cast<unsigned>(source));
  DPC_CUDA(cudaGetLastError());
  constexpr int NT = 512, V = 2;
  const void* fn = unit ? reinterpret_cast<const void*>(ssst::stream_persistent<true, NT, V>)
                        : reinterpret_cast<const void*>(ssst::stream_persistent<false, NT, V>);
  const int nt = NT;
  int per_sm = 0;
  DPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, nt, 0));
  if (per_sm < 1) return fail(DPC_E_CUDA, "frontier stream kernel does not fit on an SM");
  const int blocks = per_sm * ctx->sms;
  void* args[] = {&a};
  if (coop) DPC_CUDA(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(nt), args, 0, s));
  else DPC_CUDA(cudaLaunchKernel(fn, dim3(blocks), dim3(nt), args, 0, s));
  *host_launches += 2;
  if (met) {
    ssst::Ctr c{};
    DPC_CUDA(cudaMemcpyAsync(&c, a.ctr, sizeof(c), cudaMemcpyDeviceToHost, s));
    DPC_CUDA(cudaStreamSynchronize(s));
    *levels = c.levels;
    met->edges_processed += static_cast<int64_t>(c.relaxed);
    met->vertices_processed += static_cast<int64_t>(c.fverts);
  }
  return DPC_OK;
}

}  // namespace dpc
