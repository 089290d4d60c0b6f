// Size-class ("bin") drain for the grid-consolidated SpMV (probe).
// Parent phase: thread per RPT consecutive rows; light rows (deg <= T) done
// inline, heavier rows inserted into the worklist of their degree class
// (block-aggregated: shared atomics, one global atomic per class per block).
// One device-wide barrier.  Drain: per class a lane-group size matched to the
// degree (no per-position segmentation): G lanes x K positions per row,
// vector loads for the wide classes, fixed 512-position chunks above 512.
#pragma once

namespace lab {

constexpr int NBIN = 9;  // (0,4] (4,8] (8,16] (16,32] (32,64] (64,128] (128,256] (256,512] chunks(>512)
constexpr int kChunkBin = 8;
__host__ __device__ inline int class_of(unsigned d) {  // d >= 1
  return d > 512 ? kChunkBin : d <= 4 ? 0 : 31 - __builtin_clz(d - 1) - 1;
}
constexpr unsigned kChunk = 512;

struct BArgs {
  const unsigned* rowptr;
  const int* col;
  const float* val;
  const float* x;
  float* y;
  unsigned n, m;
  unsigned T;                 // inline threshold (<= 4)
  uint4* items;               // bins' regions: {row, s, e, chunk | flag}
  unsigned off[NBIN], cap[NBIN];
  unsigned* ctr;              // [0..8] class counts, [9] barrier, [10] exit, [11] fault
  unsigned long long* ts;
  unsigned mode;
};

template <int G, int K, bool VEC, int U>
__device__ __forceinline__ void drain_bin(const BArgs& a, const uint4* items, unsigned cnt, unsigned nw, unsigned first) {
  constexpr int R = 32 / G;  // rows per warp per unit
  const unsigned lane = threadIdx.x & 31u;
  const unsigned sub = lane / G, gl = lane % G;
  const unsigned per_step = R * U;
  const unsigned steps = (cnt + per_step - 1) / per_step;
  for (unsigned st = first; st < steps; st += nw) {
    uint4 it[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const unsigned i = (st * U + u) * R + sub;
      it[u] = i < cnt ? __ldcg(items + i) : make_uint4(0, 0, 0, 0);
    }
    float sum[U];
    if (!VEC) {
      int c[U][K];
      float v[U][K];
#pragma unroll
      for (int u = 0; u < U; u++)
#pragma unroll
        for (int k = 0; k < K; k++) {
          const unsigned p = it[u].y + gl + G * k;
          const bool ok = p < it[u].z;
          c[u][k] = ok ? __ldg(a.col + p) : 0;
          v[u][k] = ok ? __ldg(a.val + p) : 0.f;
        }
#pragma unroll
      for (int u = 0; u < U; u++) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < K; k++) s += v[u][k] * __ldg(a.x + c[u][k]);
        sum[u] = s;
      }
    } else {
      // aligned 4-position groups; chunk items cover 512 aligned positions
      int4 c[U][K];
      float4 v[U][K];
      unsigned lo[U], hi[U], gb[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const unsigned s = it[u].y, e = it[u].z, j = it[u].w & 0x7fffffffu;
        const unsigned base = (s & ~3u) + kChunk * j;
        gb[u] = base;
        lo[u] = max(s, base);
        hi[u] = (it[u].w & 0x80000000u) ? min(e, base + kChunk) : e;
#pragma unroll
        for (int k = 0; k < K; k++) {
          const unsigned q = base + 4u * (lane + 32u * k);
          if (q < hi[u]) {
            c[u][k] = __ldg(reinterpret_cast<const int4*>(a.col + q));
            v[u][k] = __ldg(reinterpret_cast<const float4*>(a.val + q));
          } else {
            c[u][k] = make_int4(0, 0, 0, 0);
            v[u][k] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < K; k++) {
          const unsigned q = gb[u] + 4u * (lane + 32u * k);
          const int cc[4] = {c[u][k].x, c[u][k].y, c[u][k].z, c[u][k].w};
          const float vv[4] = {v[u][k].x, v[u][k].y, v[u][k].z, v[u][k].w};
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const bool ok = q + e >= lo[u] && q + e < hi[u];
            s += (ok ? vv[e] : 0.f) * __ldg(a.x + (ok ? cc[e] : 0));
          }
        }
        sum[u] = s;
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      float s = sum[u];
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      const unsigned i = (st * U + u) * R + sub;
      if (gl == 0 && i < cnt) {
        if (it[u].w & 0x80000000u) atomicAdd(a.y + it[u].x, s);
        else a.y[it[u].x] = s;
      }
    }
  }
}

template <int NT, int RPT, int UI>
__global__ void __launch_bounds__(NT, 1) spmv_bins(BArgs a) {
  __shared__ unsigned s_cnt[NBIN], s_base[NBIN];
  const unsigned tid = threadIdx.x, b = blockIdx.x, GB = gridDim.x;
  if (tid == 0 && a.ts) a.ts[b * 8 + 0] = gns();
  if (tid < NBIN) s_cnt[tid] = 0;
  __syncthreads();
  const unsigned n = a.n;
  const unsigned per_pass = GB * NT * RPT;
  for (unsigned p0 = 0; p0 < n; p0 += per_pass) {
    const unsigned r0 = p0 + (b * NT + tid) * RPT;
    unsigned rs[RPT + 1];
#pragma unroll
    for (int i = 0; i <= RPT; i++) rs[i] = r0 + i <= n ? __ldg(a.rowptr + r0 + i) : 0u;
#pragma unroll
    for (int i = 0; i < RPT; i++)
      if (r0 + i >= n) rs[i + 1] = rs[i];
    unsigned slot[RPT];
    int bn[RPT];
#pragma unroll
    for (int i = 0; i < RPT; i++) {
      const unsigned d = rs[i + 1] - rs[i];
      bn[i] = -1;
      if (r0 + i < n) {
        if (d == 0) {
          a.y[r0 + i] = 0.f;
        } else {
          const int k = class_of(d);
          bn[i] = k;
          const unsigned nit = k == kChunkBin ? (rs[i + 1] - (rs[i] & ~3u) + kChunk - 1) / kChunk : 1u;
          slot[i] = atomicAdd(s_cnt + k, nit);
          if (k == kChunkBin) a.y[r0 + i] = 0.f;
        }
      }
    }
    __syncthreads();
    if (tid < NBIN) {
      const unsigned c = s_cnt[tid];
      s_base[tid] = c ? atomicAdd(a.ctr + tid, c) : 0u;
      s_cnt[tid] = 0;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < RPT; i++) {
      const int k = bn[i];
      if (k >= 0) {
        const unsigned at = s_base[k] + slot[i];
        const unsigned s = rs[i], e = rs[i + 1];
        if (k == kChunkBin) {
          const unsigned nit = (e - (s & ~3u) + kChunk - 1) / kChunk;
          for (unsigned j = 0; j < nit; j++) {
            if (at + j < a.cap[kChunkBin]) a.items[a.off[kChunkBin] + at + j] = make_uint4(r0 + i, s, e, j | 0x80000000u);
            else atomicOr(a.ctr + 11, 1u);
          }
        } else {
          if (at < a.cap[k]) a.items[a.off[k] + at] = make_uint4(r0 + i, s, e, 0u);
          else atomicOr(a.ctr + 11, 1u);
        }
      }
    }
  }
  // ---------------- device-wide barrier ----------------
  __syncthreads();
  if (tid == 0 && a.ts) a.ts[b * 8 + 2] = gns();
  if (tid == 0) {
    __threadfence();
    atomicAdd(a.ctr + 9, 1u);
    unsigned seen;
    const unsigned long long t0 = gns();
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(a.ctr + 9) : "memory");
      if (seen < GB) __nanosleep(32);
      if (gns() - t0 > 2000000000ull) {
        atomicOr(a.ctr + 11, 2u);
        break;
      }
    } while (seen < GB);
  }
  __syncthreads();
  if (tid == 0 && a.ts) a.ts[b * 8 + 3] = gns();
  // ---------------- drain: classes as one dealt sequence of warp steps ----------------
  const unsigned nw = GB * (NT / 32), gw = b * (NT / 32) + (tid >> 5);
  unsigned cnt[NBIN];
#pragma unroll
  for (int k = 0; k < NBIN; k++) cnt[k] = min(*reinterpret_cast<volatile unsigned*>(a.ctr + k), a.cap[k]);
  unsigned done = 0;  // steps of the classes dealt so far
  auto first = [&](unsigned steps) {
    const unsigned f = (gw + nw - done % nw) % nw;
    done += steps;
    return f;
  };
  // heaviest per step first
#define DRAIN(k, G, K, VEC, U) \
  drain_bin<G, K, VEC, U>(a, a.items + a.off[k], cnt[k], nw, first((cnt[k] + (32 / G) * U - 1) / ((32 / G) * U)))
  DRAIN(8, 32, 4, true, 1);
  DRAIN(7, 32, 5, true, 1);
  DRAIN(6, 32, 3, true, 1);
  DRAIN(5, 32, 2, true, UI);
  DRAIN(4, 16, 4, false, UI);
  DRAIN(3, 8, 4, false, UI);
  DRAIN(2, 4, 4, false, UI);
  DRAIN(1, 2, 4, false, UI);
  DRAIN(0, 1, 4, false, UI);
#undef DRAIN
  __syncthreads();
  if (tid == 0 && a.ts) a.ts[b * 8 + 4] = gns();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(a.ctr + 10, 1u) == GB - 1) {
      for (int k = 0; k < NBIN; k++) a.ctr[k] = 0;
      a.ctr[9] = 0;
      a.ctr[10] = 0;
      __threadfence();
    }
  }
}

}  // namespace lab

// ---------------------------------------------------------------------------
// v2: 7 classes, <= 32 registers (two 1024-thread blocks per SM), warp-
// aggregated class reservation, per-block shares of every class handed to the
// block's warps through shared counters (no static per-warp imbalance).
namespace lab {
constexpr int NB2 = 7;  // (0,4] (4,8] (8,16] (16,32] (32,64] (64,128] chunks of 256 (>128)
constexpr unsigned kChunk2 = 256;
__host__ __device__ inline int class2_of(unsigned d) {
  return d > 128 ? 6 : d <= 4 ? 0 : 31 - __builtin_clz(d - 1) - 1;
}

template <int G, int K, bool VEC>
__device__ __forceinline__ void unit2(const BArgs& a, const uint4* items, unsigned cnt, unsigned step) {
  constexpr int R = 32 / G;
  const unsigned lane = threadIdx.x & 31u, sub = lane / G, gl = lane % G;
  const unsigned i = step * R + sub;
  const uint4 it = i < cnt ? __ldcg(items + i) : make_uint4(0, 0, 0, 0);
  float s = 0.f;
  if (!VEC) {
    int c[K];
    float v[K];
#pragma unroll
    for (int k = 0; k < K; k++) {
      const unsigned p = it.y + gl + G * k;
      const bool ok = p < it.z;
      c[k] = ok ? __ldg(a.col + p) : 0;
      v[k] = ok ? __ldg(a.val + p) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < K; k++) s += v[k] * __ldg(a.x + c[k]);
  } else {
    const unsigned j = it.w & 0x7fffffffu;
    const unsigned base = (it.y & ~3u) + kChunk2 * j;
    const unsigned lo = max(it.y, base);
    const unsigned hi = (it.w & 0x80000000u) ? min(it.z, base + kChunk2) : it.z;
    int4 c[K];
    float4 v[K];
#pragma unroll
    for (int k = 0; k < K; k++) {
      const unsigned q = base + 4u * (lane + 32u * k);
      c[k] = q < hi ? __ldg(reinterpret_cast<const int4*>(a.col + q)) : make_int4(0, 0, 0, 0);
      v[k] = q < hi ? __ldg(reinterpret_cast<const float4*>(a.val + q)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < K; k++) {
      const unsigned q = base + 4u * (lane + 32u * k);
      s += (q >= lo && q < hi ? v[k].x : 0.f) * __ldg(a.x + c[k].x);
      s += (q + 1 >= lo && q + 1 < hi ? v[k].y : 0.f) * __ldg(a.x + c[k].y);
      s += (q + 2 >= lo && q + 2 < hi ? v[k].z : 0.f) * __ldg(a.x + c[k].z);
      s += (q + 3 >= lo && q + 3 < hi ? v[k].w : 0.f) * __ldg(a.x + c[k].w);
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (gl == 0 && i < cnt) {
    if (it.w & 0x80000000u) atomicAdd(a.y + it.x, s);
    else a.y[it.x] = s;
  }
}

template <int NT, int MINB, int RPT>
__global__ void __launch_bounds__(NT, MINB) spmv_bins2(BArgs a) {
  __shared__ unsigned s_cnt[NB2], s_base[NB2], s_next[NB2];
  const unsigned tid = threadIdx.x, b = blockIdx.x, GB = gridDim.x, lane = tid & 31u;
  if (tid == 0 && a.ts) a.ts[b * 8 + 0] = gns();
  if (tid < NB2) s_cnt[tid] = 0, s_next[tid] = 0;
  __syncthreads();
  const unsigned n = a.n;
  const unsigned per_pass = GB * NT * RPT;
  for (unsigned p0 = 0; p0 < n; p0 += per_pass) {
    const unsigned r0 = p0 + (b * NT + tid) * RPT;
    unsigned rs[RPT + 1];
#pragma unroll
    for (int i = 0; i <= RPT; i++) rs[i] = r0 + i <= n ? __ldg(a.rowptr + r0 + i) : 0u;
#pragma unroll
    for (int i = 0; i < RPT; i++)
      if (r0 + i >= n) rs[i + 1] = rs[i];
    unsigned slot[RPT];
#pragma unroll
    for (int i = 0; i < RPT; i++) {
      const unsigned d = rs[i + 1] - rs[i];
      int k = -1;
      unsigned nit = 0;
      if (r0 + i < n) {
        if (d == 0) a.y[r0 + i] = 0.f;
        else {
          k = class2_of(d);
          nit = k == 6 ? (rs[i + 1] - (rs[i] & ~3u) + kChunk2 - 1) / kChunk2 : 1u;
          if (k == 6) a.y[r0 + i] = 0.f;
        }
      }
      // warp-aggregated: lanes of the same class share one shared atomic
      const unsigned peers = __match_any_sync(0xffffffffu, k);
      const unsigned leader = __ffs(peers) - 1;
      unsigned base = 0;
      if (lane == leader && k >= 0 && k != 6) base = atomicAdd(s_cnt + k, __popc(peers));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (k == 6) slot[i] = atomicAdd(s_cnt + 6, nit);  // chunked rows: rare, one shared atomic each
      else slot[i] = base + __popc(peers & ((1u << lane) - 1u));
      if (k < 0) slot[i] = 0xffffffffu;
      else slot[i] = (slot[i] & 0x0fffffffu) | (static_cast<unsigned>(k) << 28);
    }
    __syncthreads();
    if (tid < NB2) {
      const unsigned c = s_cnt[tid];
      s_base[tid] = c ? atomicAdd(a.ctr + tid, c) : 0u;
      s_cnt[tid] = 0;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < RPT; i++) {
      if (slot[i] == 0xffffffffu) continue;
      const int k = static_cast<int>(slot[i] >> 28);
      const unsigned at = s_base[k] + (slot[i] & 0x0fffffffu);
      const unsigned s = rs[i], e = rs[i + 1];
      if (k == 6) {
        const unsigned nit = (e - (s & ~3u) + kChunk2 - 1) / kChunk2;
        for (unsigned j = 0; j < nit; j++) {
          if (at + j < a.cap[6]) a.items[a.off[6] + at + j] = make_uint4(r0 + i, s, e, j | 0x80000000u);
          else atomicOr(a.ctr + 11, 1u);
        }
      } else {
        if (at < a.cap[k]) a.items[a.off[k] + at] = make_uint4(r0 + i, s, e, 0u);
        else atomicOr(a.ctr + 11, 1u);
      }
    }
  }
  __syncthreads();
  if (tid == 0 && a.ts) a.ts[b * 8 + 2] = gns();
  if (tid == 0) {
    __threadfence();
    atomicAdd(a.ctr + 9, 1u);
    unsigned seen;
    const unsigned long long t0 = gns();
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(a.ctr + 9) : "memory");
      if (seen < GB) __nanosleep(32);
      if (gns() - t0 > 2000000000ull) {
        atomicOr(a.ctr + 11, 2u);
        break;
      }
    } while (seen < GB);
  }
  __syncthreads();
  if (tid == 0 && a.ts) a.ts[b * 8 + 3] = gns();
  // drain: block b owns a contiguous share of every class's steps; its
  // warps take steps from a shared counter, heaviest class first
  auto run = [&](int k, auto unitfn, unsigned per_step) {
    const unsigned cnt = min(*reinterpret_cast<volatile unsigned*>(a.ctr + k), a.cap[k]);
    const unsigned steps = (cnt + per_step - 1) / per_step;
    const unsigned lo = static_cast<unsigned>(static_cast<unsigned long long>(steps) * b / GB);
    const unsigned hi = static_cast<unsigned>(static_cast<unsigned long long>(steps) * (b + 1) / GB);
    for (;;) {
      unsigned st = 0;
      if (lane == 0) st = atomicAdd(s_next + k, 1u);
      st = __shfl_sync(0xffffffffu, st, 0) + lo;
      if (st >= hi) break;
      unitfn(a.items + a.off[k], cnt, st);
    }
  };
  run(6, [&](const uint4* it, unsigned c, unsigned st) { unit2<32, 2, true>(a, it, c, st); }, 1);
  run(5, [&](const uint4* it, unsigned c, unsigned st) { unit2<32, 2, true>(a, it, c, st); }, 1);
  run(4, [&](const uint4* it, unsigned c, unsigned st) { unit2<16, 4, false>(a, it, c, st); }, 2);
  run(3, [&](const uint4* it, unsigned c, unsigned st) { unit2<8, 4, false>(a, it, c, st); }, 4);
  run(2, [&](const uint4* it, unsigned c, unsigned st) { unit2<4, 4, false>(a, it, c, st); }, 8);
  run(1, [&](const uint4* it, unsigned c, unsigned st) { unit2<2, 4, false>(a, it, c, st); }, 16);
  run(0, [&](const uint4* it, unsigned c, unsigned st) { unit2<1, 4, false>(a, it, c, st); }, 32);
  __syncthreads();
  if (tid == 0 && a.ts) a.ts[b * 8 + 4] = gns();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(a.ctr + 10, 1u) == GB - 1) {
      for (int k = 0; k < NB2; k++) a.ctr[k] = 0;
      a.ctr[9] = 0;
      a.ctr[10] = 0;
      __threadfence();
    }
  }
}
}  // namespace lab
