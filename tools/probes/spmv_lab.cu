// SpMV drain lab (probe, not product): a TMA-staged, contiguous-tile drain for
// the grid-consolidated SpMV, A/B against the library's current kernel in one
// process.  Build: make -C tools/probes spmv_lab ; run: tools/probes/spmv_lab
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "dpc.h"

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

namespace lab {
constexpr unsigned kFull = 0xffffffffu;

struct TArgs {
  const unsigned* rowptr;
  const int* col;
  const float* val;
  const float* x;
  float* y;
  unsigned n, m;
  uint2* items;              // {row, start} of the nonempty rows, row order (+1 sentinel)
  unsigned* slice_first;     // per warp: item containing the slice start
  unsigned long long* lb;    // per block: (1 << 32 | nonempty rows), 0 = not yet published
  unsigned* ctr;             // [0] barrier, [1] exit, [2] fault, [3] items
  unsigned per;              // stream positions per warp slice (multiple of the tile)
  unsigned long long* ts;    // per block phase stamps (8 slots), or null
  unsigned mode;             // probes: 1 = gathers confined to 4 KB of x, 2 = no gathers
  unsigned nwarps;
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
__device__ __forceinline__ void tma_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Per-warp shared-memory stride: NS stages of {col, val}[TP], rows[TP],
// the tile's start bitmap and NS barriers, rounded to 128 bytes.
template <int PL, int NS>
__host__ __device__ constexpr unsigned warp_smem() {
  return (NS * 32u * PL * 8u + (32u * PL + 64u) * 4u + 32u * PL / 8u + NS * 8u + 127u) & ~127u;
}

// Persistent grid-consolidated SpMV (threshold 0): insert = ordered
// compaction of the nonempty rows into the worklist (their stream offset is
// their CSR offset), device-wide barrier, drain = equal stream slices per
// warp, TMA bulk copies of contiguous col / val tiles into a per-warp ring,
// per-lane contiguous positions with an in-lane + cross-lane segmented sum.
template <int PL, int NS, int NT>
__global__ void __launch_bounds__(NT, 1) spmv_tma(TArgs a, int phase_probe) {
  constexpr unsigned TP = 32u * PL;          // positions per tile
  constexpr int NW = NT / 32;
  extern __shared__ __align__(128) unsigned char smem[];
  // per warp: NS stages of {col[TP], val[TP]}, rows[TP], bitmap[TP/32], NS barriers
  const unsigned lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
  unsigned char* wbase = smem + wib * warp_smem<PL, NS>();
  int* s_col = reinterpret_cast<int*>(wbase);
  float* s_val = reinterpret_cast<float*>(wbase + NS * TP * 4);
  unsigned* s_rows = reinterpret_cast<unsigned*>(wbase + NS * TP * 8);
  unsigned* s_bm = reinterpret_cast<unsigned*>(wbase + NS * TP * 8 + (TP + 64) * 4);
  unsigned long long* s_bar = reinterpret_cast<unsigned long long*>(wbase + NS * TP * 8 + (TP + 64) * 4 + TP / 8);
  __shared__ unsigned s_prefix;

  const unsigned GB = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const unsigned n = a.n, m = a.m, per = a.per;
  if (tid == 0 && a.ts) a.ts[b * 8 + 0] = gns();
  // ---------------- insert: ordered compaction of nonempty rows ----------------
  // block b owns rows [r_beg, r_end); per chunk of NT * RPT rows each thread
  // owns RPT consecutive rows (their rowptr loads all in flight at once)
  constexpr int RPT = 8;
  const unsigned RB = (n + GB - 1) / GB;
  const unsigned r_beg = min(n, b * RB), r_end = min(n, r_beg + RB);
  const unsigned CH = NT * RPT;
  __shared__ unsigned s_red[NW];
  auto load_rows = [&](unsigned cb, unsigned (&rs)[RPT + 1]) {
    const unsigned r0 = cb + tid * RPT;
#pragma unroll
    for (int i = 0; i <= RPT; i++) rs[i] = r0 + i <= r_end ? __ldg(a.rowptr + r0 + i) : 0u;
#pragma unroll
    for (int i = 0; i < RPT; i++)
      if (r0 + i >= r_end) rs[i + 1] = rs[i];  // rows past the block: empty, not written
  };
  auto block_scan = [&](unsigned v, unsigned* tot) {  // exclusive; all threads call
    unsigned inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned u = __shfl_up_sync(kFull, inc, o);
      if ((tid & 31u) >= static_cast<unsigned>(o)) inc += u;
    }
    if ((tid & 31u) == 31u) s_red[tid >> 5] = inc;
    __syncthreads();
    unsigned off = 0, t = 0;
    for (int w = 0; w < NW; w++) {
      const unsigned c = s_red[w];
      off += (w < static_cast<int>(tid >> 5)) ? c : 0u;
      t += c;
    }
    __syncthreads();
    *tot = t;
    return off + inc - v;
  };
  unsigned total = 0;
  unsigned rs[RPT + 1];
  for (unsigned cb = r_beg; cb < r_end; cb += CH) {
    load_rows(cb, rs);
    unsigned cnt = 0;
    const unsigned r0 = cb + tid * RPT;
#pragma unroll
    for (int i = 0; i < RPT; i++) {
      if (rs[i + 1] > rs[i]) cnt++;
      else if (r0 + i < r_end) a.y[r0 + i] = 0.f;
    }
    unsigned t;
    block_scan(cnt, &t);
    total += t;
  }
  if (wib == 0) {  // look-back: sum of the predecessors' aggregates
    if (lane == 0) atomicExch(a.lb + b, (1ull << 32) | total);
    unsigned acc = 0;
    for (unsigned p = lane; p < b; p += 32) {
      unsigned long long v;
      const unsigned long long t0 = gns();
      while (((v = ld_acquire64(a.lb + p)) >> 32) == 0) {
        __nanosleep(32);
        if (gns() - t0 > 2000000000ull) {
          atomicOr(a.ctr + 2, 1u);
          break;
        }
      }
      acc += static_cast<unsigned>(v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if (lane == 0) {
      s_prefix = acc;
      if (b == GB - 1) {
        a.ctr[3] = acc + total;
        a.items[acc + total] = make_uint2(0xffffffffu, 0xffffffffu);  // sentinel
      }
    }
  }
  __syncthreads();
  if (tid == 0 && a.ts) a.ts[b * 8 + 1] = gns();
  unsigned P = s_prefix;
  for (unsigned cb = r_beg; cb < r_end; cb += CH) {
    if (cb != r_beg || r_end - r_beg > CH) load_rows(cb, rs);  // one chunk: still in registers
    const unsigned r0 = cb + tid * RPT;
    unsigned cnt = 0;
#pragma unroll
    for (int i = 0; i < RPT; i++) cnt += rs[i + 1] > rs[i] ? 1u : 0u;
    unsigned t;
    unsigned idx = P + block_scan(cnt, &t);
#pragma unroll
    for (int i = 0; i < RPT; i++) {
      const unsigned s = rs[i], e = rs[i + 1];
      if (e > s) {
        a.items[idx] = make_uint2(r0 + i, s);
        // slices whose first position lies in [s, e) start with this item
        const unsigned w0 = (s + per - 1) / per;
        const unsigned w1 = min((e + per - 1) / per, a.nwarps);
        for (unsigned w = w0; w < w1; w++) a.slice_first[w] = idx;
        // a slice boundary strictly inside the row: its parts are atomically added
        if ((static_cast<unsigned long long>(s / per) + 1ull) * per < e) a.y[r0 + i] = 0.f;
        idx++;
      }
    }
    P += t;
  }
  // ---------------- device-wide barrier ----------------
  __syncthreads();
  if (tid == 0 && a.ts) a.ts[b * 8 + 2] = gns();
  if (tid == 0) {
    __threadfence();
    atomicAdd(a.ctr + 0, 1u);
    unsigned seen;
    const unsigned long long t0 = gns();
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(a.ctr) : "memory");
      if (seen < GB) __nanosleep(32);
      if (gns() - t0 > 2000000000ull) {
        atomicOr(a.ctr + 2, 2u);
        break;
      }
    } while (seen < GB);
    a.lb[b] = 0;  // every look-back finished before its block arrived
  }
  __syncthreads();
  if (phase_probe == 1) goto out;
  if (tid == 0 && a.ts) a.ts[b * 8 + 3] = gns();
  {
    // ---------------- drain (software-pipelined) ----------------
    // iteration t: flags of tile t from the item window loaded during t-1;
    // reload of the window for t+1; products of t (gathers issued during
    // t-1); refill of t's stage with t+NS; t+1's col / val read and its x
    // gathers issued; segmented sums of t -- the loads of t+1 fly under t's
    // segmentation.
    const unsigned gw = b * NW + wib;
    const unsigned s0 = gw * per;
    if (s0 < m) {
      const unsigned s1 = min(m, s0 + per);
      const unsigned ntiles = (s1 - s0 + TP - 1) / TP;
      const unsigned nitems = *reinterpret_cast<volatile unsigned*>(a.ctr + 3);
      if (lane == 0) {
        for (int i = 0; i < NS; i++) mbar_init(s_bar + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      __syncwarp();
      auto issue = [&](unsigned t) {
        const unsigned k0 = s0 + t * TP;
        const unsigned cnt = min(TP, s1 - k0);
        const unsigned bytes = (cnt * 4u + 15u) & ~15u;
        const int st = t % NS;
        mbar_expect_tx(s_bar + st, 2u * bytes);
        tma_1d(s_col + st * TP, a.col + k0, bytes, s_bar + st);
        tma_1d(s_val + st * TP, a.val + k0, bytes, s_bar + st);
      };
      if (lane == 0)
        for (unsigned t = 0; t < min(ntiles, static_cast<unsigned>(NS)); t++) issue(t);
      unsigned ia = a.slice_first[gw];
      const uint2 it0 = __ldcg(a.items + ia);
      unsigned orow = it0.x;
      bool osplit = it0.y < s0;
      // item window: lane j holds items ia+1+j and ia+33+j
      auto load_win = [&](unsigned base, uint2& w0, uint2& w1) {
        const unsigned i0 = base + lane, i1 = base + 32 + lane;
        w0 = i0 <= nitems ? __ldcg(a.items + i0) : make_uint2(0xffffffffu, 0xffffffffu);
        w1 = i1 <= nitems ? __ldcg(a.items + i1) : make_uint2(0xffffffffu, 0xffffffffu);
      };
      uint2 w0, w1;
      load_win(ia + 1, w0, w1);
      // products' operands of the next tile
      float xn[PL], vn[PL];
      auto fetch = [&](unsigned t) {  // wait for tile t, read col / val, issue the x gathers
        const int st = t % NS;
        mbar_wait(s_bar + st, (t / NS) & 1u);
        const int* cp = s_col + st * TP + lane * PL;
        const float* vp = s_val + st * TP + lane * PL;
        constexpr int NQ = PL / 4;
        const int rot = NQ == 2 ? ((lane >> 2) & 1) : NQ == 4 ? ((lane >> 1) & 3) : 0;
        int4 qc[NQ];
        float4 qv[NQ];
#pragma unroll
        for (int h = 0; h < NQ; h++) {
          const int hh = (h + rot) & (NQ - 1);
          qc[h] = *reinterpret_cast<const int4*>(cp + 4 * hh);
          qv[h] = *reinterpret_cast<const float4*>(vp + 4 * hh);
        }
        const unsigned k0 = s0 + t * TP;
        const unsigned kend = min(k0 + TP, s1);
        const unsigned q0 = k0 + lane * PL;
#pragma unroll
        for (int k = 0; k < NQ; k++) {
          int4 gc = qc[k];
          float4 gv = qv[k];
#pragma unroll
          for (int r = 1; r < NQ; r++)
            if (rot == r) gc = qc[(k - r + NQ) & (NQ - 1)], gv = qv[(k - r + NQ) & (NQ - 1)];
          const int cc[4] = {gc.x, gc.y, gc.z, gc.w};
          const float vv[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const bool ok = q0 + 4 * k + e < kend;
            vn[4 * k + e] = ok ? vv[e] : 0.f;
            xn[4 * k + e] = (a.mode & 2u) ? 1.f : __ldg(a.x + ((ok ? cc[e] : 0) & ((a.mode & 1u) ? 1023 : 0x7fffffff)));
          }
        }
      };
      fetch(0);
      float carry = 0.f, lacc = 0.f;
      for (unsigned t = 0; t < ntiles; t++) {
        const int st = t % NS;
        const unsigned k0 = s0 + t * TP;
        const unsigned kend = min(k0 + TP, s1);
        // ---- flags of tile t: items ia+1.. with start < kend
        if (lane < TP / 32) s_bm[lane] = 0u;
        __syncwarp();
        unsigned nf = 0;
        {
          bool in0 = w0.y < kend, in1 = w1.y < kend;
          if (in0) {
            const unsigned o = w0.y - k0;
            atomicOr(s_bm + (o >> 5), 1u << (o & 31u));
            s_rows[lane] = w0.x;
          }
          if (in1) {
            const unsigned o = w1.y - k0;
            atomicOr(s_bm + (o >> 5), 1u << (o & 31u));
            s_rows[32 + lane] = w1.x;
          }
          nf = __popc(__ballot_sync(kFull, in0)) + __popc(__ballot_sync(kFull, in1));
          while (nf > 0 && (nf & 63u) == 0) {  // window exhausted inside the tile
            uint2 u0, u1;
            load_win(ia + 1 + nf, u0, u1);
            in0 = u0.y < kend, in1 = u1.y < kend;
            if (in0) {
              const unsigned o = u0.y - k0;
              atomicOr(s_bm + (o >> 5), 1u << (o & 31u));
              s_rows[nf + lane] = u0.x;
            }
            if (in1) {
              const unsigned o = u1.y - k0;
              atomicOr(s_bm + (o >> 5), 1u << (o & 31u));
              s_rows[nf + 32 + lane] = u1.x;
            }
            const unsigned add = __popc(__ballot_sync(kFull, in0)) + __popc(__ballot_sync(kFull, in1));
            nf += add;
            if (add < 64) break;
          }
        }
        load_win(ia + 1 + nf, w0, w1);  // next tile's window, in flight
        // ---- products of tile t
        float p[PL];
#pragma unroll
        for (int j = 0; j < PL; j++) p[j] = vn[j] * xn[j];
        __syncwarp();
        if (lane == 0 && t + NS < ntiles) issue(t + NS);  // stage st is free again
        if (t + 1 < ntiles) fetch(t + 1);                 // next tile's gathers, in flight
        (void)st;
        // ---- segmented sums of tile t
        unsigned fl;
        if (PL == 8) fl = (s_bm[lane >> 2] >> ((lane & 3u) * 8u)) & 0xffu;
        else if (PL == 16) fl = (s_bm[lane >> 1] >> ((lane & 1u) * 16u)) & 0xffffu;
        else if (PL == 4) fl = (s_bm[lane >> 3] >> ((lane & 7u) * 4u)) & 0xfu;
        else fl = s_bm[lane];
        const unsigned anyf = __ballot_sync(kFull, fl != 0);
        if (!anyf) {  // tile inside one item: lane-local accumulation
          float sum = 0.f;
#pragma unroll
          for (int j = 0; j < PL; j++) sum += p[j];
          lacc += sum;
          continue;
        }
        float la = lacc;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) la += __shfl_xor_sync(kFull, la, o);
        carry += la;
        lacc = 0.f;
        const unsigned nfl = __popc(fl);
        unsigned pre = nfl;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned u = __shfl_up_sync(kFull, pre, o);
          if (lane >= static_cast<unsigned>(o)) pre += u;
        }
        pre -= nfl;
        float run = 0.f, head = 0.f;
        unsigned seen = 0;
#pragma unroll
        for (int j = 0; j < PL; j++) {
          if ((fl >> j) & 1u) {
            if (seen == 0) head = run;
            else a.y[s_rows[pre + seen - 1]] = run;
            run = 0.f;
            seen++;
          }
          run += p[j];
        }
        if (seen == 0) head = run;
        float sv = nfl ? run : head;
        if (lane == 0 && !nfl) sv += carry;
        const unsigned lsm = anyf & ((2u << lane) - 1u);
        const unsigned ls = lsm ? 31u - __clz(lsm) : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float u = __shfl_up_sync(kFull, sv, o);
          if (lane >= ls + static_cast<unsigned>(o)) sv += u;
        }
        float cin = __shfl_up_sync(kFull, sv, 1);
        if (lane == 0) cin = carry;
        if (nfl) {
          const float tot = cin + head;
          const unsigned row = pre ? s_rows[pre - 1] : orow;
          if (!pre && osplit) atomicAdd(a.y + row, tot);
          else a.y[row] = tot;
        }
        carry = __shfl_sync(kFull, sv, 31);
        orow = s_rows[nf - 1];
        osplit = false;
        ia += nf;
        __syncwarp();
      }
      float la = lacc;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) la += __shfl_xor_sync(kFull, la, o);
      if (lane == 0) {
        const float tot = carry + la;
        const unsigned e = __ldg(a.rowptr + orow + 1);
        if (osplit || e > s1) atomicAdd(a.y + orow, tot);
        else a.y[orow] = tot;
      }
    }
  }
out:
  __syncthreads();
  if (tid == 0 && a.ts) a.ts[b * 8 + 4] = gns();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(a.ctr + 1, 1u) == GB - 1) {
      a.ctr[0] = 0;
      a.ctr[1] = 0;
      __threadfence();
    }
  }
}

}  // namespace lab

#include "spmv_bins.cuh"

static double now_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms;
  CK(cudaEventSynchronize(b));
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

template <int PL, int NS, int NT>
static double run_tma(const lab::TArgs& a0, int reps, void* flush, size_t fbytes, cudaStream_t s, cudaEvent_t e0,
                      cudaEvent_t e1, int sms, int probe = 0) {
  constexpr unsigned TP = 32u * PL;
  const size_t smem = (NT / 32) * lab::warp_smem<PL, NS>();
  auto fn = lab::spmv_tma<PL, NS, NT>;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, smem));
  if (per_sm < 1) {
    std::printf("  PL=%d NS=%d NT=%d does not fit (smem %zu)\n", PL, NS, NT, smem);
    return -1;
  }
  lab::TArgs a = a0;
  const unsigned GB = static_cast<unsigned>(sms * per_sm);
  a.nwarps = GB * (NT / 32);
  const unsigned long long per0 = (static_cast<unsigned long long>(a.m) + a.nwarps - 1) / a.nwarps;
  a.per = static_cast<unsigned>((per0 + TP - 1) / TP * TP);
  double best = 1e30, sum = 0;
  for (int i = 0; i < reps + 2; i++) {
    CK(cudaMemsetAsync(flush, i & 0xff, fbytes, s));
    CK(cudaEventRecord(e0, s));
    fn<<<GB, NT, smem, s>>>(a, probe);
    CK(cudaEventRecord(e1, s));
    CK(cudaGetLastError());
    const double ms = now_ms(e0, e1);
    if (i >= 2) {
      best = std::min(best, ms);
      sum += ms;
    }
  }
  unsigned h[4];
  CK(cudaMemcpy(h, a.ctr, 16, cudaMemcpyDeviceToHost));
  if (a.ts) {
    std::vector<unsigned long long> ts(GB * 8);
    CK(cudaMemcpy(ts.data(), a.ts, 8ull * GB * 8, cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull;
    for (unsigned i = 0; i < GB; i++) t0 = std::min(t0, ts[i * 8]);
    const char* names[5] = {"start", "pass1+scan", "lookback+pass2", "barrier", "end"};
    std::printf("    phases (us after first block start): ");
    for (int k = 0; k < 5; k++) {
      unsigned long long lo = ~0ull, hi = 0;
      for (unsigned i = 0; i < GB; i++) lo = std::min(lo, ts[i * 8 + k]), hi = std::max(hi, ts[i * 8 + k]);
      std::printf("%s %.1f-%.1f  ", names[k], (lo - t0) / 1e3, (hi - t0) / 1e3);
    }
    std::printf("\n");
  }
  std::printf("  tma PL=%d NS=%d NT=%d blocks=%u per=%u smem=%zu: mean %.2f us best %.2f us fault=%u items=%u%s\n",
              PL, NS, NT, GB, a.per, smem, sum / reps * 1e3, best * 1e3, h[2], h[3], probe ? " (insert only)" : "");
  return sum / reps;
}

template <int NT, int RPT, int UI>
static double run_bins(lab::BArgs a, int reps, void* flush, size_t fbytes, cudaStream_t s, cudaEvent_t e0,
                       cudaEvent_t e1, int sms) {
  auto fn = lab::spmv_bins<NT, RPT, UI>;
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, 0));
  const unsigned GB = static_cast<unsigned>(sms * std::max(per_sm, 1));
  double best = 1e30, sum = 0;
  for (int i = 0; i < reps + 2; i++) {
    CK(cudaMemsetAsync(flush, i & 0xff, fbytes, s));
    CK(cudaEventRecord(e0, s));
    fn<<<GB, NT, 0, s>>>(a);
    CK(cudaEventRecord(e1, s));
    CK(cudaGetLastError());
    const double ms = now_ms(e0, e1);
    if (i >= 2) best = std::min(best, ms), sum += ms;
  }
  unsigned h[12];
  CK(cudaMemcpy(h, a.ctr, 48, cudaMemcpyDeviceToHost));
  h[10] = h[11];
  std::vector<unsigned long long> ts(GB * 8);
  CK(cudaMemcpy(ts.data(), a.ts, 8ull * GB * 8, cudaMemcpyDeviceToHost));
  unsigned long long t0 = ~0ull;
  for (unsigned i = 0; i < GB; i++) t0 = std::min(t0, ts[i * 8]);
  auto rng = [&](int k, double& lo, double& hi) {
    unsigned long long l = ~0ull, h2 = 0;
    for (unsigned i = 0; i < GB; i++) l = std::min(l, ts[i * 8 + k]), h2 = std::max(h2, ts[i * 8 + k]);
    lo = (l - t0) / 1e3, hi = (h2 - t0) / 1e3;
  };
  double l2, h2, l3, h3, l4, h4;
  rng(2, l2, h2), rng(3, l3, h3), rng(4, l4, h4);
  std::printf("  bins NT=%d RPT=%d U=%d T=%u blocks=%u regs/sm=%d: mean %.2f us best %.2f us fault=%u | insert end %.1f-%.1f, "
              "barrier %.1f-%.1f, end %.1f-%.1f\n",
              NT, RPT, UI, a.T, GB, per_sm, sum / reps * 1e3, best * 1e3, h[10], l2, h2, l3, h3, l4, h4);
  return sum / reps;
}

template <int NT, int MINB, int RPT>
static double run_bins2(lab::BArgs a, int reps, void* flush, size_t fbytes, cudaStream_t s, cudaEvent_t e0,
                        cudaEvent_t e1, int sms) {
  auto fn = lab::spmv_bins2<NT, MINB, RPT>;
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, 0));
  const unsigned GB = static_cast<unsigned>(sms * std::max(per_sm, 1));
  double best = 1e30, sum = 0;
  for (int i = 0; i < reps + 2; i++) {
    CK(cudaMemsetAsync(flush, i & 0xff, fbytes, s));
    CK(cudaEventRecord(e0, s));
    fn<<<GB, NT, 0, s>>>(a);
    CK(cudaEventRecord(e1, s));
    CK(cudaGetLastError());
    const double ms = now_ms(e0, e1);
    if (i >= 2) best = std::min(best, ms), sum += ms;
  }
  unsigned h[12];
  CK(cudaMemcpy(h, a.ctr, 48, cudaMemcpyDeviceToHost));
  std::vector<unsigned long long> ts(GB * 8);
  CK(cudaMemcpy(ts.data(), a.ts, 8ull * GB * 8, cudaMemcpyDeviceToHost));
  unsigned long long t0 = ~0ull;
  for (unsigned i = 0; i < GB; i++) t0 = std::min(t0, ts[i * 8]);
  auto rng = [&](int k, double& lo, double& hi) {
    unsigned long long l = ~0ull, h2 = 0;
    for (unsigned i = 0; i < GB; i++) l = std::min(l, ts[i * 8 + k]), h2 = std::max(h2, ts[i * 8 + k]);
    lo = (l - t0) / 1e3, hi = (h2 - t0) / 1e3;
  };
  double l2, h2, l3, h3, l4, h4;
  rng(2, l2, h2), rng(3, l3, h3), rng(4, l4, h4);
  std::printf("  bins2 NT=%d MINB=%d RPT=%d blocks=%u: mean %.2f us best %.2f us fault=%u | insert end %.1f-%.1f, "
              "barrier %.1f-%.1f, end %.1f-%.1f\n",
              NT, MINB, RPT, GB, sum / reps * 1e3, best * 1e3, h[11], l2, h2, l3, h3, l4, h4);
  return sum / reps;
}

static bool check(const float* dy, const std::vector<double>& y64, const char* what) {
  const size_t n = y64.size();
  std::vector<float> y(n);
  CK(cudaMemcpy(y.data(), dy, 4 * n, cudaMemcpyDeviceToHost));
  double worst = 0;
  size_t bad = 0, at = 0;
  for (size_t i = 0; i < n; i++) {
    const double d = std::fabs(y[i] - y64[i]);
    const double r = y64[i] != 0 ? d / std::fabs(y64[i]) : d;
    if (r > worst) worst = r, at = i;
    if (r > 1e-5) bad++;
  }
  std::printf("  check %-10s max rel err %.3g at %zu (y %.9g ref %.9g), %zu rows > 1e-5 -> %s\n", what, worst, at,
              y[at], y64[at], bad, bad ? "FAIL" : "ok");
  return bad == 0;
}

int main(int argc, char** argv) {
  const int scale = argc > 1 ? std::atoi(argv[1]) : 20;
  const int reps = argc > 2 ? std::atoi(argv[2]) : 20;
  dpc_csr* g = nullptr;
  if (dpc_gen_rmat(scale, 16, 0.57, 0.19, 0.19, 1, 255, 1, DPC_GEN_VALUES, &g) != DPC_OK) {
    std::fprintf(stderr, "gen: %s\n", dpc_last_error());
    return 1;
  }
  const unsigned n = static_cast<unsigned>(g->n), m = static_cast<unsigned>(g->m);
  std::printf("R-MAT scale %d: n=%u m=%u\n", scale, n, m);
  std::vector<float> x(n);
  for (unsigned i = 0; i < n; i++) x[i] = static_cast<float>((i * 2654435761u) % 16777215u + 1) / 16777216.f;
  std::vector<double> y64(n);
  for (unsigned r = 0; r < n; r++) {
    double s = 0;
    for (int64_t k = g->rowptr[r]; k < g->rowptr[r + 1]; k++) s += static_cast<double>(g->val[k]) * x[g->col[k]];
    y64[r] = s;
  }
  dpc_ctx* ctx = nullptr;
  if (dpc_ctx_create(0, &ctx) != DPC_OK) {
    std::fprintf(stderr, "ctx: %s\n", dpc_last_error());
    return 1;
  }
  cudaStream_t s = static_cast<cudaStream_t>(dpc_ctx_stream(ctx));
  const int sms = dpc_ctx_sm_count(ctx);
  dpc_dgraph* dg = nullptr;
  if (dpc_dgraph_upload(ctx, g, &dg) != DPC_OK) {
    std::fprintf(stderr, "upload: %s\n", dpc_last_error());
    return 1;
  }
  float* dx = dpc_dgraph_x(dg);
  float* dy = dpc_dgraph_y(dg);
  CK(cudaMemcpy(dx, x.data(), 4 * n, cudaMemcpyHostToDevice));
  void* flush = nullptr;
  const size_t fbytes = size_t{512} << 20;
  CK(cudaMalloc(&flush, fbytes));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  // current library kernel
  {
    dpc_launch_cfg cfg;
    dpc_launch_cfg_default(DPC_APP_SPMV, DPC_GRID, &cfg);
    double sum = 0, best = 1e30;
    for (int i = 0; i < reps + 2; i++) {
      CK(cudaMemsetAsync(flush, i & 0xff, fbytes, s));
      CK(cudaEventRecord(e0, s));
      if (dpc_spmv_device(ctx, dg, dx, dy, &cfg, nullptr) != DPC_OK) {
        std::fprintf(stderr, "spmv: %s\n", dpc_last_error());
        return 1;
      }
      CK(cudaEventRecord(e1, s));
      const double ms = now_ms(e0, e1);
      if (i >= 2) sum += ms, best = std::min(best, ms);
    }
    std::printf("  library grid_stream: mean %.2f us best %.2f us\n", sum / reps * 1e3, best * 1e3);
    check(dy, y64, "library");
  }
  // lab kernel buffers: rowptr u32 + col/val padded to a 16-byte multiple
  // (the library's upload pads 16 bytes; TMA tails round up to 16)
  unsigned* drp;
  int* dcol;
  float* dval;
  CK(cudaMalloc(&drp, 4ull * (n + 1)));
  CK(cudaMalloc(&dcol, 4ull * (m + 64)));
  CK(cudaMalloc(&dval, 4ull * (m + 64)));
  {
    std::vector<unsigned> rp(n + 1);
    for (unsigned i = 0; i <= n; i++) rp[i] = static_cast<unsigned>(g->rowptr[i]);
    CK(cudaMemcpy(drp, rp.data(), 4ull * (n + 1), cudaMemcpyHostToDevice));
    CK(cudaMemset(dcol, 0, 4ull * (m + 64)));
    CK(cudaMemset(dval, 0, 4ull * (m + 64)));
    CK(cudaMemcpy(dcol, g->col, 4ull * m, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dval, g->val, 4ull * m, cudaMemcpyHostToDevice));
  }
  lab::TArgs a{};
  a.rowptr = drp;
  a.col = dcol;
  a.val = dval;
  a.x = dx;
  a.y = dy;
  a.n = n;
  a.m = m;
  CK(cudaMalloc(&a.items, 8ull * (n + 1)));
  CK(cudaMalloc(&a.slice_first, 4ull * 65536));
  CK(cudaMalloc(&a.lb, 8ull * 4096));
  CK(cudaMalloc(&a.ctr, 64));
  CK(cudaMalloc(&a.ts, 8ull * 8 * 4096));
  CK(cudaMemset(a.lb, 0, 8ull * 4096));
  CK(cudaMemset(a.ctr, 0, 64));
  auto reset_y = [&] { CK(cudaMemset(dy, 0xff, 4ull * n)); };  // NaN: every row must be written
  reset_y();
  run_tma<8, 2, 1024>(a, reps, flush, fbytes, s, e0, e1, sms);
  check(dy, y64, "tma8x2");
  reset_y();
  run_tma<8, 3, 768>(a, reps, flush, fbytes, s, e0, e1, sms);
  check(dy, y64, "tma8x3/768");
  reset_y();
  run_tma<16, 2, 512>(a, reps, flush, fbytes, s, e0, e1, sms);
  check(dy, y64, "tma16x2/512");
  reset_y();
  run_tma<4, 3, 1024>(a, reps, flush, fbytes, s, e0, e1, sms);
  check(dy, y64, "tma4x3");
  run_tma<8, 2, 1024>(a, reps, flush, fbytes, s, e0, e1, sms, 1);
  {
    lab::BArgs ba{};
    ba.rowptr = drp, ba.col = dcol, ba.val = dval, ba.x = dx, ba.y = dy, ba.n = n, ba.m = m, ba.T = 4;
    // exact class capacities from the degree histogram
    unsigned capk[lab::NBIN] = {};
    for (unsigned r = 0; r < n; r++) {
      const unsigned s0 = static_cast<unsigned>(g->rowptr[r]), e = static_cast<unsigned>(g->rowptr[r + 1]);
      const unsigned d = e - s0;
      if (d == 0) continue;
      const int k = lab::class_of(d);
      capk[k] += k == lab::kChunkBin ? (e - (s0 & ~3u) + lab::kChunk - 1) / lab::kChunk : 1u;
    }
    unsigned tot = 0;
    for (int k = 0; k < lab::NBIN; k++) ba.off[k] = tot, ba.cap[k] = capk[k], tot += capk[k];
    std::printf("  classes:");
    for (int k = 0; k < lab::NBIN; k++) std::printf(" %u", capk[k]);
    std::printf("\n");
    CK(cudaMalloc(&ba.items, 16ull * (tot + 1)));
    CK(cudaMalloc(&ba.ctr, 64));
    CK(cudaMemset(ba.ctr, 0, 64));
    ba.ts = a.ts;
    {
      ba.T = 0;
      reset_y();
      run_bins<1024, 8, 1>(ba, reps, flush, fbytes, s, e0, e1, sms);
      check(dy, y64, "bins1024/8/1");
      reset_y();
      run_bins<1024, 8, 2>(ba, reps, flush, fbytes, s, e0, e1, sms);
      check(dy, y64, "bins1024/8/2");
      reset_y();
      run_bins<512, 8, 2>(ba, reps, flush, fbytes, s, e0, e1, sms);
      check(dy, y64, "bins512/8/2");
      reset_y();
      run_bins<1024, 4, 2>(ba, reps, flush, fbytes, s, e0, e1, sms);
      check(dy, y64, "bins1024/4/2");
    }
  }
  {
    lab::BArgs ba{};
    ba.rowptr = drp, ba.col = dcol, ba.val = dval, ba.x = dx, ba.y = dy, ba.n = n, ba.m = m, ba.T = 0;
    unsigned capk[lab::NB2] = {};
    for (unsigned r = 0; r < n; r++) {
      const unsigned s0 = static_cast<unsigned>(g->rowptr[r]), e = static_cast<unsigned>(g->rowptr[r + 1]);
      if (e == s0) continue;
      const int k = lab::class2_of(e - s0);
      capk[k] += k == 6 ? (e - (s0 & ~3u) + lab::kChunk2 - 1) / lab::kChunk2 : 1u;
    }
    unsigned tot = 0;
    for (int k = 0; k < lab::NB2; k++) ba.off[k] = tot, ba.cap[k] = capk[k], tot += capk[k];
    CK(cudaMalloc(&ba.items, 16ull * (tot + 1)));
    CK(cudaMalloc(&ba.ctr, 64));
    CK(cudaMemset(ba.ctr, 0, 64));
    ba.ts = a.ts;
    reset_y();
    run_bins2<1024, 2, 4>(ba, reps, flush, fbytes, s, e0, e1, sms);
    check(dy, y64, "bins2/1024x2/4");
    reset_y();
    run_bins2<1024, 1, 8>(ba, reps, flush, fbytes, s, e0, e1, sms);
    check(dy, y64, "bins2/1024x1/8");
    reset_y();
    run_bins2<512, 3, 4>(ba, reps, flush, fbytes, s, e0, e1, sms);
    check(dy, y64, "bins2/512x3/4");
  }
  a.mode = 1;
  run_tma<4, 3, 1024>(a, reps, flush, fbytes, s, e0, e1, sms);
  run_tma<8, 2, 1024>(a, reps, flush, fbytes, s, e0, e1, sms);
  a.mode = 2;
  run_tma<4, 3, 1024>(a, reps, flush, fbytes, s, e0, e1, sms);
  run_tma<8, 2, 1024>(a, reps, flush, fbytes, s, e0, e1, sms);
  a.mode = 0;
  if (argc > 3) {  // ncu: a few launches of the two main shapes
    run_tma<4, 3, 1024>(a, 2, flush, fbytes, s, e0, e1, sms);
    run_tma<8, 2, 1024>(a, 2, flush, fbytes, s, e0, e1, sms);
  }
  dpc_dgraph_free(dg);
  dpc_ctx_destroy(ctx);
  dpc_csr_free(g);
  return 0;
}
