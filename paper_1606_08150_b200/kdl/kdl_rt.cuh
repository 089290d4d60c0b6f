// Device runtime of the .kdl -> sm_100a CUDA builder (paper_1606_08150_b200/kdl):
// the consolidated-program builtins (dp_buffers / dp_insert / dp_buf_* /
// dp_grid_last, ast.hpp:25-33 and 63-65) mapped onto B200 primitives.
//
//   * owner buffers (warp / block: shared-memory record; grid: per-launch
//     Inst record in HBM) hold {base, count, cap}; storage is reserved lazily,
//     once per owner, from a pre-allocated arena (the paper's "pre-alloc"
//     allocator) — owners that never insert cost nothing;
//   * dp_insert is warp-aggregated: one shared/global atomic per warp per
//     insert instruction, whatever the divergence;
//   * grid buffers alternate between two regions by launch level, so a
//     recursive grid-level chain (level L reads what L-1 wrote while it fills
//     the other region) never needs more than two;
//   * dp_grid_last is the last-block ticket (__threadfence + atomicAdd on the
//     launch's own Inst record), cached per block like sim.hpp:1708-1716;
//   * device launches are CDP2 fire-and-forget; a launch that follows
//     sync_device becomes a tail launch (runs after the whole parent grid and
//     everything it launched, which is what the postwork needs);
//   * every fault the simulator reports (sim.hpp:49-52: overflow, runtime,
//     config) sets a bit in ctr[0] instead of trapping.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>

#include "dpc_kdl.h"

namespace dk {

enum : unsigned long long {
  F_OVERFLOW = 1,   // consolidation buffer overflow / non-positive capacity
  F_POOL = 2,       // pre-allocated pool exhausted
  F_BOUNDS = 4,     // array index out of bounds
  F_DIV = 8,        // integer division / modulo by zero
  F_CONFIG = 16,    // launch extents outside [1, 2^31) x [1, 1024]
  F_LAUNCH = 32,    // device launch refused (pending-launch pool, resources)
  F_INST = 64,      // launch-record arena exhausted
  F_BUFGET = 128,   // dp_buf_get / dp_buf_cfg index out of range
};

constexpr int kMaxArrays = 64;

struct Inst {                 // one per device launch that needs it
  unsigned long long count;   // grid buffer fill
  unsigned int ticket;        // dp_grid_last counter
  unsigned int level;         // launch depth: grid buffer region = level & 1
  unsigned long long aux;     // sync_device split: phase state base (0 unset, 1 busy, else off + 2)
};

struct Inh {                  // the buffer a consolidated kernel drains
  const long long* items;     // contiguous [n][stride] words (grid regions), or nullptr
  const unsigned long long* segs;  // warp / block owners: segment table (word offset + 2)
  long long n;
  long long stride;
  long long shift;            // items per segment = 1 << shift
};

// Warp / block owner record (shared memory).  The buffer is a chain of up to
// kSegs segments of `cap` items (cap = the directive's capacity rounded up to
// a power of two), each reserved from the arena when the first item lands in
// it: the reference faults when one buffer fills (sim.hpp:1513), this runtime
// grows it by up to kSegs x before raising the same overflow fault.
constexpr int kSegs = 32;
struct Own {
  unsigned long long count;
  long long cap;              // items per segment (power of two), < 1 = invalid
  long long shift;
  unsigned long long seg[kSegs];  // 0 unset, 1 being reserved, ~0 failed, else word offset + 2
};

struct Rt {
  void* arr[kMaxArrays];
  long long len[kMaxArrays];
  unsigned long long* ctr;    // [0] fault bits [1] launches [2] arena top (words) [3] inst top
  long long* arena;
  unsigned long long arena_words;
  Inst* inst;
  unsigned long long inst_cap;
  long long* region[2];
  unsigned long long region_words;
  long long narr;
};

constexpr unsigned long long kNoBase = ~0ull;

static_assert(sizeof(Rt) == sizeof(dk_rt_t), "dk::Rt must match include/dpc_kdl.h");
static_assert(sizeof(Inst) == 24, "launch records are 24 bytes (include/dpc_kdl.h)");

}  // namespace dk

__constant__ dk::Rt dk_rt;

// DSL value widths (compile option): 64 = the simulator's Value (int64 /
// fp64, sim.hpp:72-80), 32 = int32 / fp32 arrays and scalars.  Buffer items,
// counters and launch state stay 64-bit words either way.
#ifndef DK_WIDTH
#define DK_WIDTH 64
#endif
#if DK_WIDTH == 32
typedef int dk_int;
typedef float dk_flt;
__device__ __forceinline__ dk_flt dk_word_flt(long long w) { return __int_as_float(static_cast<int>(w)); }
__device__ __forceinline__ long long dk_flt_word(dk_flt v) {
  return static_cast<long long>(static_cast<unsigned>(__float_as_int(v)));
}
#else
typedef long long dk_int;
typedef double dk_flt;
__device__ __forceinline__ dk_flt dk_word_flt(long long w) { return __longlong_as_double(w); }
__device__ __forceinline__ long long dk_flt_word(dk_flt v) { return __double_as_longlong(v); }
#endif

__device__ dk_int dk_sink_i[2];
__device__ dk_flt dk_sink_f[2];

__device__ __forceinline__ void dk_fault(unsigned long long bit) { atomicOr(&dk_rt.ctr[0], bit); }

// ---- checked array access (the simulator faults on out-of-bounds) ----
__device__ __forceinline__ bool dk_ok(long long id, long long i) {
  if (static_cast<unsigned long long>(id) >= static_cast<unsigned long long>(dk_rt.narr) ||
      static_cast<unsigned long long>(i) >= static_cast<unsigned long long>(dk_rt.len[id])) {
    dk_fault(dk::F_BOUNDS);
    return false;
  }
  return true;
}
__device__ __forceinline__ dk_int* dk_ip(long long id, long long i) {
  return dk_ok(id, i) ? static_cast<dk_int*>(dk_rt.arr[id]) + i : dk_sink_i;
}
__device__ __forceinline__ dk_flt* dk_fp(long long id, long long i) {
  return dk_ok(id, i) ? static_cast<dk_flt*>(dk_rt.arr[id]) + i : dk_sink_f;
}
// atomicAdd, warp-aggregated per address: the lanes of a warp that hit the
// same element (__match_any_sync) combine their values with shuffles and one
// lane issues the atomic; each lane still gets a distinct "old" value (the
// aggregate's old + its exclusive prefix), a valid order of the original
// atomics.  Same-address atomics serialise in L2, so this turns a hot
// ancestor / row update from 32 serial atomics into one.
template <class T>
__device__ __forceinline__ T dk_atomic_agg(T* p, T v) {
  const unsigned m = __activemask();
  const unsigned peers = __match_any_sync(m, reinterpret_cast<unsigned long long>(p));
  const unsigned lane = threadIdx.x & 31u;
  if (peers == (1u << lane)) return atomicAdd(p, v);
  const int leader = __ffs(peers) - 1;
  T total = T(0), pre = T(0);
  for (unsigned r = peers; r; r &= r - 1) {
    const int l = __ffs(r) - 1;
    const T x = __shfl_sync(peers, v, l);
    total += x;
    if (static_cast<unsigned>(l) < lane) pre += x;
  }
  T old = T(0);
  if (lane == static_cast<unsigned>(leader)) old = atomicAdd(p, total);
  return __shfl_sync(peers, old, leader) + pre;
}
// Statement form (result unused): when every active lane of the warp hits
// the same element, the lanes combine first and one lane issues the atomic
// (ints: redux.sync — for int64 on 16/16/32-bit pieces, exact mod 2^64;
// floats: a butterfly for a full warp, a shuffle loop otherwise); mixed
// addresses go out as plain fire-and-forget REDs.
__device__ __forceinline__ void dk_add_i(long long* p, long long v) {
  const unsigned m = __activemask();
  unsigned long long* q = reinterpret_cast<unsigned long long*>(p);
  if (__match_any_sync(m, reinterpret_cast<unsigned long long>(p)) != m) {
    atomicAdd(q, static_cast<unsigned long long>(v));
    return;
  }
  const unsigned long long u = static_cast<unsigned long long>(v);
  const unsigned lo16 = __reduce_add_sync(m, static_cast<unsigned>(u & 0xffffu));
  const unsigned hi16 = __reduce_add_sync(m, static_cast<unsigned>((u >> 16) & 0xffffu));
  const unsigned hi32 = __reduce_add_sync(m, static_cast<unsigned>(u >> 32));
  if ((threadIdx.x & 31u) == static_cast<unsigned>(__ffs(m) - 1))
    atomicAdd(q, (static_cast<unsigned long long>(hi32) << 32) + (static_cast<unsigned long long>(hi16) << 16) +
                     lo16);
}
__device__ __forceinline__ void dk_add_i(int* p, int v) {
  const unsigned m = __activemask();
  if (__match_any_sync(m, reinterpret_cast<unsigned long long>(p)) != m) {
    atomicAdd(p, v);
    return;
  }
  const unsigned t = __reduce_add_sync(m, static_cast<unsigned>(v));
  if ((threadIdx.x & 31u) == static_cast<unsigned>(__ffs(m) - 1)) atomicAdd(p, static_cast<int>(t));
}
template <class F>
__device__ __forceinline__ void dk_add_f(F* p, F v) {
  const unsigned m = __activemask();
  if (__match_any_sync(m, reinterpret_cast<unsigned long long>(p)) != m) {
    atomicAdd(p, v);
    return;
  }
  if (m == 0xffffffffu) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(m, v, o);
  } else {
    F t = F(0);
    for (unsigned r = m; r; r &= r - 1) t += __shfl_sync(m, v, __ffs(r) - 1);
    v = t;
  }
  if ((threadIdx.x & 31u) == static_cast<unsigned>(__ffs(m) - 1)) atomicAdd(p, v);
}
__device__ __forceinline__ long long dk_atomic_i(long long* p, long long v) {
  return static_cast<long long>(dk_atomic_agg(reinterpret_cast<unsigned long long*>(p),
                                              static_cast<unsigned long long>(v)));
}
__device__ __forceinline__ int dk_atomic_i(int* p, int v) { return dk_atomic_agg(p, v); }
template <class F>
__device__ __forceinline__ F dk_atomic_f(F* p, F v) { return dk_atomic_agg(p, v); }

// ---- arithmetic with the simulator's fault rules (sim.hpp:1574-1590) ----
// (64-bit division is a long software sequence on the GPU; operands that fit
// in 31 bits take the 32-bit unsigned path, same result)
__device__ __forceinline__ long long dk_idiv(long long a, long long b) {
  if (b == 0) { dk_fault(dk::F_DIV); return 0; }
  if (((a | b) >> 31) == 0) return static_cast<long long>(static_cast<unsigned>(a) / static_cast<unsigned>(b));
  return a / b;
}
__device__ __forceinline__ long long dk_imod(long long a, long long b) {
  if (b == 0) { dk_fault(dk::F_DIV); return 0; }
  if (((a | b) >> 31) == 0) return static_cast<long long>(static_cast<unsigned>(a) % static_cast<unsigned>(b));
  return a % b;
}
__device__ __forceinline__ int dk_idiv(int a, int b) {
  if (b == 0) { dk_fault(dk::F_DIV); return 0; }
  return a / b;
}
__device__ __forceinline__ int dk_imod(int a, int b) {
  if (b == 0) { dk_fault(dk::F_DIV); return 0; }
  return a % b;
}
template <class T> __device__ __forceinline__ T dk_min(T a, T b) { return b < a ? b : a; }
template <class T> __device__ __forceinline__ T dk_max(T a, T b) { return a < b ? b : a; }

// ---- owner buffers ----
__device__ __forceinline__ unsigned dk_lane() { return threadIdx.x & 31u; }

// Owner init (dp_buffers, block- or warp-convergent, one thread per owner).
__device__ __forceinline__ void dk_own_init(dk::Own* o, long long cap) {
  long long sh = 0;
  while (sh < 40 && (1LL << sh) < cap) sh++;
  o->count = 0;
  o->cap = cap < 1 ? 0 : (1LL << sh);
  o->shift = sh;
  for (int j = 0; j < dk::kSegs; j++) o->seg[j] = 0;
}

// Segment j of an owner: reserved once from the arena (the first lane to need
// it wins the CAS; the others wait for the pointer).
__device__ __noinline__ unsigned long long dk_seg_base(dk::Own* o, long long j, long long stride) {
  unsigned long long b = atomicCAS(&o->seg[j], 0ull, 1ull);
  if (b == 0) {
    b = dk::kNoBase;
    const unsigned long long words = static_cast<unsigned long long>(o->cap) * stride;
    const unsigned long long off = atomicAdd(&dk_rt.ctr[2], words);
    if (off + words > dk_rt.arena_words) dk_fault(dk::F_POOL);
    else b = off + 2;
    atomicExch(&o->seg[j], b);
    return b;
  }
  while (b == 1) {
    __nanosleep(32);
    b = atomicAdd(&o->seg[j], 0ull);
  }
  return b;
}

// Warp-aggregated slot reservation in a shared-memory owner (warp or block).
__device__ __forceinline__ long long* dk_reserve_own(dk::Own* o, long long stride) {
  const unsigned m = __activemask();
  const unsigned lane = dk_lane();
  const int leader = __ffs(m) - 1;
  unsigned long long pos = 0;
  if (lane == static_cast<unsigned>(leader))
    pos = atomicAdd(&o->count, static_cast<unsigned long long>(__popc(m)));
  pos = __shfl_sync(m, pos, leader) + __popc(m & ((1u << lane) - 1u));
  if (o->cap < 1 || pos >= static_cast<unsigned long long>(o->cap) * dk::kSegs) {
    dk_fault(dk::F_OVERFLOW);
    return nullptr;
  }
  const long long j = static_cast<long long>(pos >> o->shift);
  unsigned long long b = *reinterpret_cast<volatile unsigned long long*>(&o->seg[j]);
  if (b < 2) b = dk_seg_base(o, j, stride);
  if (b == dk::kNoBase) return nullptr;
  return dk_rt.arena + (b - 2) + (pos & static_cast<unsigned long long>(o->cap - 1)) * stride;
}

__device__ __forceinline__ long long dk_grid_cap(long long total_bytes, long long nv, long long stride) {
  const long long c = total_bytes / (nv * 8);
  const long long r = static_cast<long long>(dk_rt.region_words) / stride;
  return c < r ? c : r;
}

// Grid owner: the launch's Inst record, storage = region[level & 1].
__device__ __forceinline__ long long* dk_reserve_grid(dk::Inst* in, long long stride, long long cap) {
  const unsigned m = __activemask();
  const unsigned lane = dk_lane();
  const int leader = __ffs(m) - 1;
  unsigned long long pos = 0;
  if (lane == static_cast<unsigned>(leader))
    pos = atomicAdd(&in->count, static_cast<unsigned long long>(__popc(m)));
  pos = __shfl_sync(m, pos, leader) + __popc(m & ((1u << lane) - 1u));
  if (cap < 1 || pos >= static_cast<unsigned long long>(cap)) {
    dk_fault(dk::F_OVERFLOW);
    return nullptr;
  }
  return dk_rt.region[in->level & 1u] + pos * stride;
}

__device__ __forceinline__ long long dk_clamp_count(unsigned long long c, long long cap) {
  return static_cast<long long>(c) < cap ? static_cast<long long>(c) : cap;
}

__device__ __forceinline__ long long dk_pending_own(dk::Own* o) {
  __syncwarp(__activemask());
  return dk_clamp_count(*reinterpret_cast<volatile unsigned long long*>(&o->count), o->cap * dk::kSegs);
}
__device__ __forceinline__ long long dk_pending_grid(dk::Inst* in, long long cap) {
  return dk_clamp_count(*reinterpret_cast<volatile unsigned long long*>(&in->count), cap);
}

// The buffer a launch from this owner hands to its child (sim.hpp:1530-1541):
// the launching thread copies the owner's segment table (shared memory) into
// the arena so the child can index item i as segs[i >> shift].
__device__ __forceinline__ dk::Inh dk_inherit_own(dk::Own* o, long long stride) {
  __threadfence();
  const long long n = dk_pending_own(o);
  if (n <= 0 || o->cap < 1) return dk::Inh{nullptr, nullptr, 0, stride, 0};
  const long long nseg = (n + o->cap - 1) >> o->shift;
  const unsigned long long off = atomicAdd(&dk_rt.ctr[2], static_cast<unsigned long long>(nseg));
  if (off + nseg > dk_rt.arena_words) {
    dk_fault(dk::F_POOL);
    return dk::Inh{nullptr, nullptr, 0, stride, 0};
  }
  unsigned long long* t = reinterpret_cast<unsigned long long*>(dk_rt.arena + off);
  for (long long j = 0; j < nseg; j++) t[j] = *reinterpret_cast<volatile unsigned long long*>(&o->seg[j]);
  __threadfence();
  return dk::Inh{nullptr, t, n, stride, o->shift};
}
__device__ __forceinline__ dk::Inh dk_inherit_grid(dk::Inst* in, long long stride, long long cap) {
  __threadfence();
  return dk::Inh{dk_rt.region[in->level & 1u], nullptr, dk_pending_grid(in, cap), stride, 0};
}

__device__ __forceinline__ long long dk_buf_word(const dk::Inh& h, long long i, long long w) {
  if (i < 0 || i >= h.n) {
    dk_fault(dk::F_BUFGET);
    return 0;
  }
  if (h.items) return h.items[i * h.stride + w];
  const unsigned long long b = h.segs[i >> h.shift];
  if (b < 2 || b == dk::kNoBase) {
    dk_fault(dk::F_BUFGET);
    return 0;
  }
  return dk_rt.arena[(b - 2) + (i & ((1LL << h.shift) - 1)) * h.stride + w];
}

// ---- launches ----
__device__ __forceinline__ dk::Inst* dk_new_inst(const dk::Inst* parent) {
  const unsigned long long i = atomicAdd(&dk_rt.ctr[3], 1ull);
  if (i >= dk_rt.inst_cap) {
    dk_fault(dk::F_INST);
    return nullptr;
  }
  dk::Inst* r = dk_rt.inst + i;
  r->count = 0;
  r->ticket = 0;
  r->level = parent ? parent->level + 1 : 1;
  r->aux = 0;
  return r;
}

// State area of one split phase (one reservation per launch, CAS on aux).
__device__ __noinline__ long long* dk_state_base(dk::Inst* in, long long words) {
  unsigned long long b = atomicCAS(&in->aux, 0ull, 1ull);
  if (b == 0) {
    b = dk::kNoBase;
    const unsigned long long off = atomicAdd(&dk_rt.ctr[2], static_cast<unsigned long long>(words));
    if (off + words > dk_rt.arena_words) dk_fault(dk::F_POOL);
    else b = off + 2;
    atomicExch(&in->aux, b);
  }
  while (b == 1) {
    __nanosleep(32);
    b = atomicAdd(&in->aux, 0ull);
  }
  return b == dk::kNoBase ? nullptr : dk_rt.arena + (b - 2);
}

__device__ __forceinline__ bool dk_launch_ok(long long g, long long b) {
  if (g < 1 || g > 0x7fffffffLL || b < 1 || b > 1024) {
    dk_fault(dk::F_CONFIG);
    return false;
  }
  return true;
}

__device__ __forceinline__ void dk_launched(cudaError_t e) {
  if (e != cudaSuccess) dk_fault(dk::F_LAUNCH);
  else atomicAdd(&dk_rt.ctr[1], 1ull);
}

// Last-block election of one launch (transform.hpp:620-633 counter/exit
// protocol); block-convergent, evaluated once per block.
__device__ __forceinline__ long long dk_grid_last(dk::Inst* in, int* cache) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0 && *cache < 0) {
    const unsigned t = atomicAdd(&in->ticket, 1u);
    *cache = (t == gridDim.x - 1) ? 1 : 0;
    __threadfence();
  }
  __syncthreads();
  return *cache;
}
