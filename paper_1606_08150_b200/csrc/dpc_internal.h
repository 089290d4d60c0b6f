// Internal host-side helpers shared by the host (generators / IO) and CUDA
// translation units of libdpc.so.  Not part of the ABI.
#pragma once

#include <cstdint>
#include <string>

#include "dpc.h"

namespace dpc {

// Thread-local last-error slot behind dpc_last_error().
void set_error(const std::string& msg);
void clear_error();
dpc_status fail(dpc_status st, const std::string& msg);

// splitmix64 finalizer: the counter-based hash every generator draws from.
// A pure function of its input, so generation is independent of thread count.
inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Stream ids keep the draws of different quantities independent.
enum : uint64_t {
  kStreamRmat = 0x1000000000000000ull,
  kStreamWeight = 0x2000000000000000ull,
  kStreamValue = 0x3000000000000000ull,
  kStreamPerm = 0x4000000000000000ull,
  kStreamDegree = 0x5000000000000000ull,
  kStreamNbr = 0x6000000000000000ull,
  kStreamTree = 0x7000000000000000ull,
  kStreamTreeSel = 0x8000000000000000ull,
};

inline uint64_t draw(uint64_t seed, uint64_t stream, uint64_t counter) {
  return mix64(mix64(seed ^ stream) ^ counter);
}

// fp32 value in (0, 1] with 24 random bits: exact in fp32 and fp64.
inline float unit_value(uint64_t h) {
  return static_cast<float>((h >> 40) + 1) * (1.0f / 16777216.0f);
}

// GC priority (SPEC.md:468 canonical order, made explicit): vertices are
// colored in descending (hash64(v ^ seed), v) order.  Shared verbatim with the
// device code (gc.cu) and the oracle (oracle/oracle.c).
inline uint64_t gc_priority(uint64_t v, uint64_t seed) { return mix64(v ^ seed); }

int host_threads();

}  // namespace dpc
