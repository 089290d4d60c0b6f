/* C ABI of a module produced by the .kdl -> sm_100a compiler
 * (paper_1606_08150_b200/kdl): every generated shared object exports exactly
 * these entry points.  Together with the Python front end (parse ->
 * consolidate -> CUDA builder -> nvcc) they replace the reference's
 * compile-and-simulate pair:
 *
 *   dpcons::parse_program   (parser.hpp:783)    -> kdl.parse_program
 *   dpcons::consolidate     (transform.hpp:971) -> kdl.consolidate
 *   dpcons::simulate        (sim.hpp:1746)      -> dk_set_rt + dk_launch_entry
 *                                                  (real execution on the B200)
 *   SimResult.metrics.childLaunchCount (sim.hpp:34-47) -> ctr[1] of dk_rt_t
 *   SimFault kinds overflow / runtime / config (sim.hpp:49-52) -> ctr[0] bits
 *
 * The module keeps the consolidated program's device state in one runtime
 * record (dk_rt_t, copied to __constant__ memory by dk_set_rt): the global
 * arrays (int -> int64, float -> float64, as the simulator's Value), the
 * counters, the pre-allocated buffer arena, the launch-record arena and the
 * two grid-buffer regions.  All pointers are device pointers.
 */
#ifndef DPC_KDL_H_
#define DPC_KDL_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DK_MAX_ARRAYS 64

/* ctr[0] fault bits */
#define DK_F_OVERFLOW 1u  /* consolidation buffer overflow (sim "overflow") */
#define DK_F_POOL 2u      /* pre-allocated pool exhausted (sim "overflow") */
#define DK_F_BOUNDS 4u    /* array index out of bounds (sim "runtime") */
#define DK_F_DIV 8u       /* integer division / modulo by zero (sim "runtime") */
#define DK_F_CONFIG 16u   /* launch extents out of range (sim "config") */
#define DK_F_LAUNCH 32u   /* device launch refused (pending-launch pool) */
#define DK_F_INST 64u     /* launch-record arena exhausted */
#define DK_F_BUFGET 128u  /* dp_buf_get / dp_buf_cfg index out of range (sim "runtime") */

typedef struct dk_rt_t {
  void* arr[DK_MAX_ARRAYS];      /* global arrays in declaration order */
  int64_t len[DK_MAX_ARRAYS];    /* their lengths (evaluated `global T a[len]`) */
  uint64_t* ctr;                 /* [0] faults [1] device launches [2] arena top [3] launch records used (start 1) */
  int64_t* arena;                /* owner buffers + sync_device phase state */
  uint64_t arena_words;
  void* inst;                    /* launch records, 24 bytes each; record 0 = the entry launch (zeroed per run) */
  uint64_t inst_cap;
  int64_t* region[2];            /* grid buffers, alternating by launch depth */
  uint64_t region_words;
  int64_t narr;
} dk_rt_t;

/* Select the device, size the CDP2 pending-launch pool (pending > 0) and
 * resolve every consolidated launch's KC_X block count from the compiled
 * kernel's occupancy: B = max(1, blocksPerSM * SMs / X) (config.hpp:63-72).
 * Returns 0, or 1 with dk_error() set. */
int dk_init(int device, long long pending);

/* sizeof(dk_rt_t) as compiled, for binding layout checks. */
int dk_sizeof_rt(void);

/* Copy the runtime record to the module's __constant__ dk_rt. */
int dk_set_rt(const void* rt);

/* Number of consolidated launch sites with a KC_X size, and their resolved
 * block counts (after dk_init). */
int dk_kc_count(void);
int dk_kc_values(long long* out);

/* Launch the program's entry `k<<<grid, block>>>(args)` on `stream`
 * (a cudaStream_t).  args: one 64-bit word per entry parameter (int value,
 * float64 bit pattern, or array index for array parameters); inst0: device
 * pointer to launch record 0.  Returns 0, 2 for bad extents, 1 for a launch
 * error (dk_error()). */
int dk_launch_entry(long long grid, long long block, const long long* args, void* inst0, void* stream);

const char* dk_error(void);

#ifdef __cplusplus
}
#endif

#endif /* DPC_KDL_H_ */
