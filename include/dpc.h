/*
 * dpc.h — C ABI of the B200-native workload-consolidation library (libdpc.so).
 *
 * This is the drop-in boundary for the hot path named by BASELINE.json's
 * north_star: the reference's application layer (CSR graph/matrix loaders and
 * generators, per-app run functions) fronting sm_100a kernels that run the
 * irregular-loop apps (SSSP, SpMV, graph coloring) and the parallel-recursion
 * apps (tree descendants / heights) in five variants: flat, basic-DP, and
 * warp / block / grid workload consolidation (arXiv 1606.08150 §IV).
 *
 * The reference ships this layer only as a specification
 * (module `workloads`); its code-level
 * boundary is `dpcons::simulate(Program, Workload, SimConfig) -> SimResult`
 * (/root/reference/proj/include/dpcons/sim.hpp:1746) fed by
 * `dpcons::consolidate` (transform.hpp:971).  Each entry point below cites the
 * reference interface it replaces.
 *
 * Conventions
 *  - Every function returns dpc_status; on failure dpc_last_error() returns a
 *    thread-local message.  Status kinds mirror SimFault.kind
 *    (sim.hpp:49-52: nesting | overflow | deadlock | oom | runtime | config).
 *  - Plain pointers and sizes only.  Host buffers are caller-owned.  Objects
 *    returned through `**out` are library-owned and released with the
 *    matching *_free / *_destroy.
 *  - Run calls are synchronous.  One dpc_ctx per host thread.
 *  - There is no CPU fallback: a run call on a machine without a usable
 *    sm_100 device fails with DPC_E_CUDA.
 */
#ifndef DPC_H_
#define DPC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DPC_ABI_VERSION 1

/* ---- status (SimFault.kind, sim.hpp:49-52; Diag, diag.hpp:16-20) ------- */
typedef enum dpc_status {
  DPC_OK = 0,
  DPC_E_INVALID = 1,  /* bad argument / invariant violation ("config")       */
  DPC_E_OVERFLOW = 2, /* consolidation buffer overflow (sim.hpp:1512-1517)    */
  DPC_E_NESTING = 3,  /* device nesting limit (sim.hpp:696-699)               */
  DPC_E_CUDA = 4,     /* CUDA runtime error / no device ("runtime")           */
  DPC_E_NCCL = 5,     /* NCCL error                                           */
  DPC_E_OOM = 6,      /* device or host allocation failed (sim.hpp:1139-1144) */
  DPC_E_IO = 7,       /* file I/O or parse error            */
  DPC_E_DEADLOCK = 8  /* watchdog fired (sim.hpp:946-955)                     */
} dpc_status;

/* Thread-local description of the last failure (empty string if none). */
const char* dpc_last_error(void);
int dpc_abi_version(void);

/* ---- variants (Granularity, ast.hpp:68; SPEC.md cli modes) ------------- */
typedef enum dpc_variant {
  DPC_FLAT = 0,  /* no-dp: thread-mapped loops, no device launches          */
  DPC_BASIC = 1, /* basic-dp: one CDP2 child launch per qualifying thread   */
  DPC_WARP = 2,  /* warp-level consolidation: <= 1 launch per warp          */
  DPC_BLOCK = 3, /* block-level consolidation: <= 1 launch per block        */
  DPC_GRID = 4   /* grid-level consolidation: 1 launch per parent grid      */
} dpc_variant;

typedef enum dpc_app {
  DPC_APP_SSSP = 0,
  DPC_APP_SPMV = 1,
  DPC_APP_COLOR = 2,
  DPC_APP_TREE_DESC = 3,
  DPC_APP_TREE_HEIGHT = 4
} dpc_app;

/* ---- data (SPEC.md:411-418 CsrGraph / Tree) ---------------------------- */
/* CSR graph or matrix.  rowptr has n+1 entries (rowptr[0]=0, rowptr[n]=m).
 * w (int32 edge weights) and val (fp32 matrix values) are optional (NULL). */
typedef struct dpc_csr {
  int64_t n;
  int64_t m;
  int64_t* rowptr;
  int32_t* col;
  int32_t* w;
  float* val;
  int64_t ncols; /* columns; 0 = square (n).  Row slices of a partitioned
                    matrix keep global column ids and set ncols. */
} dpc_csr;

/* Rooted tree.  parent[root] = -1.  Children of v are
 * clist[cstart[v] .. cstart[v+1]).  depth = number of levels. */
typedef struct dpc_tree {
  int64_t n;
  int32_t root;
  int32_t depth;
  int32_t* parent;
  int64_t* cstart;
  int32_t* clist;
} dpc_tree;

/* generator flags */
#define DPC_GEN_WEIGHTS 1u    /* fill w[] uniform in [wmin, wmax]            */
#define DPC_GEN_VALUES 2u     /* fill val[] uniform in (0, 1]                */
#define DPC_GEN_PERMUTE 4u    /* random vertex relabelling                   */
#define DPC_GEN_SYMMETRIC 8u  /* add reverse arcs, drop self loops + dups    */

/* R-MAT graph: n = 2^scale, m = edgefactor * n arcs (before symmetrize),
 * quadrant probabilities (a, b, c, 1-a-b-c).  Counter-based hashing makes the
 * output a pure function of the arguments (any thread count).
 * Replaces SPEC.md:435-444 gen_graph for the paper's Kron/R-MAT datasets. */
dpc_status dpc_gen_rmat(int scale, int edgefactor, double a, double b, double c,
                        int32_t wmin, int32_t wmax, uint64_t seed, uint32_t flags,
                        dpc_csr** out);

/* Rows [r0, r1) of exactly the graph dpc_gen_rmat(scale, ...) returns (same
 * arguments; DPC_GEN_SYMMETRIC not supported), with global column ids:
 * out->n = r1 - r0, out->ncols = 2^scale.  Each rank of a row-partitioned run
 * generates only its slice (BASELINE config 5). */
dpc_status dpc_gen_rmat_rows(int scale, int edgefactor, double a, double b, double c,
                             int32_t wmin, int32_t wmax, uint64_t seed, uint32_t flags,
                             int64_t r0, int64_t r1, dpc_csr** out);

/* SPEC.md:435-444 gen_graph(nodeCount, uniform(min,max), seed). */
dpc_status dpc_gen_graph_uniform(int64_t n, int32_t dmin, int32_t dmax, int32_t wmin,
                                 int32_t wmax, uint64_t seed, uint32_t flags,
                                 dpc_csr** out);

/* SPEC.md:435-444 gen_graph(nodeCount, powerlaw(alpha, maxDeg), seed). */
dpc_status dpc_gen_graph_powerlaw(int64_t n, double alpha, int32_t maxdeg, int32_t wmin,
                                  int32_t wmax, uint64_t seed, uint32_t flags,
                                  dpc_csr** out);

/* SPEC.md:425-433 gen_tree(depth, minChildren, maxChildren,
 * nonLeafFillFraction, seed).  Nodes are numbered level by level. */
dpc_status dpc_gen_tree(int32_t depth, int32_t min_children, int32_t max_children,
                        double fill, uint64_t seed, dpc_tree** out);

/* Copies caller arrays into a library-owned graph, validating the CSR
 * invariants.  w / val may be NULL. */
dpc_status dpc_csr_create(int64_t n, int64_t m, const int64_t* rowptr, const int32_t* col,
                          const int32_t* w, const float* val, dpc_csr** out);
/* The same for a row slice of a larger matrix (ncols > 0: column ids index
 * the whole matrix's columns, as the partitioned multi-GPU paths need for a
 * rank's row block of the caller's own graph). */
dpc_status dpc_csr_create_rows(int64_t n, int64_t ncols, int64_t m, const int64_t* rowptr, const int32_t* col,
                               const int32_t* w, const float* val, dpc_csr** out);
dpc_status dpc_csr_validate(const dpc_csr* g);
void dpc_csr_free(dpc_csr* g);

/* Copies a parent array into a library-owned tree (validates: one root,
 * acyclic, parents in range). */
dpc_status dpc_tree_create(int64_t n, const int32_t* parent, dpc_tree** out);
void dpc_tree_free(dpc_tree* t);

/* SPEC.md:446-450 load_csr / save_csr; text format SPEC.md:473
 * (line 1 "nodes edges [weighted]", line 2 row offsets, line 3 column
 * indices, line 4 optional weights).  A ".bin" suffix selects the binary
 * form (magic "DPCCSR01"). */
dpc_status dpc_load_csr(const char* path, dpc_csr** out);
dpc_status dpc_save_csr(const dpc_csr* g, const char* path);
/* DIMACS ingest (the paper's datasets; SPEC.md:475 names a
 * converter as the extension): the 9th challenge shortest-path format
 * ("c" comments, "p sp n m", "a u v w" arcs, 1-based; weights kept) or the
 * 10th challenge / METIS graph format (CiteSeer, Kron_log16: header
 * "n m [fmt [ncon]]", then one line of 1-based neighbours per vertex, "%"
 * comments; fmt 1 / 11 edge weights kept, vertex sizes / weights skipped;
 * m counts undirected edges, so the CSR holds 2m arcs).  The format is taken
 * from the first non-comment line.  Arcs keep file order within a row. */
dpc_status dpc_load_dimacs(const char* path, dpc_csr** out);
/* Tree text format SPEC.md:473: line 1 nodeCount, line 2 parent per node. */
dpc_status dpc_load_tree(const char* path, dpc_tree** out);
dpc_status dpc_save_tree(const dpc_tree* t, const char* path);

/* ---- launch configuration (Directive ast.hpp:90-111; KC_X config.hpp:68-84) */
typedef struct dpc_launch_cfg {
  int32_t variant;        /* dpc_variant                                    */
  int32_t threshold;      /* child work when degree > threshold (SPEC 469)  */
  int32_t parent_threads; /* parent block size                              */
  int32_t child_threads;  /* consolidated child block size                  */
  int32_t child_blocks;   /* 0 = derive from kc_x and measured occupancy    */
  int32_t kc_x;           /* KC_X concurrency divisor (config.hpp:68-75); 0 = "1-1" (B = pending items) */
  int32_t chunk;          /* edges per consolidated work item (load balance) */
  int32_t flags;          /* DPC_CFG_* bits                                  */
} dpc_launch_cfg;

/* dpc_launch_cfg.flags */
#define DPC_CFG_GRID_CDP 1 /* grid variant: last block launches the child via
                              CDP2 (else: one persistent cooperative kernel
                              with a device-wide barrier) */
#define DPC_CFG_GRID_CHUNKED 2 /* persistent grid variant, comparison forms: SpMV
                                  drains fixed-size chunk items warp by warp
                                  instead of the stream-balanced drain; SSSP
                                  takes two device-wide barriers per level
                                  (insert | drain) instead of one */
#define DPC_CFG_GRID_ASYNC 8 /* GC / SSSP persistent grid variant: asynchronous
                                worklist (device FIFO, no barrier between
                                rounds) instead of round-synchronous grid
                                barriers; GC default */
#define DPC_CFG_ALLOC_MALLOC 16 /* SpMV warp / block variants: per-owner buffers from
                                  the device heap (malloc / tail-launched free)
                                  instead of the pre-allocated pool -- the
                                  paper's allocator study, PAPER.md:296 */
#define DPC_CFG_X_PEER_GATHER 32 /* fused multi-GPU SpMV: every x gather goes to its
                                    owner's memory (default: the kernel first pulls the
                                    owners' x slices into the local x with coalesced
                                    peer reads, before the device-wide barrier it
                                    already has, then gathers locally) */
#define DPC_CFG_GRID_STREAM 64 /* SSSP / BFS persistent grid variant: force the
                                  frontier stream form -- each level's frontier
                                  edges cut into equal per-warp slices, bitmap
                                  dedup (sssp_stream.cu); default when the graph
                                  has >= 2^24 edges (measured faster there) */
#define DPC_CFG_GRID_LEVEL 128 /* SSSP / BFS persistent grid variant: force the
                                  light-list + chunk-item level form (default
                                  below 2^24 edges) */
#define DPC_CFG_SPMV_STREAM 256 /* SpMV grid variant: the per-call stream kernel
                                   (insert phase + item-table drain, round 1)
                                   instead of the default drain with the cached
                                   per-matrix window plan (row-start bits per
                                   256 nonzeros, built once per uploaded matrix,
                                   spmv_plan.cu); the fused multi-GPU forms
                                   always run the stream kernel */
#define DPC_CFG_GC_HASH (1 << 28) /* GC: greedy order = the seeded hash order
                                    (mix64(v ^ seed), v) instead of the canonical
                                    node order 0, 1, ..., n-1 (SPEC.md:454's GC
                                    oracle, the default) */
#define DPC_CFG_GC_LLF (1 << 29) /* GC: largest-log-degree-first order (ties by
                                   the seeded hash): shorter dependency chains
                                   and fewer colors on power-law graphs */
#define DPC_CFG_COOP_LAUNCH 4 /* persistent grid kernels: cudaLaunchCooperativeKernel
                                 + grid.sync instead of a normal launch of a
                                 co-resident grid + software barrier */

/* Bits 8-31 of dpc_launch_cfg.flags select measured alternative kernel
 * shapes of the same computation (stream drain shapes, GC server bounds,
 * ...): every value gives the same results.  Timing probes
 * that skip work are compiled out of the library.  SpMV grid plan form:
 * bit 9 / bit 12 = the 128-nonzero-window register / TMA-ring drains, bit 13
 * = the 256-nonzero drain without the hot-column x cache (the default keeps
 * the 32K most used columns' x in shared memory; DPC_SPMV_HOT_CAP in the
 * environment overrides the slot count, 0 disables it). */

/* Fills the measured default for (app, variant) (profiles/r02_launch_cfg.json,
 * compiled in as paper_1606_08150_b200/csrc/launch_table.inc).  Replaces
 * resolve_config, transform.hpp:417-475. */
dpc_status dpc_launch_cfg_default(int32_t app, int32_t variant, dpc_launch_cfg* cfg);

/* ---- metrics (Metrics, sim.hpp:34-47) ---------------------------------- */
typedef struct dpc_metrics {
  int64_t child_launch_count;   /* device-side launches (counter in HBM)     */
  int64_t buffer_items_inserted;/* consolidation-buffer items (chunks)       */
  int64_t pool_peak;            /* peak items held in the pre-allocated pool */
  int64_t iterations;           /* SSSP / GC rounds, tree levels             */
  int64_t edges_processed;      /* relaxed edges / nnz / scanned arcs        */
  int64_t host_launches;        /* kernels launched from the host            */
  double device_ms;             /* CUDA-event time of the run's kernels      */
  int32_t overflow;             /* nonzero: a buffer overflowed              */
  int32_t result_count;         /* colors used (GC), reached vertices (SSSP); basic TD/TH: children computed inline when the device pending-launch pool was full */
  int64_t vertices_processed;   /* SSSP / BFS: sum of the frontier sizes     */
} dpc_metrics;

/* ---- context ------------------------------------------------------------ */
typedef struct dpc_ctx dpc_ctx;

/* Creates a context bound to CUDA device `device` with its own stream.
 * Fails with DPC_E_CUDA when no sm_100 device is present. */
dpc_status dpc_ctx_create(int32_t device, dpc_ctx** out);
void dpc_ctx_destroy(dpc_ctx* ctx);
/* The context's cudaStream_t (as void*), for callers that time or order work. */
void* dpc_ctx_stream(dpc_ctx* ctx);
/* Number of SMs on the context's device (148 on B200). */
int32_t dpc_ctx_sm_count(dpc_ctx* ctx);
/* Timing helpers on the context stream: record event slot i (0..63), and
 * elapsed milliseconds between slots a and b (synchronizes on b). */
dpc_status dpc_ctx_event_record(dpc_ctx* ctx, int32_t slot);
dpc_status dpc_ctx_event_elapsed(dpc_ctx* ctx, int32_t a, int32_t b, float* ms);
dpc_status dpc_ctx_synchronize(dpc_ctx* ctx);
/* Writes a buffer larger than L2 on the context stream (timing hygiene). */
dpc_status dpc_ctx_flush_l2(dpc_ctx* ctx);

/* ---- host-buffer runs: the reference-facing API ------------------------
 * Each call uploads the inputs, runs the variant, downloads the result.
 * They replace benchmark(name) + simulate() (sim.hpp:1746)
 * for one app.  cfg may be NULL (measured default for cfg->variant = GRID).
 */
/* y = A x (fp32).  Replaces the SpMV benchmark. */
dpc_status dpc_run_spmv(dpc_ctx* ctx, const dpc_csr* A, const float* x, float* y,
                        const dpc_launch_cfg* cfg, dpc_metrics* met);
/* Single-source shortest paths with int32 weights >= 0; dist[v] = UINT32_MAX
 * when unreachable.  Replaces the SSSP benchmark. */
dpc_status dpc_run_sssp(dpc_ctx* ctx, const dpc_csr* g, int32_t source, uint32_t* dist,
                        const dpc_launch_cfg* cfg, dpc_metrics* met);
/* Greedy first-fit coloring in the canonical node order 0, 1, ..., n-1
 * (SPEC.md:454's GC oracle) -- or, with cfg->flags DPC_CFG_GC_HASH, in
 * descending (hash64(v ^ seed), v) order, or with DPC_CFG_GC_LLF
 * largest-log-degree-first (seed breaks ties); g must be symmetric without
 * self loops.  *ncolors receives the number of colors. */
/* BFS levels from `source` (the paper's BFS-Rec benchmark; SPEC.md:454 oracle
 * "BFS levels"): the SSSP consolidation with unit edge weights, weights in
 * G ignored.  level[v] = hops from source, UINT32_MAX if unreachable. */
dpc_status dpc_run_bfs(dpc_ctx* ctx, const dpc_csr* G, int32_t source, uint32_t* level,
                       const dpc_launch_cfg* cfg, dpc_metrics* met);
dpc_status dpc_run_color(dpc_ctx* ctx, const dpc_csr* g, uint64_t seed, int32_t* color,
                         int32_t* ncolors, const dpc_launch_cfg* cfg, dpc_metrics* met);
/* desc[v] = number of proper descendants of v (TD). */
dpc_status dpc_run_tree_desc(dpc_ctx* ctx, const dpc_tree* t, int32_t* desc,
                             const dpc_launch_cfg* cfg, dpc_metrics* met);
/* height[v] = max edges from v down to a leaf (TH). */
dpc_status dpc_run_tree_height(dpc_ctx* ctx, const dpc_tree* t, int32_t* height,
                               const dpc_launch_cfg* cfg, dpc_metrics* met);

/* ---- device-resident runs (inputs already in HBM; used by bench.py) ----- */
typedef struct dpc_dgraph dpc_dgraph;
typedef struct dpc_dtree dpc_dtree;

/* Uploads a graph once; the handle owns all device buffers of the app. */
dpc_status dpc_dgraph_upload(dpc_ctx* ctx, const dpc_csr* g, dpc_dgraph** out);
void dpc_dgraph_free(dpc_dgraph* dg);
/* Device pointers of the handle's x (n floats) and y (n floats) vectors. */
float* dpc_dgraph_x(dpc_dgraph* dg);
float* dpc_dgraph_y(dpc_dgraph* dg);
/* Device pointer of the handle's SSSP distance / GC color vector. */
uint32_t* dpc_dgraph_dist(dpc_dgraph* dg);
int32_t* dpc_dgraph_color(dpc_dgraph* dg);

/* %globaltimer stamps (ns) of the last persistent-kernel run whose metrics
 * were read: kernel start, device-wide barrier, end (phase split). */
dpc_status dpc_dgraph_phase_ns(dpc_dgraph* dg, uint64_t out[3]);
/* Runs called without metrics return once their work is enqueued; a fault
 * they raise is reported by the next call on the graph or by this check
 * (synchronises the context stream). */
dpc_status dpc_dgraph_check(dpc_ctx* ctx, dpc_dgraph* dg);
/* Tree persistent grid: kernel start, end of the top-down levels, end of the
 * count-down postwork (%globaltimer ns) of the last run. */
dpc_status dpc_dtree_phase_ns(dpc_dtree* dt, uint64_t out[3]);
/* Fault check of the last dpc_tree_device run made without metrics. */
dpc_status dpc_dtree_check(dpc_ctx* ctx, dpc_dtree* dt);

/* Asynchronous on the context stream (no host sync, no copies). */
dpc_status dpc_spmv_device(dpc_ctx* ctx, dpc_dgraph* dg, const float* d_x, float* d_y,
                           const dpc_launch_cfg* cfg, dpc_metrics* met);
/* Synchronous at the end (termination is device-driven; the host reads the
 * iteration count once). */
/* BFS levels on a device-resident graph (weights not needed). */
dpc_status dpc_bfs_device(dpc_ctx* ctx, dpc_dgraph* dg, int32_t source, const dpc_launch_cfg* cfg,
                          dpc_metrics* met);
dpc_status dpc_sssp_device(dpc_ctx* ctx, dpc_dgraph* dg, int32_t source,
                           const dpc_launch_cfg* cfg, dpc_metrics* met);
dpc_status dpc_color_device(dpc_ctx* ctx, dpc_dgraph* dg, uint64_t seed,
                            const dpc_launch_cfg* cfg, dpc_metrics* met);

dpc_status dpc_dtree_upload(dpc_ctx* ctx, const dpc_tree* t, dpc_dtree** out);
void dpc_dtree_free(dpc_dtree* dt);
/* which = DPC_APP_TREE_DESC or DPC_APP_TREE_HEIGHT; result stays on device. */
dpc_status dpc_tree_device(dpc_ctx* ctx, dpc_dtree* dt, int32_t which,
                           const dpc_launch_cfg* cfg, dpc_metrics* met);
int32_t* dpc_dtree_result(dpc_dtree* dt);

/* SpMV through the operator-resident handle with HOST vectors: copies x in,
 * runs, copies y out (synchronous).  This is the end-to-end path. */
dpc_status dpc_spmv_host(dpc_ctx* ctx, dpc_dgraph* dg, const float* x_host, float* y_host,
                         const dpc_launch_cfg* cfg, dpc_metrics* met);

/* The same over `count` independent host vectors, pipelined: vector i+1's
 * host->device copy and vector i-1's device->host copy overlap vector i's
 * SpMV (two copy streams + the context stream, two device slots).  Returns
 * when every y is in host memory.  Host vectors should be pinned
 * (dpc_host_alloc) for the copies to overlap.  Serving form of the
 * reference's per-call simulate() (sim.hpp:1746). */
dpc_status dpc_spmv_host_batch(dpc_ctx* ctx, dpc_dgraph* dg, const float* const* x_host, float* const* y_host,
                               int64_t count, const dpc_launch_cfg* cfg, dpc_metrics* met);
/* The same over `count` vectors stored back to back in host memory (x_host:
 * count x ncols floats, y_host: count x n floats, pinned for overlap):
 * the copies move `group` vectors at a time (0 = about 32 MB per copy) --
 * PCIe copies of a few MB each run well below the link rate when both
 * directions are busy (measured: 4 MB pairs 58 GB/s aggregate, 64 MB pairs
 * 83 GB/s) -- double-buffered, group k+1 coming in and group k-1 going out
 * while group k is multiplied.  Returns when every y is in host memory. */
dpc_status dpc_spmv_host_batch_contig(dpc_ctx* ctx, dpc_dgraph* dg, const float* x_host, float* y_host,
                                      int64_t count, int64_t group, const dpc_launch_cfg* cfg, dpc_metrics* met);

/* ---- fused multi-GPU path over peer memory (BASELINE config 5) ----
 * CUDA IPC export / import of a device buffer; the caller moves the 64-byte
 * handles between ranks (NCCL, MPI, torch.distributed). */
dpc_status dpc_ipc_handle(const void* d_ptr, uint8_t out[64]);
dpc_status dpc_ipc_open(dpc_ctx* ctx, const uint8_t handle[64], void** d_out);
dpc_status dpc_ipc_close(void* d_ptr);
/* Device-side barrier over peer memory: d_flag_tab is a DEVICE array of
 * `world` pointers to the ranks' flag arrays (2 x world u64 each, zeroed
 * once); epochs must increase by one per barrier (1, 2, ...) and stay below
 * 2^32.  Enqueued on the context stream. */
dpc_status dpc_p2p_barrier(dpc_ctx* ctx, uint64_t* const* d_flag_tab, int32_t world, int32_t me, uint64_t epoch);
/* The same barrier carrying one u32 per rank: *sum = the sum over ranks
 * (synchronous; an all-reduce riding on the flags, e.g. frontier sizes). */
dpc_status dpc_p2p_barrier_sum(dpc_ctx* ctx, uint64_t* const* d_flag_tab, int32_t world, int32_t me,
                               uint64_t epoch, uint32_t value, uint64_t* sum);
/* Reports DPC_E_DEADLOCK if a barrier timed out (synchronises the stream). */
dpc_status dpc_p2p_check(dpc_ctx* ctx);
/* Fused partitioned SSSP (dpc_msssp_* with no send buffers): relaxations of
 * remote vertices go straight into their owner's distance / stamp / next
 * frontier through peer pointers.  dpc_msssp_buffers gives the 5 device
 * buffers this rank exports (dist, stamp, front0, front1, counters; IPC-able
 * cudaMalloc bases); d_peer_table is a DEVICE array of `world` such 5-pointer
 * records, own and IPC-mapped.  Per iteration: relax, peer barrier, apply
 * (0 pairs), dpc_p2p_barrier_sum of the next-frontier sizes. */
dpc_status dpc_msssp_buffers(dpc_dgraph* dg, void* out[5]);
dpc_status dpc_msssp_set_peers(dpc_dgraph* dg, const void* d_peer_table);
/* Grid stream SpMV of this rank's row block with x read from the owners:
 * d_xpeer is a DEVICE array of `world` pointers, x entry i at
 * d_xpeer[i / rows_per_rank][i % rows_per_rank] (replaces ncclAllGather +
 * dpc_spmv_device, multi.cu).  Needs the grid variant with threshold 0.
 * Uses the local graph's x buffer (ncols entries) as the pulled copy of x
 * unless DPC_CFG_X_PEER_GATHER. */
dpc_status dpc_multi_spmv_fused(dpc_ctx* ctx, dpc_dgraph* local, const float* const* d_xpeer, int32_t world,
                                int64_t rows_per_rank, float* d_y_local, const dpc_launch_cfg* cfg,
                                dpc_metrics* met);

/* Device memory on the context's GPU (caller-owned vectors for the
 * device-pointer entry points). */
void* dpc_dev_alloc(dpc_ctx* ctx, size_t bytes);
void dpc_dev_free(dpc_ctx* ctx, void* p);

/* Pinned host memory (for copy bandwidth on the end-to-end path). */
void* dpc_host_alloc(size_t bytes);
void dpc_host_free(void* p);

/* Copies between caller host memory and library device memory on the
 * context stream (synchronous). */
dpc_status dpc_copy_h2d(dpc_ctx* ctx, void* dst_dev, const void* src_host, size_t bytes);
dpc_status dpc_copy_d2h(dpc_ctx* ctx, void* dst_host, const void* src_dev, size_t bytes);
/* Fills device memory with a byte value on the context stream (asynchronous;
 * ordered before the stream's later work). */
dpc_status dpc_dev_memset(dpc_ctx* ctx, void* dst_dev, int32_t value, size_t bytes);

/* Diagnostics: with DPC_TRACE=1 in the environment, the coloring kernels
 * record per vertex %globaltimer (ns) at its color write [0, n), at its
 * enqueue [n, 2n) and at its dequeue [2n, 3n) (asynchronous form); copies
 * the first `n` words of that record from the handle's last run. */
dpc_status dpc_dgraph_trace(dpc_dgraph* g, uint64_t* out, int64_t n);

/* ---- PageRank (the paper's PR benchmark; SPEC.md:454 / :468) ------------
 * `iters` power iterations with damping d from r = 1/n:
 *   r'[v] = (1-d)/n + d (sum over edges u->v of r[u] / outdeg(u) + D / n),
 * D = rank mass of the vertices without out-edges.  Each iteration is one
 * SpMV over the transposed graph with the SpMV variant of `cfg`
 * (dpc_launch_cfg_default(DPC_APP_SPMV, ...)), built once per handle. */
typedef struct dpc_prgraph dpc_prgraph;
dpc_status dpc_pr_upload(dpc_ctx* ctx, const dpc_csr* g, dpc_prgraph** out);
void dpc_pr_free(dpc_prgraph* h);
dpc_status dpc_pr_device(dpc_ctx* ctx, dpc_prgraph* h, int32_t iters, double damping,
                         const dpc_launch_cfg* cfg, dpc_metrics* met);
/* Device pointer to the n ranks of the last dpc_pr_device run. */
float* dpc_pr_rank(dpc_prgraph* h);
dpc_status dpc_run_pagerank(dpc_ctx* ctx, const dpc_csr* g, int32_t iters, double damping, float* rank,
                            const dpc_launch_cfg* cfg, dpc_metrics* met);

/* ---- multi-GPU (one process per GPU; NCCL over NVLink) ------------------
 * Row / vertex partition of a graph across `world` ranks (BASELINE config 5).
 */
typedef struct dpc_comm dpc_comm;
/* NCCL unique id (128 bytes) created on rank 0 and broadcast by the caller. */
dpc_status dpc_comm_unique_id(uint8_t id[128]);
dpc_status dpc_comm_init(dpc_ctx* ctx, int32_t rank, int32_t world, const uint8_t id[128],
                         dpc_comm** out);
void dpc_comm_destroy(dpc_comm* comm);
int32_t dpc_comm_rank(dpc_comm* comm);
int32_t dpc_comm_world(dpc_comm* comm);
/* Equal-nnz row split of a CSR into `world` parts: bounds[0..world]. */
dpc_status dpc_partition_rows(const dpc_csr* g, int32_t world, int64_t* bounds);
/* One distributed SpMV step on a 1-D row partition with equal row blocks
 * (rank p owns rows / x entries [p*R, (p+1)*R), R = local->n,
 * local->ncols = R * world): ncclAllGather of every rank's x slice (d_x_local,
 * R floats) into the handle's x (R * world floats) over NVLink, then
 * y_local = A_local x with the variant in cfg.  Asynchronous on the context
 * stream. */
dpc_status dpc_multi_spmv(dpc_ctx* ctx, dpc_comm* comm, dpc_dgraph* local, const float* d_x_local,
                          float* d_y_local, const dpc_launch_cfg* cfg, dpc_metrics* met);

/* Vertex-partitioned SSSP (BASELINE config 5; the reference's Fig. 1(b)
 * irregular loop, run level-synchronously across ranks).
 * `local` is this rank's row block [rank*R, rank*R + local->n) of an
 * n_global-vertex graph with global column ids (dpc_gen_rmat_rows), R =
 * ceil(n_global / world).  Each iteration relaxes the local frontier with
 * the cfg variant (the grid variant runs in its CDP form: one exchange per
 * iteration), sends {vertex, distance} pairs for remote targets to their
 * owners with grouped ncclSend/ncclRecv over NVLink, applies what it
 * receives, and stops when the all-reduced next-frontier size is 0.
 * Distances of the local vertices are left in the handle (dpc_dgraph_dist).
 * met->result_count = pairs this rank sent. */
dpc_status dpc_multi_sssp(dpc_ctx* ctx, dpc_comm* comm, dpc_dgraph* local, int64_t n_global, int64_t source,
                          const dpc_launch_cfg* cfg, dpc_metrics* met);

/* The steps of dpc_multi_sssp, for callers that drive the exchange with
 * their own transport (and for single-GPU tests of the partitioned path):
 *   dpc_msssp_begin : init distances of the rank's block (r0 = rank * R,
 *                     rows_per_rank = R), clear the remote filter
 *   dpc_msssp_relax : relax the current frontier; send_counts[q] = pairs
 *                     queued for owner q (host array of `world` entries)
 *   dpc_msssp_send_buffer(q) : device pointer to those pairs
 *                     ({uint32 global vertex, uint32 distance} each)
 *   dpc_msssp_recv_buffer : device receive area; it holds
 *                     dpc_msssp_recv_capacity pairs (world x local edges
 *                     at begin).  A rank can receive more than that (its
 *                     peers' edge counts bound what they send), so callers
 *                     that know the incoming count call
 *                     dpc_msssp_recv_reserve, which grows the area
 *   dpc_msssp_send_counts : device copy of send_counts (for collectives)
 *   dpc_msssp_apply : apply `count` received pairs (device pointer), close
 *                     the iteration; *next_fsize = local |F_it+1|
 *   dpc_msssp_end   : fault check and metrics */
dpc_status dpc_msssp_begin(dpc_ctx* ctx, dpc_dgraph* local, int64_t r0, int64_t rows_per_rank,
                           int64_t n_global, int32_t world, int64_t source, const dpc_launch_cfg* cfg);
dpc_status dpc_msssp_relax(dpc_ctx* ctx, dpc_dgraph* local, uint32_t* send_counts);
const void* dpc_msssp_send_buffer(dpc_dgraph* local, int32_t owner);
void* dpc_msssp_recv_buffer(dpc_dgraph* local);
uint64_t dpc_msssp_recv_capacity(dpc_dgraph* local);
dpc_status dpc_msssp_recv_reserve(dpc_ctx* ctx, dpc_dgraph* local, uint64_t pairs, void** d_out);
const uint32_t* dpc_msssp_send_counts(dpc_dgraph* local);
dpc_status dpc_msssp_apply(dpc_ctx* ctx, dpc_dgraph* local, const void* d_pairs, uint64_t count,
                           uint32_t* next_fsize);
dpc_status dpc_msssp_end(dpc_ctx* ctx, dpc_dgraph* local, dpc_metrics* met);

#ifdef __cplusplus
}
#endif
#endif /* DPC_H_ */
