/* TEST INFRASTRUCTURE ONLY — the CPU checker.  Only tests/, bench.py's
 * cpu_baseline / --impl reference legs and __graft_entry__.smoke() may load
 * liboracle.so; libdpc.so never links it and has no CPU fallback.
 *
 * Plain-C restatement of the sequential oracles the reference specifies for
 * the hot-path apps ("SSSP = level-synchronous relaxation
 * distances; SpMV = y = A·x; GC = greedy first-fit coloring under canonical
 * node order; TH = per-subtree height; TD = per-subtree descendant counts"),
 * plus multi-threaded CPU versions used as the CPU baseline.
 * Pinned by tests/test_oracle.py against (1) SPEC.md:457-459 golden examples,
 * (2) tests/golden/*.json vectors produced by running the reference simulator
 * itself (oracle/_ref, tests/golden/make_golden.py).
 */
#ifndef DPC_ORACLE_H_
#define DPC_ORACLE_H_
#include <stdint.h>

uint64_t orc_mix64(uint64_t z);

/* y64 = A x in fp64, row by row in column order. */
void orc_spmv_f64(int64_t n, const int64_t* rowptr, const int32_t* col, const float* val,
                  const float* x, double* y);
/* fp32 CSR SpMV over `threads` OpenMP threads (CPU baseline). */
void orc_spmv_f32_mt(int64_t n, const int64_t* rowptr, const int32_t* col, const float* val,
                     const float* x, float* y, int threads);

/* Dijkstra with a binary heap; dist = UINT32_MAX for unreachable.  Equal to
 * the fixpoint of level-synchronous relaxation. */
int orc_sssp_dijkstra(int64_t n, const int64_t* rowptr, const int32_t* col, const int32_t* w,
                      int32_t source, uint32_t* dist);
/* Frontier Bellman-Ford over `threads` threads (CPU baseline); returns rounds. */
int64_t orc_sssp_bf_mt(int64_t n, const int64_t* rowptr, const int32_t* col, const int32_t* w,
                       int32_t source, uint32_t* dist, int threads);

/* Sequential greedy first-fit in descending (mix64(v ^ seed), v) order
 * (SPEC.md:454, 468).  Returns the number of colors, -1 on alloc failure. */
int32_t orc_color_greedy(int64_t n, const int64_t* rowptr, const int32_t* col, uint64_t seed,
                         int32_t* color);
/* ... under order 0 = hash (above), 1 = canonical node order,
 * 2 = largest-log-degree-first (see oracle.c). */
int32_t orc_color_greedy_order(int64_t n, const int64_t* rowptr, const int32_t* col, uint64_t seed,
                               int order, int32_t* color);
/* 1 iff color is a proper coloring with colors in [0, ncolors). */
int orc_color_valid(int64_t n, const int64_t* rowptr, const int32_t* col, const int32_t* color,
                    int32_t ncolors);

/* TD: desc[v] = number of proper descendants; TH: height[v] = edges to the
 * deepest leaf below v.  Bottom-up over a BFS order. */
int orc_tree_desc(int64_t n, const int32_t* parent, int32_t* desc);
int orc_tree_height(int64_t n, const int32_t* parent, int32_t* height);

/* BFS levels from source (UINT32_MAX = unreachable). */
int orc_bfs(int64_t n, const int64_t* rowptr, const int32_t* col, int32_t source, uint32_t* level);
/* PageRank: iters power iterations, damping d, fp64. */
int orc_pagerank(int64_t n, const int64_t* rowptr, const int32_t* col, int32_t iters, double d,
                 double* rank);
/* Directed R-MAT graph, the same graph as dpc_gen_rmat for the
 * same arguments: rowptr[2^scale + 1], col/w/val[2^scale * edgefactor]
 * caller-allocated (w / val may be NULL).  0 on success, -1 on alloc failure. */
int orc_gen_rmat(int scale, int edgefactor, double a, double b, double c, int32_t wmin, int32_t wmax,
                 uint64_t seed, int permute, int64_t* rowptr, int32_t* col, int32_t* w, float* val);
#endif
