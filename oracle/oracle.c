/* TEST INFRASTRUCTURE ONLY — see oracle.h.  CPU restatement of the
 * reference's sequential oracles for the hot-path apps. */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* Minimal pthread parallel-for: fn(arg, lo, hi) on `threads` contiguous or
 * dynamically claimed chunks of [0, n). */
typedef void (*range_fn)(void* arg, int64_t lo, int64_t hi);
typedef struct {
  range_fn fn;
  void* arg;
  int64_t n, chunk;
  int64_t next; /* atomic cursor */
} pfor_t;

static void* pfor_worker(void* p) {
  pfor_t* t = (pfor_t*)p;
  for (;;) {
    int64_t lo = __atomic_fetch_add(&t->next, t->chunk, __ATOMIC_RELAXED);
    if (lo >= t->n) break;
    int64_t hi = lo + t->chunk < t->n ? lo + t->chunk : t->n;
    t->fn(t->arg, lo, hi);
  }
  return NULL;
}

static void parallel_for(int64_t n, int64_t chunk, int threads, range_fn fn, void* arg) {
  pfor_t t = {fn, arg, n, chunk > 0 ? chunk : 1, 0};
  if (threads <= 1 || n <= chunk) {
    if (n > 0) fn(arg, 0, n);
    return;
  }
  if (threads > 256) threads = 256;
  pthread_t th[256];
  int started = 0;
  for (int i = 1; i < threads; i++)
    if (pthread_create(&th[started], NULL, pfor_worker, &t) == 0) started++;
  pfor_worker(&t);
  for (int i = 0; i < started; i++) pthread_join(th[i], NULL);
}

/* Same counter hash as the product (paper_1606_08150_b200/csrc/dpc_internal.h). */
uint64_t orc_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* ---------------- SpMV (SPEC.md:454 "SpMV = y = A·x", :459) ------------- */
void orc_spmv_f64(int64_t n, const int64_t* rowptr, const int32_t* col, const float* val,
                  const float* x, double* y) {
  for (int64_t i = 0; i < n; i++) {
    double s = 0.0;
    for (int64_t k = rowptr[i]; k < rowptr[i + 1]; k++) s += (double)val[k] * (double)x[col[k]];
    y[i] = s;
  }
}

typedef struct {
  const int64_t* rowptr;
  const int32_t* col;
  const float* val;
  const float* x;
  float* y;
} spmv_arg_t;

static void spmv_range(void* p, int64_t lo, int64_t hi) {
  const spmv_arg_t* a = (const spmv_arg_t*)p;
  const int64_t* rowptr = a->rowptr;
  const int32_t* col = a->col;
  const float* val = a->val;
  const float* x = a->x;
  for (int64_t i = lo; i < hi; i++) {
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    int64_t k = rowptr[i], e = rowptr[i + 1];
    for (; k + 3 < e; k += 4) {
      s0 += val[k] * x[col[k]];
      s1 += val[k + 1] * x[col[k + 1]];
      s2 += val[k + 2] * x[col[k + 2]];
      s3 += val[k + 3] * x[col[k + 3]];
    }
    for (; k < e; k++) s0 += val[k] * x[col[k]];
    a->y[i] = (s0 + s1) + (s2 + s3);
  }
}

void orc_spmv_f32_mt(int64_t n, const int64_t* rowptr, const int32_t* col, const float* val,
                     const float* x, float* y, int threads) {
  spmv_arg_t a = {rowptr, col, val, x, y};
  parallel_for(n, 1024, threads, spmv_range, &a);
}

/* ---------------- SSSP ------------------- */
typedef struct {
  uint64_t* a;
  int64_t len, cap;
} heap_t;

static int heap_push(heap_t* h, uint64_t key) {
  if (h->len == h->cap) {
    int64_t nc = h->cap ? 2 * h->cap : 1024;
    uint64_t* na = (uint64_t*)realloc(h->a, (size_t)nc * sizeof(uint64_t));
    if (!na) return -1;
    h->a = na;
    h->cap = nc;
  }
  int64_t i = h->len++;
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (h->a[p] <= key) break;
    h->a[i] = h->a[p];
    i = p;
  }
  h->a[i] = key;
  return 0;
}

static uint64_t heap_pop(heap_t* h) {
  uint64_t top = h->a[0], last = h->a[--h->len];
  int64_t i = 0;
  for (;;) {
    int64_t c = 2 * i + 1;
    if (c >= h->len) break;
    if (c + 1 < h->len && h->a[c + 1] < h->a[c]) c++;
    if (h->a[c] >= last) break;
    h->a[i] = h->a[c];
    i = c;
  }
  if (h->len) h->a[i] = last;
  return top;
}

int orc_sssp_dijkstra(int64_t n, const int64_t* rowptr, const int32_t* col, const int32_t* w,
                      int32_t source, uint32_t* dist) {
  for (int64_t i = 0; i < n; i++) dist[i] = UINT32_MAX;
  if (source < 0 || source >= n) return -1;
  heap_t h = {0, 0, 0};
  dist[source] = 0;
  if (heap_push(&h, (uint64_t)source)) return -1;
  while (h.len) {
    uint64_t k = heap_pop(&h);
    uint32_t d = (uint32_t)(k >> 32), u = (uint32_t)k;
    if (d != dist[u]) continue;
    for (int64_t e = rowptr[u]; e < rowptr[u + 1]; e++) {
      uint64_t nd = (uint64_t)d + (uint64_t)(uint32_t)w[e];
      uint32_t v = (uint32_t)col[e];
      if (nd < dist[v]) {
        dist[v] = (uint32_t)nd;
        if (heap_push(&h, (nd << 32) | v)) {
          free(h.a);
          return -1;
        }
      }
    }
  }
  free(h.a);
  return 0;
}

static inline int atomic_min_u32(uint32_t* p, uint32_t v) {
  uint32_t old = __atomic_load_n(p, __ATOMIC_RELAXED);
  while (v < old) {
    if (__atomic_compare_exchange_n(p, &old, v, 1, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) return 1;
  }
  return 0;
}

typedef struct {
  const int64_t* rowptr;
  const int32_t* col;
  const int32_t* w;
  uint32_t* dist;
  uint32_t* stamp;
  const uint32_t* front;
  uint32_t* next;
  int64_t nn;
  uint32_t it;
} bf_arg_t;

static void bf_range(void* p, int64_t lo, int64_t hi) {
  bf_arg_t* a = (bf_arg_t*)p;
  for (int64_t i = lo; i < hi; i++) {
    uint32_t u = a->front[i];
    uint32_t du = __atomic_load_n(&a->dist[u], __ATOMIC_RELAXED);
    for (int64_t e = a->rowptr[u]; e < a->rowptr[u + 1]; e++) {
      uint64_t nd = (uint64_t)du + (uint64_t)(uint32_t)a->w[e];
      if (nd >= UINT32_MAX) continue;
      uint32_t v = (uint32_t)a->col[e];
      if (atomic_min_u32(&a->dist[v], (uint32_t)nd)) {
        if (__atomic_exchange_n(&a->stamp[v], a->it, __ATOMIC_RELAXED) != a->it) {
          int64_t q = __atomic_fetch_add(&a->nn, 1, __ATOMIC_RELAXED);
          a->next[q] = v;
        }
      }
    }
  }
}

int64_t orc_sssp_bf_mt(int64_t n, const int64_t* rowptr, const int32_t* col, const int32_t* w,
                       int32_t source, uint32_t* dist, int threads) {
  if (threads < 1) threads = 1;
  if (source < 0 || source >= n) return -1;
  uint32_t* front = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n ? n : 1));
  uint32_t* next = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n ? n : 1));
  uint32_t* stamp = (uint32_t*)calloc((size_t)(n ? n : 1), sizeof(uint32_t));
  if (!front || !next || !stamp) {
    free(front), free(next), free(stamp);
    return -1;
  }
  for (int64_t i = 0; i < n; i++) dist[i] = UINT32_MAX;
  dist[source] = 0;
  front[0] = (uint32_t)source;
  int64_t fn = 1, rounds = 0;
  while (fn > 0) {
    bf_arg_t a = {rowptr, col, w, dist, stamp, front, next, 0, (uint32_t)(rounds + 1)};
    parallel_for(fn, 64, threads, bf_range, &a);
    uint32_t* t = front;
    front = next;
    next = t;
    fn = a.nn;
    rounds++;
  }
  free(front), free(next), free(stamp);
  return rounds;
}

/* ---------------- GC -------------------------------- */
typedef struct {
  uint64_t p;
  int32_t v;
} prio_t;

static int prio_desc(const void* a, const void* b) {
  const prio_t* x = (const prio_t*)a;
  const prio_t* y = (const prio_t*)b;
  if (x->p != y->p) return x->p < y->p ? 1 : -1;
  return x->v < y->v ? 1 : (x->v > y->v ? -1 : 0);
}

/* Greedy first-fit in descending priority order under one of three orders
 * (the GPU kernels' DPC_CFG_GC_* flags):
 *   ORC_GC_HASH      priority (mix64(v ^ seed), v)            -- the default
 *   ORC_GC_CANONICAL canonical node order 0, 1, ..., n-1: SPEC.md:454's GC
 *                    oracle ("greedy first-fit coloring under canonical
 *                    node order"), priority (~v)
 *   ORC_GC_LLF       largest-log-degree-first: priority
 *                    (bits(deg(v)) << 58 | mix64(v ^ seed) >> 6, v), with
 *                    bits(d) = 32 - clz(d) (0 for d = 0) -- the LLF order of
 *                    Hasenplaugh et al. (SPAA 2014) */
static uint64_t orc_gc_prio(int64_t v, int64_t deg, uint64_t seed, int order) {
  if (order == 1) return ~(uint64_t)v;
  if (order == 2) {
    uint64_t bits = 0;
    while (bits < 32 && ((uint64_t)deg >> bits)) bits++;
    return (bits << 58) | (orc_mix64((uint64_t)v ^ seed) >> 6);
  }
  return orc_mix64((uint64_t)v ^ seed);
}

int32_t orc_color_greedy_order(int64_t n, const int64_t* rowptr, const int32_t* col, uint64_t seed,
                               int order, int32_t* color) {
  prio_t* ord = (prio_t*)malloc(sizeof(prio_t) * (size_t)(n ? n : 1));
  int64_t maxdeg = 0;
  for (int64_t v = 0; v < n; v++)
    if (rowptr[v + 1] - rowptr[v] > maxdeg) maxdeg = rowptr[v + 1] - rowptr[v];
  int64_t* mark = (int64_t*)malloc(sizeof(int64_t) * (size_t)(maxdeg + 2));
  if (!ord || !mark) {
    free(ord), free(mark);
    return -1;
  }
  for (int64_t v = 0; v < n; v++) {
    ord[v].p = orc_gc_prio(v, rowptr[v + 1] - rowptr[v], seed, order);
    ord[v].v = (int32_t)v;
    color[v] = -1;
  }
  qsort(ord, (size_t)n, sizeof(prio_t), prio_desc);
  for (int64_t i = 0; i < maxdeg + 2; i++) mark[i] = -1;
  int32_t ncolors = 0;
  for (int64_t i = 0; i < n; i++) {
    int32_t v = ord[i].v;
    for (int64_t e = rowptr[v]; e < rowptr[v + 1]; e++) {
      int32_t c = color[col[e]];
      if (c >= 0 && c <= maxdeg) mark[c] = v;
    }
    int32_t c = 0;
    while (mark[c] == v) c++;
    color[v] = c;
    if (c + 1 > ncolors) ncolors = c + 1;
  }
  free(ord), free(mark);
  return ncolors;
}

int32_t orc_color_greedy(int64_t n, const int64_t* rowptr, const int32_t* col, uint64_t seed,
                         int32_t* color) {
  return orc_color_greedy_order(n, rowptr, col, seed, 0, color);
}

int orc_color_valid(int64_t n, const int64_t* rowptr, const int32_t* col, const int32_t* color,
                    int32_t ncolors) {
  for (int64_t v = 0; v < n; v++) {
    if (color[v] < 0 || color[v] >= ncolors) return 0;
    for (int64_t e = rowptr[v]; e < rowptr[v + 1]; e++)
      if (col[e] != v && color[col[e]] == color[v]) return 0;
  }
  return 1;
}

/* ---------------- TD / TH ---------------------- */
/* BFS order from the root over the children lists built from parent[]. */
static int32_t* bfs_order(int64_t n, const int32_t* parent) {
  int64_t* cs = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int32_t* cl = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  int32_t* q = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  if (!cs || !cl || !q) {
    free(cs), free(cl), free(q);
    return NULL;
  }
  int32_t root = -1;
  for (int64_t v = 0; v < n; v++) {
    if (parent[v] < 0) root = (int32_t)v;
    else cs[parent[v] + 1]++;
  }
  for (int64_t v = 0; v < n; v++) cs[v + 1] += cs[v];
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  if (!cur || root < 0) {
    free(cs), free(cl), free(q), free(cur);
    return NULL;
  }
  memcpy(cur, cs, sizeof(int64_t) * (size_t)n);
  for (int64_t v = 0; v < n; v++)
    if (parent[v] >= 0) cl[cur[parent[v]]++] = (int32_t)v;
  int64_t head = 0, tail = 0;
  q[tail++] = root;
  while (head < tail) {
    int32_t v = q[head++];
    for (int64_t k = cs[v]; k < cs[v + 1]; k++) q[tail++] = cl[k];
  }
  free(cs), free(cl), free(cur);
  return q;
}

int orc_tree_desc(int64_t n, const int32_t* parent, int32_t* desc) {
  int32_t* q = bfs_order(n, parent);
  if (!q) return -1;
  for (int64_t v = 0; v < n; v++) desc[v] = 0;
  for (int64_t i = n - 1; i > 0; i--) {
    int32_t v = q[i];
    desc[parent[v]] += desc[v] + 1;
  }
  free(q);
  return 0;
}

int orc_tree_height(int64_t n, const int32_t* parent, int32_t* height) {
  int32_t* q = bfs_order(n, parent);
  if (!q) return -1;
  for (int64_t v = 0; v < n; v++) height[v] = 0;
  for (int64_t i = n - 1; i > 0; i--) {
    int32_t v = q[i];
    if (height[v] + 1 > height[parent[v]]) height[parent[v]] = height[v] + 1;
  }
  free(q);
  return 0;
}

/* BFS levels ("BFS-Rec = BFS levels"): hops from source by a
 * FIFO sweep; UINT32_MAX = unreachable. */
int orc_bfs(int64_t n, const int64_t* rowptr, const int32_t* col, int32_t source, uint32_t* level) {
  for (int64_t i = 0; i < n; i++) level[i] = UINT32_MAX;
  if (source < 0 || source >= n) return -1;
  int32_t* q = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  if (!q) return -1;
  int64_t head = 0, tail = 0;
  level[source] = 0;
  q[tail++] = source;
  while (head < tail) {
    int32_t u = q[head++];
    for (int64_t e = rowptr[u]; e < rowptr[u + 1]; e++) {
      int32_t v = col[e];
      if (level[v] == UINT32_MAX) {
        level[v] = level[u] + 1;
        q[tail++] = v;
      }
    }
  }
  free(q);
  return 0;
}

/* PageRank, SPEC.md:454 ("PR = one-or-more power iterations with damping
 * 0.85") with the fixed iteration count of SPEC.md:468: r0 = 1/n,
 * r'[v] = (1-d)/n + d (sum_{u->v} r[u]/outdeg(u) + D/n), D = dangling mass.
 * fp64, push order over the CSR. */
int orc_pagerank(int64_t n, const int64_t* rowptr, const int32_t* col, int32_t iters, double d,
                 double* rank) {
  if (n <= 0) return 0;
  double* nxt = (double*)malloc(sizeof(double) * (size_t)n);
  if (!nxt) return -1;
  for (int64_t v = 0; v < n; v++) rank[v] = 1.0 / (double)n;
  for (int32_t it = 0; it < iters; it++) {
    double dm = 0.0;
    for (int64_t v = 0; v < n; v++) nxt[v] = 0.0;
    for (int64_t u = 0; u < n; u++) {
      const int64_t deg = rowptr[u + 1] - rowptr[u];
      if (deg == 0) { dm += rank[u]; continue; }
      const double c = rank[u] / (double)deg;
      for (int64_t e = rowptr[u]; e < rowptr[u + 1]; e++) nxt[col[e]] += c;
    }
    for (int64_t v = 0; v < n; v++) rank[v] = (1.0 - d) / (double)n + d * (nxt[v] + dm / (double)n);
  }
  free(nxt);
  return 0;
}

/* ---------------- R-MAT generator --------------------- */
/* Independent restatement of the synthetic R-MAT graph the product generates
 * ("R-MAT (a,b,c,d); duplicates and self loops kept"), drawn from
 * the same counter hash so both sides produce the same graph: arc e descends
 * `scale` quadrant levels, each consuming 16 bits of
 * mix64(mix64(seed ^ STREAM_RMAT) ^ (e*8 + level/4)); a level picks the
 * source bit (u >= a+b) and the destination bit (a <= u < a+b or u >= a+b+c)
 * with the probabilities quantised to 1/65536.  Optional vertex permutation
 * (Fisher-Yates from the top, j = draw(PERM, i) mod (i+1)).  Rows list their
 * arcs in (dst, arc id) order; weights = wmin + draw(WEIGHT, e) mod range,
 * values = ((draw(VALUE, e) >> 40) + 1) / 2^24.  Directed only.  Used by the
 * reference arm of bench.py so that leg builds its input without libdpc.so,
 * and by tests/test_oracle.py to check the product generator. */
#define ORC_STREAM_RMAT 0x1000000000000000ull
#define ORC_STREAM_WEIGHT 0x2000000000000000ull
#define ORC_STREAM_VALUE 0x3000000000000000ull
#define ORC_STREAM_PERM 0x4000000000000000ull

static inline uint64_t orc_draw(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return orc_mix64(orc_mix64(seed ^ stream) ^ ctr);
}

static int key_cmp(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

int orc_gen_rmat(int scale, int edgefactor, double a, double b, double c, int32_t wmin, int32_t wmax,
                 uint64_t seed, int permute, int64_t* rowptr, int32_t* col, int32_t* w, float* val) {
  const int64_t n = (int64_t)1 << scale, m = n * edgefactor;
  const uint32_t ta = (uint32_t)llround(a * 65536.0), tb = (uint32_t)llround((a + b) * 65536.0),
                 tc = (uint32_t)llround((a + b + c) * 65536.0);
  uint32_t* perm = NULL;
  uint32_t* src = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(m ? m : 1));
  uint64_t* key = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(m ? m : 1));
  if (!src || !key) goto oom;
  if (permute) {
    perm = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
    if (!perm) goto oom;
    for (int64_t i = 0; i < n; i++) perm[i] = (uint32_t)i;
    for (int64_t i = n - 1; i > 0; i--) {
      uint64_t j = orc_draw(seed, ORC_STREAM_PERM, (uint64_t)i) % (uint64_t)(i + 1);
      uint32_t t = perm[i];
      perm[i] = perm[j], perm[j] = t;
    }
  }
  for (int64_t i = 0; i <= n; i++) rowptr[i] = 0;
  for (int64_t e = 0; e < m; e++) {
    uint32_t s = 0, d = 0;
    uint64_t h = 0;
    for (int lv = 0; lv < scale; lv++) {
      if ((lv & 3) == 0) h = orc_draw(seed, ORC_STREAM_RMAT, (uint64_t)e * 8 + (uint64_t)(lv / 4));
      uint32_t u = (uint32_t)(h >> (16 * (lv & 3))) & 0xffffu;
      s = (s << 1) | (u >= tb);
      d = (d << 1) | ((u >= ta && u < tb) || u >= tc);
    }
    if (perm) s = perm[s], d = perm[d];
    src[e] = s;
    key[e] = ((uint64_t)d << 32) | (uint64_t)e;
    rowptr[s + 1]++;
  }
  for (int64_t i = 0; i < n; i++) rowptr[i + 1] += rowptr[i];
  {
    /* counting sort by source, then each row by (dst, arc id) */
    int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    uint64_t* sorted = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(m ? m : 1));
    if (!cur || !sorted) {
      free(cur), free(sorted);
      goto oom;
    }
    memcpy(cur, rowptr, sizeof(int64_t) * (size_t)n);
    for (int64_t e = 0; e < m; e++) sorted[cur[src[e]]++] = key[e];
    for (int64_t i = 0; i < n; i++)
      qsort(sorted + rowptr[i], (size_t)(rowptr[i + 1] - rowptr[i]), sizeof(uint64_t), key_cmp);
    const uint64_t wr = (uint64_t)((int64_t)wmax - wmin + 1);
    for (int64_t p = 0; p < m; p++) {
      uint64_t e = sorted[p] & 0xffffffffull;
      col[p] = (int32_t)(sorted[p] >> 32);
      if (w) w[p] = wmin + (int32_t)(orc_draw(seed, ORC_STREAM_WEIGHT, e) % wr);
      if (val) val[p] = (float)((orc_draw(seed, ORC_STREAM_VALUE, e) >> 40) + 1) * (1.0f / 16777216.0f);
    }
    free(cur), free(sorted);
  }
  free(perm), free(src), free(key);
  return 0;
oom:
  free(perm), free(src), free(key);
  return -1;
}
