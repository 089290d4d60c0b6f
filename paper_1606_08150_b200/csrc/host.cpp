// Host side of libdpc.so: error slot, CSR / tree containers, synthetic
// generators and file I/O.  This is the data layer the reference specifies
// but does not ship (module `workloads`): CsrGraph, Tree,
// gen_graph, gen_tree, load_csr, save_csr.
//
// All generators draw from a counter-based hash (dpc::mix64), so outputs are a
// pure function of the arguments, independent of the host thread count
// (SPEC.md:431 / :441 "fixed seed -> identical ... across runs and platforms").
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "dpc_internal.h"

namespace dpc {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
void clear_error() { g_last_error.clear(); }
dpc_status fail(dpc_status st, const std::string& msg) {
  set_error(msg);
  return st;
}

int host_threads() {
  static int n = [] {
    const char* e = std::getenv("DPC_HOST_THREADS");
    if (e && std::atoi(e) > 0) return std::atoi(e);
    unsigned h = std::thread::hardware_concurrency();
    return h == 0 ? 1 : static_cast<int>(std::min(h, 64u));
  }();
  return n;
}

// Runs f(lo, hi) over [0, n) split into contiguous ranges, one per thread.
static void parallel_for(int64_t n, const std::function<void(int64_t, int64_t)>& f) {
  int t = host_threads();
  if (n < 1 << 16 || t <= 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  int64_t per = (n + t - 1) / t;
  for (int i = 0; i < t; i++) {
    int64_t lo = i * per, hi = std::min<int64_t>(n, lo + per);
    if (lo >= hi) break;
    th.emplace_back([=, &f] { f(lo, hi); });
  }
  for (auto& x : th) x.join();
}

template <class T>
static T* xalloc(int64_t count) {
  if (count <= 0) count = 1;
  T* p = static_cast<T*>(std::malloc(sizeof(T) * static_cast<size_t>(count)));
  if (!p) throw std::bad_alloc();
  return p;
}

static dpc_csr* new_csr() {
  auto* g = static_cast<dpc_csr*>(std::calloc(1, sizeof(dpc_csr)));
  if (!g) throw std::bad_alloc();
  return g;
}

static dpc_tree* new_tree() {
  auto* t = static_cast<dpc_tree*>(std::calloc(1, sizeof(dpc_tree)));
  if (!t) throw std::bad_alloc();
  return t;
}

// Generic edge-list -> CSR builder.  edge(e, &src, &dst) yields arc e.
// Row entries are ordered by (dst, arc id): deterministic for any thread
// count.  With symmetric, arc e contributes (s,d) and (d,s); self loops and
// duplicate (row, col) pairs are dropped keeping the smallest arc id, so both
// directions of an undirected pair share one weight.
struct EdgeSrc {
  int64_t n;
  int64_t m;
  std::function<void(int64_t, uint32_t*, uint32_t*)> edge;
};

// Rows [r0, r1) only (r1 < 0: all rows); a slice keeps global column ids.
static dpc_csr* build_csr(const EdgeSrc& es, int32_t wmin, int32_t wmax, uint64_t seed,
                          uint32_t flags, int64_t r0 = 0, int64_t r1 = -1) {
  if (r1 < 0) r1 = es.n;
  const int64_t n = r1 - r0;
  const uint32_t lo32 = static_cast<uint32_t>(r0), hi32 = static_cast<uint32_t>(r1);
  auto in_slice = [&](uint32_t s) { return s >= lo32 && s < hi32; };
  const bool sym = flags & DPC_GEN_SYMMETRIC;
  const int64_t arcs = sym ? 2 * es.m : es.m;
  std::vector<uint32_t> src(static_cast<size_t>(arcs)), dst(static_cast<size_t>(arcs));
  parallel_for(es.m, [&](int64_t lo, int64_t hi) {
    for (int64_t e = lo; e < hi; e++) {
      uint32_t s, d;
      es.edge(e, &s, &d);
      if (sym) {
        src[2 * e] = s, dst[2 * e] = d;
        src[2 * e + 1] = d, dst[2 * e + 1] = s;
      } else {
        src[e] = s, dst[e] = d;
      }
    }
  });
  // degree count
  std::vector<int64_t> rowptr(static_cast<size_t>(n + 1), 0);
  {
    std::vector<std::atomic<uint32_t>> deg(static_cast<size_t>(n));
    parallel_for(n, [&](int64_t lo, int64_t hi) {
      for (int64_t i = lo; i < hi; i++) deg[i].store(0, std::memory_order_relaxed);
    });
    parallel_for(arcs, [&](int64_t lo, int64_t hi) {
      for (int64_t e = lo; e < hi; e++) {
        if ((sym && src[e] == dst[e]) || !in_slice(src[e])) continue;
        deg[src[e] - lo32].fetch_add(1, std::memory_order_relaxed);
      }
    });
    for (int64_t i = 0; i < n; i++) rowptr[i + 1] = rowptr[i] + deg[i].load();
  }
  int64_t m1 = rowptr[n];
  std::vector<uint64_t> keys(static_cast<size_t>(std::max<int64_t>(m1, 1)));
  {
    std::vector<std::atomic<int64_t>> cur(static_cast<size_t>(n));
    parallel_for(n, [&](int64_t lo, int64_t hi) {
      for (int64_t i = lo; i < hi; i++) cur[i].store(rowptr[i], std::memory_order_relaxed);
    });
    parallel_for(arcs, [&](int64_t lo, int64_t hi) {
      for (int64_t e = lo; e < hi; e++) {
        if ((sym && src[e] == dst[e]) || !in_slice(src[e])) continue;
        int64_t p = cur[src[e] - lo32].fetch_add(1, std::memory_order_relaxed);
        keys[p] = (static_cast<uint64_t>(dst[e]) << 32) | static_cast<uint64_t>(e);
      }
    });
  }
  std::vector<uint32_t>().swap(src);
  std::vector<uint32_t>().swap(dst);
  // sort each row, then (symmetric) drop duplicates
  std::vector<int64_t> newdeg(static_cast<size_t>(n), 0);
  parallel_for(n, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; i++) {
      uint64_t* b = keys.data() + rowptr[i];
      uint64_t* e = keys.data() + rowptr[i + 1];
      std::sort(b, e);
      if (sym) {
        int64_t k = 0;
        for (uint64_t* p = b; p < e; p++)
          if (k == 0 || (b[k - 1] >> 32) != (*p >> 32)) b[k++] = *p;
        newdeg[i] = k;
      } else {
        newdeg[i] = e - b;
      }
    }
  });
  dpc_csr* g = new_csr();
  g->n = n;
  if (n != es.n) g->ncols = es.n;
  g->rowptr = xalloc<int64_t>(n + 1);
  g->rowptr[0] = 0;
  for (int64_t i = 0; i < n; i++) g->rowptr[i + 1] = g->rowptr[i] + newdeg[i];
  g->m = g->rowptr[n];
  g->col = xalloc<int32_t>(g->m);
  const bool wts = flags & DPC_GEN_WEIGHTS, vals = flags & DPC_GEN_VALUES;
  if (wts) g->w = xalloc<int32_t>(g->m);
  if (vals) g->val = xalloc<float>(g->m);
  const uint64_t wr = static_cast<uint64_t>(static_cast<int64_t>(wmax) - wmin + 1);
  parallel_for(n, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; i++) {
      const uint64_t* kb = keys.data() + rowptr[i];
      int64_t o = g->rowptr[i];
      for (int64_t j = 0; j < newdeg[i]; j++) {
        uint64_t key = kb[j];
        uint64_t arc = key & 0xffffffffull;
        uint64_t eid = sym ? (arc >> 1) : arc;
        g->col[o + j] = static_cast<int32_t>(key >> 32);
        if (wts) g->w[o + j] = wmin + static_cast<int32_t>(draw(seed, kStreamWeight, eid) % wr);
        if (vals) g->val[o + j] = unit_value(draw(seed, kStreamValue, eid));
      }
    }
  });
  return g;
}

static std::vector<uint32_t> random_permutation(int64_t n, uint64_t seed) {
  std::vector<uint32_t> p(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; i++) p[i] = static_cast<uint32_t>(i);
  for (int64_t i = n - 1; i > 0; i--) {
    uint64_t j = draw(seed, kStreamPerm, static_cast<uint64_t>(i)) % static_cast<uint64_t>(i + 1);
    std::swap(p[i], p[j]);
  }
  return p;
}

}  // namespace dpc

using namespace dpc;

#define DPC_TRY_BEGIN \
  clear_error();      \
  try {
#define DPC_TRY_END                                                  \
  }                                                                  \
  catch (const std::bad_alloc&) {                                    \
    return fail(DPC_E_OOM, "host allocation failed");                \
  }                                                                  \
  catch (const std::exception& ex) {                                 \
    return fail(DPC_E_INVALID, std::string("exception: ") + ex.what()); \
  }

extern "C" {

const char* dpc_last_error(void) { return g_last_error.c_str(); }
int dpc_abi_version(void) { return DPC_ABI_VERSION; }

dpc_status dpc_gen_rmat_rows(int scale, int edgefactor, double a, double b, double c,
                             int32_t wmin, int32_t wmax, uint64_t seed, uint32_t flags, int64_t r0,
                             int64_t r1, dpc_csr** out) {
  DPC_TRY_BEGIN
  if (!out) return fail(DPC_E_INVALID, "out is NULL");
  if (scale < 1 || scale > 31) return fail(DPC_E_INVALID, "scale must be in [1, 31]");
  if (edgefactor < 0) return fail(DPC_E_INVALID, "edgefactor must be >= 0");
  if (a < 0 || b < 0 || c < 0 || a + b + c > 1.0)
    return fail(DPC_E_INVALID, "R-MAT probabilities must be >= 0 with a+b+c <= 1");
  if ((flags & DPC_GEN_WEIGHTS) && (wmin < 0 || wmax < wmin))
    return fail(DPC_E_INVALID, "weights need 0 <= wmin <= wmax");
  const int64_t n = int64_t{1} << scale;
  const int64_t m = n * edgefactor;
  if (m >= (int64_t{1} << 32) || (flags & DPC_GEN_SYMMETRIC && 2 * m >= (int64_t{1} << 32)))
    return fail(DPC_E_INVALID, "arc count must stay below 2^32");
  const uint32_t ta = static_cast<uint32_t>(std::lround(a * 65536.0));
  const uint32_t tb = static_cast<uint32_t>(std::lround((a + b) * 65536.0));
  const uint32_t tc = static_cast<uint32_t>(std::lround((a + b + c) * 65536.0));
  std::vector<uint32_t> perm;
  if (flags & DPC_GEN_PERMUTE) perm = random_permutation(n, seed);
  EdgeSrc es{n, m, nullptr};
  es.edge = [&](int64_t e, uint32_t* s, uint32_t* d) {
    uint32_t si = 0, di = 0;
    uint64_t h = 0;
    for (int lv = 0; lv < scale; lv++) {
      if ((lv & 3) == 0) h = draw(seed, kStreamRmat, static_cast<uint64_t>(e) * 8 + lv / 4);
      uint32_t u = static_cast<uint32_t>(h >> (16 * (lv & 3))) & 0xffffu;
      uint32_t sb = u >= tb, db = (u >= ta && u < tb) || u >= tc;
      si = (si << 1) | sb;
      di = (di << 1) | db;
    }
    if (!perm.empty()) si = perm[si], di = perm[di];
    *s = si;
    *d = di;
  };
  if (r1 < 0) r1 = n;
  if (r0 < 0 || r0 > r1 || r1 > n) return fail(DPC_E_INVALID, "row slice out of range");
  if ((flags & DPC_GEN_SYMMETRIC) && (r0 != 0 || r1 != n))
    return fail(DPC_E_INVALID, "row slices of symmetrized graphs are not supported");
  *out = build_csr(es, wmin, wmax, seed, flags, r0, r1);
  return DPC_OK;
  DPC_TRY_END
}

dpc_status dpc_gen_rmat(int scale, int edgefactor, double a, double b, double c, int32_t wmin,
                        int32_t wmax, uint64_t seed, uint32_t flags, dpc_csr** out) {
  return dpc_gen_rmat_rows(scale, edgefactor, a, b, c, wmin, wmax, seed, flags, 0, -1, out);
}

dpc_status dpc_gen_graph_uniform(int64_t n, int32_t dmin, int32_t dmax, int32_t wmin, int32_t wmax,
                                 uint64_t seed, uint32_t flags, dpc_csr** out) {
  DPC_TRY_BEGIN
  if (!out) return fail(DPC_E_INVALID, "out is NULL");
  if (n < 1 || n >= (int64_t{1} << 31)) return fail(DPC_E_INVALID, "nodeCount must be in [1, 2^31)");
  if (dmin < 0 || dmax < dmin) return fail(DPC_E_INVALID, "uniform degrees need 0 <= min <= max");
  if ((flags & DPC_GEN_WEIGHTS) && (wmin < 0 || wmax < wmin))
    return fail(DPC_E_INVALID, "weights need 0 <= wmin <= wmax");
  std::vector<int64_t> off(static_cast<size_t>(n + 1), 0);
  const uint64_t r = static_cast<uint64_t>(dmax - dmin + 1);
  for (int64_t v = 0; v < n; v++)
    off[v + 1] = off[v] + dmin + static_cast<int64_t>(draw(seed, kStreamDegree, v) % r);
  const int64_t m = off[n];
  if (m >= (int64_t{1} << 31)) return fail(DPC_E_INVALID, "too many edges");
  std::vector<uint32_t> srcs(static_cast<size_t>(std::max<int64_t>(m, 1)));
  for (int64_t v = 0; v < n; v++)
    for (int64_t k = off[v]; k < off[v + 1]; k++) srcs[k] = static_cast<uint32_t>(v);
  EdgeSrc es{n, m, nullptr};
  es.edge = [&](int64_t e, uint32_t* s, uint32_t* d) {
    *s = srcs[e];
    *d = static_cast<uint32_t>(draw(seed, kStreamNbr, e) % static_cast<uint64_t>(n));
  };
  *out = build_csr(es, wmin, wmax, seed, flags);
  return DPC_OK;
  DPC_TRY_END
}

dpc_status dpc_gen_graph_powerlaw(int64_t n, double alpha, int32_t maxdeg, int32_t wmin,
                                  int32_t wmax, uint64_t seed, uint32_t flags, dpc_csr** out) {
  DPC_TRY_BEGIN
  if (!out) return fail(DPC_E_INVALID, "out is NULL");
  if (n < 1 || n >= (int64_t{1} << 31)) return fail(DPC_E_INVALID, "nodeCount must be in [1, 2^31)");
  if (!(alpha > 0) || maxdeg < 1) return fail(DPC_E_INVALID, "powerlaw needs alpha > 0, maxDeg >= 1");
  if ((flags & DPC_GEN_WEIGHTS) && (wmin < 0 || wmax < wmin))
    return fail(DPC_E_INVALID, "weights need 0 <= wmin <= wmax");
  // P(d) ~ d^-alpha on [1, maxdeg]; inverse CDF on a 53-bit uniform.
  std::vector<double> cdf(static_cast<size_t>(maxdeg));
  double acc = 0;
  for (int32_t d = 1; d <= maxdeg; d++) acc += std::pow(static_cast<double>(d), -alpha), cdf[d - 1] = acc;
  for (auto& x : cdf) x /= acc;
  std::vector<int64_t> off(static_cast<size_t>(n + 1), 0);
  for (int64_t v = 0; v < n; v++) {
    double u = static_cast<double>(draw(seed, kStreamDegree, v) >> 11) * (1.0 / 9007199254740992.0);
    int64_t d = std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin() + 1;
    off[v + 1] = off[v] + std::min<int64_t>(d, maxdeg);
  }
  const int64_t m = off[n];
  if (m >= (int64_t{1} << 31)) return fail(DPC_E_INVALID, "too many edges");
  std::vector<uint32_t> srcs(static_cast<size_t>(std::max<int64_t>(m, 1)));
  for (int64_t v = 0; v < n; v++)
    for (int64_t k = off[v]; k < off[v + 1]; k++) srcs[k] = static_cast<uint32_t>(v);
  EdgeSrc es{n, m, nullptr};
  es.edge = [&](int64_t e, uint32_t* s, uint32_t* d) {
    *s = srcs[e];
    *d = static_cast<uint32_t>(draw(seed, kStreamNbr, e) % static_cast<uint64_t>(n));
  };
  *out = build_csr(es, wmin, wmax, seed, flags);
  return DPC_OK;
  DPC_TRY_END
}

dpc_status dpc_csr_validate(const dpc_csr* g) {
  clear_error();
  if (!g) return fail(DPC_E_INVALID, "graph is NULL");
  if (g->n < 0 || g->m < 0) return fail(DPC_E_INVALID, "negative sizes");
  if (g->n >= (int64_t{1} << 31)) return fail(DPC_E_INVALID, "nodeCount must be < 2^31");
  if (!g->rowptr) return fail(DPC_E_INVALID, "rowptr is NULL");
  if (g->m > 0 && !g->col) return fail(DPC_E_INVALID, "col is NULL");
  if (g->rowptr[0] != 0) return fail(DPC_E_INVALID, "rowOffsets[0] must be 0");
  for (int64_t i = 0; i < g->n; i++)
    if (g->rowptr[i + 1] < g->rowptr[i])
      return fail(DPC_E_INVALID, "rowOffsets must be nondecreasing (row " + std::to_string(i) + ")");
  if (g->rowptr[g->n] != g->m) return fail(DPC_E_INVALID, "rowOffsets[nodeCount] must equal edgeCount");
  if (g->ncols < 0 || g->ncols >= (int64_t{1} << 31)) return fail(DPC_E_INVALID, "bad column count");
  const int64_t nc = g->ncols ? g->ncols : g->n;
  for (int64_t k = 0; k < g->m; k++)
    if (g->col[k] < 0 || g->col[k] >= nc)
      return fail(DPC_E_INVALID, "column index out of range at " + std::to_string(k));
  return DPC_OK;
}

static dpc_status make_csr(int64_t n, int64_t ncols, int64_t m, const int64_t* rowptr, const int32_t* col,
                           const int32_t* w, const float* val, dpc_csr** out) {
  if (!out) return fail(DPC_E_INVALID, "out is NULL");
  dpc_csr tmp{n, m, const_cast<int64_t*>(rowptr), const_cast<int32_t*>(col), nullptr, nullptr, ncols};
  dpc_status st = dpc_csr_validate(&tmp);
  if (st != DPC_OK) return st;
  std::unique_ptr<dpc_csr, void (*)(dpc_csr*)> g(new_csr(), dpc_csr_free);
  g->n = n;
  g->m = m;
  g->ncols = ncols;
  g->rowptr = xalloc<int64_t>(n + 1);
  std::memcpy(g->rowptr, rowptr, sizeof(int64_t) * (n + 1));
  g->col = xalloc<int32_t>(m);
  if (m) std::memcpy(g->col, col, sizeof(int32_t) * m);
  if (w) {
    g->w = xalloc<int32_t>(m);
    if (m) std::memcpy(g->w, w, sizeof(int32_t) * m);
  }
  if (val) {
    g->val = xalloc<float>(m);
    if (m) std::memcpy(g->val, val, sizeof(float) * m);
  }
  *out = g.release();
  return DPC_OK;
}

dpc_status dpc_csr_create(int64_t n, int64_t m, const int64_t* rowptr, const int32_t* col,
                          const int32_t* w, const float* val, dpc_csr** out) {
  DPC_TRY_BEGIN
  return make_csr(n, 0, m, rowptr, col, w, val, out);
  DPC_TRY_END
}

dpc_status dpc_csr_create_rows(int64_t n, int64_t ncols, int64_t m, const int64_t* rowptr, const int32_t* col,
                               const int32_t* w, const float* val, dpc_csr** out) {
  DPC_TRY_BEGIN
  if (ncols <= 0) return fail(DPC_E_INVALID, "a row slice needs ncols > 0");
  return make_csr(n, ncols, m, rowptr, col, w, val, out);
  DPC_TRY_END
}

void dpc_csr_free(dpc_csr* g) {
  if (!g) return;
  std::free(g->rowptr);
  std::free(g->col);
  std::free(g->w);
  std::free(g->val);
  std::free(g);
}

// Builds cstart/clist/depth from parent[]; validates one root, acyclic.
static dpc_status finish_tree(dpc_tree* t) {
  const int64_t n = t->n;
  int64_t roots = 0;
  t->root = -1;
  for (int64_t v = 0; v < n; v++) {
    int32_t p = t->parent[v];
    if (p == -1) {
      roots++;
      t->root = static_cast<int32_t>(v);
    } else if (p < 0 || p >= n || p == v) {
      return fail(DPC_E_INVALID, "parent index out of range at node " + std::to_string(v));
    }
  }
  if (roots != 1) return fail(DPC_E_INVALID, "tree must have exactly one root (parent = -1)");
  t->cstart = xalloc<int64_t>(n + 1);
  t->clist = xalloc<int32_t>(n);
  std::fill(t->cstart, t->cstart + n + 1, 0);
  for (int64_t v = 0; v < n; v++)
    if (t->parent[v] >= 0) t->cstart[t->parent[v] + 1]++;
  for (int64_t v = 0; v < n; v++) t->cstart[v + 1] += t->cstart[v];
  std::vector<int64_t> cur(t->cstart, t->cstart + n);
  for (int64_t v = 0; v < n; v++)
    if (t->parent[v] >= 0) t->clist[cur[t->parent[v]]++] = static_cast<int32_t>(v);
  // BFS from the root: every node reached exactly once <=> acyclic
  std::vector<int32_t> q;
  q.reserve(static_cast<size_t>(n));
  q.push_back(t->root);
  int32_t depth = 0;
  size_t lo = 0;
  while (lo < q.size()) {
    size_t hi = q.size();
    depth++;
    for (size_t i = lo; i < hi; i++) {
      int32_t v = q[i];
      for (int64_t k = t->cstart[v]; k < t->cstart[v + 1]; k++) q.push_back(t->clist[k]);
    }
    lo = hi;
    if (static_cast<int64_t>(q.size()) > n) break;
  }
  if (static_cast<int64_t>(q.size()) != n) return fail(DPC_E_INVALID, "parent array contains a cycle");
  t->depth = depth;
  return DPC_OK;
}

dpc_status dpc_tree_create(int64_t n, const int32_t* parent, dpc_tree** out) {
  DPC_TRY_BEGIN
  if (!out || !parent) return fail(DPC_E_INVALID, "NULL argument");
  if (n < 1 || n >= (int64_t{1} << 31)) return fail(DPC_E_INVALID, "nodeCount must be in [1, 2^31)");
  std::unique_ptr<dpc_tree, void (*)(dpc_tree*)> t(new_tree(), dpc_tree_free);
  t->n = n;
  t->parent = xalloc<int32_t>(n);
  std::memcpy(t->parent, parent, sizeof(int32_t) * n);
  dpc_status st = finish_tree(t.get());
  if (st != DPC_OK) return st;
  *out = t.release();
  return DPC_OK;
  DPC_TRY_END
}

void dpc_tree_free(dpc_tree* t) {
  if (!t) return;
  std::free(t->parent);
  std::free(t->cstart);
  std::free(t->clist);
  std::free(t);
}

// SPEC.md:425-433.  Level L (0-based) expands k = floor(fill * |level|)
// candidates (at least one while fill > 0, so the tree has exactly `depth`
// levels), chosen by ascending (hash(id), id); each expanding node draws its
// child count uniformly in [min, max] (the first expanding node of a level
// gets at least one child).  Children are numbered level by level in parent
// id order, so ids are a BFS order.
dpc_status dpc_gen_tree(int32_t depth, int32_t minc, int32_t maxc, double fill, uint64_t seed,
                        dpc_tree** out) {
  DPC_TRY_BEGIN
  if (!out) return fail(DPC_E_INVALID, "out is NULL");
  if (depth < 1) return fail(DPC_E_INVALID, "depth must be >= 1");
  if (minc < 0 || maxc < minc) return fail(DPC_E_INVALID, "children need 0 <= min <= max");
  if (!(fill >= 0.0 && fill <= 1.0)) return fail(DPC_E_INVALID, "fill fraction must be in [0, 1]");
  std::vector<int32_t> parent{-1};
  int64_t lo = 0, hi = 1;  // current level id range
  const uint64_t r = static_cast<uint64_t>(maxc - minc + 1);
  for (int32_t lv = 0; lv + 1 < depth && maxc > 0; lv++) {
    int64_t cnt = hi - lo;
    int64_t k = static_cast<int64_t>(std::floor(fill * static_cast<double>(cnt)));
    if (k == 0 && fill > 0.0) k = 1;
    if (k == 0) break;
    std::vector<uint64_t> sel;
    if (k < cnt) {
      std::vector<std::pair<uint64_t, int64_t>> key(static_cast<size_t>(cnt));
      for (int64_t i = 0; i < cnt; i++) key[i] = {draw(seed, kStreamTreeSel, lo + i), lo + i};
      std::nth_element(key.begin(), key.begin() + k, key.end());
      sel.resize(static_cast<size_t>(k));
      for (int64_t i = 0; i < k; i++) sel[i] = static_cast<uint64_t>(key[i].second);
      std::sort(sel.begin(), sel.end());
    } else {
      for (int64_t i = lo; i < hi; i++) sel.push_back(static_cast<uint64_t>(i));
    }
    int64_t next_lo = static_cast<int64_t>(parent.size());
    bool first = true;
    for (uint64_t p : sel) {
      int64_t c = minc + static_cast<int64_t>(draw(seed, kStreamTree, p) % r);
      if (first && c == 0) c = 1;
      first = false;
      if (static_cast<int64_t>(parent.size()) + c >= (int64_t{1} << 31) - 1)
        return fail(DPC_E_INVALID, "tree exceeds 2^31 nodes");
      for (int64_t j = 0; j < c; j++) parent.push_back(static_cast<int32_t>(p));
    }
    lo = next_lo;
    hi = static_cast<int64_t>(parent.size());
    if (lo == hi) break;
  }
  std::unique_ptr<dpc_tree, void (*)(dpc_tree*)> t(new_tree(), dpc_tree_free);
  t->n = static_cast<int64_t>(parent.size());
  t->parent = xalloc<int32_t>(t->n);
  std::memcpy(t->parent, parent.data(), sizeof(int32_t) * t->n);
  dpc_status st = finish_tree(t.get());
  if (st != DPC_OK) return st;
  *out = t.release();
  return DPC_OK;
  DPC_TRY_END
}

// ---------------- file I/O ----------------

static bool ends_with(const std::string& s, const char* suf) {
  size_t k = std::strlen(suf);
  return s.size() >= k && s.compare(s.size() - k, k, suf) == 0;
}

// Minimal fast whitespace tokenizer over a whole file.
struct TextReader {
  std::string buf;
  size_t pos = 0;
  bool load(const char* path) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return false;
    std::fseek(f, 0, SEEK_END);
    long sz = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    buf.resize(sz > 0 ? static_cast<size_t>(sz) : 0);
    size_t rd = sz > 0 ? std::fread(&buf[0], 1, buf.size(), f) : 0;
    std::fclose(f);
    return rd == buf.size();
  }
  // next line as [b, e); returns false at EOF
  bool line(size_t* b, size_t* e) {
    if (pos >= buf.size()) return false;
    *b = pos;
    size_t nl = buf.find('\n', pos);
    if (nl == std::string::npos) nl = buf.size();
    *e = nl;
    pos = nl + 1;
    return true;
  }
  // parses integers in [b, e) into out; returns count or -1 on junk
  int64_t ints(size_t b, size_t e, std::vector<int64_t>& out) {
    const char* p = buf.data() + b;
    const char* end = buf.data() + e;
    int64_t cnt = 0;
    while (p < end) {
      while (p < end && (*p == ' ' || *p == '\t' || *p == '\r')) p++;
      if (p >= end) break;
      bool neg = false;
      if (*p == '-') neg = true, p++;
      if (p >= end || *p < '0' || *p > '9') return -1;
      int64_t v = 0;
      while (p < end && *p >= '0' && *p <= '9') {
        if (v > (INT64_MAX - 9) / 10) return -1;
        v = v * 10 + (*p++ - '0');
      }
      out.push_back(neg ? -v : v);
      cnt++;
    }
    return cnt;
  }
};

dpc_status dpc_load_csr(const char* path, dpc_csr** out) {
  DPC_TRY_BEGIN
  if (!path || !out) return fail(DPC_E_INVALID, "NULL argument");
  std::string p(path);
  if (ends_with(p, ".bin")) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return fail(DPC_E_IO, "cannot open " + p);
    char magic[8];
    int64_t hdr[3];
    bool ok = std::fread(magic, 1, 8, f) == 8 && std::memcmp(magic, "DPCCSR01", 8) == 0 &&
              std::fread(hdr, sizeof(int64_t), 3, f) == 3;
    if (!ok || hdr[0] < 0 || hdr[1] < 0) {
      std::fclose(f);
      return fail(DPC_E_IO, "bad binary CSR header in " + p);
    }
    std::unique_ptr<dpc_csr, void (*)(dpc_csr*)> g(new_csr(), dpc_csr_free);
    g->n = hdr[0];
    g->m = hdr[1];
    g->rowptr = xalloc<int64_t>(g->n + 1);
    g->col = xalloc<int32_t>(g->m);
    ok = std::fread(g->rowptr, sizeof(int64_t), g->n + 1, f) == static_cast<size_t>(g->n + 1) &&
         std::fread(g->col, sizeof(int32_t), g->m, f) == static_cast<size_t>(g->m);
    if (ok && (hdr[2] & 1)) {
      g->w = xalloc<int32_t>(g->m);
      ok = std::fread(g->w, sizeof(int32_t), g->m, f) == static_cast<size_t>(g->m);
    }
    if (ok && (hdr[2] & 2)) {
      g->val = xalloc<float>(g->m);
      ok = std::fread(g->val, sizeof(float), g->m, f) == static_cast<size_t>(g->m);
    }
    std::fclose(f);
    if (!ok) return fail(DPC_E_IO, "truncated binary CSR " + p);
    dpc_status st = dpc_csr_validate(g.get());
    if (st != DPC_OK) return fail(DPC_E_IO, std::string("invalid CSR in file: ") + dpc_last_error());
    *out = g.release();
    return DPC_OK;
  }
  TextReader r;
  if (!r.load(path)) return fail(DPC_E_IO, "cannot read " + p);
  size_t b, e;
  if (!r.line(&b, &e)) return fail(DPC_E_IO, "empty CSR file");
  std::string head = r.buf.substr(b, e - b);
  long long n = -1, m = -1;
  char word[32] = {0};
  int got = std::sscanf(head.c_str(), "%lld %lld %31s", &n, &m, word);
  if (got < 2 || n < 0 || m < 0) return fail(DPC_E_IO, "malformed CSR header line");
  bool weighted = got == 3 && std::strcmp(word, "weighted") == 0;
  if (got == 3 && !weighted) return fail(DPC_E_IO, "unknown header token '" + std::string(word) + "'");
  std::vector<int64_t> rp, cl, wt;
  rp.reserve(static_cast<size_t>(n + 1));
  if (!r.line(&b, &e) || r.ints(b, e, rp) != n + 1) return fail(DPC_E_IO, "row offsets line must hold nodes+1 integers");
  cl.reserve(static_cast<size_t>(m));
  if (m > 0 || r.pos < r.buf.size()) {
    if (!r.line(&b, &e) || r.ints(b, e, cl) != m) return fail(DPC_E_IO, "column line must hold edges integers");
  }
  if (weighted) {
    wt.reserve(static_cast<size_t>(m));
    if (!r.line(&b, &e) || r.ints(b, e, wt) != m) return fail(DPC_E_IO, "weight line must hold edges integers");
  }
  std::vector<int32_t> c32(cl.begin(), cl.end()), w32(wt.begin(), wt.end());
  for (int64_t k = 0; k < m; k++)
    if (cl[k] < 0 || cl[k] >= n) return fail(DPC_E_IO, "column index out of range in file");
  dpc_status st = dpc_csr_create(n, m, rp.data(), c32.data(), weighted ? w32.data() : nullptr,
                                 nullptr, out);
  if (st != DPC_OK) return fail(DPC_E_IO, std::string("invalid CSR in file: ") + dpc_last_error());
  return DPC_OK;
  DPC_TRY_END
}

dpc_status dpc_load_dimacs(const char* path, dpc_csr** out) {
  DPC_TRY_BEGIN
  if (!path || !out) return fail(DPC_E_INVALID, "NULL argument");
  std::string p(path);
  TextReader r;
  if (!r.load(path)) return fail(DPC_E_IO, "cannot read " + p);
  size_t b, e;
  auto skip = [&](char c) { return b < e && r.buf[b] == c; };
  // first non-comment line decides the format
  bool found = false;
  while (r.line(&b, &e)) {
    while (b < e && (r.buf[b] == ' ' || r.buf[b] == '\t' || r.buf[b] == '\r')) b++;
    if (b == e || skip('c') || skip('%')) continue;
    found = true;
    break;
  }
  if (!found) return fail(DPC_E_IO, "empty DIMACS file");
  std::vector<int64_t> cnt;  // per-row arc counts, then offsets
  std::vector<int32_t> src, dst, wt;
  int64_t n = 0;
  bool weighted = false;
  if (skip('p')) {  // 9th challenge: p sp n m / a u v w
    long long nn = -1, mm = -1;
    char kind[16] = {0};
    std::string head = r.buf.substr(b, e - b);
    if (std::sscanf(head.c_str(), "p %15s %lld %lld", kind, &nn, &mm) != 3 || nn < 0 || mm < 0)
      return fail(DPC_E_IO, "malformed DIMACS problem line");
    n = nn;
    if (n > INT32_MAX) return fail(DPC_E_IO, "DIMACS graph has more than 2^31 - 1 vertices");
    weighted = true;
    src.reserve(static_cast<size_t>(mm));
    std::vector<int64_t> t;
    while (r.line(&b, &e)) {
      while (b < e && (r.buf[b] == ' ' || r.buf[b] == '\t' || r.buf[b] == '\r')) b++;
      if (b == e || skip('c')) continue;
      if (!skip('a')) return fail(DPC_E_IO, "DIMACS arc line expected ('a u v w')");
      t.clear();
      if (r.ints(b + 1, e, t) != 3) return fail(DPC_E_IO, "DIMACS arc line must hold u v w");
      if (t[0] < 1 || t[0] > n || t[1] < 1 || t[1] > n) return fail(DPC_E_IO, "DIMACS arc endpoint out of range");
      if (t[2] < 0 || t[2] > INT32_MAX) return fail(DPC_E_IO, "DIMACS arc weight out of range");
      src.push_back(static_cast<int32_t>(t[0] - 1));
      dst.push_back(static_cast<int32_t>(t[1] - 1));
      wt.push_back(static_cast<int32_t>(t[2]));
    }
    if (static_cast<long long>(src.size()) != mm) return fail(DPC_E_IO, "DIMACS arc count differs from the problem line");
  } else {  // 10th challenge / METIS: n m [fmt [ncon]], then n adjacency lines
    std::vector<int64_t> h;
    if (r.ints(b, e, h) < 2 || h[0] < 0 || h[1] < 0) return fail(DPC_E_IO, "malformed METIS header line");
    n = h[0];
    if (n > INT32_MAX) return fail(DPC_E_IO, "METIS graph has more than 2^31 - 1 vertices");
    const int64_t fmt = h.size() > 2 ? h[2] : 0, ncon = h.size() > 3 ? h[3] : 1;
    const bool vsize = (fmt / 100) % 10 == 1, vwgt = (fmt / 10) % 10 == 1;
    weighted = fmt % 10 == 1;
    if (fmt != 0 && fmt != 1 && fmt != 10 && fmt != 11 && fmt != 100 && fmt != 101 && fmt != 110 && fmt != 111)
      return fail(DPC_E_IO, "unknown METIS fmt field");
    const int64_t skipv = (vsize ? 1 : 0) + (vwgt ? ncon : 0);
    src.reserve(static_cast<size_t>(2 * h[1]));
    std::vector<int64_t> t;
    int64_t v = 0;
    while (v < n && r.line(&b, &e)) {
      size_t bb = b;
      while (bb < e && (r.buf[bb] == ' ' || r.buf[bb] == '\t' || r.buf[bb] == '\r')) bb++;
      if (bb < e && r.buf[bb] == '%') continue;
      t.clear();
      if (r.ints(b, e, t) < 0) return fail(DPC_E_IO, "non-integer token in METIS adjacency line");
      if (static_cast<int64_t>(t.size()) < skipv) return fail(DPC_E_IO, "METIS line shorter than its vertex fields");
      const int64_t per = weighted ? 2 : 1;
      if ((static_cast<int64_t>(t.size()) - skipv) % per) return fail(DPC_E_IO, "METIS neighbour / weight pairs incomplete");
      for (size_t k = static_cast<size_t>(skipv); k < t.size(); k += per) {
        if (t[k] < 1 || t[k] > n) return fail(DPC_E_IO, "METIS neighbour out of range");
        src.push_back(static_cast<int32_t>(v));
        dst.push_back(static_cast<int32_t>(t[k] - 1));
        if (weighted) {
          if (t[k + 1] < 0 || t[k + 1] > INT32_MAX) return fail(DPC_E_IO, "METIS edge weight out of range");
          wt.push_back(static_cast<int32_t>(t[k + 1]));
        }
      }
      v++;
    }
    if (v != n) return fail(DPC_E_IO, "METIS file ends before its n adjacency lines");
    if (static_cast<int64_t>(src.size()) != 2 * h[1]) return fail(DPC_E_IO, "METIS arc count differs from 2 m");
  }
  if (n > INT32_MAX) return fail(DPC_E_IO, "DIMACS graph has more than 2^31 - 1 vertices");
  // counting sort by source, stable (file order within a row)
  const int64_t m = static_cast<int64_t>(src.size());
  std::vector<int64_t> rp(static_cast<size_t>(n + 1), 0);
  for (int64_t k = 0; k < m; k++) rp[src[k] + 1]++;
  for (int64_t i = 0; i < n; i++) rp[i + 1] += rp[i];
  std::vector<int64_t> at(rp.begin(), rp.end() - 1);
  std::vector<int32_t> c(static_cast<size_t>(m)), w(weighted ? static_cast<size_t>(m) : 0);
  for (int64_t k = 0; k < m; k++) {
    const int64_t q = at[src[k]]++;
    c[q] = dst[k];
    if (weighted) w[q] = wt[k];
  }
  dpc_status st = dpc_csr_create(n, m, rp.data(), c.data(), weighted ? w.data() : nullptr, nullptr, out);
  if (st != DPC_OK) return fail(DPC_E_IO, std::string("invalid graph in file: ") + dpc_last_error());
  return DPC_OK;
  DPC_TRY_END
}

dpc_status dpc_save_csr(const dpc_csr* g, const char* path) {
  DPC_TRY_BEGIN
  if (!path) return fail(DPC_E_INVALID, "path is NULL");
  dpc_status st = dpc_csr_validate(g);
  if (st != DPC_OK) return st;
  std::string p(path);
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(DPC_E_IO, "cannot open " + p + " for writing");
  bool ok = true;
  if (ends_with(p, ".bin")) {
    int64_t hdr[3] = {g->n, g->m, (g->w ? 1 : 0) | (g->val ? 2 : 0)};
    ok = std::fwrite("DPCCSR01", 1, 8, f) == 8 && std::fwrite(hdr, sizeof(int64_t), 3, f) == 3 &&
         std::fwrite(g->rowptr, sizeof(int64_t), g->n + 1, f) == static_cast<size_t>(g->n + 1) &&
         std::fwrite(g->col, sizeof(int32_t), g->m, f) == static_cast<size_t>(g->m);
    if (ok && g->w) ok = std::fwrite(g->w, sizeof(int32_t), g->m, f) == static_cast<size_t>(g->m);
    if (ok && g->val) ok = std::fwrite(g->val, sizeof(float), g->m, f) == static_cast<size_t>(g->m);
  } else {
    std::fprintf(f, "%lld %lld%s\n", static_cast<long long>(g->n), static_cast<long long>(g->m),
                 g->w ? " weighted" : "");
    for (int64_t i = 0; i <= g->n; i++) std::fprintf(f, i ? " %lld" : "%lld", static_cast<long long>(g->rowptr[i]));
    std::fputc('\n', f);
    for (int64_t k = 0; k < g->m; k++) std::fprintf(f, k ? " %d" : "%d", g->col[k]);
    std::fputc('\n', f);
    if (g->w) {
      for (int64_t k = 0; k < g->m; k++) std::fprintf(f, k ? " %d" : "%d", g->w[k]);
      std::fputc('\n', f);
    }
  }
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) return fail(DPC_E_IO, "write failed for " + p);
  return DPC_OK;
  DPC_TRY_END
}

dpc_status dpc_load_tree(const char* path, dpc_tree** out) {
  DPC_TRY_BEGIN
  if (!path || !out) return fail(DPC_E_INVALID, "NULL argument");
  TextReader r;
  if (!r.load(path)) return fail(DPC_E_IO, std::string("cannot read ") + path);
  size_t b, e;
  std::vector<int64_t> head, par;
  if (!r.line(&b, &e) || r.ints(b, e, head) != 1 || head[0] < 1)
    return fail(DPC_E_IO, "tree header must be a positive nodeCount");
  if (!r.line(&b, &e) || r.ints(b, e, par) != head[0])
    return fail(DPC_E_IO, "parent line must hold nodeCount integers");
  std::vector<int32_t> p32(par.size());
  for (size_t i = 0; i < par.size(); i++) {
    if (par[i] < -1 || par[i] >= head[0]) return fail(DPC_E_IO, "parent index out of range in file");
    p32[i] = static_cast<int32_t>(par[i]);
  }
  dpc_status st = dpc_tree_create(head[0], p32.data(), out);
  if (st != DPC_OK) return fail(DPC_E_IO, std::string("invalid tree in file: ") + dpc_last_error());
  return DPC_OK;
  DPC_TRY_END
}

dpc_status dpc_save_tree(const dpc_tree* t, const char* path) {
  DPC_TRY_BEGIN
  if (!t || !path) return fail(DPC_E_INVALID, "NULL argument");
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(DPC_E_IO, std::string("cannot open ") + path);
  std::fprintf(f, "%lld\n", static_cast<long long>(t->n));
  for (int64_t v = 0; v < t->n; v++) std::fprintf(f, v ? " %d" : "%d", t->parent[v]);
  std::fputc('\n', f);
  if (std::fclose(f) != 0) return fail(DPC_E_IO, "write failed");
  return DPC_OK;
  DPC_TRY_END
}

}  // extern "C"
