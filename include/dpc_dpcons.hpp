// dpc_dpcons.hpp -- the reference-side adapter:
// runs a hot-path benchmark on the B200 through libdpc.so's C ABI from the
// reference's own data boundary, a dpcons::Workload (sim.hpp:27-32), and
// returns a dpcons::SimResult (sim.hpp:34-66) shaped like simulate()'s, so a
// GPU run diffs global-by-global against dpcons::simulate() (sim.hpp:1746).
//
// Header-only C++20.  Include it in a translation unit that can see the
// reference headers (-I/root/reference/proj/include) and this repo's
// include/, and link libdpc.so.  The Workload layouts are the ones the
// bundled .kdl formulations use (paper_1606_08150_b200/kdl/programs/), i.e.
// exactly what simulate() consumes for the same benchmark:
//   spmv : int rowptr[n+1], col[m]; float val[m], x[nx]        -> float y[n]
//   sssp : int rowptr[n+1], col[m], w[m], dist[n] (source = the
//          vertex with dist 0, others >= 2^40)                  -> int dist[n]
//   bfs  : int rowptr[n+1], col[m], level[n] (source level 0)   -> int level[n]
//   td   : int cstart[n+1], clist[n], parent[n]                 -> int desc[n]
//   th   : int cstart[n+1], clist[n], parent[n]                 -> int height[n]
// Unreached vertices come back as 2^40, the value the .kdl programs use.
// Metrics: childLaunchCount (device launches), bufferItemsInserted and
// fixedPoolPeak are filled from dpc_metrics; the simulator's cycle, DRAM and
// occupancy models have no GPU counterpart here (ncu measures those,
// tools/compare_metrics.py) and stay at their defaults.
// Faults map dpc_status -> SimFault.kind (sim.hpp:49-52).
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "dpc.h"
#include "dpcons/sim.hpp"

namespace dpc_dpcons {

constexpr std::int64_t kUnreached = std::int64_t{1} << 40;

// Granularity override of consolidate() (transform.hpp:971) -> variant;
// no override = the program as written (basic-dp).
inline dpc_variant variant_of(std::optional<dpcons::ast::Granularity> g) {
  if (!g) return DPC_BASIC;
  switch (*g) {
    case dpcons::ast::Granularity::Warp: return DPC_WARP;
    case dpcons::ast::Granularity::Block: return DPC_BLOCK;
    default: return DPC_GRID;
  }
}

inline const char* fault_kind(dpc_status s) {
  switch (s) {
    case DPC_E_OVERFLOW: return "overflow";
    case DPC_E_NESTING: return "nesting";
    case DPC_E_OOM: return "oom";
    case DPC_E_DEADLOCK: return "deadlock";
    case DPC_E_INVALID: return "config";
    default: return "runtime";
  }
}

namespace detail {

inline const std::vector<std::int64_t>& ints(const dpcons::Workload& wl, const char* k) { return wl.intArrays.at(k); }
inline const std::vector<double>& floats(const dpcons::Workload& wl, const char* k) { return wl.floatArrays.at(k); }

inline void set_fault(dpcons::SimResult& r, dpc_status st) {
  if (st != DPC_OK && !r.fault) r.fault = dpcons::SimFault{fault_kind(st), dpc_last_error()};
}

inline void set_metrics(dpcons::SimResult& r, const dpc_metrics& m) {
  r.metrics.childLaunchCount = m.child_launch_count;
  r.metrics.bufferItemsInserted = m.buffer_items_inserted;
  r.metrics.fixedPoolPeak = m.pool_peak;
}

inline dpcons::GlobalArrayState int_global(const char* name, std::vector<std::int64_t> v) {
  dpcons::GlobalArrayState g;
  g.name = name;
  g.isFloat = false;
  g.ints = std::move(v);
  return g;
}

// CSR from the Workload's rowptr / col (+ w or val); nullptr + fault on error.
inline dpc_csr* csr(const dpcons::Workload& wl, const char* wname, const char* vname, dpcons::SimResult& r) {
  const auto& rp = ints(wl, "rowptr");
  const auto& cl = ints(wl, "col");
  std::vector<std::int64_t> rowptr(rp.begin(), rp.end());
  std::vector<std::int32_t> col(cl.begin(), cl.end()), w;
  std::vector<float> val;
  if (wname) {
    const auto& ws = ints(wl, wname);
    w.assign(ws.begin(), ws.end());
  }
  if (vname) {
    const auto& vs = floats(wl, vname);
    val.assign(vs.begin(), vs.end());
  }
  dpc_csr* g = nullptr;
  set_fault(r, dpc_csr_create(static_cast<std::int64_t>(rowptr.size()) - 1, static_cast<std::int64_t>(col.size()),
                              rowptr.data(), col.data(), wname ? w.data() : nullptr,
                              vname ? val.data() : nullptr, &g));
  return g;
}

inline int32_t source_of(const std::vector<std::int64_t>& d) {
  for (std::size_t i = 0; i < d.size(); i++)
    if (d[i] == 0) return static_cast<int32_t>(i);
  return 0;
}

inline std::vector<std::int64_t> widen(const std::vector<std::uint32_t>& d) {
  std::vector<std::int64_t> out(d.size());
  for (std::size_t i = 0; i < d.size(); i++) out[i] = d[i] == UINT32_MAX ? kUnreached : d[i];
  return out;
}

inline dpc_launch_cfg cfg_for(int32_t app, dpc_variant v, dpcons::SimResult& r) {
  dpc_launch_cfg c{};
  set_fault(r, dpc_launch_cfg_default(app, v, &c));
  return c;
}

}  // namespace detail

// SpMV benchmark: y = A x in fp32 on the GPU, reported as fp64.
inline dpcons::SimResult run_spmv(dpc_ctx* ctx, const dpcons::Workload& wl,
                                  std::optional<dpcons::ast::Granularity> g = std::nullopt) {
  dpcons::SimResult r;
  dpc_csr* A = detail::csr(wl, nullptr, "val", r);
  const auto& xs = detail::floats(wl, "x");
  std::vector<float> x(xs.begin(), xs.end()), y(A ? static_cast<std::size_t>(A->n) : 0);
  dpc_metrics m{};
  dpc_launch_cfg c = detail::cfg_for(DPC_APP_SPMV, variant_of(g), r);
  if (A && !r.fault) detail::set_fault(r, dpc_run_spmv(ctx, A, x.data(), y.data(), &c, &m));
  dpcons::GlobalArrayState out;
  out.name = "y";
  out.isFloat = true;
  out.floats.assign(y.begin(), y.end());
  r.globals.push_back(std::move(out));
  detail::set_metrics(r, m);
  dpc_csr_free(A);
  return r;
}

// SSSP / BFS benchmarks: shortest distances
// (levels) from the vertex whose initial dist (level) is 0.
inline dpcons::SimResult run_sssp(dpc_ctx* ctx, const dpcons::Workload& wl,
                                  std::optional<dpcons::ast::Granularity> g = std::nullopt, bool bfs = false) {
  dpcons::SimResult r;
  const char* dname = bfs ? "level" : "dist";
  dpc_csr* G = detail::csr(wl, bfs ? nullptr : "w", nullptr, r);
  const int32_t src = detail::source_of(detail::ints(wl, dname));
  std::vector<std::uint32_t> d(G ? static_cast<std::size_t>(G->n) : 0);
  dpc_metrics m{};
  dpc_launch_cfg c = detail::cfg_for(DPC_APP_SSSP, variant_of(g), r);
  if (G && !r.fault)
    detail::set_fault(r, bfs ? dpc_run_bfs(ctx, G, src, d.data(), &c, &m)
                             : dpc_run_sssp(ctx, G, src, d.data(), &c, &m));
  r.globals.push_back(detail::int_global(dname, detail::widen(d)));
  detail::set_metrics(r, m);
  dpc_csr_free(G);
  return r;
}

// TD / TH benchmarks: per-node descendants / heights.
inline dpcons::SimResult run_tree(dpc_ctx* ctx, const dpcons::Workload& wl, bool height,
                                  std::optional<dpcons::ast::Granularity> g = std::nullopt) {
  dpcons::SimResult r;
  const auto& ps = detail::ints(wl, "parent");
  std::vector<std::int32_t> parent(ps.begin(), ps.end()), out(parent.size());
  dpc_tree* T = nullptr;
  detail::set_fault(r, dpc_tree_create(static_cast<std::int64_t>(parent.size()), parent.data(), &T));
  dpc_metrics m{};
  const int32_t app = height ? DPC_APP_TREE_HEIGHT : DPC_APP_TREE_DESC;
  dpc_launch_cfg c = detail::cfg_for(app, variant_of(g), r);
  if (T && !r.fault)
    detail::set_fault(r, height ? dpc_run_tree_height(ctx, T, out.data(), &c, &m)
                                : dpc_run_tree_desc(ctx, T, out.data(), &c, &m));
  r.globals.push_back(detail::int_global(height ? "height" : "desc",
                                         std::vector<std::int64_t>(out.begin(), out.end())));
  detail::set_metrics(r, m);
  dpc_tree_free(T);
  return r;
}

// benchmark(name) dispatch: "spmv", "sssp", "bfs", "td", "th".
inline dpcons::SimResult run(dpc_ctx* ctx, const std::string& name, const dpcons::Workload& wl,
                             std::optional<dpcons::ast::Granularity> g = std::nullopt) {
  if (name == "spmv") return run_spmv(ctx, wl, g);
  if (name == "sssp") return run_sssp(ctx, wl, g, false);
  if (name == "bfs") return run_sssp(ctx, wl, g, true);
  if (name == "td") return run_tree(ctx, wl, false, g);
  if (name == "th") return run_tree(ctx, wl, true, g);
  dpcons::SimResult r;
  r.fault = dpcons::SimFault{"config", "unknown benchmark " + name};
  return r;
}

}  // namespace dpc_dpcons
