// TEST INFRASTRUCTURE ONLY -- never linked into libdpc.so.
//
// Exercises the reference-side adapter include/dpc_dpcons.hpp (SURVEY.md
// §8(a) row a15) end to end: one dpcons::Workload is (1) simulated by the
// UNMODIFIED reference -- parse_program (parser.hpp:781) -> consolidate
// (transform.hpp:971) -> simulate (sim.hpp:1746), repeated to a fixpoint for
// the programs that need it -- and (2) run on the B200 through the adapter
// (libdpc.so's C ABI); the two SimResults are diffed global by global.
// Built by oracle/Makefile into oracle/_ref/libsim_adapter.so (needs the
// reference headers here; the built .so travels to the GPU box).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <set>
#include <string>

namespace dpcons {
inline std::set<std::int64_t> runningSet_;  // sim.hpp:817 shim, see ref_sim.cpp
}

#include "dpcons/parser.hpp"
#include "dpcons/sim.hpp"
#include "dpcons/transform.hpp"
#include "dpcons/validate.hpp"
#include "dpc_dpcons.hpp"

namespace {
void put_err(char* err, int errlen, const std::string& s) {
  if (err && errlen > 0) {
    std::strncpy(err, s.c_str(), static_cast<size_t>(errlen - 1));
    err[errlen - 1] = 0;
  }
}
const dpcons::GlobalArrayState* find(const dpcons::SimResult& r, const std::string& name) {
  for (const auto& g : r.globals)
    if (g.name == name) return &g;
  return nullptr;
}
}  // namespace

extern "C" {

// bench: "spmv" | "sssp" | "bfs" | "td" | "th"; out: the global to diff;
// mode 0 = as written (basic-dp), 1 warp, 2 block, 3 grid; fixpoint: repeat
// simulate() feeding `out` back until it stops changing.
// Returns 0 and fills mismatches / max_rel on success; 1 reference error,
// 2 GPU fault, 3 missing output.
int adapter_diff(const char* bench, const char* src, int mode, const char* out, int fixpoint, int n_scal,
                 const char** snames, const int64_t* svals, int n_iarr, const char** inames,
                 const int64_t* const* iptrs, const int64_t* ilens, int n_farr, const char** fnames,
                 const double* const* fptrs, const int64_t* flens, int64_t* mismatches, double* max_rel,
                 int64_t* gpu_launches, int64_t* sim_launches, char* err, int errlen) {
  dpcons::Workload wl;
  for (int i = 0; i < n_scal; i++) wl.intScalars[snames[i]] = svals[i];
  for (int i = 0; i < n_iarr; i++) wl.intArrays[inames[i]].assign(iptrs[i], iptrs[i] + ilens[i]);
  for (int i = 0; i < n_farr; i++) wl.floatArrays[fnames[i]].assign(fptrs[i], fptrs[i] + flens[i]);
  auto pr = dpcons::parse_program(src);
  if (!pr.ok()) {
    put_err(err, errlen, "parse failed");
    return 1;
  }
  dpcons::ast::Program prog = *pr.program;
  std::optional<dpcons::ast::Granularity> gran;
  if (mode >= 1 && mode <= 3) {
    gran = mode == 1 ? dpcons::ast::Granularity::Warp
           : mode == 2 ? dpcons::ast::Granularity::Block
                       : dpcons::ast::Granularity::Grid;
    dpcons::TransformOptions opt;
    opt.granularityOverride = gran;
    auto tr = dpcons::consolidate(prog, opt);
    if (!tr.ok()) {
      put_err(err, errlen, "consolidate failed");
      return 1;
    }
    prog = *tr.program;
  }
  // (1) the reference simulator, to a fixpoint when asked
  dpcons::Workload sw = wl;
  dpcons::SimResult sim;
  *sim_launches = 0;
  for (int run = 0; run < 1000; run++) {
    dpcons::runningSet_.clear();
    sim = dpcons::simulate(prog, sw, dpcons::SimConfig{});
    if (!sim.ok()) {
      put_err(err, errlen, "simulate: " + sim.fault->kind + ": " + sim.fault->message);
      return 1;
    }
    *sim_launches += sim.metrics.childLaunchCount;
    const auto* g = find(sim, out);
    if (!g) {
      put_err(err, errlen, std::string("simulator has no global ") + out);
      return 3;
    }
    if (!fixpoint || g->isFloat || g->ints == sw.intArrays[out]) break;
    sw.intArrays[out] = g->ints;
  }
  // (2) the B200 through the adapter, from the ORIGINAL workload
  dpc_ctx* ctx = nullptr;
  if (dpc_ctx_create(0, &ctx) != DPC_OK) {
    put_err(err, errlen, std::string("dpc_ctx_create: ") + dpc_last_error());
    return 2;
  }
  dpcons::SimResult gpu = dpc_dpcons::run(ctx, bench, wl, gran);
  dpc_ctx_destroy(ctx);
  if (!gpu.ok()) {
    put_err(err, errlen, "gpu: " + gpu.fault->kind + ": " + gpu.fault->message);
    return 2;
  }
  *gpu_launches = gpu.metrics.childLaunchCount;
  const auto* a = find(sim, out);
  const auto* b = find(gpu, out);
  if (!a || !b || a->isFloat != b->isFloat) {
    put_err(err, errlen, std::string("output ") + out + " missing or of another type");
    return 3;
  }
  int64_t bad = 0;
  double worst = 0.0;
  if (a->isFloat) {
    if (a->floats.size() != b->floats.size()) bad = -1;
    for (size_t i = 0; bad >= 0 && i < a->floats.size(); i++) {
      const double d = std::fabs(a->floats[i] - b->floats[i]);
      const double rel = a->floats[i] != 0.0 ? d / std::fabs(a->floats[i]) : d;
      worst = std::max(worst, rel);
      if (rel > 1e-5) bad++;
    }
  } else {
    if (a->ints.size() != b->ints.size()) bad = -1;
    for (size_t i = 0; bad >= 0 && i < a->ints.size(); i++) bad += a->ints[i] != b->ints[i];
  }
  *mismatches = bad;
  *max_rel = worst;
  return 0;
}

}  // extern "C"
