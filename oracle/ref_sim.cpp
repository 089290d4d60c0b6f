// TEST INFRASTRUCTURE ONLY — never linked into libdpc.so.
//
// C-ABI driver around the UNMODIFIED reference (dpcons, compiled in place from
// /root/reference/proj/include by oracle/Makefile into oracle/_ref/).  It runs
// the reference pipeline parse_program (parser.hpp:781) -> consolidate
// (transform.hpp:971, granularity override) -> simulate (sim.hpp:1746) on one
// of our .kdl formulations (oracle/kdl/) and a Workload of named int64/fp64
// arrays (sim.hpp:27-32), then returns one output global and the Metrics
// (sim.hpp:34-47).  Used by tests/ to pin the CPU restatement (oracle.c) and by
// bench.py --impl reference as the reference's own CPU path.
//
// Shim: sim.hpp uses `runningSet_` without declaring it
// (sim.hpp:817, :832).  Unqualified lookup from the member function falls back
// to namespace scope, so a namespace-scope set makes the header compile.  It is
// cleared before every simulate() because instance sequence numbers restart.
#include <cstdint>
#include <cstring>
#include <set>
#include <string>

namespace dpcons {
inline std::set<std::int64_t> runningSet_;
}

#include "dpcons/config.hpp"
#include "dpcons/memplan.hpp"
#include "dpcons/parser.hpp"
#include "dpcons/sim.hpp"
#include "dpcons/transform.hpp"
#include "dpcons/unparse.hpp"
#include "dpcons/validate.hpp"

namespace {
void put_err(char* err, int errlen, const std::string& s) {
  if (err && errlen > 0) {
    std::strncpy(err, s.c_str(), static_cast<size_t>(errlen - 1));
    err[errlen - 1] = 0;
  }
}
std::string diags_text(const dpcons::DiagList& d) {
  std::string s;
  for (const auto& x : d) s += dpcons::format_diag(x) + "\n";
  return s;
}
}  // namespace

extern "C" {

// mode: 0 = as written (basic-dp / flat programs), 1 = warp, 2 = block, 3 = grid.
// metrics_out (12 int64): childLaunchCount, fixedPoolPeak, virtualPoolPeak,
// simulatedCycles, parentSwapEvents, maxConcurrentObserved,
// bufferItemsInserted, allocCyclesCharged, dramTransactions, deadlockDetected,
// warpExecEfficiency*1e6, smOccupancyAchieved*1e6.
// Returns 0 on success, 1 on parse/transform error, 2 on a simulator fault,
// 3 on a bad output request.
int ref_run(const char* src, int mode, int n_scal, const char** snames, const int64_t* svals,
            int n_iarr, const char** inames, const int64_t* const* iptrs, const int64_t* ilens,
            int n_farr, const char** fnames, const double* const* fptrs, const int64_t* flens,
            const char* out_name, void* out_buf, int64_t out_len, int64_t* metrics_out, char* err,
            int errlen) {
  auto pr = dpcons::parse_program(src);
  if (!pr.ok()) {
    put_err(err, errlen, "parse: " + diags_text(pr.diags));
    return 1;
  }
  auto vd = dpcons::validate(*pr.program);
  if (!vd.empty()) {
    put_err(err, errlen, "validate: " + diags_text(vd));
    return 1;
  }
  dpcons::ast::Program prog = *pr.program;
  if (mode >= 1 && mode <= 3) {
    dpcons::TransformOptions opt;
    opt.granularityOverride = mode == 1   ? dpcons::ast::Granularity::Warp
                              : mode == 2 ? dpcons::ast::Granularity::Block
                                          : dpcons::ast::Granularity::Grid;
    auto tr = dpcons::consolidate(prog, opt);
    if (!tr.ok()) {
      put_err(err, errlen, "transform: " + diags_text(tr.diags));
      return 1;
    }
    prog = *tr.program;
  }
  dpcons::Workload wl;
  for (int i = 0; i < n_scal; i++) wl.intScalars[snames[i]] = svals[i];
  for (int i = 0; i < n_iarr; i++) wl.intArrays[inames[i]].assign(iptrs[i], iptrs[i] + ilens[i]);
  for (int i = 0; i < n_farr; i++) wl.floatArrays[fnames[i]].assign(fptrs[i], fptrs[i] + flens[i]);
  dpcons::runningSet_.clear();
  dpcons::SimConfig cfg;
  auto res = dpcons::simulate(prog, wl, cfg);
  const auto& m = res.metrics;
  if (metrics_out) {
    int64_t mv[12] = {m.childLaunchCount,      m.fixedPoolPeak,        m.virtualPoolPeak,
                      m.simulatedCycles,       m.parentSwapEvents,     m.maxConcurrentObserved,
                      m.bufferItemsInserted,   m.allocCyclesCharged,   m.dramTransactions,
                      m.deadlockDetected ? 1 : 0,
                      static_cast<int64_t>(m.warpExecEfficiency * 1e6),
                      static_cast<int64_t>(m.smOccupancyAchieved * 1e6)};
    std::memcpy(metrics_out, mv, sizeof(mv));
  }
  if (!res.ok()) {
    put_err(err, errlen, res.fault->kind + ": " + res.fault->message);
    return 2;
  }
  if (out_name && out_buf) {
    for (const auto& g : res.globals) {
      if (g.name != out_name) continue;
      int64_t len = g.isFloat ? static_cast<int64_t>(g.floats.size()) : static_cast<int64_t>(g.ints.size());
      if (len != out_len) {
        put_err(err, errlen, "output length mismatch");
        return 3;
      }
      if (g.isFloat) std::memcpy(out_buf, g.floats.data(), sizeof(double) * static_cast<size_t>(len));
      else std::memcpy(out_buf, g.ints.data(), sizeof(int64_t) * static_cast<size_t>(len));
      return 0;
    }
    put_err(err, errlen, std::string("no global named ") + out_name);
    return 3;
  }
  return 0;
}

// Reference policy functions, exposed so tests can pin our B200 policy code
// (launch configuration, buffer sizing) against the reference's own KATs.
// config.hpp:68-75 kc_config(B, T, X) -> (blocks, threads)
void ref_kc_config(int64_t b, int64_t t, int64_t x, int64_t* out_b, int64_t* out_t) {
  auto r = dpcons::kc_config(b, t, x);
  *out_b = r.blocks;
  *out_t = r.threadsPerBlock;
}

// memplan.hpp:61-66 per_buffer_size(totalThread, totalBuffVar, const)
int64_t ref_per_buffer_size(int64_t threads, int64_t nvars, int64_t k) {
  try {
    return dpcons::per_buffer_size(threads, nvars, k);
  } catch (...) {
    return -1;
  }
}

// Round-trips the consolidated program as text (transform.hpp:971 ->
// unparse.hpp:344) so tests can show the reference's generated code shape.
int ref_consolidate_text(const char* src, int mode, char* out, int outlen) {
  auto pr = dpcons::parse_program(src);
  if (!pr.ok()) {
    put_err(out, outlen, "parse: " + diags_text(pr.diags));
    return 1;
  }
  dpcons::TransformOptions opt;
  opt.granularityOverride = mode == 1   ? dpcons::ast::Granularity::Warp
                            : mode == 2 ? dpcons::ast::Granularity::Block
                                        : dpcons::ast::Granularity::Grid;
  auto tr = dpcons::consolidate(*pr.program, opt);
  if (!tr.ok()) {
    put_err(out, outlen, "transform: " + diags_text(tr.diags));
    return 1;
  }
  put_err(out, outlen, dpcons::unparse(*tr.program));
  return 0;
}

}  // extern "C"
