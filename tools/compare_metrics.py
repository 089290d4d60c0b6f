"""Metrics parity / compare tool (the reference spec's
cmd_compare): the paper's Fig. 6-10 evaluation analogue.

For each app and variant it reports, relative to basic-DP:
  * child launches         (B200: device launch counter; simulator: Metrics.childLaunchCount)
  * warp execution efficiency   (B200: ncu smsp__thread_inst_executed_per_inst_executed / 32;
                                 simulator: Metrics.warpExecEfficiency)
  * achieved SM occupancy  (B200: ncu sm__warps_active pct; simulator: smOccupancyAchieved)
  * DRAM transactions      (B200: ncu dram__sectors_read + write; simulator: 32-B segment proxy)
  * time                   (B200: device time of the range; simulator: simulatedCycles)
next to the paper's published K20c numbers.

The B200 side needs ncu range replay (CDP children included):
  ncu --replay-mode app-range --csv --log-file gpurun_out/compare_ncu.csv \\
      --metrics gpu__time_duration.sum,smsp__thread_inst_executed_per_inst_executed.ratio,\\
sm__warps_active.avg.pct_of_peak_sustained_active,dram__sectors_read.sum,dram__sectors_write.sum \\
      python tools/compare_metrics.py collect
  python tools/compare_metrics.py report gpurun_out/compare_ncu.csv profiles/r01_compare.md
`collect` writes gpurun_out/compare_launches.json; `report` runs the
reference simulator (oracle/_ref) on the same inputs and writes the table.
"""
import csv
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

VARIANTS = ["flat", "basic", "warp", "block", "grid"]
OUT = os.path.join(ROOT, "gpurun_out")
PAPER = {  # PAPER.md:318-334, K20c, averaged over the paper's benchmarks
    "launches_pct_of_basic": "0.07-14.48 %",
    "warp_eff": {"basic": 33.2, "warp": 69.3, "block": 75.0, "grid": 83.1},
    "occupancy": {"basic": 27.9, "warp": 39.3, "block": 60.3, "grid": 82.9},
    "dram_pct_of_basic": {"warp": 60, "block": 34, "grid": 36},
    "speedup_vs_basic_mean": {"warp": 999, "block": 1357, "grid": 1459},
}


def inputs():
    import paper_1606_08150_b200 as dpc
    g = dpc.gen_rmat(12, 16, seed=3, weights=False, values=True)
    t = dpc.gen_tree(4, 16, 64, 0.5, seed=2)
    return g, t


def collect():
    import torch

    import paper_1606_08150_b200 as dpc
    ctx = dpc.Context(0)
    g, t = inputs()
    x = (np.arange(g.n, dtype=np.float32) % 97 + 1) / 97.0
    dg = dpc.DeviceGraph(ctx, g)
    dg.set_x(x)
    dt = dpc.DeviceTree(ctx, t)
    order, launches = [], {}
    runs = [("spmv", v, lambda v=v: dg.spmv(v, metrics=True)) for v in VARIANTS]
    runs += [("td", v, lambda v=v: dt.run("tree_desc", v, metrics=True)) for v in VARIANTS]
    for app, v, fn in runs:
        fn()
        ctx.synchronize()
        torch.cuda.profiler.start()
        met = fn()
        ctx.synchronize()
        torch.cuda.profiler.stop()
        order.append([app, v])
        launches[f"{app}/{v}"] = int(met.child_launch_count)
    # the compiler's output for the same programs the simulator runs
    import paper_1606_08150_b200.kdl as kdl
    x64 = (np.arange(g.n) % 97 + 1) / 97.0
    kruns = []
    for v in ["basic", "warp", "block", "grid"]:
        mod = kdl.compile(kdl.read_program("spmv.kdl"), v, name="spmv")
        kruns.append(("kdl-spmv", v, lambda mod=mod: mod.run({"n": g.n, "m": g.m, "nx": g.n, "thr": 32},
                                                             {"rowptr": g.rowptr, "col": g.col, "val": g.val,
                                                              "x": x64})))
    kids = np.diff(t.cstart)
    for v in ["basic", "warp", "block", "grid"]:
        mod = kdl.compile(kdl.read_program("td.kdl"), v, name="td")
        kruns.append(("kdl-td", v, lambda mod=mod: mod.run({"n": t.n, "root": t.root, "rootnc": int(kids[t.root])},
                                                           {"cstart": t.cstart, "clist": t.clist,
                                                            "parent": t.parent})))
    for app, v, fn in kruns:
        fn()
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        res = fn()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        order.append([app, v])
        launches[f"{app}/{v}"] = int(res.launches)
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "compare_launches.json"), "w") as f:
        json.dump({"order": order, "launches": launches, "spmv_rows": g.n, "spmv_nnz": g.m, "td_nodes": t.n}, f)
    print("collected", len(order), "ranges")


def parse_ncu(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Metric Name" in r][0]
    h = rows[hi]
    ii, ni, vi = h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
    ranges = {}
    for r in rows[hi + 1:]:
        if len(r) > vi:
            ranges.setdefault(int(r[ii]), {})[r[ni]] = float(r[vi].replace(",", ""))
    return [ranges[k] for k in sorted(ranges)]


def simulate():
    from tests._oracle import RefSim
    ref = RefSim()
    g, t = inputs()
    x = (np.arange(g.n, dtype=np.float64) % 97 + 1) / 97.0
    out = {}
    src = ref.kdl("spmv.kdl")
    for v in ["basic", "warp", "block", "grid"]:
        rc, _, met, err = ref.run(src, v, {"n": g.n, "m": g.m, "nx": g.n, "thr": 32},
                                  {"rowptr": g.rowptr, "col": g.col}, {"val": g.val, "x": x},
                                  out="y", out_len=g.n, out_float=True)
        out[f"spmv/{v}"] = met if rc == 0 else {"fault": err}
    src = ref.kdl("td.kdl")
    kids = np.diff(t.cstart)
    for v in ["basic", "warp", "block", "grid"]:
        rc, _, met, err = ref.run(src, v, {"n": t.n, "root": t.root, "rootnc": int(kids[t.root])},
                                  {"cstart": t.cstart, "clist": t.clist, "parent": t.parent}, {},
                                  out="desc", out_len=t.n)
        out[f"td/{v}"] = met if rc == 0 else {"fault": err}
    return out


def report(ncu_csv, out_md):
    info = json.load(open(os.path.join(OUT, "compare_launches.json")))
    nc = parse_ncu(ncu_csv)
    b200 = {}
    for (app, v), m in zip(info["order"], nc):
        b200[f"{app}/{v}"] = {
            "launches": info["launches"][f"{app}/{v}"],
            "warp_eff_pct": round(100 * m.get("smsp__thread_inst_executed_per_inst_executed.ratio", 0) / 32, 1),
            "occupancy_pct": round(m.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0), 1),
            "dram_sectors": int(m.get("dram__sectors_read.sum", 0) + m.get("dram__sectors_write.sum", 0)),
            "time_us": round(m.get("gpu__time_duration.sum", 0) / 1e3, 1)}
    sim = simulate()
    lines = ["# Consolidation metrics vs basic-DP: B200 (ncu range replay, CDP children included),",
             "# the reference simulator (oracle/_ref, same inputs) and the paper (K20c, PAPER.md:318-334)", "",
             f"SpMV: R-MAT scale 12 ({info['spmv_rows']} rows, {info['spmv_nnz']} nnz); "
             f"TD: gen_tree(4, 16, 64, 0.5, 2) = {info['td_nodes']} nodes.", "",
             "| app / variant | B200 launches | B200 warp eff % | B200 occupancy % | B200 DRAM sectors (x basic) "
             "| B200 range time us (x faster; includes host API time) | sim launches | sim warp eff % | sim occupancy % "
             "| sim DRAM tx (x basic) | sim cycles (x faster) |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for app in ["spmv", "td", "kdl-spmv", "kdl-td"]:
        simapp = app.replace("kdl-", "")
        bb, sb = b200.get(f"{app}/basic", {}), sim.get(f"{simapp}/basic", {})
        for v in VARIANTS:
            if f"{app}/{v}" not in b200:
                continue
            b, sm = b200.get(f"{app}/{v}", {}), sim.get(f"{simapp}/{v}", {})
            dr = f"{b['dram_sectors']} ({b['dram_sectors'] / max(1, bb.get('dram_sectors', 1)):.2f})" if b else "-"
            tm = f"{b['time_us']} ({bb.get('time_us', 0) / max(1e-9, b['time_us']):.1f})" if b else "-"
            if "childLaunchCount" in sm:
                sl = sm["childLaunchCount"]
                sw = round(sm["warpExecEfficiency_1e6"] / 1e4, 1)
                so = round(sm["smOccupancyAchieved_1e6"] / 1e4, 1)
                sd = f"{sm['dramTransactions']} ({sm['dramTransactions'] / max(1, sb.get('dramTransactions', 1)):.2f})"
                sc = f"{sm['simulatedCycles']} ({sb.get('simulatedCycles', 0) / max(1, sm['simulatedCycles']):.1f})"
            elif "fault" in sm:
                sl = sw = so = sd = sc = "fault: " + sm["fault"][:40]
            else:
                sl = sw = so = sd = sc = "-"
            lines.append(f"| {app} / {v} | {b.get('launches', '-')} | {b.get('warp_eff_pct', '-')} | "
                         f"{b.get('occupancy_pct', '-')} | {dr} | {tm} | {sl} | {sw} | {so} | {sd} | {sc} |")
    lines += ["", "kdl-* rows: the same .kdl programs the simulator runs, compiled for sm_100a by "
              "paper_1606_08150_b200.kdl (int64 / fp64 values, CDP2 launches); the other B200 rows are the "
              "hand-written kernels (fp32 / int32).",
              "", "Paper (K20c, mean over its benchmarks): launches after consolidation "
              f"{PAPER['launches_pct_of_basic']} of basic; warp efficiency {PAPER['warp_eff']}; "
              f"occupancy {PAPER['occupancy']}; DRAM % of basic {PAPER['dram_pct_of_basic']}; "
              f"mean speed-up vs basic {PAPER['speedup_vs_basic_mean']}."]
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "collect":
        collect()
    else:
        report(sys.argv[2], sys.argv[3])
