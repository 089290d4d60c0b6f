"""Times every app x variant at its BASELINE configuration (device-resident,
CUDA events, L2 flushed) and checks each result against the CPU oracle.

usage: python tools/prof_apps.py [--apps sssp gc td th] [--reps N] [--json out.json]
Also importable: run_apps(ctx, apps, reps) -> dict (used by bench.py)."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1606_08150_b200 as dpc  # noqa: E402

VARIANTS = ["flat", "basic", "warp", "block", "grid"]
TREE = dict(depth=24, lo=1, hi=4, fill=0.851, seed=1)     # BASELINE config 4: 4,246,411 nodes, depth 24
TREE_PAPER = dict(depth=5, lo=32, hi=128, fill=0.4, seed=1)  # paper-shaped, ~2.7M nodes
# depth 24 at the size basic-DP still fits in the device pending-launch pool
# (599,186 on B200; 196,634 internal nodes -> ~394K outstanding launches)
TREE_DEEP_FIT = dict(depth=24, lo=1, hi=4, fill=0.75, seed=1)  # 491,454 nodes


def _time(ctx, fn, reps):
    ts = []
    for _ in range(reps):
        ctx.flush_l2()
        ctx.synchronize()
        ctx.record(4)
        fn()
        ctx.record(5)
        ts.append(ctx.elapsed_ms(4, 5))
    return float(np.median(ts))


def _variants(ctx, reps, run, check, extra):
    """run(variant, metrics) -> Metrics; check() -> bool; extra(Metrics) -> dict."""
    res = {}
    for v in VARIANTS:
        try:
            met = run(v, True)
            ok = bool(check())
            ms = _time(ctx, lambda: run(v, False), reps if v != "basic" else 1)
            res[v] = {"ms": round(ms, 4), "bit_exact": ok, "device_launches": met.child_launch_count,
                      **extra(met)}
        except dpc.DpcError as e:
            res[v] = {"error": str(e)}
    return res


def _summ(res, unit_count, unit):
    for r in res.values():
        if "ms" in r:
            r["g" + unit] = round(unit_count / (r["ms"] * 1e-3) / 1e9, 4)
    out = {"variants": res}
    timed = [(r["ms"], v) for v, r in res.items() if "ms" in r and v in ("warp", "block", "grid")]
    if timed:
        best = min(timed)
        out["best_consolidated"] = best[1]
        if "ms" in res.get("basic", {}):
            out["best_vs_basic"] = round(res["basic"]["ms"] / best[0], 2)
        if "ms" in res.get("flat", {}):
            out["best_vs_flat"] = round(res["flat"]["ms"] / best[0], 2)
    return out


def app_sssp(ctx, orc, reps, scale=16):
    g = dpc.gen_rmat(scale, 16, seed=1)
    s = int(np.argmax(g.degrees()))
    ref = orc.sssp(g.rowptr, g.col, g.w, s)
    m_reached = int(g.degrees()[ref != np.uint32(0xFFFFFFFF)].sum())
    dg = dpc.DeviceGraph(ctx, g)
    res = _variants(ctx, reps, lambda v, m: dg.sssp(s, v, metrics=m),
                    lambda: np.array_equal(dg.get_dist(), ref),
                    lambda met: {"iterations": met.iterations, "relaxed_edges": met.edges_processed})
    dg.close()
    out = _summ(res, m_reached, "teps")
    out.update({"workload": f"SSSP R-MAT scale {scale}, int weights [1,255], source = max-degree vertex",
                "unit": "GTEPS (edges of the reached component / time, Graph500)",
                "m_reached": m_reached})
    return out


def app_bfs(ctx, orc, reps, scale=16):
    """BFS-Rec (the paper's seventh benchmark): config-1 graph, unit weights."""
    g = dpc.gen_rmat(scale, 16, seed=1, weights=False)
    s = int(np.argmax(g.degrees()))
    ref = orc.bfs(g.rowptr, g.col, s)
    m_reached = int(g.degrees()[ref != np.uint32(0xFFFFFFFF)].sum())
    dg = dpc.DeviceGraph(ctx, g)
    res = _variants(ctx, reps, lambda v, m: dg.bfs(s, v, metrics=m),
                    lambda: np.array_equal(dg.get_dist(), ref),
                    lambda met: {"iterations": met.iterations})
    dg.close()
    out = _summ(res, m_reached, "teps")
    out.update({"workload": f"BFS R-MAT scale {scale}, source = max-degree vertex",
                "unit": "GTEPS (edges of the reached component / time, Graph500)",
                "m_reached": m_reached, "levels": int(ref[ref != np.uint32(0xFFFFFFFF)].max())})
    return out


def app_pr(ctx, orc, reps, scale=20, iters=20):
    """PageRank (the paper's PR benchmark): 20 power iterations on the config-2
    graph pattern (directed R-MAT scale 20), each one SpMV of the transpose."""
    g = dpc.gen_rmat(scale, 16, seed=1, weights=False)
    ref = orc.pagerank(g.rowptr, g.col, iters, 0.85)
    pg = dpc.PageRankGraph(ctx, g)
    res = _variants(ctx, reps, lambda v, m: pg.run(iters, 0.85, v, metrics=m),
                    lambda: bool(np.max(np.abs(pg.rank() - ref) / ref) <= 1e-4),
                    lambda met: {"iterations": iters})
    pg.close()
    out = _summ(res, iters * g.m, "teps")
    out.update({"workload": f"PageRank R-MAT scale {scale} directed ({g.m} arcs), {iters} iterations, d = 0.85",
                "unit": "GTEPS (arcs x iterations / time)", "check": "max rel err vs fp64 oracle <= 1e-4"})
    for r in out["variants"].values():
        if "bit_exact" in r:
            r["within_1e-4"] = r.pop("bit_exact")
    return out


def app_gc(ctx, orc, reps, scale=20):
    g = dpc.gen_rmat(scale, 16, seed=1, weights=False, symmetric=True)
    ref, k = orc.color(g.rowptr, g.col, 1)
    dg = dpc.DeviceGraph(ctx, g)
    res = _variants(ctx, reps, lambda v, m: dg.color(1, v, metrics=m),
                    lambda: np.array_equal(dg.get_color(), ref),
                    lambda met: {"colors": met.result_count, "rounds": met.iterations})
    dg.close()
    out = _summ(res, 2 * g.m, "teps")
    out.update({"workload": f"GC R-MAT scale {scale} symmetrized ({g.m} arcs), JP priorities mix64(v^1)",
                "unit": "G scanned arcs/s (2 scans per arc)", "colors": k, "arcs": g.m})
    return out


def app_tree(ctx, orc, reps, which, shape=TREE):
    t = dpc.gen_tree(shape["depth"], shape["lo"], shape["hi"], shape["fill"], shape["seed"])
    ref = orc.tree_desc(t.parent) if which == "tree_desc" else orc.tree_height(t.parent)
    dt = dpc.DeviceTree(ctx, t)
    res = _variants(ctx, reps, lambda v, m: dt.run(which, v, metrics=m),
                    lambda: np.array_equal(dt.result(), ref),
                    lambda met: {"levels": met.iterations})
    dt.close()
    out = _summ(res, t.n - 1, "edges_per_s")
    out.update({"workload": f"{which}: gen_tree({shape['depth']}, {shape['lo']}, {shape['hi']}, "
                            f"{shape['fill']}, {shape['seed']}) = {t.n} nodes, depth {t.depth}",
                "unit": "G tree edges/s"})
    return out


def run_apps(ctx, apps, reps=3):
    from tests._oracle import Oracle
    orc = Oracle()
    out = {}
    for a in apps:
        t0 = time.time()
        if a == "sssp":
            out[a] = app_sssp(ctx, orc, reps)
        elif a == "gc":
            out[a] = app_gc(ctx, orc, reps)
        elif a == "bfs":
            out[a] = app_bfs(ctx, orc, reps)
        elif a == "pr":
            out[a] = app_pr(ctx, orc, reps)
        elif a in ("td", "th"):
            out[a] = app_tree(ctx, orc, reps, "tree_desc" if a == "td" else "tree_height")
        elif a in ("td_paper", "th_paper"):
            out[a] = app_tree(ctx, orc, reps, "tree_desc" if a == "td_paper" else "tree_height",
                              TREE_PAPER)
        elif a in ("td_deep_fit", "th_deep_fit"):
            out[a] = app_tree(ctx, orc, reps, "tree_desc" if a == "td_deep_fit" else "tree_height",
                              TREE_DEEP_FIT)
        out[a]["wall_s"] = round(time.time() - t0, 1)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--apps", nargs="*", default=["sssp", "bfs", "pr", "gc", "td", "th", "td_paper", "th_paper",
                                                  "td_deep_fit", "th_deep_fit"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    ctx = dpc.Context(0)
    r = run_apps(ctx, a.apps, a.reps)
    print(json.dumps(r, indent=1))
    if a.json:
        with open(a.json, "w") as f:
            json.dump(r, f, indent=1)
