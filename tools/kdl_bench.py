"""Times the compiler's output: the bundled .kdl programs compiled for
sm_100a in basic / warp / block / grid mode, run on the B200 (device time of
the entry launch and everything it launches, CUDA events), next to the
hand-written consolidated kernels of libdpc on the same inputs — the paper's
evaluation done on compiler-generated code.

    python tools/kdl_bench.py [--json out.json] [--scale-spmv 18] [--scale-sssp 16]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1606_08150_b200 as dpc  # noqa: E402
import paper_1606_08150_b200.kdl as kdl  # noqa: E402

MODES = ["basic", "warp", "block", "grid"]
# (mode, drain schedule): "block" is the B200 default, "reference" the
# reference's multi-block drain (transform.hpp:538-566)
RUNS = [("basic", "block"), ("warp", "block"), ("block", "block"), ("grid", "block"),
        ("warp", "reference"), ("block", "reference"), ("grid", "reference")]
INF = 2**40


def key(mode, sch):
    return mode if sch == "block" else f"{mode}/reference-drain"


def best(fn, reps):
    ms = []
    out = None
    for _ in range(reps):
        out = fn()
        ms.append(out.ms)
    return min(ms), out


def spmv(scale, reps, orc, runs=None, width=64):
    g = dpc.gen_rmat(scale, 16, seed=7, weights=False, values=True)
    x = ((np.arange(g.n) % 97) + 1) / 128.0
    want = orc.spmv_f64(g.rowptr, g.col, g.val, x)
    rows = {}
    for mode, sch in runs or RUNS:
        mod = kdl.compile(kdl.read_program("spmv.kdl"), mode, name="spmv", schedule=sch, width=width)
        try:
            ms, res = best(lambda: mod.run({"n": g.n, "m": g.m, "nx": g.n, "thr": 32},
                                           {"rowptr": g.rowptr, "col": g.col, "val": g.val, "x": x},
                                           timed=True), reps)
            err = float(np.max(np.abs(res.arrays["y"] - want) / np.maximum(1e-30, np.abs(want))))
            rows[key(mode, sch)] = {"ms": round(ms, 4), "launches": res.launches, "max_rel_err": err,
                                    "kc": res.kc}
        except Exception as e:  # noqa: BLE001 - report the fault per mode
            rows[key(mode, sch)] = {"error": str(e)[:200]}
    return {"workload": f"spmv.kdl, R-MAT scale {scale} ef 16 ({g.n} rows, {g.m} nnz), thr 32, "
                        f"{'int64 / fp64' if width == 64 else 'int32 / fp32'}", "modes": rows}


def sssp(scale, reps, orc, runs=None):
    g = dpc.gen_rmat(scale, 16, seed=3)
    s = int(np.argmax(g.degrees()))
    want = orc.sssp(g.rowptr, g.col, g.w, s)
    rows = {}
    for mode, sch in runs or RUNS:
        mod = kdl.compile(kdl.read_program("sssp.kdl"), mode, name="sssp", schedule=sch)
        dist = np.full(g.n, INF, np.int64)
        dist[s] = 0
        try:
            ms, res = best(lambda: mod.run({"n": g.n, "m": g.m, "thr": 32},
                                           {"rowptr": g.rowptr, "col": g.col, "w": g.w, "dist": dist},
                                           until_stable="dist", timed=True), reps)
            d = np.where(res.arrays["dist"] >= INF, 2**32 - 1, res.arrays["dist"])
            rows[key(mode, sch)] = {"ms": round(ms, 4), "sweeps": res.runs, "launches": res.launches,
                                    "bit_exact": bool(np.array_equal(d, want.astype(np.int64)))}
        except Exception as e:  # noqa: BLE001
            rows[key(mode, sch)] = {"error": str(e)[:200]}
    return {"workload": f"sssp.kdl (Bellman-Ford sweeps to a fixpoint), R-MAT scale {scale} ef 16 "
                        f"({g.n} V, {g.m} E)", "modes": rows}


def tree(shape, reps, orc, name="td.kdl", out="desc", width=64):
    t = dpc.gen_tree(*shape)
    want = orc.tree_desc(t.parent) if out == "desc" else orc.tree_height(t.parent)
    rows = {}
    for mode in MODES:
        mod = kdl.compile(kdl.read_program(name), mode, name=name[:-4], width=width)
        arrs = {"cstart": t.cstart, "clist": t.clist, "parent": t.parent, out: np.zeros(t.n, np.int64)}
        try:
            ms, res = best(lambda: mod.run({"n": t.n, "root": t.root, "rootnc": len(t.children(t.root))}, arrs,
                                           until_stable=out if out == "height" else None, timed=True), reps)
            rows[mode] = {"ms": round(ms, 4), "launches": res.launches, "runs": res.runs,
                          "bit_exact": bool(np.array_equal(res.arrays[out], want))}
        except Exception as e:  # noqa: BLE001
            rows[mode] = {"error": str(e)[:200]}
    return {"workload": f"{name}, gen_tree{tuple(shape)} = {t.n} nodes, {'int64' if width == 64 else 'int32'}",
            "modes": rows}


def bfs(scale, reps, orc):
    g = dpc.gen_rmat(scale, 16, seed=3)
    s = int(np.argmax(g.degrees()))
    want = orc.bfs(g.rowptr, g.col, s).astype(np.int64)
    rows = {}
    for mode in MODES:
        mod = kdl.compile(kdl.read_program("bfs.kdl"), mode, name="bfs")
        lev = np.full(g.n, INF, np.int64)
        lev[s] = 0
        try:
            ms, res = best(lambda: mod.run({"n": g.n, "m": g.m, "src": s, "srcs": int(g.rowptr[s]),
                                            "srce": int(g.rowptr[s + 1])},
                                           {"rowptr": g.rowptr, "col": g.col, "level": lev},
                                           until_stable="level", timed=True), reps)
            got = np.where(res.arrays["level"] >= INF, 2**32 - 1, res.arrays["level"])
            rows[mode] = {"ms": round(ms, 4), "runs": res.runs, "launches": res.launches,
                          "bit_exact": bool(np.array_equal(got, want))}
        except Exception as e:  # noqa: BLE001
            rows[mode] = {"error": str(e)[:200]}
    return {"workload": f"bfs.kdl (BFS-Rec, recursive, runs to a fixpoint), R-MAT scale {scale} ef 16 "
                        f"({g.n} V, {g.m} E)", "modes": rows}


def hand_written(scale_spmv, scale_sssp, shape):
    """libdpc's hand-written kernels on the same inputs (grid variant)."""
    ctx = dpc.Context(0)
    out = {}
    g = dpc.gen_rmat(scale_spmv, 16, seed=7, weights=False, values=True)
    x = (((np.arange(g.n) % 97) + 1) / 128.0).astype(np.float32)
    dg = dpc.DeviceGraph(ctx, g)
    dg.set_x(x)
    for v in MODES:
        dg.spmv(v)
        ctx.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            dg.spmv(v)
        ctx.synchronize()
        out[f"spmv/{v}"] = round((time.perf_counter() - t0) / 5 * 1e3, 4)
    g = dpc.gen_rmat(scale_sssp, 16, seed=3)
    s = int(np.argmax(g.degrees()))
    dg = dpc.DeviceGraph(ctx, g)
    for v in MODES:
        dg.sssp(s, v)
        ctx.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            dg.sssp(s, v)
        ctx.synchronize()
        out[f"sssp/{v}"] = round((time.perf_counter() - t0) / 3 * 1e3, 4)
    t = dpc.gen_tree(*shape)
    dt = dpc.DeviceTree(ctx, t)
    for v in MODES:
        dt.run("tree_desc", v)
        ctx.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            dt.run("tree_desc", v)
        ctx.synchronize()
        out[f"td/{v}"] = round((time.perf_counter() - t0) / 3 * 1e3, 4)
    ctx.close()
    return out


def summarize(app):
    ms = {k: v["ms"] for k, v in app["modes"].items() if "ms" in v}
    if "basic" in ms:
        best = min((v, k) for k, v in ms.items() if k in ("warp", "block", "grid"))
        app["best_consolidated"] = best[1]
        app["best_vs_basic"] = round(ms["basic"] / best[0], 2)
    return app


def run_compiled(reps=2, scale_spmv=18, scale_sssp=16, shape=(5, 32, 128, 0.4, 1)):
    """bench.py's `kdl` object: the compiler's output for the bundled
    programs (B200 drain schedule), each checked against the oracle."""
    from tests._oracle import Oracle
    orc = Oracle()
    runs = [(m, "block") for m in MODES]
    return {"spmv": summarize(spmv(scale_spmv, reps, orc, runs)),
            "sssp": summarize(sssp(scale_sssp, reps, orc, runs)),
            "td": summarize(tree(list(shape), reps, orc)),
            "bfs": summarize(bfs(scale_sssp, reps, orc)),
            "spmv_w32": summarize(spmv(scale_spmv, reps, orc, runs, width=32)),
            "td_w32": summarize(tree(list(shape), reps, orc, width=32)),
            "note": "generated by paper_1606_08150_b200.kdl from the .kdl programs (int64 / fp64 data, "
                    "CDP2 device launches); device time of the entry launch tree, CUDA events"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json")
    ap.add_argument("--scale-spmv", type=int, default=18)
    ap.add_argument("--scale-sssp", type=int, default=16)
    ap.add_argument("--tree", default="5,32,128,0.4,1")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    from tests._oracle import Oracle
    orc = Oracle()
    shape = [float(v) if "." in v else int(v) for v in a.tree.split(",")]
    res = {"spmv": spmv(a.scale_spmv, a.reps, orc), "sssp": sssp(a.scale_sssp, a.reps, orc),
           "td": tree(shape, a.reps, orc), "bfs": bfs(a.scale_sssp, a.reps, orc),
           "spmv_w32": spmv(a.scale_spmv, a.reps, orc, [(m, "block") for m in MODES], width=32),
           "td_w32": tree(shape, a.reps, orc, width=32)}
    try:
        res["hand_written_wall_ms"] = hand_written(a.scale_spmv, a.scale_sssp, shape)
    except Exception as e:  # noqa: BLE001
        res["hand_written_wall_ms"] = {"error": str(e)[:200]}
    print(json.dumps(res, indent=1))
    if a.json:
        with open(a.json, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
