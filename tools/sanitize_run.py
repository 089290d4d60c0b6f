"""Small runs of every app x variant (and every grid form) for
compute-sanitizer (tools/gpu/sanitize.sh): memcheck / racecheck / synccheck /
initcheck.  Each run is checked against the oracle; exits non-zero on a
mismatch.  Persistent grid kernels run in both barrier forms (software
barrier on a co-resident normal launch, and cooperative launch + grid.sync).

usage: python tools/sanitize_run.py [--apps ...] [--quick]"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1606_08150_b200 as dpc  # noqa: E402
from tests._oracle import Oracle  # noqa: E402

VARIANTS = ["flat", "basic", "warp", "block", "grid"]
COOP = 4


def cfgs(app, v):
    """(name, cfg) pairs to run for one variant: every grid form."""
    base = dpc.launch_cfg(app, v)
    out = [(v, base)]
    if v != "grid":
        return out
    coop = dpc.launch_cfg(app, v)
    coop.flags |= COOP
    out.append(("grid+coop", coop))
    out.append(("grid_cdp", dpc.launch_cfg(app, v, grid_cdp=True)))
    if app == "sssp":
        out.append(("grid_stream", dpc.launch_cfg(app, v, grid_stream=True)))
        out.append(("grid_level", dpc.launch_cfg(app, v, grid_level=True)))
        out.append(("grid_async", dpc.launch_cfg(app, v, grid_async=True)))
    if app == "color":
        out.append(("grid_rounds", dpc.launch_cfg(app, v, grid_async=False)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--apps", nargs="*", default=["spmv", "sssp", "bfs", "color", "tree_desc", "tree_height"])
    ap.add_argument("--scale", type=int, default=9)
    a = ap.parse_args()
    ctx, orc = dpc.Context(0), Oracle()
    bad = 0
    for app in a.apps:
        if app in ("spmv",):
            g = dpc.gen_rmat(a.scale, 16, seed=2, weights=False, values=True)
            x = ((np.arange(g.n) % 89) + 1).astype(np.float32) / 89
            y64 = orc.spmv_f64(g.rowptr, g.col, g.val, x)
            for v in VARIANTS:
                for name, cfg in cfgs("spmv", v):
                    y, _ = dpc.run_spmv(g, x, cfg=cfg, ctx=ctx)
                    ok = bool(np.all(np.abs(y - y64) <= 1e-5 * np.abs(y64)))
                    bad += not ok
                    print(f"spmv {name}: {'ok' if ok else 'MISMATCH'}", flush=True)
        elif app in ("sssp", "bfs"):
            g = dpc.gen_rmat(a.scale, 16, seed=3, weights=app == "sssp")
            s = int(np.argmax(g.degrees()))
            ref = orc.sssp(g.rowptr, g.col, g.w, s) if app == "sssp" else orc.bfs(g.rowptr, g.col, s)
            for v in VARIANTS:
                for name, cfg in cfgs("sssp", v):
                    if app == "bfs" and name == "grid_async":
                        continue
                    fn = dpc.run_sssp if app == "sssp" else dpc.run_bfs
                    d, _ = fn(g, s, cfg=cfg, ctx=ctx)
                    ok = bool(np.array_equal(d, ref))
                    bad += not ok
                    print(f"{app} {name}: {'ok' if ok else 'MISMATCH'}", flush=True)
        elif app == "color":
            g = dpc.gen_rmat(a.scale, 16, seed=4, weights=False, symmetric=True)
            ref, k = orc.color(g.rowptr, g.col, 1)
            for v in VARIANTS:
                for name, cfg in cfgs("color", v):
                    c, kk, _ = dpc.run_color(g, 1, cfg=cfg, ctx=ctx)
                    ok = bool(np.array_equal(c, ref)) and kk == k
                    bad += not ok
                    print(f"color {name}: {'ok' if ok else 'MISMATCH'}", flush=True)
        else:
            t = dpc.gen_tree(8, 1, 4, 0.8, 2)
            ref = orc.tree_desc(t.parent) if app == "tree_desc" else orc.tree_height(t.parent)
            fn = dpc.run_tree_desc if app == "tree_desc" else dpc.run_tree_height
            for v in VARIANTS:
                for name, cfg in cfgs(app, v):
                    r, _ = fn(t, cfg=cfg, ctx=ctx)
                    ok = bool(np.array_equal(r, ref))
                    bad += not ok
                    print(f"{app} {name}: {'ok' if ok else 'MISMATCH'}", flush=True)
    ctx.close()
    print(f"sanitize_run: {bad} mismatches", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
