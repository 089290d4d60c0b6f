"""Measured launch-configuration sweep for SpMV (config 2) — the B200
replacement of the occupancy-calculator KC_X choice (config.hpp:28-84) and of
the reference's cmd_sweep.

Times each (variant, chunk, kc_x / child_blocks, experiment flags) point with
CUDA events (median of --reps, L2 flushed) and prints one JSON document; the
best point per variant is what configs/launch_cfg.json / launch_table.inc take.
"""
import argparse
import itertools
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_08150_b200 as dpc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--variants", nargs="*", default=["grid", "grid_cdp", "block", "warp"])
ap.add_argument("--chunks", nargs="*", type=int, default=[256, 512, 1024, 2048, 4096])
ap.add_argument("--kcx", nargs="*", type=int, default=[1, 4, 16, 32, 0])
ap.add_argument("--flags", nargs="*", type=int, default=[0, 256, 512, 768, 1024])
ap.add_argument("--thresholds", nargs="*", type=int, default=[32])
ap.add_argument("--json", default=None)
a = ap.parse_args()

ctx = dpc.Context(0)
g = dpc.gen_rmat(a.scale, 16, seed=1, weights=False, values=True)
dg = dpc.DeviceGraph(ctx, g)
x = (np.random.default_rng(1).integers(1, 1 << 24, g.n) / float(1 << 24)).astype(np.float32)
dg.set_x(x)
from tests._oracle import Oracle  # noqa: E402
y64 = Oracle().spmv_f64(g.rowptr, g.col, g.val, x)


def timeit(cfg):
    dg.spmv(cfg=cfg)
    ts = []
    for _ in range(a.reps):
        ctx.flush_l2()
        ctx.record(0)
        dg.spmv(cfg=cfg)
        ctx.record(1)
        ts.append(ctx.elapsed_ms(0, 1))
    y = dg.get_y().astype(np.float64)
    err = np.abs(y - y64) / np.maximum(np.abs(y64), 1e-300)
    ok = bool(np.all(err <= 1e-5))
    if not ok:
        bad = np.argsort(-err)[:5]
        deg = np.diff(g.rowptr)
        print("  worst rows", [(int(r), int(deg[r]), float(y[r]), float(y64[r])) for r in bad],
              "nbad", int((err > 1e-5).sum()), flush=True)
    return float(np.median(ts)), ok


res = []
for v in a.variants:
    base = "grid" if v == "grid_cdp" else v
    if v == "grid":
        space = itertools.product(a.chunks, [1], a.flags, a.thresholds)
    else:
        space = itertools.product(a.chunks, a.kcx, [0], a.thresholds)
    for chunk, kcx, flags, thr in space:
        over = dict(chunk=chunk, kc_x=kcx, threshold=thr)
        cfg = dpc.launch_cfg("spmv", base, **over)
        cfg.flags = flags | (1 if v == "grid_cdp" else 0)
        try:
            ms, ok = timeit(cfg)
        except dpc.DpcError as e:
            res.append({"variant": v, **over, "flags": flags, "error": str(e)})
            continue
        res.append({"variant": v, **over, "flags": flags, "ms": round(ms, 4),
                    "gteps": round(g.m / ms / 1e6, 2), "ok": ok})
        print(json.dumps(res[-1]), flush=True)
best = {}
for r in res:
    if "ms" in r and r["ok"] and (r["variant"] not in best or r["ms"] < best[r["variant"]]["ms"]):
        best[r["variant"]] = r
print(json.dumps({"best": best}, indent=1))
if a.json:
    with open(a.json, "w") as f:
        json.dump({"points": res, "best": best, "scale": a.scale, "nnz": g.m}, f, indent=1)
