"""Runs SpMV variants on the config-2 matrix a few times (for ncu captures).
usage: python tools/prof_spmv.py [variant ...] [--reps N] [--scale S]"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_08150_b200 as dpc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("variants", nargs="*", default=["grid"])
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--cdp", action="store_true")
ap.add_argument("--chunk", type=int, default=0)
ap.add_argument("--flags", type=int, default=0)
ap.add_argument("--threshold", type=int, default=-1)
ap.add_argument("--burst", type=int, default=0)
ap.add_argument("--permute", action="store_true", help="vertex-permuted R-MAT (config 5 shape)")
a = ap.parse_args()
ctx = dpc.Context(0)
g = dpc.gen_rmat(a.scale, 16, seed=1, weights=False, values=True, permute=a.permute)
dg = dpc.DeviceGraph(ctx, g)
dg.set_x((np.arange(g.n) % 1000 + 1).astype(np.float32) / 1000)
for v in a.variants:
    over = {}
    if a.cdp:
        over["grid_cdp"] = True
    if a.chunk:
        over["chunk"] = a.chunk
    if a.threshold >= 0:
        over["threshold"] = a.threshold
    cfg = dpc.launch_cfg("spmv", v, **over)
    cfg.flags |= a.flags
    for _ in range(a.reps):
        ctx.flush_l2()
        ctx.record(0)
        dg.spmv(v, cfg=cfg)
        ctx.record(1)
        print(v, f"{ctx.elapsed_ms(0, 1):.4f} ms")
    if a.burst:
        for nb in (1, a.burst):
            ctx.flush_l2()
            ctx.record(0)
            for _ in range(nb):
                dg.spmv(v, cfg=cfg)
            ctx.record(1)
            print(f"  burst {nb}: {ctx.elapsed_ms(0, 1) / nb * 1e3:.1f} us per run")
    if v == "grid" and not a.cdp:
        ctx.flush_l2()
        dg.spmv(v, cfg=cfg, metrics=True)
        t0, t1, t2 = dg.phase_ns()
        print(f"  phase split: insert+inline {(t1 - t0) / 1e3:.1f} us, drain {(t2 - t1) / 1e3:.1f} us")
ctx.synchronize()
