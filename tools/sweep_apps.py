"""Measured chunk / threshold sweep for SSSP (config 1) and GC (config 3):
median device time per (variant, chunk, threshold), results checked against
the oracle.  Feeds launch_table.inc (the KC_X / buffer-size policy the
reference picks with an occupancy formula, config.hpp:68-84)."""
import argparse
import itertools
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_08150_b200 as dpc  # noqa: E402
from tests._oracle import Oracle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--apps", nargs="*", default=["sssp", "gc"])
ap.add_argument("--variants", nargs="*", default=["grid", "block"])
ap.add_argument("--chunks", nargs="*", type=int, default=[32, 64, 128, 256, 512])
ap.add_argument("--thresholds", nargs="*", type=int, default=[32])
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--json", default=None)
a = ap.parse_args()
ctx = dpc.Context(0)
orc = Oracle()
out = []


def timed(fn):
    fn()
    ts = []
    for _ in range(a.reps):
        ctx.flush_l2()
        ctx.synchronize()
        ctx.record(0)
        fn()
        ctx.record(1)
        ts.append(ctx.elapsed_ms(0, 1))
    return float(np.median(ts))


for app in a.apps:
    if app == "sssp":
        g = dpc.gen_rmat(16, 16, seed=1)
        s = int(np.argmax(g.degrees()))
        ref = orc.sssp(g.rowptr, g.col, g.w, s)
        dg = dpc.DeviceGraph(ctx, g)
        run = lambda cfg: dg.sssp(s, cfg=cfg, metrics=False)  # noqa: E731
        check = lambda: np.array_equal(dg.get_dist(), ref)  # noqa: E731
    else:
        g = dpc.gen_rmat(20, 16, seed=1, weights=False, symmetric=True)
        ref, _ = orc.color(g.rowptr, g.col, 1)
        dg = dpc.DeviceGraph(ctx, g)
        run = lambda cfg: dg.color(1, cfg=cfg, metrics=False)  # noqa: E731
        check = lambda: np.array_equal(dg.get_color(), ref)  # noqa: E731
    for v, chunk, thr in itertools.product(a.variants, a.chunks, a.thresholds):
        cfg = dpc.launch_cfg("sssp" if app == "sssp" else "color", v, chunk=max(32, chunk), threshold=thr)
        try:
            ms = timed(lambda: run(cfg))
            r = {"app": app, "variant": v, "chunk": chunk, "threshold": thr, "ms": round(ms, 4),
                 "ok": bool(check())}
        except dpc.DpcError as e:
            r = {"app": app, "variant": v, "chunk": chunk, "threshold": thr, "error": str(e)}
        out.append(r)
        print(json.dumps(r), flush=True)
    dg.close()
if a.json:
    with open(a.json, "w") as f:
        json.dump(out, f, indent=1)
