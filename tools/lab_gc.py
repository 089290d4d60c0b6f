"""GC lab: config 3 (R-MAT scale 20 symmetrized) under the hash, canonical
 and largest-log-degree-first orders; time, colors and rounds of
each variant, bit-exact against the oracle under the same order.
usage: python tools/lab_gc.py [--scale S] [--variants grid block ...] [--reps N]"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_08150_b200 as dpc  # noqa: E402
from tests._oracle import Oracle  # noqa: E402  (checker only)

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--variants", nargs="*", default=["grid", "block", "basic"])
ap.add_argument("--orders", nargs="*", default=["hash", "canonical", "llf"])
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--flags", type=int, nargs="*", default=[0], help="extra dpc_launch_cfg.flags values to sweep")
a = ap.parse_args()
orc = Oracle()
ctx = dpc.Context(0)
g = dpc.gen_rmat(a.scale, 16, seed=1, weights=False, symmetric=True)
dg = dpc.DeviceGraph(ctx, g)
for order in a.orders:
    t0 = time.time()
    ref, k = orc.color(g.rowptr, g.col, 1, order={"hash": 0, "canonical": 1, "llf": 2}[order])
    print(f"order {order}: oracle colors {k} ({time.time() - t0:.1f} s)", flush=True)
    for v, fl in [(v, f) for v in a.variants for f in a.flags]:
        cfg = dpc.launch_cfg("color", v, gc_order=order)
        cfg.flags |= fl
        met = dg.color(1, v, cfg=cfg)
        ok = np.array_equal(dg.get_color(), ref)
        ts = []
        for _ in range(a.reps):
            ctx.flush_l2()
            ctx.record(0)
            dg.color(1, v, cfg=cfg, metrics=False)
            ctx.record(1)
            ts.append(ctx.elapsed_ms(0, 1))
        print(f"  {v:6s} flags={fl:#x} exact={ok} colors={met.result_count} rounds={met.iterations} "
              f"launches={met.child_launch_count} min {min(ts):.3f} ms mean {np.mean(ts):.3f} ms", flush=True)
dg.close()
