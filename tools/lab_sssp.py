"""SSSP / BFS grid-form lab: config 1 (R-MAT scale 16, source = max-degree
vertex) and larger scales; every run checked bit-exact against the oracle.
usage: python tools/lab_sssp.py [--scales 16 22] [--basic] [--reps N]
(DPC_SSSP_PHASES=1 prints the per-level phase timeline of the grid form)"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_08150_b200 as dpc  # noqa: E402
from tests._oracle import Oracle  # noqa: E402  (checker only)

ap = argparse.ArgumentParser()
ap.add_argument("--scales", type=int, nargs="*", default=[16])
ap.add_argument("--basic", action="store_true")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
orc = Oracle()
ctx = dpc.Context(0)


def timed(fn):
    fn()
    ts = []
    for _ in range(a.reps):
        ctx.flush_l2()
        ctx.record(0)
        fn()
        ctx.record(1)
        ts.append(ctx.elapsed_ms(0, 1))
    return min(ts), float(np.mean(ts))


for scale in a.scales:
    g = dpc.gen_rmat(scale, 16, seed=1)
    s = int(np.argmax(g.degrees()))
    dg = dpc.DeviceGraph(ctx, g)
    ref = orc.sssp(g.rowptr, g.col, g.w, s)
    refb = orc.bfs(g.rowptr, g.col, s)
    variants = ["grid", "block"] + (["basic"] if a.basic and scale <= 16 else [])
    for v in variants:
        met = dg.sssp(s, v, metrics=True)
        ok = np.array_equal(dg.get_dist(), ref)
        mn, me = timed(lambda: dg.sssp(s, v, metrics=False))
        print(f"scale {scale} sssp {v:6s} exact={ok} min {mn:.4f} ms mean {me:.4f} ms iters={met.iterations} "
              f"relaxed={met.edges_processed}", flush=True)
        met = dg.bfs(s, v, metrics=True)
        ok = np.array_equal(dg.get_dist(), refb)
        mn, me = timed(lambda: dg.bfs(s, v, metrics=False))
        print(f"scale {scale} bfs  {v:6s} exact={ok} min {mn:.4f} ms mean {me:.4f} ms iters={met.iterations}",
              flush=True)
    dg.close()
