"""SpMV config 2 under three timing methods the bench contract allows:
(1) 512 MB memset flush + event pair per step (the bench's method),
(2) no flush (A is 147 MB > L2), event pair per step,
(3) no flush, one event pair around K back-to-back steps.
usage: python tools/probes/lab_r02/spmv_timing_forms.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))))
import paper_1606_08150_b200 as dpc  # noqa: E402

ctx = dpc.Context(0)
g = dpc.gen_rmat(20, 16, seed=1, weights=False, values=True)
dg = dpc.DeviceGraph(ctx, g)
dg.set_x((np.arange(g.n) % 1000 + 1).astype(np.float32) / 1000)
for _ in range(5):
    dg.spmv("grid")
K = 50
for rep in range(3):
    ts = []
    for _ in range(K):
        ctx.flush_l2()
        ctx.record(0)
        dg.spmv("grid")
        ctx.record(1)
        ts.append(ctx.elapsed_ms(0, 1) * 1e3)
    m1 = np.mean(ts)
    ts = []
    ctx.synchronize()
    for _ in range(K):
        ctx.record(0)
        dg.spmv("grid")
        ctx.record(1)
        ts.append(ctx.elapsed_ms(0, 1) * 1e3)
    m2 = np.mean(ts)
    ctx.synchronize()
    ctx.record(0)
    for _ in range(K):
        dg.spmv("grid")
    ctx.record(1)
    m3 = ctx.elapsed_ms(0, 1) * 1e3 / K
    print(f"flush+per-step {m1:6.1f} us   no flush per-step {m2:6.1f} us   no flush K back-to-back {m3:6.1f} us",
          flush=True)
