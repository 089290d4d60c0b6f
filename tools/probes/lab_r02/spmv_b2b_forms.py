"""Back-to-back SpMV timing forms for K = 10 / 20 / 50: (a) 512 MB flush
enqueued right before the event pair, (b) flush before the W warm-up steps,
synchronize, then the event pair (no flush in front of the region).
usage: python tools/probes/lab_r02/spmv_b2b_forms.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))))
import paper_1606_08150_b200 as dpc  # noqa: E402

ctx = dpc.Context(0)
g = dpc.gen_rmat(20, 16, seed=1, weights=False, values=True)
dg = dpc.DeviceGraph(ctx, g)
dg.set_x((np.arange(g.n) % 1000 + 1).astype(np.float32) / 1000)
for _ in range(3):
    dg.spmv("grid")
for rep in range(3):
    for K in (10, 20, 50):
        ctx.synchronize()
        ctx.flush_l2()
        ctx.record(0)
        for _ in range(K):
            dg.spmv("grid")
        ctx.record(1)
        a = ctx.elapsed_ms(0, 1) * 1e3 / K
        ctx.flush_l2()
        for _ in range(3):
            dg.spmv("grid")
        ctx.synchronize()
        ctx.record(0)
        for _ in range(K):
            dg.spmv("grid")
        ctx.record(1)
        b = ctx.elapsed_ms(0, 1) * 1e3 / K
        print(f"K={K:3d}  (a) flush in front {a:6.1f} us   (b) flush before warm-up, sync {b:6.1f} us", flush=True)
