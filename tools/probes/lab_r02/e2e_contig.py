"""dpc_spmv_host_batch_contig: per-vector time vs group size and batch length (config 2)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))))
import paper_1606_08150_b200 as dpc  # noqa: E402

ctx = dpc.Context(0)
g = dpc.gen_rmat(20, 16, seed=1, weights=False, values=True)
n = g.n
dg = dpc.DeviceGraph(ctx, g)
K = 256
xp, yp = dpc._lib.dpc_host_alloc(4 * n * K), dpc._lib.dpc_host_alloc(4 * n * K)
xs = np.frombuffer((C.c_float * (n * K)).from_address(xp), np.float32).reshape(K, n)
ys = np.frombuffer((C.c_float * (n * K)).from_address(yp), np.float32).reshape(K, n)
xs[:] = (np.arange(n) % 97 + 1) / 97.0
for k in (64, 128, 256):
    for grp in (2, 4, 8, 16, 32):
        dg.spmv_host_batch_contig(xs[:grp], ys[:grp], group=grp)
        ts = []
        for _ in range(3):
            ctx.flush_l2()
            ctx.record(0)
            dg.spmv_host_batch_contig(xs[:k], ys[:k], group=grp)
            ctx.record(1)
            ts.append(ctx.elapsed_ms(0, 1) / k)
        print(f"K={k:3d} group={grp:2d} ms/vector {min(ts):.4f} GTEPS {g.m / (min(ts) * 1e-3) / 1e9:.1f}", flush=True)
