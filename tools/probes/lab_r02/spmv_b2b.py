"""SpMV config 2, K launches back to back after one L2 flush (the bench's
headline timing form); under `ncu --cache-control none` the per-launch DRAM
bytes show whether anything survives in L2 from one step to the next.
usage: python tools/probes/lab_r02/spmv_b2b.py [K]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))))
import paper_1606_08150_b200 as dpc  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ctx = dpc.Context(0)
g = dpc.gen_rmat(20, 16, seed=1, weights=False, values=True)
dg = dpc.DeviceGraph(ctx, g)
dg.set_x((np.arange(g.n) % 1000 + 1).astype(np.float32) / 1000)
for _ in range(3):
    dg.spmv("grid")
ctx.flush_l2()
ctx.record(0)
for _ in range(K):
    dg.spmv("grid")
ctx.record(1)
print(f"{K} back-to-back steps: {ctx.elapsed_ms(0, 1) * 1e3 / K:.1f} us per step")
