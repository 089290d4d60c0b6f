"""Probe for ncu: a few SpMV grid runs of one form on config 2.
usage: python tools/probes/spmv_one.py [plan8|plan_reg|stream] [scale[:p]]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1606_08150_b200 as dpc  # noqa: E402

form = sys.argv[1] if len(sys.argv) > 1 else "plan"
arg = sys.argv[2] if len(sys.argv) > 2 else "20"
g = dpc.gen_rmat(int(arg.split(":")[0]), 16, seed=1, weights=False, values=True, permute=arg.endswith(":p"))
ctx = dpc.Context(0)
dg = dpc.DeviceGraph(ctx, g)
dg.set_x((np.random.default_rng(1).integers(1, 1 << 24, g.n) / float(1 << 24)).astype(np.float32))
cfg = dpc.launch_cfg("spmv", "grid", spmv_stream=form == "stream")
if form == "plan_reg":
    cfg.flags |= 1 << 9
for _ in range(int(os.environ.get("REPS", "3"))):
    ctx.flush_l2()
    dg.spmv("grid", cfg=cfg)
ctx.synchronize()
dg.check()
