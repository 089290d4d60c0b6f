"""SpMV grid plan form lab: time and check the grid variant over the
cartesian product of environment knobs (DPC_SPMV_HOT_CAP = hot-column slots)
on config 2 (or, with --scale 24
--permute, the config-5 matrix on one GPU).
usage: python tools/lab_spmv_hot.py [--scale S] [--permute] --set DPC_SPMV_HOT_CAP=0,32768 [--flags F]
(timing-probe builds, DPC_LIB_PATH=tools/probes/ab/libdpc_probe.so: --flags (P << 16) selects probe P)"""
import argparse
import itertools
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_08150_b200 as dpc  # noqa: E402
from tests._oracle import Oracle  # noqa: E402  (checker only)

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--permute", action="store_true")
ap.add_argument("--set", action="append", default=[], help="NAME=v1,v2,...")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--flags", type=int, default=0)
a = ap.parse_args()
knobs = [(kv.split("=")[0], kv.split("=")[1].split(",")) for kv in a.set]
ctx = dpc.Context(0)
g = dpc.gen_rmat(a.scale, 16, seed=1, weights=False, values=True, permute=a.permute)
x = (np.arange(g.n) % 1000 + 1).astype(np.float32) / 1000
dg = dpc.DeviceGraph(ctx, g)
dg.set_x(x)
y64 = Oracle().spmv_f64(g.rowptr, g.col, g.val, x) if a.scale <= 22 else None
deg = np.sort(np.bincount(g.col, minlength=g.n))[::-1]
for combo in itertools.product(*[v for _, v in knobs]):
    for (name, _), val in zip(knobs, combo):
        os.environ[name] = val
    cfg = dpc.launch_cfg("spmv", "grid")
    cfg.flags |= a.flags
    dg.spmv("grid", cfg=cfg)  # builds the plan
    ts = []
    for _ in range(a.reps):
        ctx.flush_l2()
        ctx.record(0)
        dg.spmv("grid", cfg=cfg)
        ctx.record(1)
        ts.append(ctx.elapsed_ms(0, 1) * 1e3)
    ok = ""
    if y64 is not None:
        y = dg.get_y()
        err = np.abs(y - y64) / np.maximum(np.abs(y64), 1e-30)
        ok = f"maxrel {err.max():.2e} {'OK' if err.max() <= 1e-5 else 'FAIL'}"
    cap = int(os.environ.get("DPC_SPMV_HOT_CAP", "53248"))
    hit = deg[:cap][deg[:cap] >= 2].sum() / g.m if cap else 0.0
    tag = " ".join(f"{n}={v}" for (n, _), v in zip(knobs, combo))
    print(f"{tag:40s} hit {hit:.3f}  mean {np.mean(ts):7.1f} us  min {np.min(ts):7.1f} us  "
          f"GTEPS {g.m / np.mean(ts) / 1e3:6.1f}  {ok}", flush=True)
