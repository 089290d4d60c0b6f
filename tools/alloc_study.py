"""Allocator study (Fig. 5; memplan.hpp:45-58):
warp- and block-consolidated SpMV with per-owner buffers from the
pre-allocated pool (default) vs the CUDA device heap (malloc in the parent,
free in a tail-launched grid), device-timed, checked against fp64."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_08150_b200 as dpc  # noqa: E402
from tests._oracle import Oracle  # noqa: E402

ctx = dpc.Context(0)
orc = Oracle()
out = []
for scale in (16, 20):
    g = dpc.gen_rmat(scale, 16, seed=1, weights=False, values=True)
    x = (np.arange(g.n, dtype=np.float32) % 97 + 1) / 97.0
    y64 = orc.spmv_f64(g.rowptr, g.col, g.val, x)
    dg = dpc.DeviceGraph(ctx, g)
    dg.set_x(x)
    for v in ("warp", "block"):
        for alloc, flag in (("pool", 0), ("malloc", 16)):
            cfg = dpc.launch_cfg("spmv", v)
            cfg.flags |= flag
            met = dg.spmv(v, cfg=cfg, metrics=True)
            ok = bool(np.all(np.abs(dg.get_y().astype(np.float64) - y64) <= 1e-5 * np.abs(y64)))
            ts = []
            for _ in range(5):
                ctx.flush_l2()
                ctx.record(0)
                dg.spmv(v, cfg=cfg)
                ctx.record(1)
                ts.append(ctx.elapsed_ms(0, 1))
            r = {"scale": scale, "variant": v, "allocator": alloc, "ms": round(float(np.median(ts)), 4),
                 "launches": int(met.child_launch_count), "ok": ok}
            out.append(r)
            print(json.dumps(r), flush=True)
    dg.close()
for scale in (16, 20):
    for v in ("warp", "block"):
        p = [r for r in out if r["scale"] == scale and r["variant"] == v]
        print(f"scale {scale} {v}: malloc / pool = {p[1]['ms'] / p[0]['ms']:.2f}x")
