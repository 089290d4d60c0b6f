"""Probe: SpMV grid forms (stream kernel vs cached-plan kernel): parity vs
the fp64 oracle and device time (L2 flushed) on config 2 and other shapes."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1606_08150_b200 as dpc  # noqa: E402
from tests._oracle import Oracle  # noqa: E402

orc = Oracle()
ctx = dpc.Context(0)
for arg in sys.argv[1:] or ["20", "20:p", "24:p", "12", "16"]:
    scale, perm = int(arg.split(":")[0]), arg.endswith(":p")
    g = dpc.gen_rmat(scale, 16, seed=1, weights=False, values=True, permute=perm)
    x = (np.random.default_rng(1).integers(1, 1 << 24, g.n) / float(1 << 24)).astype(np.float32)
    y64 = orc.spmv_f64(g.rowptr, g.col, g.val, x)
    dg = dpc.DeviceGraph(ctx, g)
    dg.set_x(x)
    res = {"scale": arg, "nnz": g.m}
    reg = dpc.launch_cfg("spmv", "grid")
    reg.flags |= 1 << 9
    tma = dpc.launch_cfg("spmv", "grid")
    tma.flags |= 1 << 12
    for name, cfg in (("stream", dpc.launch_cfg("spmv", "grid", spmv_stream=True)), ("plan8", dpc.launch_cfg("spmv", "grid")),
                      ("plan_reg", reg), ("plan_tma", tma)):
        t0 = time.time()
        dg.spmv("grid", cfg=cfg, metrics=True)
        first_s = time.time() - t0
        y = dg.get_y().astype(np.float64)
        err = float(np.max(np.abs(y - y64) / np.maximum(np.abs(y64), 1e-30)))
        ts = []
        for _ in range(20):
            ctx.flush_l2()
            ctx.record(0)
            dg.spmv("grid", cfg=cfg)
            ctx.record(1)
            ts.append(ctx.elapsed_ms(0, 1))
        dg.check()
        ms = float(np.mean(ts))
        byt = g.m * 8 + (g.n + 1) * 4 + 8 * g.n
        res[name] = {"ms": round(ms, 4), "max_rel_err": err, "ok": err <= 1e-5, "gteps": round(g.m / ms / 1e6, 1),
                     "frac": round(byt / ms / 1e6 / 6549.1, 3), "first_call_s": round(first_s, 3)}
    dg.close()
    print(json.dumps(res), flush=True)
