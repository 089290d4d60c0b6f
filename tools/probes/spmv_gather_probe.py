"""Timing probe (wrong results by design): the plan drains with x gathers
normal / confined to 4 KB / dropped, to split the time between the gathers
and the rest.  Needs the probe build:  make -C paper_1606_08150_b200/csrc probe
  DPC_LIB_PATH=tools/probes/ab/libdpc_probe.so python tools/probes/spmv_gather_probe.py"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1606_08150_b200 as dpc  # noqa: E402

ctx = dpc.Context(0)
g = dpc.gen_rmat(int(sys.argv[1]) if len(sys.argv) > 1 else 20, 16, seed=1, weights=False, values=True)
dg = dpc.DeviceGraph(ctx, g)
dg.set_x((np.random.default_rng(1).integers(1, 1 << 24, g.n) / float(1 << 24)).astype(np.float32))
out = {}
for form, fbits in (("reg", 1 << 9), ("tma", 1 << 12)):
    for probe, pname in ((0, "gathers"), (1, "gathers_4KB"), (2, "no_gathers")):
        cfg = dpc.launch_cfg("spmv", "grid")
        cfg.flags |= fbits | (probe << 10)
        dg.spmv("grid", cfg=cfg)
        ts = []
        for _ in range(20):
            ctx.flush_l2()
            ctx.record(0)
            dg.spmv("grid", cfg=cfg)
            ctx.record(1)
            ts.append(ctx.elapsed_ms(0, 1))
        out[f"{form}/{pname}"] = round(float(np.mean(ts)) * 1e3, 1)
print(json.dumps({"us": out, "lib": dpc.lib_path()}))
