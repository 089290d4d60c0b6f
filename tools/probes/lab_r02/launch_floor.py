"""Launch floor of the SpMV plan kernel under the bench's timing method:
probe 5 (return at entry, timing-probe build) after the 512 MB memset flush,
after a flush kernel that runs with the max-shared carveout, and back to back
without a flush.  usage: DPC_LIB_PATH=tools/probes/ab/libdpc_probe.so python tools/probes/lab_r02/launch_floor.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))))
import paper_1606_08150_b200 as dpc  # noqa: E402

ctx = dpc.Context(0)
g = dpc.gen_rmat(20, 16, seed=1, weights=False, values=True)
dg = dpc.DeviceGraph(ctx, g)
dg.set_x((np.arange(g.n) % 1000 + 1).astype(np.float32) / 1000)
for probe in (5, 0):
    cfg = dpc.launch_cfg("spmv", "grid")
    cfg.flags |= probe << 16
    dg.spmv("grid", cfg=cfg)
    for mode in ("memset", "kernel", "none"):
        os.environ["DPC_FLUSH_KERNEL"] = "1" if mode == "kernel" else "0"
        ts = []
        for _ in range(20):
            if mode != "none":
                ctx.flush_l2()
            ctx.record(0)
            dg.spmv("grid", cfg=cfg)
            ctx.record(1)
            ts.append(ctx.elapsed_ms(0, 1) * 1e3)
        print(f"probe {probe} flush {mode:7s}: mean {np.mean(ts):6.1f} us min {np.min(ts):6.1f} us", flush=True)
