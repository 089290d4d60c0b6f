"""SSSP config 1 level form: cooperative-launch grid.sync (launch-table
default, DPC_CFG_COOP_LAUNCH) vs the software barrier; bit-exact check."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))))
import paper_1606_08150_b200 as dpc  # noqa: E402
from tests._oracle import Oracle  # noqa: E402

orc = Oracle()
ctx = dpc.Context(0)
for scale in (16, 18):
    g = dpc.gen_rmat(scale, 16, seed=1)
    s = int(np.argmax(g.degrees()))
    ref = orc.sssp(g.rowptr, g.col, g.w, s)
    dg = dpc.DeviceGraph(ctx, g)
    for name, toggle in (("coop grid.sync", 0), ("soft barrier", 4)):
        cfg = dpc.launch_cfg("sssp", "grid")
        cfg.flags ^= toggle
        for app in ("sssp", "bfs"):
            run = (lambda: dg.sssp(s, "grid", cfg=cfg, metrics=False)) if app == "sssp" else \
                  (lambda: dg.bfs(s, "grid", cfg=cfg, metrics=False))
            run()
            ok = np.array_equal(dg.get_dist(), ref if app == "sssp" else orc.bfs(g.rowptr, g.col, s))
            ts = []
            for _ in range(7):
                ctx.flush_l2(); ctx.record(0); run(); ctx.record(1); ts.append(ctx.elapsed_ms(0, 1))
            print(f"scale {scale} {app:4s} {name:15s} exact={ok} min {min(ts):.4f} ms mean {np.mean(ts):.4f}", flush=True)
    dg.close()
