"""SSSP config 1, grid form: threshold x chunk sweep (min of 5)."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_1606_08150_b200 as dpc
from tests._oracle import Oracle
orc = Oracle(); ctx = dpc.Context(0)
g = dpc.gen_rmat(16, 16, seed=1)
s = int(np.argmax(g.degrees()))
ref = orc.sssp(g.rowptr, g.col, g.w, s)
dg = dpc.DeviceGraph(ctx, g)
for thr in [4, 8, 16, 32, 64]:
    for ch in [32, 64, 128]:
        cfg = dpc.launch_cfg("sssp", "grid", threshold=thr, chunk=ch)
        dg.sssp(s, "grid", cfg=cfg)
        ok = np.array_equal(dg.get_dist(), ref)
        ts = []
        for _ in range(5):
            ctx.flush_l2(); ctx.record(0); dg.sssp(s, "grid", cfg=cfg, metrics=False); ctx.record(1)
            ts.append(ctx.elapsed_ms(0, 1))
        print(f"thr {thr:3d} chunk {ch:4d} exact {ok} ms {min(ts):.4f}", flush=True)
dg.close(); ctx.close()
