"""SSSP config 1: levels, relaxed edges and time of the grid forms."""
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
def coop():
    c = dpc.launch_cfg("sssp", "grid")
    c.flags = c.flags ^ 4   # DPC_CFG_COOP_LAUNCH toggled
    return c


for name, cfg in [("grid soft", None), ("grid coop-toggled", coop()),
                  ("grid two-barrier", dpc.launch_cfg("sssp", "grid", grid_chunked=True)),
                  ("block", dpc.launch_cfg("sssp", "block"))]:
    v = "block" if name == "block" else "grid"
    met = dg.sssp(s, v, cfg=cfg)
    ok = np.array_equal(dg.get_dist(), ref)
    ts = []
    for _ in range(5):
        ctx.flush_l2(); ctx.record(0); dg.sssp(s, v, cfg=cfg, metrics=False); ctx.record(1); ts.append(ctx.elapsed_ms(0, 1))
    print(f"{name:18s} exact={ok} ms={min(ts):.4f} iterations={met.iterations} relaxed={met.edges_processed} "
          f"launches={met.child_launch_count}", flush=True)
dg.close(); ctx.close()
