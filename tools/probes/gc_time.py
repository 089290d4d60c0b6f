"""GC config 3 grid: device time of the whole run (ctx events)."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_1606_08150_b200 as dpc
ctx = dpc.Context(0)
g = dpc.gen_rmat(20, 16, seed=1, weights=False, symmetric=True)
dg = dpc.DeviceGraph(ctx, g)
dg.color(1, "grid")
for _ in range(3):
    ctx.flush_l2(); ctx.record(0); dg.color(1, "grid", metrics=False); ctx.record(1)
    print("grid ms", round(ctx.elapsed_ms(0, 1), 3), flush=True)
dg.close(); ctx.close()
