import sys, numpy as np
sys.path.insert(0, '.')
import paper_1606_08150_b200 as dpc
ctx = dpc.Context(0)
for scale in [16, 20]:
    g = dpc.gen_rmat(scale, 16, seed=1, weights=False, symmetric=True)
    dg = dpc.DeviceGraph(ctx, g)
    dg.color(1, 'grid')
    ts = []
    for _ in range(3):
        ctx.flush_l2(); ctx.record(0); dg.color(1, 'grid', metrics=False); ctx.record(1); ts.append(ctx.elapsed_ms(0, 1))
    print(scale, 'ms', round(min(ts), 3), flush=True)
    dg.close()
