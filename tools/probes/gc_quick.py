import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_1606_08150_b200 as dpc
from tests._oracle import Oracle
orc = Oracle(); ctx = dpc.Context(0)
for scale in [8, 12, 16, 20]:
    g = dpc.gen_rmat(scale, 16, seed=1, weights=False, symmetric=True)
    ref, nref = orc.color(g.rowptr, g.col, 1)
    dg = dpc.DeviceGraph(ctx, g)
    for v in ['grid']:
        t0 = time.time(); met = dg.color(1, v); t1 = time.time()
        c = dg.get_color()
        ctx.flush_l2(); ctx.record(0); dg.color(1, v, metrics=False); ctx.record(1)
        print(scale, v, 'exact', np.array_equal(c, ref), 'colors', met.result_count, nref, 'ms', round(ctx.elapsed_ms(0,1),3), flush=True)
    dg.close()
