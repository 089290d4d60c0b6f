import sys, numpy as np
sys.path.insert(0, '.')
import paper_1606_08150_b200 as dpc
from tests._oracle import Oracle
orc = Oracle(); ctx = dpc.Context(0)
g = dpc.gen_rmat(20, 16, seed=1, weights=False, symmetric=True)
ref, nref = orc.color(g.rowptr, g.col, 1)
dg = dpc.DeviceGraph(ctx, g)
for k in [0, 1, 2, 3, 4, 5, 6, 8]:
    cfg = dpc.launch_cfg('color', 'grid'); cfg.flags |= k << 24
    met = dg.color(1, 'grid', cfg=cfg)
    ok = np.array_equal(dg.get_color(), ref)
    ts = []
    for _ in range(3):
        ctx.flush_l2(); ctx.record(0); dg.color(1, 'grid', cfg=cfg, metrics=False); ctx.record(1); ts.append(ctx.elapsed_ms(0, 1))
    print('bmax', (256 << k) if k else 2048, 'exact', ok, 'ms', round(min(ts), 3), flush=True)
dg.close(); ctx.close()
