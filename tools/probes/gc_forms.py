import sys, numpy as np
sys.path.insert(0, '.')
import paper_1606_08150_b200 as dpc
from tests._oracle import Oracle
orc = Oracle(); ctx = dpc.Context(0)
for scale in [8, 12, 16, 20]:
    g = dpc.gen_rmat(scale, 16, seed=1, weights=False, symmetric=True)
    ref, nref = orc.color(g.rowptr, g.col, 1)
    dg = dpc.DeviceGraph(ctx, g)
    for name, extra in [('blocks+warps', 0), ('warps only', 1 << 19)]:
        cfg = dpc.launch_cfg('color', 'grid'); cfg.flags |= extra
        try:
            met = dg.color(1, 'grid', cfg=cfg)
            ok = np.array_equal(dg.get_color(), ref)
            ctx.flush_l2(); ctx.record(0); dg.color(1, 'grid', cfg=cfg, metrics=False); ctx.record(1)
            print(scale, name, 'exact', ok, 'ms', round(ctx.elapsed_ms(0, 1), 3), flush=True)
        except dpc.DpcError as e:
            print(scale, name, 'error', e, flush=True)
    dg.close()
