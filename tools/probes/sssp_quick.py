import sys, numpy as np
sys.path.insert(0, '.')
import paper_1606_08150_b200 as dpc
from tests._oracle import Oracle
orc = Oracle(); ctx = dpc.Context(0)
for scale in [8, 12, 16, 20]:
    g = dpc.gen_rmat(scale, 16, seed=1)
    s = int(np.argmax(g.degrees()))
    ref = orc.sssp(g.rowptr, g.col, g.w, s)
    dg = dpc.DeviceGraph(ctx, g)
    for v, cfg in [('grid', None), ('grid-rounds', dpc.launch_cfg('sssp', 'grid', grid_chunked=True)), ('basic', None)]:
        if v == 'basic' and scale > 16: continue
        vv = 'basic' if v == 'basic' else 'grid'
        met = dg.sssp(s, vv, cfg=cfg)
        ok = np.array_equal(dg.get_dist(), ref)
        ts = []
        for _ in range(3):
            ctx.flush_l2(); ctx.record(0); dg.sssp(s, vv, cfg=cfg, metrics=False); ctx.record(1); ts.append(ctx.elapsed_ms(0, 1))
        print(scale, v, 'exact', ok, 'ms', round(min(ts), 4), 'relaxed', met.edges_processed, flush=True)
    dg.close()
