import sys, numpy as np
sys.path.insert(0, '.')
import paper_1606_08150_b200 as dpc
ctx = dpc.Context(0)
g = dpc.gen_rmat(16, 16, seed=1)
s = int(np.argmax(g.degrees()))
dg = dpc.DeviceGraph(ctx, g)
for flags in [0, 4, 2]:
    cfg = dpc.launch_cfg('sssp', 'grid'); cfg.flags |= flags
    met = dg.sssp(s, 'grid', cfg=cfg)
    ctx.flush_l2(); ctx.record(0); dg.sssp(s, 'grid', cfg=cfg, metrics=False); ctx.record(1)
    print('flags', flags, 'iters', met.iterations, 'ms', ctx.elapsed_ms(0,1), 'items', met.buffer_items_inserted, flush=True)
