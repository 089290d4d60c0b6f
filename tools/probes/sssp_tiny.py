import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_1606_08150_b200 as dpc
from tests._oracle import Oracle
orc = Oracle(); ctx = dpc.Context(0)
flags = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for scale in [6]:
    g = dpc.gen_rmat(scale, 16, seed=1)
    s = int(np.argmax(g.degrees()))
    cfg = dpc.launch_cfg('sssp', 'grid'); cfg.flags |= flags
    t0 = time.time()
    try:
        d, met = dpc.run_sssp(g, s, 'grid', cfg=cfg, ctx=ctx)
        print(scale, flags, 'ok', np.array_equal(d, orc.sssp(g.rowptr, g.col, g.w, s)), met.iterations, time.time() - t0, flush=True)
    except dpc.DpcError as e:
        print(scale, flags, 'error', e, time.time() - t0, flush=True)
