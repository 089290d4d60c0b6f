import sys, ctypes, numpy as np
sys.path.insert(0, '.')
import paper_1606_08150_b200 as dpc
rt = ctypes.CDLL("libcudart.so.12") if False else None
import torch
ctx = dpc.Context(0)
g = dpc.gen_rmat(12, 16, seed=1, weights=False, values=True)
dg = dpc.DeviceGraph(ctx, g)
dg.set_x(np.ones(g.n, np.float32))
for v in ["basic", "block"]:
    dg.spmv(v); ctx.synchronize()
    torch.cuda.profiler.start()
    dg.spmv(v); ctx.synchronize()
    torch.cuda.profiler.stop()
print("done")
