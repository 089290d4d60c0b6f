"""Per-vector time of dpc_spmv_host_batch vs batch length (config 2)."""
import ctypes as C
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_1606_08150_b200 as dpc
ctx = dpc.Context(0)
g = dpc.gen_rmat(20, 16, seed=1, weights=False, values=True)
n = g.n
dg = dpc.DeviceGraph(ctx, g)
nb = 4
xs = [np.frombuffer((C.c_float * n).from_address(dpc._lib.dpc_host_alloc(4 * n)), np.float32) for _ in range(nb)]
ys = [np.frombuffer((C.c_float * n).from_address(dpc._lib.dpc_host_alloc(4 * n)), np.float32) for _ in range(nb)]
for x in xs:
    x[:] = (np.arange(n) % 97 + 1) / 97.0
dg.spmv_host_batch(xs[:2], ys[:2])
for k in [1, 2, 4, 10, 20, 40, 80]:
    ts = []
    for _ in range(3):
        ctx.record(0)
        dg.spmv_host_batch([xs[i % nb] for i in range(k)], [ys[i % nb] for i in range(k)])
        ctx.record(1)
        ts.append(ctx.elapsed_ms(0, 1) / k)
    print(f"K={k:3d} ms/vector {min(ts):.4f} GTEPS {g.m / (min(ts) * 1e-3) / 1e9:.1f}", flush=True)
# copy-only reference
import torch
xh = torch.empty(n, dtype=torch.float32).pin_memory(); xd = torch.empty(n, dtype=torch.float32, device="cuda")
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); xd.copy_(xh, non_blocking=True); e1.record(); torch.cuda.synchronize()
print("H2D 4 MB ms", e0.elapsed_time(e1))
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); xh.copy_(xd, non_blocking=True); e1.record(); torch.cuda.synchronize()
print("D2H 4 MB ms", e0.elapsed_time(e1))
dg.close(); ctx.close()
