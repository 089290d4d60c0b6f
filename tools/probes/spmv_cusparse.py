"""Context only (not a product path): cuSPARSE CSR SpMV (through torch.sparse)
on the config-2 matrix, CUDA-event timed with an L2 flush, to calibrate what a
library kernel reaches on B200."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1606_08150_b200 as dpc  # noqa: E402

g = dpc.gen_rmat(20, 16, seed=1, weights=False, values=True)
dev = torch.device("cuda:0")
crow = torch.from_numpy(g.rowptr.astype(np.int32)).to(dev)
col = torch.from_numpy(g.col.astype(np.int32)).to(dev)
val = torch.from_numpy(g.val).to(dev)
A = torch.sparse_csr_tensor(crow, col, val, size=(g.n, g.n))
x = torch.rand(g.n, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
for _ in range(5):
    y = A @ x
torch.cuda.synchronize()
ts = []
for _ in range(20):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    y = A @ x
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
byts = g.m * 8 + (g.n + 1) * 4 + g.n * 8
print(f"cusparse spmv: {ms*1e3:.1f} us  {g.m/ms/1e6:.1f} GTEPS  {byts/ms/1e6:.0f} GB/s")
