"""Pinned host -> device / device -> host copy bandwidth vs copy size on this box."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))))
import paper_1606_08150_b200 as dpc  # noqa: E402

ctx = dpc.Context(0)
L = dpc._lib
for mb in (1, 4, 16, 64, 256):
    nb = mb << 20
    h = L.dpc_host_alloc(nb)
    d = ctx.alloc(nb)
    for direction in ("h2d", "d2h"):
        ts = []
        for _ in range(5):
            ctx.record(0)
            if direction == "h2d":
                dpc._check(L.dpc_copy_h2d(ctx.handle, d, h, nb))
            else:
                dpc._check(L.dpc_copy_d2h(ctx.handle, h, d, nb))
            ctx.record(1)
            ts.append(ctx.elapsed_ms(0, 1))
        print(f"{mb:4d} MB {direction}: {nb / (min(ts) * 1e-3) / 1e9:6.1f} GB/s", flush=True)
    ctx.free(d)
    L.dpc_host_free(h)
