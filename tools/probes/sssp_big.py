"""Probe: one grid-consolidated SSSP on a large R-MAT graph (for ncu).
usage: python tools/probes/sssp_big.py [scale] [p] [stream]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1606_08150_b200 as dpc  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
perm = "p" in sys.argv[2:]
cfg = dpc.launch_cfg("sssp", "grid", grid_stream="stream" in sys.argv[2:])
ctx = dpc.Context(0)
g = dpc.gen_rmat(scale, 16, seed=1, weights=True, permute=perm)
s = int(np.argmax(g.degrees()))
dg = dpc.DeviceGraph(ctx, g)
for _ in range(int(os.environ.get("REPS", "2"))):
    met = dg.sssp(s, "grid", cfg=cfg, metrics=True)
print("iters", met.iterations, "relaxed", met.edges_processed, "fverts", met.vertices_processed)
