"""Runs the grid variant of SSSP (config 1), GC (config 3) and TD / TH
(config 4, depth-24 tree) a few times each -- the command the round's ncu
launch list and full captures are taken on."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_08150_b200 as dpc  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ctx = dpc.Context(0)
g = dpc.gen_rmat(16, 16, seed=1)
dg = dpc.DeviceGraph(ctx, g)
s = int(np.argmax(g.degrees()))
for _ in range(reps):
    dg.sssp(s, "grid")
dg.close()
g = dpc.gen_rmat(20, 16, seed=1, weights=False, symmetric=True)
dg = dpc.DeviceGraph(ctx, g)
for _ in range(reps):
    dg.color(1, "grid")
dg.close()
t = dpc.gen_tree(24, 1, 4, 0.84, 1)
dt = dpc.DeviceTree(ctx, t)
for _ in range(reps):
    dt.run("tree_desc", "grid")
    dt.run("tree_height", "grid")
ctx.synchronize()
print("done")
