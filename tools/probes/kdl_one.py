"""One compiled .kdl program run (for ncu): python tools/probes/kdl_one.py spmv grid"""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_1606_08150_b200 as dpc
import paper_1606_08150_b200.kdl as kdl
prog, mode = sys.argv[1], sys.argv[2]
if prog == "spmv":
    g = dpc.gen_rmat(18, 16, seed=7, weights=False, values=True)
    x = ((np.arange(g.n) % 97) + 1) / 128.0
    mod = kdl.compile(kdl.read_program("spmv.kdl"), mode, name="spmv")
    for _ in range(2):
        r = mod.run({"n": g.n, "m": g.m, "nx": g.n, "thr": 32}, {"rowptr": g.rowptr, "col": g.col, "val": g.val, "x": x},
                    timed=True)
        print(mode, r.ms, r.launches)
