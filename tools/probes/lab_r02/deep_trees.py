"""Trees deeper than the BASELINE depth-24 bound, every variant: exact or a
clean DpcError (never a wrong result or a hang).  Chain depths 100..2000,
a deep + wide comb."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))))
import paper_1606_08150_b200 as dpc  # noqa: E402
from tests._oracle import Oracle  # noqa: E402

orc = Oracle()
ctx = dpc.Context(0)
cases = {}
for d in (100, 500, 2000):
    cases[f"chain{d}"] = np.concatenate([[-1], np.arange(d - 1)]).astype(np.int32)
# comb: a chain of 300 with 50 leaves on every chain node
par = [-1] + list(range(299))
for v in range(300):
    par += [v] * 50
cases["comb300x50"] = np.array(par, np.int32)
for name, parent in cases.items():
    t = dpc.tree_from_parent(parent)
    for v in ["flat", "basic", "warp", "block", "grid"]:
        for app, fn, ref in (("td", dpc.run_tree_desc, orc.tree_desc), ("th", dpc.run_tree_height, orc.tree_height)):
            try:
                r, _ = fn(t, v, ctx=ctx)
                ok = np.array_equal(r, ref(parent))
                print(f"{name:12s} {app} {v:6s} {'exact' if ok else 'WRONG'}", flush=True)
            except dpc.DpcError as e:
                print(f"{name:12s} {app} {v:6s} refused: {str(e)[:90]}", flush=True)
