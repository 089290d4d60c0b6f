"""Config-4 tree, persistent grid: top-down vs count-down postwork time."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_1606_08150_b200 as dpc
ctx = dpc.Context(0)
for shape in [(24, 1, 4, 0.84, 1), (5, 32, 128, 0.4, 1)]:
    t = dpc.gen_tree(*shape)
    dt = dpc.DeviceTree(ctx, t)
    for which in ["tree_desc", "tree_height"]:
        dt.run(which, "grid")
        for _ in range(3):
            ctx.record(0); dt.run(which, "grid", metrics=False); ctx.record(1)
            ms = ctx.elapsed_ms(0, 1)
            p = dt.phase_ns()
            print(f"{shape} {which}: total {ms * 1e3:.1f} us, top-down {(p[1] - p[0]) / 1e3:.1f} us, "
                  f"postwork {(p[2] - p[1]) / 1e3:.1f} us", flush=True)
    dt.close()
ctx.close()
