"""Probe: SSSP / BFS grid forms (level form vs frontier stream form) on R-MAT
graphs of several scales: bit-exactness against the oracle and device time."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1606_08150_b200 as dpc  # noqa: E402
from tests._oracle import Oracle  # noqa: E402

orc = Oracle()
ctx = dpc.Context(0)
threads = os.cpu_count()
for arg in sys.argv[1:] or ["12", "16", "20", "22", "24:p"]:
    scale, perm = int(arg.split(":")[0]), arg.endswith(":p")
    g = dpc.gen_rmat(scale, 16, seed=1, weights=True, permute=perm)
    deg = g.degrees()
    s = int(np.argmax(deg))
    ref, _ = orc.sssp_mt(g.rowptr, g.col, g.w, s, threads)
    mr = int(deg[ref != np.uint32(0xFFFFFFFF)].sum())
    dg = dpc.DeviceGraph(ctx, g)
    res = {"scale": arg}
    forms = {"level": dpc.launch_cfg("sssp", "grid", grid_level=True), "stream": dpc.launch_cfg("sssp", "grid", grid_stream=True)}
    for name, cfg in forms.items():
        met = dg.sssp(s, "grid", cfg=cfg, metrics=True)
        ok = bool(np.array_equal(dg.get_dist(), ref))
        ts = []
        for _ in range(5):
            ctx.flush_l2()
            ctx.record(0)
            dg.sssp(s, "grid", cfg=cfg, metrics=False)
            ctx.record(1)
            ts.append(ctx.elapsed_ms(0, 1))
        dg.check()
        ms = float(np.median(ts))
        res[name] = {"ok": ok, "ms": round(ms, 4), "gteps": round(mr / ms / 1e6, 2), "levels": met.iterations,
                     "relaxed": met.edges_processed, "fverts": met.vertices_processed}
    # BFS through the stream form
    bref = orc.bfs(g.rowptr, g.col, s)
    met = dg.bfs(s, "grid", cfg=forms["stream"], metrics=True)
    res["bfs_stream_ok"] = bool(np.array_equal(dg.get_dist(), bref))
    dg.close()
    print(json.dumps(res), flush=True)
