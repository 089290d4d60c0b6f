"""Probe: single-GPU SpMV and SSSP on large R-MAT graphs (scales 22 / 24),
generation and oracle times, device time per run (CUDA events), parity."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1606_08150_b200 as dpc  # noqa: E402
from tests._oracle import Oracle  # noqa: E402

orc = Oracle()
ctx = dpc.Context(0)
threads = os.cpu_count()
out = {"threads": threads}
for scale, permute in [(int(a.split(":")[0]), a.endswith(":p")) for a in (sys.argv[1:] or ["22", "24:p"])]:
    r = {}
    t0 = time.time()
    g = dpc.gen_rmat(scale, 16, seed=1, weights=True, values=True, permute=permute)
    r["gen_s"] = round(time.time() - t0, 2)
    deg = g.degrees()
    s = int(np.argmax(deg))
    t0 = time.time()
    ref, rounds = orc.sssp_mt(g.rowptr, g.col, g.w, s, threads)
    r["oracle_sssp_mt_s"] = round(time.time() - t0, 2)
    r["oracle_rounds"] = int(rounds)
    reached = ref != np.uint32(0xFFFFFFFF)
    mr = int(deg[reached].sum())
    r["m_reached"] = mr
    t0 = time.time()
    dg = dpc.DeviceGraph(ctx, g)
    r["upload_s"] = round(time.time() - t0, 2)
    for v in ("grid", "block"):
        try:
            met = dg.sssp(s, v, metrics=True)
            ok = bool(np.array_equal(dg.get_dist(), ref))
            ts = []
            for _ in range(3):
                ctx.flush_l2()
                ctx.record(0)
                dg.sssp(s, v, metrics=False)
                ctx.record(1)
                ts.append(ctx.elapsed_ms(0, 1))
            ms = float(np.median(ts))
            r[f"sssp_{v}"] = {"ms": round(ms, 3), "ok": ok, "gteps": round(mr / ms / 1e6, 2),
                             "iters": met.iterations, "relaxed": met.edges_processed}
        except dpc.DpcError as e:
            r[f"sssp_{v}"] = {"error": str(e)}
    x = ((np.arange(g.n) % 97) + 1).astype(np.float32) / 97
    dg.set_x(x)
    t0 = time.time()
    y64 = orc.spmv_f64(g.rowptr, g.col, g.val, x)
    r["oracle_spmv_s"] = round(time.time() - t0, 2)
    dg.spmv("grid")
    y = dg.get_y().astype(np.float64)
    ok = bool(np.all(np.abs(y - y64) <= 1e-5 * np.abs(y64)))
    ts = []
    for _ in range(5):
        ctx.flush_l2()
        ctx.record(0)
        dg.spmv("grid")
        ctx.record(1)
        ts.append(ctx.elapsed_ms(0, 1))
    ms = float(np.mean(ts))
    byt = g.m * 8 + (g.n + 1) * 4 + 8 * g.n
    r["spmv_grid"] = {"ms": round(ms, 4), "ok": ok, "gteps": round(g.m / ms / 1e6, 2),
                      "hbm_frac": round(byt / ms / 1e6 / 6549, 3)}
    dg.close()
    out[f"scale{scale}{'p' if permute else ''}"] = r
    print(json.dumps(out), flush=True)
