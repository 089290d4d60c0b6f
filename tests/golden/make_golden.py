"""Generates the golden fixtures in this directory by running the REFERENCE
itself: the unmodified dpcons simulator (oracle/_ref/libref_sim.so, compiled
in place from /root/reference/proj/include) executing our .kdl formulations
(paper_1606_08150_b200/kdl/programs/) in basic / warp / block / grid mode.  Run here (the container
with /root/reference); the JSON fixtures are committed so the CPU tests can
pin oracle/oracle.c without the reference present.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import paper_1606_08150_b200 as dpc  # noqa: E402
from tests._oracle import RefSim  # noqa: E402

MODES = ["basic", "warp", "block", "grid"]
INF = 2**40


def run_fix(ref, src, mode, scal, ints, floats, out, n, is_float, fixpoint):
    cur = ints.get(out) if not is_float else None
    runs = 0
    metrics = None
    while True:
        rc, res, met, err = ref.run(src, mode, scal, ints, floats, out=out, out_len=n, out_float=is_float)
        if rc != 0:
            raise RuntimeError(f"{mode}: {err}")
        runs += 1
        metrics = metrics or met
        if not fixpoint or np.array_equal(res, cur):
            return res, metrics, runs
        cur = res
        ints = dict(ints)
        ints[out] = res


def spmv_cases(ref):
    src = ref.kdl("spmv.kdl")
    cases = []
    for scale, seed in [(6, 1), (8, 2)]:
        g = dpc.gen_rmat(scale, 8, seed=seed, weights=False, values=True)
        x = ((np.arange(g.n) * 7919 % 1000) + 1).astype(np.float32) / 1000.0
        outs = {}
        for mode in MODES:
            y, met, _ = run_fix(ref, src, mode, {"n": g.n, "m": g.m, "nx": g.n, "thr": 32},
                                {"rowptr": g.rowptr, "col": g.col},
                                {"val": g.val.astype(np.float64), "x": x.astype(np.float64)},
                                "y", g.n, True, False)
            outs[mode] = {"y": y.tolist(), "childLaunchCount": met["childLaunchCount"]}
        cases.append({"scale": scale, "seed": seed, "rowptr": g.rowptr.tolist(),
                      "col": g.col.tolist(), "val": g.val.tolist(), "x": x.tolist(), "ref": outs})
    return cases


def sssp_cases(ref):
    src = ref.kdl("sssp.kdl")
    cases = []
    for scale, ef, seed in [(6, 8, 3), (8, 8, 4)]:
        g = dpc.gen_rmat(scale, ef, seed=seed)
        s = int(np.argmax(g.degrees()))
        outs = {}
        for mode in MODES:
            dist = np.full(g.n, INF, np.int64)
            dist[s] = 0
            d, met, sweeps = run_fix(ref, src, mode, {"n": g.n, "m": g.m, "thr": 32},
                                     {"rowptr": g.rowptr, "col": g.col, "w": g.w, "dist": dist},
                                     {}, "dist", g.n, False, True)
            d = np.where(d >= INF, 2**32 - 1, d)
            outs[mode] = {"dist": d.tolist(), "sweeps": sweeps,
                          "childLaunchCount": met["childLaunchCount"]}
        cases.append({"scale": scale, "seed": seed, "source": s, "rowptr": g.rowptr.tolist(),
                      "col": g.col.tolist(), "w": g.w.tolist(), "ref": outs})
    return cases


def tree_cases(ref):
    cases = []
    for shape in [(4, 2, 5, 0.9, 1), (6, 1, 4, 0.8, 2)]:
        t = dpc.gen_tree(*shape)
        rec = {"shape": list(shape), "parent": t.parent.tolist(), "ref": {}}
        for name, out, fix in [("td.kdl", "desc", False), ("th.kdl", "height", True)]:
            src = ref.kdl(name)
            for mode in MODES:
                r, met, runs = run_fix(ref, src, mode,
                                       {"n": t.n, "root": t.root, "rootnc": len(t.children(t.root))},
                                       {"cstart": t.cstart, "clist": t.clist, "parent": t.parent,
                                        out: np.zeros(t.n, np.int64)}, {}, out, t.n, False, fix)
                rec["ref"].setdefault(mode, {})[out] = r.tolist()
                rec["ref"][mode][f"{out}_childLaunchCount"] = met["childLaunchCount"]
        cases.append(rec)
    return cases


def main():
    ref = RefSim()
    data = {
        "generator": "tests/golden/make_golden.py (reference dpcons simulator via oracle/_ref)",
        "spmv": spmv_cases(ref),
        "sssp": sssp_cases(ref),
        "tree": tree_cases(ref),
        "policy": {
            "kc_config": [[b, t, x, *ref.kc_config(b, t, x)]
                          for b, t, x in [(64, 256, 16), (64, 256, 1), (20, 128, 32), (104, 256, 16),
                                          (1184, 256, 1), (1184, 256, 16), (1184, 256, 32)]],
            "per_buffer_size": [[a, b, c, ref.per_buffer_size(a, b, c)]
                                for a, b, c in [(1024, 1, 4), (256, 2, 4), (32, 3, 4), (256, 3, 8)]],
        },
    }
    with open(os.path.join(HERE, "reference_runs.json"), "w") as f:
        json.dump(data, f, separators=(",", ":"))
    print("wrote", os.path.join(HERE, "reference_runs.json"))


if __name__ == "__main__":
    main()
