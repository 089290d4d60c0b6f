"""Golden fixtures for the .kdl -> CUDA compiler, made by running the
REFERENCE itself (oracle/_ref/libref_sim.so, compiled in place from
/root/reference/proj/include):

* `consolidated`: the reference's consolidate() output (transform.hpp:971,
  printed by unparse.hpp) for every bundled program and every test program
  in warp / block / grid mode — the CPU tests compare this package's
  rewrite with it node for node;
* `runs`: the reference simulator's results for the test programs
  (tests/kdl/*.kdl) on small seeded inputs in basic / warp / block / grid
  mode — the GPU tests run the generated CUDA on the same inputs.

    python tests/golden/make_kdl_golden.py
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
KDL_TESTS = os.path.join(ROOT, "tests", "kdl")
PROGRAMS = os.path.join(ROOT, "paper_1606_08150_b200", "kdl", "programs")


def sources():
    out = {}
    for d in (PROGRAMS, KDL_TESTS):
        for f in sorted(os.listdir(d)):
            if f.endswith(".kdl"):
                with open(os.path.join(d, f)) as fh:
                    out[f] = fh.read()
    return out


def test_inputs():
    """Small seeded CSR inputs for solo / mold / post (scale 7, R-MAT)."""
    g = dpc.gen_rmat(7, 8, seed=11, weights=False, values=True)
    return g


def main():
    ref = RefSim()
    srcs = sources()
    cons = {}
    for name, src in srcs.items():
        for mode in ["warp", "block", "grid"]:
            rc, txt = ref.consolidate_text(src, mode)
            cons.setdefault(name, {})[mode] = txt if rc == 0 else {"error": txt}
    g = test_inputs()
    runs = {"rowptr": g.rowptr.tolist(), "col": g.col.tolist(), "val": g.val.tolist(), "t": 16}
    scal = {"n": g.n, "m": g.m, "t": 16}
    z = np.zeros(g.n, np.int64)
    zm = np.zeros(g.m, np.float64)
    for name, out, ints, floats in [
            ("solo.kdl", "sum", {"rowptr": g.rowptr, "col": g.col, "sum": z}, {}),
            ("mold.kdl", "scaled", {"rowptr": g.rowptr}, {"val": g.val.astype(np.float64), "scaled": zm}),
            ("post.kdl", "out", {"rowptr": g.rowptr, "col": g.col, "cnt": z, "out": z}, {})]:
        is_float = out == "scaled"
        n_out = g.m if is_float else g.n
        for mode in MODES:
            rc, res, met, err = ref.run(srcs[name], mode, scal, ints, floats, out=out, out_len=n_out,
                                        out_float=is_float)
            runs.setdefault(name, {})[mode] = ({"out": res.tolist(), "childLaunchCount": met["childLaunchCount"]}
                                               if rc == 0 else {"error": err})
    # BFS-Rec (bundled bfs.kdl): sweeps to a fixpoint; first-run launches
    gb = dpc.gen_rmat(8, 8, seed=4)
    s = int(np.argmax(gb.degrees()))
    bfs = {"rowptr": gb.rowptr.tolist(), "col": gb.col.tolist(), "src": s}
    for mode in MODES:
        lev = np.full(gb.n, 2**40, np.int64)
        lev[s] = 0
        first = None
        while True:
            rc, res, met, err = ref.run(srcs["bfs.kdl"], mode,
                                        {"n": gb.n, "m": gb.m, "src": s, "srcs": int(gb.rowptr[s]),
                                         "srce": int(gb.rowptr[s + 1])},
                                        {"rowptr": gb.rowptr, "col": gb.col, "level": lev}, {},
                                        out="level", out_len=gb.n)
            if rc != 0:
                raise RuntimeError(err)
            first = met["childLaunchCount"] if first is None else first
            if np.array_equal(res, lev):
                break
            lev = res
        bfs[mode] = {"level": lev.tolist(), "childLaunchCount_first_run": first}
    runs["bfs.kdl"] = bfs
    data = {"generator": "tests/golden/make_kdl_golden.py (reference consolidate() + simulator via oracle/_ref)",
            "consolidated": cons, "runs": runs}
    path = os.path.join(HERE, "kdl_reference.json")
    with open(path, "w") as f:
        json.dump(data, f, separators=(",", ":"))
    print("wrote", path)


if __name__ == "__main__":
    main()
