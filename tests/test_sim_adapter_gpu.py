"""the reference-side adapter include/dpc_dpcons.hpp,
compiled against the reference headers (oracle/_ref/libsim_adapter.so, see
oracle/sim_adapter.cpp), runs SpMV / SSSP / BFS / TD / TH on the B200 from a
dpcons::Workload and returns a dpcons::SimResult; the same Workload goes
through the UNMODIFIED reference consolidate() + simulate() (sim.hpp:1746).
The two SimResults must agree global by global: bit-exact for the integer
apps, <= 1e-5 relative for the fp32 SpMV (the simulator computes in fp64)."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_1606_08150_b200 as dpc
from tests._oracle import ORACLE_DIR, RefSim

pytestmark = pytest.mark.gpu
LIB = os.path.join(ORACLE_DIR, "_ref", "libsim_adapter.so")
MODES = {"basic": 0, "warp": 1, "block": 2, "grid": 3}
INF = 1 << 40


@pytest.fixture(scope="module")
def adapter():
    if not os.path.exists(LIB):
        pytest.skip("oracle/_ref/libsim_adapter.so not built (needs the reference headers at build time)")
    L = C.CDLL(LIB)
    P = C.c_void_p
    L.adapter_diff.restype = C.c_int
    L.adapter_diff.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_char_p, C.c_int, C.c_int, P, P, C.c_int, P, P,
                               P, C.c_int, P, P, P, P, P, P, P, C.c_char_p, C.c_int]
    return L


def diff(L, bench, prog, mode, out, fixpoint, scalars, ints, floats):
    keep = []

    def names(keys):
        a = (C.c_char_p * max(1, len(keys)))(*[k.encode() for k in keys])
        keep.append(a)
        return a

    sk = list(scalars)
    sv = (C.c_int64 * max(1, len(sk)))(*[int(scalars[k]) for k in sk])
    ik = list(ints)
    iarrs = [np.ascontiguousarray(ints[k], np.int64) for k in ik]
    ip = (C.c_void_p * max(1, len(ik)))(*[a.ctypes.data for a in iarrs])
    il = (C.c_int64 * max(1, len(ik)))(*[len(a) for a in iarrs])
    fk = list(floats)
    farrs = [np.ascontiguousarray(floats[k], np.float64) for k in fk]
    fp = (C.c_void_p * max(1, len(fk)))(*[a.ctypes.data for a in farrs])
    fl = (C.c_int64 * max(1, len(fk)))(*[len(a) for a in farrs])
    mism, rel = C.c_int64(), C.c_double()
    gl, sl = C.c_int64(), C.c_int64()
    err = C.create_string_buffer(512)
    rc = L.adapter_diff(bench.encode(), RefSim.kdl(prog).encode(), MODES[mode], out.encode(), int(fixpoint),
                        len(sk), names(sk), sv, len(ik), names(ik), ip, il, len(fk), names(fk), fp, fl,
                        C.byref(mism), C.byref(rel), C.byref(gl), C.byref(sl), err, 512)
    assert rc == 0, err.value.decode()
    return mism.value, rel.value, gl.value, sl.value


@pytest.mark.parametrize("mode", list(MODES))
def test_adapter_spmv(adapter, mode):
    g = dpc.gen_rmat(9, 8, seed=3, weights=False, values=True)
    x = ((np.arange(g.n) % 97) + 1) / 97.0
    m, rel, _, _ = diff(adapter, "spmv", "spmv.kdl", mode, "y", False,
                        {"n": g.n, "m": g.m, "nx": g.n, "thr": 32}, {"rowptr": g.rowptr, "col": g.col},
                        {"val": g.val.astype(np.float64), "x": x.astype(np.float32).astype(np.float64),
                         "y": np.zeros(g.n)})
    assert m == 0 and rel <= 1e-5


@pytest.mark.parametrize("mode", list(MODES))
def test_adapter_sssp(adapter, mode):
    g = dpc.gen_rmat(9, 8, seed=5)
    s = int(np.argmax(g.degrees()))
    dist = np.full(g.n, INF, np.int64)
    dist[s] = 0
    m, _, _, _ = diff(adapter, "sssp", "sssp.kdl", mode, "dist", True, {"n": g.n, "m": g.m, "thr": 32},
                      {"rowptr": g.rowptr, "col": g.col, "w": g.w, "dist": dist}, {})
    assert m == 0


@pytest.mark.parametrize("mode", list(MODES))
def test_adapter_bfs(adapter, mode):
    g = dpc.gen_rmat(9, 8, seed=6, weights=False)
    s = int(np.argmax(g.degrees()))
    lev = np.full(g.n, INF, np.int64)
    lev[s] = 0
    m, _, _, _ = diff(adapter, "bfs", "bfs.kdl", mode, "level", True, {"n": g.n, "m": g.m},
                      {"rowptr": g.rowptr, "col": g.col, "level": lev}, {})
    assert m == 0


@pytest.mark.parametrize("which", ["td", "th"])
@pytest.mark.parametrize("mode", list(MODES))
def test_adapter_trees(adapter, which, mode):
    t = dpc.gen_tree(6, 2, 5, 0.6, 3)
    out = "desc" if which == "td" else "height"
    m, _, gl, sl = diff(adapter, which, f"{which}.kdl", mode, out, which == "th",
                        {"n": t.n, "root": t.root, "rootnc": len(t.children(t.root))},
                        {"cstart": t.cstart, "clist": t.clist, "parent": t.parent, out: np.zeros(t.n, np.int64)},
                        {})
    assert m == 0
    if mode == "basic":  # one device launch per internal non-root node on both sides
        internal = int((np.diff(t.cstart) > 0).sum())
        assert gl == internal - 1
