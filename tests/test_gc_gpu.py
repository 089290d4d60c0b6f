"""Graph-coloring parity on the B200: every variant returns exactly the
sequential greedy first-fit coloring in canonical node order (
oracle/oracle.c orc_color_greedy_order), which is also checked for validity; the
color count is reported (BASELINE north_star: "a valid coloring with its color
count reported")."""
import numpy as np
import pytest

import paper_1606_08150_b200 as dpc

pytestmark = pytest.mark.gpu

VARIANTS = ["flat", "basic", "warp", "block", "grid"]


def _check(orc, g, seed, color, ncolors):
    ref, k = orc.color(g.rowptr, g.col, seed)
    assert np.array_equal(color, ref)
    assert ncolors == k
    assert orc.color_valid(g.rowptr, g.col, color, ncolors)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("scale", [8, 12, 14])
def test_gc_rmat(ctx, orc, variant, scale):
    g = dpc.gen_rmat(scale, 16, seed=scale, weights=False, symmetric=True)
    color, k, met = dpc.run_color(g, 7, variant, ctx=ctx)
    _check(orc, g, 7, color, k)
    assert met.result_count == k


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("chunk,threshold", [(32, 0), (100, 70), (4096, 32)])
def test_gc_cfg_sweep(ctx, orc, variant, chunk, threshold):
    g = dpc.gen_graph(3000, powerlaw=(1.4, 2900), seed=4, weights=False, symmetric=True)
    cfg = dpc.launch_cfg("color", variant, chunk=chunk, threshold=threshold)
    color, k, _ = dpc.run_color(g, 3, cfg=cfg, ctx=ctx)
    _check(orc, g, 3, color, k)


@pytest.mark.parametrize("variant", VARIANTS)
def test_gc_edge_cases(ctx, orc, variant):
    g = dpc.csr_from_arrays([0, 0], [])
    color, k, _ = dpc.run_color(g, 1, variant, ctx=ctx)
    assert color.tolist() == [0] and k == 1
    # clique of 70 (colors >= 64 exercise the windowed mex) + isolated vertex
    n = 71
    rows = [[j for j in range(70) if j != i] for i in range(70)] + [[]]
    rowptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])])
    g = dpc.csr_from_arrays(rowptr, np.concatenate(rows[:70]).astype(np.int32))
    color, k, _ = dpc.run_color(g, 5, variant, ctx=ctx)
    _check(orc, g, 5, color, k)
    assert k == 70
    # star with a 40k-leaf hub
    leaves = 40_000
    rowptr = np.concatenate([[0, leaves], leaves + np.arange(1, leaves + 1)])
    col = np.concatenate([np.arange(1, leaves + 1), np.zeros(leaves)]).astype(np.int32)
    g = dpc.csr_from_arrays(rowptr, col)
    color, k, _ = dpc.run_color(g, 9, variant, ctx=ctx)
    _check(orc, g, 9, color, k)
    assert k == 2


def test_gc_asymmetric_rejected(ctx):
    g = dpc.csr_from_arrays([0, 1, 1], [1])
    with pytest.raises(dpc.DpcError) as e:
        dpc.run_color(g, 1, "grid", ctx=ctx)
    assert e.value.kind == "invalid"


def test_gc_config3_full(ctx, orc):
    """BASELINE config 3: R-MAT scale 20 symmetrized, warp/block/grid sweep."""
    g = dpc.gen_rmat(20, 16, seed=1, weights=False, symmetric=True)
    ref, k = orc.color(g.rowptr, g.col, 1)
    dg = dpc.DeviceGraph(ctx, g)
    for v in ["flat", "basic", "warp", "block", "grid"]:
        met = dg.color(1, v)
        assert np.array_equal(dg.get_color(), ref), v
        assert met.result_count == k
    dg.close()


def _clique(n):
    rows = [[j for j in range(n) if j != i] for i in range(n)]
    rowptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])])
    return dpc.csr_from_arrays(rowptr, np.concatenate(rows).astype(np.int32))


@pytest.mark.parametrize("form", ["async", "rounds"])
def test_gc_grid_forms(ctx, orc, form):
    """The persistent grid variant's two forms: the asynchronous worklist
    (default) and the round-synchronous one, on heavy vertices (chunk tasks),
    a 1030-clique (colors >= 1024: windowed mex) and R-MAT."""
    cfg = dpc.launch_cfg("color", "grid", grid_async=(form == "async"))
    for g in (_clique(1030), dpc.gen_rmat(15, 16, seed=2, weights=False, symmetric=True),
              dpc.gen_graph(5000, powerlaw=(1.3, 4900), seed=8, weights=False, symmetric=True)):
        color, k, met = dpc.run_color(g, 11, cfg=cfg, ctx=ctx)
        _check(orc, g, 11, color, k)
        assert met.child_launch_count == 0


ORDERS = {"hash": 0, "llf": 2}


@pytest.mark.parametrize("order", list(ORDERS))
@pytest.mark.parametrize("variant", VARIANTS)
def test_gc_orders(ctx, orc, order, variant):
    """The seeded hash order (DPC_CFG_GC_HASH) and largest-log-degree-first
    (DPC_CFG_GC_LLF) -- the canonical default is what every other test checks -- in every variant, both grid
    forms, on R-MAT, a power-law graph with heavy vertices, a 1030-clique and
    a star: bit-identical to the oracle under the same order."""
    graphs = [dpc.gen_rmat(13, 16, seed=3, weights=False, symmetric=True),
              dpc.gen_graph(4000, powerlaw=(1.3, 3900), seed=6, weights=False, symmetric=True),
              _clique(1030)]
    leaves = 5000
    graphs.append(dpc.csr_from_arrays(np.concatenate([[0, leaves], leaves + np.arange(1, leaves + 1)]),
                                      np.concatenate([np.arange(1, leaves + 1), np.zeros(leaves)]).astype(np.int32)))
    forms = [True, False] if variant == "grid" else [None]
    for g in graphs:
        ref, k = orc.color(g.rowptr, g.col, 5, order=ORDERS[order])
        for form in forms:
            kw = {"gc_order": order}
            if form is not None:
                kw["grid_async"] = form
            color, kk, met = dpc.run_color(g, 5, cfg=dpc.launch_cfg("color", variant, **kw), ctx=ctx)
            assert np.array_equal(color, ref), (order, variant, form)
            assert kk == k == met.result_count
            assert orc.color_valid(g.rowptr, g.col, color, kk)


@pytest.mark.parametrize("order", list(ORDERS))
def test_gc_orders_config3_full(ctx, orc, order):
    """BASELINE config 3 (R-MAT scale 20 symmetrized) under the hash and LLF
    orders: every variant bit-exact, color count reported."""
    g = dpc.gen_rmat(20, 16, seed=1, weights=False, symmetric=True)
    ref, k = orc.color(g.rowptr, g.col, 1, order=ORDERS[order])
    dg = dpc.DeviceGraph(ctx, g)
    for v in VARIANTS:
        met = dg.color(1, v, cfg=dpc.launch_cfg("color", v, gc_order=order))
        assert np.array_equal(dg.get_color(), ref), v
        assert met.result_count == k
    dg.close()


def test_gc_orders_exclusive(ctx):
    g = dpc.gen_rmat(8, 8, seed=1, weights=False, symmetric=True)
    cfg = dpc.launch_cfg("color", "grid")
    cfg.flags |= dpc.CFG_GC_HASH | dpc.CFG_GC_LLF
    with pytest.raises(dpc.DpcError) as e:
        dpc.run_color(g, 1, cfg=cfg, ctx=ctx)
    assert e.value.kind == "invalid"
