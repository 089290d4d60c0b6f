"""SSSP parity on the B200: every variant bit-exact against Dijkstra
(oracle/oracle.c), including edge cases (unreachable vertices, zero weights,
self loops, duplicate edges, a single hub)."""
import numpy as np
import pytest

import paper_1606_08150_b200 as dpc

pytestmark = pytest.mark.gpu

VARIANTS = ["flat", "basic", "warp", "block", "grid"]


def _source(g):
    return int(np.argmax(g.degrees()))


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("scale", [8, 12, 14])
def test_sssp_rmat(ctx, orc, variant, scale):
    g = dpc.gen_rmat(scale, 16, seed=scale + 100)
    s = _source(g)
    d, met = dpc.run_sssp(g, s, variant, ctx=ctx)
    assert np.array_equal(d, orc.sssp(g.rowptr, g.col, g.w, s))
    if variant == "flat":
        assert met.child_launch_count == 0


def test_sssp_grid_cdp(ctx, orc):
    g = dpc.gen_rmat(13, 16, seed=9)
    s = _source(g)
    cfg = dpc.launch_cfg("sssp", "grid", grid_cdp=True)
    d, met = dpc.run_sssp(g, s, cfg=cfg, ctx=ctx)
    assert np.array_equal(d, orc.sssp(g.rowptr, g.col, g.w, s))
    assert 1 <= met.child_launch_count <= met.iterations  # <= 1 launch per parent grid


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("chunk,threshold", [(32, 0), (100, 7), (4096, 32)])
def test_sssp_cfg_sweep(ctx, orc, variant, chunk, threshold):
    g = dpc.gen_graph(4000, powerlaw=(1.5, 3000), seed=5, wmin=0, wmax=20)
    cfg = dpc.launch_cfg("sssp", variant, chunk=chunk, threshold=threshold)
    d, _ = dpc.run_sssp(g, 0, cfg=cfg, ctx=ctx)
    assert np.array_equal(d, orc.sssp(g.rowptr, g.col, g.w, 0))


@pytest.mark.parametrize("variant", VARIANTS)
def test_sssp_edge_cases(ctx, orc, variant):
    # single vertex, no edges
    g = dpc.csr_from_arrays([0, 0], [], w=[])
    d, _ = dpc.run_sssp(g, 0, variant, ctx=ctx)
    assert d.tolist() == [0]
    # disconnected + self loop + duplicate edges + zero weight
    g = dpc.csr_from_arrays([0, 3, 4, 4, 5], [0, 1, 1, 2, 3], w=[5, 0, 7, 1, 2])
    d, _ = dpc.run_sssp(g, 0, variant, ctx=ctx)
    assert d.tolist() == [0, 0, 1, 2**32 - 1]
    # hub with 50k out-edges into a chain
    n = 50_001
    rowptr = np.concatenate([[0], np.full(n, n - 1)]).astype(np.int64)
    col = np.arange(1, n, dtype=np.int32)
    w = (np.arange(1, n) % 13 + 1).astype(np.int32)
    g = dpc.csr_from_arrays(rowptr, col, w=w)
    d, _ = dpc.run_sssp(g, 0, variant, ctx=ctx)
    assert np.array_equal(d, orc.sssp(g.rowptr, g.col, g.w, 0))


def test_sssp_config1_full(ctx, orc):
    """BASELINE config 1: R-MAT scale 16, int weights [1,255], all variants."""
    g = dpc.gen_rmat(16, 16, seed=1)
    s = _source(g)
    ref = orc.sssp(g.rowptr, g.col, g.w, s)
    dg = dpc.DeviceGraph(ctx, g)
    for v in VARIANTS:
        met = dg.sssp(s, v)
        assert np.array_equal(dg.get_dist(), ref), v
        assert met.iterations > 0
    dg.close()


def test_sssp_invalid(ctx):
    g = dpc.gen_rmat(6, 4, seed=1)
    with pytest.raises(dpc.DpcError) as e:
        dpc.run_sssp(g, g.n + 5, "grid", ctx=ctx)
    assert e.value.kind == "invalid"
    g2 = dpc.gen_rmat(6, 4, seed=1, weights=False, values=True)
    with pytest.raises(dpc.DpcError):
        dpc.run_sssp(g2, 0, "grid", ctx=ctx)


@pytest.mark.parametrize("form", ["one_barrier", "one_barrier_soft", "two_barrier", "async"])
@pytest.mark.parametrize("scale", [10, 14])
def test_sssp_grid_forms(ctx, orc, form, scale):
    """The persistent grid variant's two forms (level-synchronous default and
    the asynchronous worklist) are bit-exact against Dijkstra, including an
    isolated source and zero-weight edges."""
    g = dpc.gen_rmat(scale, 16, seed=scale + 1, wmin=0, wmax=3)
    cfg = dpc.launch_cfg("sssp", "grid", grid_async=(form == "async"), grid_chunked=(form == "two_barrier"))
    if form == "one_barrier_soft":
        cfg.flags &= ~4                      # normal launch + software grid barrier
    for s in (int(np.argmax(g.degrees())), int(np.flatnonzero(g.degrees() == 0)[0])):
        d, met = dpc.run_sssp(g, s, "grid", cfg=cfg, ctx=ctx)
        assert np.array_equal(d, orc.sssp(g.rowptr, g.col, g.w, s))
        assert met.child_launch_count == 0


@pytest.mark.gpu
def test_async_runs_without_metrics(ctx, orc):
    """Runs without metrics return once enqueued; results and the deferred
    fault check (dpc_dgraph_check / dpc_dtree_check) are read afterwards."""
    g = dpc.gen_rmat(12, 16, seed=4)
    s = int(np.argmax(g.degrees()))
    dg = dpc.DeviceGraph(ctx, g)
    for _ in range(3):
        assert dg.sssp(s, "grid", metrics=False) is None
    dg.check()
    assert np.array_equal(dg.get_dist(), orc.sssp(g.rowptr, g.col, g.w, s))
    dg.close()
    t = dpc.gen_tree(8, 1, 4, 0.8, 2)
    dt = dpc.DeviceTree(ctx, t)
    dt.run("tree_desc", "grid", metrics=False)
    dt.run("tree_desc", "grid", metrics=False)
    assert np.array_equal(dt.result(), orc.tree_desc(t.parent))
    dt.close()


# ---- the frontier stream form of the grid variant (sssp_stream.cu) -------
STREAM = dict(grid_stream=True)


@pytest.mark.parametrize("scale,permute", [(6, False), (10, True), (12, False), (14, True)])
def test_sssp_stream_form_rmat(ctx, orc, scale, permute):
    g = dpc.gen_rmat(scale, 16, seed=scale + 7, permute=permute)
    s = _source(g)
    for coop in (False, True):
        cfg = dpc.launch_cfg("sssp", "grid", **STREAM)
        if coop:
            cfg.flags |= 4  # DPC_CFG_COOP_LAUNCH
        d, met = dpc.run_sssp(g, s, cfg=cfg, ctx=ctx)
        assert np.array_equal(d, orc.sssp(g.rowptr, g.col, g.w, s))
        assert met.child_launch_count == 0 and met.vertices_processed >= 1


def test_sssp_stream_form_edge_cases(ctx, orc):
    cfg = dpc.launch_cfg("sssp", "grid", **STREAM)
    g = dpc.csr_from_arrays([0, 0], [], w=[])
    d, _ = dpc.run_sssp(g, 0, cfg=cfg, ctx=ctx)
    assert d.tolist() == [0]
    g = dpc.csr_from_arrays([0, 3, 4, 4, 5], [0, 1, 1, 2, 3], w=[5, 0, 7, 1, 2])
    d, _ = dpc.run_sssp(g, 0, cfg=cfg, ctx=ctx)
    assert d.tolist() == [0, 0, 1, 2**32 - 1]
    # a hub whose stream spans every warp, then a chain (one vertex per level)
    n = 50_001
    rowptr = np.concatenate([[0], np.full(n, n - 1)]).astype(np.int64)
    col = np.arange(1, n, dtype=np.int32)
    w = (np.arange(1, n) % 13 + 1).astype(np.int32)
    g = dpc.csr_from_arrays(rowptr, col, w=w)
    d, _ = dpc.run_sssp(g, 0, cfg=cfg, ctx=ctx)
    assert np.array_equal(d, orc.sssp(g.rowptr, g.col, g.w, 0))
    chain = 3000
    g = dpc.csr_from_arrays(np.arange(chain + 1).clip(0, chain - 1).astype(np.int64),
                            np.arange(1, chain, dtype=np.int32), w=np.full(chain - 1, 3, np.int32))
    d, met = dpc.run_sssp(g, 0, cfg=cfg, ctx=ctx)
    assert np.array_equal(d, orc.sssp(g.rowptr, g.col, g.w, 0))
    assert met.iterations >= chain - 1


@pytest.mark.parametrize("wmax", [0, 1, 20])
def test_sssp_stream_form_powerlaw(ctx, orc, wmax):
    g = dpc.gen_graph(6000, powerlaw=(1.5, 5000), seed=11, wmin=0, wmax=wmax)
    d, _ = dpc.run_sssp(g, 0, cfg=dpc.launch_cfg("sssp", "grid", **STREAM), ctx=ctx)
    assert np.array_equal(d, orc.sssp(g.rowptr, g.col, g.w, 0))


def test_bfs_stream_form(ctx, orc):
    g = dpc.gen_rmat(13, 16, seed=4, weights=False)
    s = _source(g)
    d, _ = dpc.run_bfs(g, s, cfg=dpc.launch_cfg("sssp", "grid", **STREAM), ctx=ctx)
    assert np.array_equal(d, orc.bfs(g.rowptr, g.col, s))


def test_sssp_scale22_default_grid_is_stream_form(ctx, orc):
    """At >= 2^24 edges the grid default is the stream form: scale 22, bit-exact,
    with the level form forced beside it."""
    import os
    g = dpc.gen_rmat(22, 16, seed=1)
    s = _source(g)
    ref, _ = orc.sssp_mt(g.rowptr, g.col, g.w, s, os.cpu_count() or 1)
    dg = dpc.DeviceGraph(ctx, g)
    met = dg.sssp(s, "grid")
    assert np.array_equal(dg.get_dist(), ref)
    assert met.vertices_processed > 0  # only the stream form counts frontier visits
    dg.sssp(s, "grid", cfg=dpc.launch_cfg("sssp", "grid", grid_level=True))
    assert np.array_equal(dg.get_dist(), ref)
    dg.close()


def test_sssp_on_dimacs_ingested_graph(ctx, orc, tmp_path):
    """A DIMACS 9th-challenge .gr file (the paper's dataset format) through
    dpc_load_dimacs, then every SSSP variant on the GPU: bit-exact."""
    g = dpc.gen_rmat(12, 16, seed=21)
    src = np.repeat(np.arange(g.n), g.degrees())
    p = tmp_path / "g.gr"
    lines = [f"p sp {g.n} {g.m}"] + [f"a {u + 1} {v + 1} {w}" for u, v, w in zip(src, g.col, g.w)]
    p.write_text("\n".join(lines) + "\n")
    h = dpc.load_dimacs(str(p))
    s = int(np.argmax(h.degrees()))
    ref = orc.sssp(h.rowptr, h.col, h.w, s)
    for v in ["flat", "basic", "warp", "block", "grid"]:
        d, _ = dpc.run_sssp(h, s, v, ctx=ctx)
        assert np.array_equal(d, ref), v


@pytest.mark.parametrize("unit", [False, True])
def test_sssp_hub_spills_level_form(ctx, orc, unit):
    """A hub with 2^20 out-edges: its chunk items push more vertices into
    each block's shared queue than it holds (2048), so the level form's
    spill path classifies them (and records their row bounds for the light
    pass) -- then a second hub level and a tail of light vertices."""
    L = 1 << 20
    n = L + 64 + 2
    hub, hub2 = 0, L + 1
    rng = np.random.default_rng(5)
    # hub -> leaves 1..L; every leaf -> hub2, every 64th leaf also -> one of
    # the 64 tail vertices; hub2 -> the 64 tail vertices
    deg = np.ones(n, np.int64)
    deg[hub] = L
    deg[1:L + 1] = 1 + (np.arange(1, L + 1) % 64 == 0)
    deg[hub2] = 64
    deg[L + 2:] = 0
    rowptr = np.concatenate([[0], np.cumsum(deg)])
    col = np.empty(rowptr[-1], np.int64)
    col[:L] = np.arange(1, L + 1)
    leaf_start = rowptr[1:L + 1]
    col[leaf_start] = hub2
    extra = np.nonzero(deg[1:L + 1] == 2)[0] + 1
    col[rowptr[extra] + 1] = L + 2 + (extra // 64) % 64
    col[rowptr[hub2]:rowptr[hub2] + 64] = L + 2 + np.arange(64)
    w = rng.integers(1, 256, len(col)).astype(np.int32)
    g = dpc.csr_from_arrays(rowptr, col.astype(np.int32), w=w)
    if unit:
        d, _ = dpc.run_bfs(g, hub, "grid", ctx=ctx)
        assert np.array_equal(d, orc.bfs(g.rowptr, g.col, hub))
    else:
        d, _ = dpc.run_sssp(g, hub, "grid", ctx=ctx)
        assert np.array_equal(d, orc.sssp(g.rowptr, g.col, g.w, hub))
