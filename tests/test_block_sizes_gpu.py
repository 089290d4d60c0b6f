"""Launch geometries a caller may request through dpc_launch_cfg
(parent_threads / child_threads: multiples of 32 in [32, 1024]): every
app x variant either runs them exactly or refuses with a DpcError -- a
wrong result is never returned.  (Round 2 found the shared block scan
writing the block total over warp 31's offset in 1024-thread blocks.)"""
import numpy as np
import pytest

import paper_1606_08150_b200 as dpc

pytestmark = pytest.mark.gpu

VARIANTS = ["flat", "basic", "warp", "block", "grid"]
THREADS = [64, 512, 1024]


def _x(n):
    return ((np.arange(n) % 97 + 1) / 97.0).astype(np.float32)


def _run_or_refuse(fn):
    try:
        return fn()
    except dpc.DpcError as e:  # (on the B200 every geometry here runs)
        assert e.kind in ("invalid", "cuda"), e
        return None


@pytest.mark.parametrize("threads", THREADS)
@pytest.mark.parametrize("variant", VARIANTS)
def test_spmv_block_sizes(ctx, orc, variant, threads):
    g = dpc.gen_rmat(13, 16, seed=7, weights=False, values=True)
    x = _x(g.n)
    y64 = orc.spmv_f64(g.rowptr, g.col, g.val, x)
    cfg = dpc.launch_cfg("spmv", variant, parent_threads=threads, child_threads=threads, threshold=8)
    r = _run_or_refuse(lambda: dpc.run_spmv(g, x, variant, cfg=cfg, ctx=ctx))
    if r is not None:
        y = r[0].astype(np.float64)
        assert np.all(np.abs(y - y64) <= 1e-5 * np.abs(y64) + 1e-30)


@pytest.mark.parametrize("threads", THREADS)
@pytest.mark.parametrize("variant", VARIANTS)
def test_sssp_block_sizes(ctx, orc, variant, threads):
    g = dpc.gen_rmat(13, 16, seed=8)
    s = int(np.argmax(g.degrees()))
    ref = orc.sssp(g.rowptr, g.col, g.w, s)
    cfg = dpc.launch_cfg("sssp", variant, parent_threads=threads, child_threads=threads, threshold=8)
    r = _run_or_refuse(lambda: dpc.run_sssp(g, s, variant, cfg=cfg, ctx=ctx))
    if r is not None:
        assert np.array_equal(r[0], ref)


@pytest.mark.parametrize("threads", THREADS)
@pytest.mark.parametrize("variant", VARIANTS)
def test_tree_block_sizes(ctx, orc, variant, threads):
    t = dpc.gen_tree(10, 1, 6, 0.8, 3)
    cfg_d = dpc.launch_cfg("tree_desc", variant, parent_threads=threads, child_threads=threads)
    cfg_h = dpc.launch_cfg("tree_height", variant, parent_threads=threads, child_threads=threads)
    r = _run_or_refuse(lambda: dpc.run_tree_desc(t, variant, cfg=cfg_d, ctx=ctx))
    if r is not None:
        assert np.array_equal(r[0], orc.tree_desc(t.parent))
    r = _run_or_refuse(lambda: dpc.run_tree_height(t, variant, cfg=cfg_h, ctx=ctx))
    if r is not None:
        assert np.array_equal(r[0], orc.tree_height(t.parent))


@pytest.mark.parametrize("kc", [(0, 0), (1, 0), (32, 0), (0, 1), (0, 7), (0, 1000)])
@pytest.mark.parametrize("variant", ["warp", "block", "grid"])
def test_child_geometry(ctx, orc, variant, kc):
    """KC_X divisor (0 = "1-1") and explicit child block counts, down to a
    single child block, for SpMV / SSSP / GC / TD: exact."""
    kc_x, blocks = kc
    over = {"kc_x": kc_x}
    if blocks:
        over["child_blocks"] = blocks
    g = dpc.gen_rmat(12, 16, seed=9, weights=True, values=True)
    x = _x(g.n)
    y64 = orc.spmv_f64(g.rowptr, g.col, g.val, x)
    y, _ = dpc.run_spmv(g, x, variant, cfg=dpc.launch_cfg("spmv", variant, threshold=8, **over), ctx=ctx)
    assert np.all(np.abs(y.astype(np.float64) - y64) <= 1e-5 * np.abs(y64) + 1e-30)
    s = int(np.argmax(g.degrees()))
    d, _ = dpc.run_sssp(g, s, variant, cfg=dpc.launch_cfg("sssp", variant, threshold=8, **over), ctx=ctx)
    assert np.array_equal(d, orc.sssp(g.rowptr, g.col, g.w, s))
    gs = dpc.gen_rmat(12, 16, seed=9, weights=False, symmetric=True)
    c, k, _ = dpc.run_color(gs, 1, variant, cfg=dpc.launch_cfg("color", variant, **over), ctx=ctx)
    ref, kr = orc.color(gs.rowptr, gs.col, 1)
    assert np.array_equal(c, ref) and k == kr
    t = dpc.gen_tree(9, 1, 5, 0.8, 4)
    r, _ = dpc.run_tree_desc(t, variant, cfg=dpc.launch_cfg("tree_desc", variant, **over), ctx=ctx)
    assert np.array_equal(r, orc.tree_desc(t.parent))
