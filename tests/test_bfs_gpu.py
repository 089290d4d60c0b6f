"""BFS-Rec (the paper's seventh benchmark; SPEC.md:454 oracle "BFS levels"):
the SSSP consolidation with unit weights, bit-exact against a FIFO BFS on
every variant and grid form."""
import numpy as np
import pytest

import paper_1606_08150_b200 as dpc

pytestmark = pytest.mark.gpu

VARIANTS = ["flat", "basic", "warp", "block", "grid"]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("scale", [8, 12, 15])
def test_bfs_rmat(ctx, orc, variant, scale):
    g = dpc.gen_rmat(scale, 16, seed=scale + 3, weights=False)
    for s in (int(np.argmax(g.degrees())), int(np.flatnonzero(g.degrees() == 0)[0])):
        lv, met = dpc.run_bfs(g, s, variant, ctx=ctx)
        assert np.array_equal(lv, orc.bfs(g.rowptr, g.col, s))


@pytest.mark.parametrize("form", ["async", "two_barrier"])
def test_bfs_grid_forms(ctx, orc, form):
    g = dpc.gen_graph(4000, powerlaw=(1.5, 3000), seed=5, weights=False)
    cfg = dpc.launch_cfg("sssp", "grid", grid_async=(form == "async"), grid_chunked=(form == "two_barrier"))
    lv, _ = dpc.run_bfs(g, 0, "grid", cfg=cfg, ctx=ctx)
    assert np.array_equal(lv, orc.bfs(g.rowptr, g.col, 0))


def test_bfs_path_and_edge_cases(ctx, orc):
    n = 3000                                   # a path: n levels, one vertex per level
    g = dpc.csr_from_arrays(np.arange(n + 1).clip(max=n - 1), np.arange(1, n).astype(np.int32))
    lv, met = dpc.run_bfs(g, 0, "grid", ctx=ctx)
    assert lv.tolist() == list(range(n))
    g = dpc.csr_from_arrays([0, 0], [])
    lv, _ = dpc.run_bfs(g, 0, "grid", ctx=ctx)
    assert lv.tolist() == [0]
