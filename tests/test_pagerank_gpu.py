"""PageRank (the paper's PR benchmark, fixed iteration count
:468): every SpMV variant drives the power iteration over the transposed
graph; ranks within 1e-4 relative of the fp64 oracle (fp32 arithmetic over
20 iterations), mass conserved."""
import numpy as np
import pytest

import paper_1606_08150_b200 as dpc

pytestmark = pytest.mark.gpu

VARIANTS = ["flat", "basic", "warp", "block", "grid"]
RTOL = 1e-4


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("scale", [8, 13])
def test_pagerank_rmat(ctx, orc, variant, scale):
    g = dpc.gen_rmat(scale, 16, seed=scale, weights=False)   # directed, with dangling vertices
    r, met = dpc.run_pagerank(g, 20, 0.85, variant, ctx=ctx)
    ref = orc.pagerank(g.rowptr, g.col, 20, 0.85)
    err = np.abs(r.astype(np.float64) - ref) / ref
    assert err.max() <= RTOL, err.max()
    assert abs(r.astype(np.float64).sum() - 1.0) < 1e-4


def test_pagerank_resident_and_edge_cases(ctx, orc):
    g = dpc.gen_graph(3000, powerlaw=(1.5, 2000), seed=3, weights=False)
    pg = dpc.PageRankGraph(ctx, g)
    for it in (0, 1, 5):
        pg.run(it)
        ref = orc.pagerank(g.rowptr, g.col, it, 0.85)
        assert np.max(np.abs(pg.rank() - ref) / ref) <= RTOL
    pg.close()
    g = dpc.csr_from_arrays([0, 0, 0], [])                   # all dangling: uniform
    r, _ = dpc.run_pagerank(g, 3, 0.85, ctx=ctx)
    assert np.allclose(r, 0.5)
