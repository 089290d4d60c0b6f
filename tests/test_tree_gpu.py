"""TD / TH parity on the B200: every variant bit-exact against the bottom-up
CPU oracle, on generated trees of both paper shapes and on hand-built edge
cases (SPEC.md:457-458 examples, single node, path, star)."""
import numpy as np
import pytest

import paper_1606_08150_b200 as dpc

pytestmark = pytest.mark.gpu

VARIANTS = ["flat", "basic", "warp", "block", "grid"]
WHICH = ["tree_desc", "tree_height"]


def _run(ctx, t, which, variant, cfg=None):
    fn = dpc.run_tree_desc if which == "tree_desc" else dpc.run_tree_height
    return fn(t, variant, cfg=cfg, ctx=ctx)


def _ref(orc, t, which):
    return orc.tree_desc(t.parent) if which == "tree_desc" else orc.tree_height(t.parent)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("which", WHICH)
@pytest.mark.parametrize("shape", [(6, 1, 4, 0.9), (5, 8, 16, 0.5), (4, 32, 64, 0.5), (12, 1, 3, 0.8)])
def test_tree_generated(ctx, orc, variant, which, shape):
    t = dpc.gen_tree(*shape, seed=sum(shape[:3]))
    r, met = _run(ctx, t, which, variant)
    assert np.array_equal(r, _ref(orc, t, which))


@pytest.mark.parametrize("variant", VARIANTS)
def test_tree_spec_examples(ctx, variant):
    # SPEC.md:457 TD on root with 3 leaf children -> 3
    t = dpc.tree_from_parent([-1, 0, 0, 0])
    r, _ = dpc.run_tree_desc(t, variant, ctx=ctx)
    assert r.tolist() == [3, 0, 0, 0]
    # SPEC.md:458 TH on a path of 5 nodes -> 4
    t = dpc.tree_from_parent([-1, 0, 1, 2, 3])
    r, _ = dpc.run_tree_height(t, variant, ctx=ctx)
    assert r.tolist() == [4, 3, 2, 1, 0]
    # single node
    t = dpc.tree_from_parent([-1])
    assert dpc.run_tree_desc(t, variant, ctx=ctx)[0].tolist() == [0]
    # root not at index 0, star with a 5000-wide fan-out (multi-block children)
    par = np.full(5001, 5000, np.int32)
    par[5000] = -1
    t = dpc.tree_from_parent(par)
    assert dpc.run_tree_desc(t, variant, ctx=ctx)[0][5000] == 5000
    assert dpc.run_tree_height(t, variant, ctx=ctx)[0][5000] == 1


@pytest.mark.parametrize("variant", VARIANTS)
def test_tree_deep_path_24(ctx, orc, variant):
    """Depth-24 chain-ish tree (BASELINE 'depth up to 24')."""
    t = dpc.gen_tree(24, 1, 2, 0.6, seed=3)
    assert t.depth == 24
    for which in WHICH:
        r, _ = _run(ctx, t, which, variant)
        assert np.array_equal(r, _ref(orc, t, which))


def test_tree_grid_cdp(ctx, orc):
    t = dpc.gen_tree(10, 1, 6, 0.7, seed=9)
    cfg = dpc.launch_cfg("tree_desc", "grid", grid_cdp=True)
    r, met = dpc.run_tree_desc(t, cfg=cfg, ctx=ctx)
    assert np.array_equal(r, orc.tree_desc(t.parent))
    # one consolidated launch per level below the root + one postwork per grid
    assert met.child_launch_count <= 2 * t.depth


def test_tree_config4_full(ctx, orc):
    """BASELINE config 4: 4M nodes (4,246,411: within 5% of 4,194,304), depth 24,
    every variant including basic-DP (child-side count-down postwork)."""
    t = dpc.gen_tree(24, 1, 4, 0.851, seed=1)
    assert t.depth == 24 and abs(t.n - 4_194_304) <= 0.05 * 4_194_304
    dt = dpc.DeviceTree(ctx, t)
    ref_d, ref_h = orc.tree_desc(t.parent), orc.tree_height(t.parent)
    for v in ["flat", "basic", "warp", "block", "grid"]:
        dt.run("tree_desc", v)
        assert np.array_equal(dt.result(), ref_d), v
        dt.run("tree_height", v)
        assert np.array_equal(dt.result(), ref_h), v
    dt.close()


@pytest.mark.parametrize("variant", ["flat", "basic", "warp", "block", "grid"])
def test_tree_deeper_than_baseline(ctx, orc, variant):
    """Depths far past BASELINE config 4's 24 (chains of 100 / 2000 nodes, a
    300-deep comb with 50 leaves per spine node): exact in every variant
    (basic-DP nests a device launch per level)."""
    cases = [np.concatenate([[-1], np.arange(d - 1)]).astype(np.int32) for d in (100, 2000)]
    par = [-1] + list(range(299))
    for v in range(300):
        par += [v] * 50
    cases.append(np.array(par, np.int32))
    for parent in cases:
        t = dpc.tree_from_parent(parent)
        r, _ = dpc.run_tree_desc(t, variant, ctx=ctx)
        assert np.array_equal(r, orc.tree_desc(parent))
        h, _ = dpc.run_tree_height(t, variant, ctx=ctx)
        assert np.array_equal(h, orc.tree_height(parent))
