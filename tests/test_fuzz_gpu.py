"""Seeded random-structure parity sweep: CSR graphs with mixed degree
profiles (many empty rows, a few hubs up to thousands of edges, self loops,
duplicate edges, zero weights), random trees of mixed fan-out, run through
every variant of every app and compared with the oracle (bit-exact; SpMV
within 1e-5)."""
import numpy as np
import pytest

import paper_1606_08150_b200 as dpc

pytestmark = pytest.mark.gpu

VARIANTS = ["flat", "basic", "warp", "block", "grid"]
SEEDS = list(range(12))


def _graph(seed, symmetric=False):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 3000))
    kind = rng.random(n)
    deg = np.where(kind < 0.35, 0, np.where(kind < 0.95, rng.integers(1, 24, n), rng.integers(24, 3000, n)))
    if symmetric:  # an undirected edge list, both directions, no self loops
        m = int(deg.sum() // 2)
        u = rng.integers(0, n, m)
        v = rng.integers(0, n, m)
        keep = u != v
        u, v = u[keep], v[keep]
        src = np.concatenate([u, v])
        dst = np.concatenate([v, u])
    else:
        src = np.repeat(np.arange(n), deg)
        dst = rng.integers(0, n, len(src))
        hub = int(rng.integers(0, n))  # skew: a share of the edges point at one vertex
        dst[rng.random(len(dst)) < 0.1] = hub
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    rowptr = np.concatenate([[0], np.cumsum(np.bincount(src, minlength=n))]).astype(np.int64)
    w = rng.integers(0, 256, len(dst)).astype(np.int32)
    val = (rng.integers(1, 1 << 20, len(dst)) / float(1 << 20)).astype(np.float32)
    return dpc.csr_from_arrays(rowptr, dst.astype(np.int32), w=w, val=val), rng


@pytest.mark.parametrize("seed", SEEDS)
def test_fuzz_spmv_sssp(ctx, orc, seed):
    g, rng = _graph(seed)
    x = (rng.integers(1, 1 << 20, g.n) / float(1 << 20)).astype(np.float32)
    y64 = orc.spmv_f64(g.rowptr, g.col, g.val, x)
    s = int(rng.integers(0, g.n))
    ref = orc.sssp(g.rowptr, g.col, g.w, s)
    refb = orc.bfs(g.rowptr, g.col, s)
    for v in VARIANTS:
        y, _ = dpc.run_spmv(g, x, v, ctx=ctx)
        assert np.all(np.abs(y.astype(np.float64) - y64) <= 1e-5 * np.abs(y64) + 1e-30), v
        d, _ = dpc.run_sssp(g, s, v, ctx=ctx)
        assert np.array_equal(d, ref), v
        b, _ = dpc.run_bfs(g, s, v, ctx=ctx)
        assert np.array_equal(b, refb), v


@pytest.mark.parametrize("seed", SEEDS)
def test_fuzz_gc(ctx, orc, seed):
    g, _ = _graph(seed, symmetric=True)
    for order, o in (("canonical", 1), ("hash", 0), ("llf", 2)):
        ref, k = orc.color(g.rowptr, g.col, seed, order=o)
        for v in VARIANTS:
            c, kk, _ = dpc.run_color(g, seed, v, cfg=dpc.launch_cfg("color", v, gc_order=order), ctx=ctx)
            assert np.array_equal(c, ref) and kk == k, (order, v)


@pytest.mark.parametrize("seed", SEEDS)
def test_fuzz_trees(ctx, orc, seed):
    rng = np.random.default_rng(100 + seed)
    depth = int(rng.integers(1, 25))  # the config-4 depth bound
    parents = [-1]
    level = [0]
    for _ in range(depth):
        if len(parents) > 20000:
            break
        width = int(rng.integers(1, 3000))
        # skewed choice of parents: some nodes get a wide fan-out
        pick = np.minimum((rng.pareto(1.2, width) * len(level) / 8).astype(np.int64), len(level) - 1)
        nxt = list(range(len(parents), len(parents) + width))
        parents += [level[int(p)] for p in pick]
        level = nxt
    parent = np.array(parents, np.int32)
    t = dpc.tree_from_parent(parent)
    for v in VARIANTS:
        r, _ = dpc.run_tree_desc(t, v, ctx=ctx)
        assert np.array_equal(r, orc.tree_desc(parent)), v
        h, _ = dpc.run_tree_height(t, v, ctx=ctx)
        assert np.array_equal(h, orc.tree_height(parent)), v


@pytest.mark.parametrize("seed", SEEDS[:8])
def test_fuzz_partitioned_sssp_spmv(ctx, orc, seed):
    """The caller's own graph cut into `world` row blocks
    (dpc_csr_create_rows, global column ids): partitioned SSSP with the host
    transport, bit-exact; fused SpMV partitions pulling x from the owners,
    within 1e-5."""
    g, rng = _graph(seed)
    n = g.n
    world = int(rng.integers(2, 6))
    R = -(-n // world)
    s = int(rng.integers(0, n))
    want = orc.sssp(g.rowptr, g.col, g.w, s)
    blocks = []
    for p in range(world):
        r0, r1 = min(n, p * R), min(n, (p + 1) * R)
        lo, hi = g.rowptr[r0], g.rowptr[r1]
        blocks.append(dpc.csr_rows_from_arrays(g.rowptr[r0:r1 + 1] - lo, g.col[lo:hi], ncols=n,
                                               w=g.w[lo:hi], val=g.val[lo:hi]))
    dgs = [dpc.DeviceGraph(ctx, b) for b in blocks]
    try:
        ranks = [dpc.PartitionedSSSP(dg, p, world, n, s, "grid") for p, dg in enumerate(dgs)]
        for _ in range(n + 1):
            counts = [r.relax() for r in ranks]
            inbox = [[] for _ in range(world)]
            for p, r in enumerate(ranks):
                for q in range(world):
                    if q != p and counts[p][q]:
                        inbox[q].append(r.outgoing(q, int(counts[p][q])))
            nxt = [r.apply(np.concatenate(inbox[q]) if inbox[q] else np.zeros((0, 2), np.uint32))
                   for q, r in enumerate(ranks)]
            if sum(nxt) == 0:
                break
        for r in ranks:
            r.end()
        got = np.concatenate([dg.get_dist() for dg in dgs])[:n]
        np.testing.assert_array_equal(got, want)
        # fused SpMV over the same blocks: x slices in a pointer table
        x = (rng.integers(1, 1 << 20, n) / float(1 << 20)).astype(np.float32)
        y64 = orc.spmv_f64(g.rowptr, g.col, g.val, x)
        bufs = []
        xs = []
        for p in range(world):
            d = ctx.alloc(4 * R)
            bufs.append(d)
            sl = np.zeros(R, np.float32)
            part = x[p * R:min(n, (p + 1) * R)]
            sl[:len(part)] = part
            ctx.h2d(d, sl)
            xs.append(d)
        tab = ctx.alloc(8 * world)
        bufs.append(tab)
        ctx.h2d(tab, np.array(xs, np.uint64))
        for p, dg in enumerate(dgs):
            r0, r1 = min(n, p * R), min(n, (p + 1) * R)
            if r1 == r0:
                continue
            yd = ctx.alloc(4 * (r1 - r0))
            bufs.append(yd)
            dg.spmv_fused(tab, world, R, yd, cfg=dpc.launch_cfg("spmv", "grid"))
            y = ctx.d2h(yd, r1 - r0).astype(np.float64)
            ref = y64[r0:r1]
            assert np.all(np.abs(y - ref) <= 1e-5 * np.abs(ref) + 1e-30), p
        for b in bufs:
            ctx.free(b)
    finally:
        for dg in dgs:
            dg.close()
