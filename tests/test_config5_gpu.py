"""BASELINE config 5 at full size on one B200: the fixed vertex-permuted
R-MAT scale-24 graph (16,777,216 vertices, 268,435,456 arcs; seed 1, the
bench's graph) split into two row blocks that run as two partitions in one
process -- the multi-GPU data paths minus NVLink (this pool has one GPU):

* fused SpMV (owners' x slices pulled inside the kernel through a pointer
  table), per rank within 1e-5 of the fp64 oracle;
* partitioned SSSP with the host transport standing in for grouped NCCL
  send/recv, and the fused form (remote relaxations straight into the other
  partition's arrays), bit-exact against the oracle on the whole graph.

Slow (host generation of the whole graph for the oracle, ~3 GB)."""
import os

import numpy as np
import pytest

import paper_1606_08150_b200 as dpc

pytestmark = pytest.mark.gpu

SCALE, SEED, WORLD = 24, 1, 2
N = 1 << SCALE
R = N // WORLD


@pytest.fixture(scope="module")
def full():
    g = dpc.gen_rmat(SCALE, 16, seed=SEED, weights=True, values=True, permute=True)
    return g


@pytest.fixture(scope="module")
def blocks():
    return [dpc.gen_rmat_rows(SCALE, p * R, (p + 1) * R, 16, seed=SEED, weights=True, values=True, permute=True)
            for p in range(WORLD)]


@pytest.fixture(scope="module")
def sssp_ref(full, orc):
    src = int(np.argmax(full.degrees()))
    d, _ = orc.sssp_mt(full.rowptr, full.col, full.w, src, os.cpu_count() or 1)
    return src, d


def test_config5_blocks_are_the_graph(full, blocks):
    """The row blocks each rank generates are exactly the whole graph's rows."""
    for p, b in enumerate(blocks):
        lo, hi = full.rowptr[p * R], full.rowptr[(p + 1) * R]
        assert np.array_equal(b.rowptr, full.rowptr[p * R:(p + 1) * R + 1] - lo)
        assert np.array_equal(b.col, full.col[lo:hi]) and np.array_equal(b.w, full.w[lo:hi])


def test_config5_fused_spmv_two_partitions(ctx, orc, full, blocks):
    x = (((np.arange(N) * 7) % 89 + 1) / 89.0).astype(np.float32)
    y64 = orc.spmv_f64(full.rowptr, full.col, full.val, x)
    bufs = []
    try:
        xs = []
        for p in range(WORLD):
            d = ctx.alloc(4 * R)
            bufs.append(d)
            ctx.h2d(d, x[p * R:(p + 1) * R])
            xs.append(d)
        tab = ctx.alloc(8 * WORLD)
        bufs.append(tab)
        ctx.h2d(tab, np.array(xs, np.uint64))
        for p, A in enumerate(blocks):
            dg = dpc.DeviceGraph(ctx, A)
            yd = ctx.alloc(4 * R)
            bufs.append(yd)
            dg.spmv_fused(tab, WORLD, R, yd, cfg=dpc.launch_cfg("spmv", "grid"))
            y = ctx.d2h(yd, R).astype(np.float64)
            ref = y64[p * R:(p + 1) * R]
            assert np.all(np.abs(y - ref) <= 1e-5 * np.abs(ref) + 1e-30), f"rank {p}"
            dg.close()
    finally:
        for b in bufs:
            ctx.free(b)


def test_config5_partitioned_sssp_host_transport(ctx, blocks, sssp_ref):
    src, want = sssp_ref
    dgs = [dpc.DeviceGraph(ctx, b) for b in blocks]
    ranks = [dpc.PartitionedSSSP(dg, p, WORLD, N, src, "grid") for p, dg in enumerate(dgs)]
    try:
        for _ in range(N + 1):
            counts = [r.relax() for r in ranks]
            inbox = [[] for _ in range(WORLD)]
            for p, r in enumerate(ranks):
                for q in range(WORLD):
                    if q != p and counts[p][q]:
                        inbox[q].append(r.outgoing(q, int(counts[p][q])))
            nxt = [r.apply(np.concatenate(inbox[q]) if inbox[q] else np.zeros((0, 2), np.uint32))
                   for q, r in enumerate(ranks)]
            if sum(nxt) == 0:
                break
        for r in ranks:
            r.end()
        got = np.concatenate([dg.get_dist() for dg in dgs])
        np.testing.assert_array_equal(got, want)
    finally:
        for dg in dgs:
            dg.close()


def test_config5_fused_sssp_two_partitions(ctx, blocks, sssp_ref):
    src, want = sssp_ref
    dgs = [dpc.DeviceGraph(ctx, b) for b in blocks]
    ps = [dpc.PartitionedSSSP(dg, p, WORLD, N, src) for p, dg in enumerate(dgs)]
    tab = ctx.alloc(8 * 5 * WORLD)
    try:
        ctx.h2d(tab, np.array([b for p in ps for b in p.buffers()], np.uint64))
        for p in ps:
            p.set_peers(tab)
        for _ in range(N + 1):
            for p in ps:
                assert not p.relax().any()   # nothing goes through send buffers
            if sum(p.apply(np.zeros((0, 2), np.uint32)) for p in ps) == 0:
                break
        for p in ps:
            p.end()
        got = np.concatenate([dg.get_dist() for dg in dgs])
        np.testing.assert_array_equal(got, want)
    finally:
        ctx.free(tab)
        for dg in dgs:
            dg.close()
