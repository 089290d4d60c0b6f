"""Vertex-partitioned SSSP (BASELINE config 5) on one B200.

World sizes 2..5 run as that many row blocks in ONE process on one GPU: each
block is its own device graph, the {vertex, distance} exchange goes through
host copies (the transport dpc_multi_sssp replaces with grouped NCCL
send/recv), and the concatenated distances must equal Dijkstra on the whole
graph bit for bit.  world = 1 runs the NCCL driver itself (a one-rank
communicator)."""
import numpy as np
import pytest

import paper_1606_08150_b200 as dpc

pytestmark = pytest.mark.gpu

VARIANTS = ["flat", "basic", "warp", "block", "grid"]


def _run_partitioned(ctx, scale, world, source, variant, seed=3):
    n = 1 << scale
    R = -(-n // world)
    blocks = [dpc.gen_rmat_rows(scale, p * R, min(n, (p + 1) * R), 16, seed=seed, permute=True)
              for p in range(world)]
    dgs = [dpc.DeviceGraph(ctx, b) for b in blocks]
    ranks = [dpc.PartitionedSSSP(dg, p, world, n, source, variant) for p, dg in enumerate(dgs)]
    sent = 0
    for _ in range(n + 1):
        counts = [r.relax() for r in ranks]
        inbox = [[] for _ in range(world)]
        for p, r in enumerate(ranks):
            assert counts[p][p] == 0          # local targets never leave the rank
            for q in range(world):
                if counts[p][q]:
                    pairs = r.outgoing(q, int(counts[p][q]))
                    assert np.all(pairs[:, 0] // R == q)   # routed to the owner
                    inbox[q].append(pairs)
                    sent += int(counts[p][q])
        nxt = [r.apply(np.concatenate(inbox[q]) if inbox[q] else np.zeros((0, 2), np.uint32))
               for q, r in enumerate(ranks)]
        if sum(nxt) == 0:
            break
    mets = [r.end() for r in ranks]
    dist = np.concatenate([dg.get_dist() for dg in dgs])
    for dg in dgs:
        dg.close()
    return dist, mets, sent


@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("variant", VARIANTS)
def test_partitioned_sssp_matches_dijkstra(ctx, orc, world, variant):
    scale = 11
    g = dpc.gen_rmat(scale, 16, seed=3, permute=True)
    source = int(np.argmax(g.degrees()))
    ref = orc.sssp(g.rowptr, g.col, g.w, source)
    dist, mets, sent = _run_partitioned(ctx, scale, world, source, variant)
    assert np.array_equal(dist, ref)
    assert sent > 0
    assert sum(m.result_count for m in mets) == sent


def test_partitioned_sssp_unreachable_and_isolated_source(ctx, orc):
    scale = 10
    g = dpc.gen_rmat(scale, 16, seed=3, permute=True)
    iso = int(np.flatnonzero(g.degrees() == 0)[0])          # an isolated source
    dist, _, sent = _run_partitioned(ctx, scale, 4, iso, "grid")
    assert np.array_equal(dist, orc.sssp(g.rowptr, g.col, g.w, iso))
    assert sent == 0 and (dist == 0xFFFFFFFF).sum() == g.n - 1


def test_multi_sssp_nccl_one_rank(ctx, orc):
    """dpc_multi_sssp through a one-rank NCCL communicator."""
    scale = 12
    g = dpc.gen_rmat(scale, 16, seed=4, permute=True)
    blk = dpc.gen_rmat_rows(scale, 0, g.n, 16, seed=4, permute=True)
    dg = dpc.DeviceGraph(ctx, blk)
    comm = dpc.Comm(ctx, 0, 1, dpc.Comm.unique_id())
    s = int(np.argmax(g.degrees()))
    met = comm.sssp(dg, g.n, s)
    assert np.array_equal(dg.get_dist(), orc.sssp(g.rowptr, g.col, g.w, s))
    assert met.iterations > 1 and met.result_count == 0
    comm.close()
    dg.close()
