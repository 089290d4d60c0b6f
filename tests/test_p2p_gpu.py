"""Fused multi-GPU SpMV over peer memory (BASELINE config 5):
x gathered from the owners inside the SpMV (dpc_multi_spmv_fused), the
device-side peer barrier (dpc_p2p_barrier) and CUDA IPC mapping
(dpc_ipc_*).  One GPU in this pool, so the tests run the ranks' partitions
(a) in one process with direct pointers and one context (stream) per rank,
(b) in two processes on the same GPU with IPC-mapped buffers — the same
code path as across GPUs, minus NVLink.  Results against the oracle
(fp32 SpMV within 1e-5 of the fp64 reference)."""
import os
import socket

import numpy as np
import pytest

import paper_1606_08150_b200 as dpc

pytestmark = pytest.mark.gpu

SCALE, SEED = 12, 3


def full_matrix():
    return dpc.gen_rmat(SCALE, 16, seed=SEED, weights=False, values=True, permute=True)


def x_vector(n, step=1):
    return (((np.arange(n) * (7 + step)) % 89 + 1) / 89.0).astype(np.float32)


def close(y, y64):
    return np.all(np.abs(y.astype(np.float64) - y64) <= 1e-5 * np.abs(y64) + 1e-30)


@pytest.mark.parametrize("mode", ["pull", "gather", "gather_hot"])
@pytest.mark.parametrize("world", [1, 3, 4])
def test_fused_spmv_partitions_one_process(orc, world, mode):
    """world row blocks; x entry i lives on block i // R (R a power of two
    for world 1 / 4, not for 3: the shift and the division paths; R % 4 != 0
    for world 3: the pull's scalar path).  Modes: the in-kernel pull of the
    owners' slices (default), per-gather peer reads, and per-gather reads
    behind shape 4's hot-column cache (filled from the owners)."""
    g = full_matrix()
    n = g.n
    R = (n + world - 1) // world
    x = x_vector(n)
    y64 = orc.spmv_f64(g.rowptr, g.col, g.val, x)
    ctx = dpc.Context(0)
    bufs = []
    try:
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
        for p in range(world):
            r0, r1 = p * R, min(n, (p + 1) * R)
            A = dpc.gen_rmat_rows(SCALE, r0, r1, 16, seed=SEED, weights=False, values=True, permute=True)
            dg = dpc.DeviceGraph(ctx, A)
            yd = ctx.alloc(4 * max(1, r1 - r0))
            bufs.append(yd)
            cfg = dpc.launch_cfg("spmv", "grid")
            if mode != "pull":
                cfg.flags |= dpc.CFG_X_PEER_GATHER | ((4 << 20) if mode == "gather_hot" else 0)
            dg.spmv_fused(tab, world, R, yd, cfg=cfg)
            y = ctx.d2h(yd, r1 - r0)
            assert close(y, y64[r0:r1]), f"rank {p}"
            dg.close()
    finally:
        for b in bufs:
            ctx.free(b)
        ctx.close()


def test_fused_spmv_rejects_non_stream_config():
    g = full_matrix()
    ctx = dpc.Context(0)
    dg = dpc.DeviceGraph(ctx, g)
    xd, yd, tab = ctx.alloc(4 * g.n), ctx.alloc(4 * g.n), ctx.alloc(8)
    ctx.h2d(tab, np.array([xd], np.uint64))
    with pytest.raises(dpc.DpcError):
        dg.spmv_fused(tab, 1, g.n, yd, variant="block")
    with pytest.raises(dpc.DpcError):
        dg.spmv_fused(tab, 1, g.n, yd, cfg=dpc.launch_cfg("spmv", "grid", threshold=8))
    for b in (xd, yd, tab):
        ctx.free(b)
    dg.close()
    ctx.close()


def test_p2p_barrier_contexts_one_process():
    """Three ranks as three contexts (streams) on one device: every epoch
    completes once all three signalled."""
    world = 3
    ctxs = [dpc.Context(0) for _ in range(world)]
    flags = [ctxs[0].alloc(16 * world) for _ in range(world)]
    for f in flags:
        ctxs[0].h2d(f, np.zeros(2 * world, np.uint64))
    tab = ctxs[0].alloc(8 * world)
    ctxs[0].h2d(tab, np.array(flags, np.uint64))
    ctxs[0].synchronize()
    for epoch in (1, 2, 3):
        for q in range(world):
            dpc.p2p_barrier(ctxs[q], tab, world, q, epoch)
        for q in range(world):
            dpc.p2p_check(ctxs[q])
            got = ctxs[q].d2h(flags[q], 2 * world, np.uint64).reshape(2, world)[epoch & 1]
            assert np.all((got >> 32) == epoch)
    for b in flags + [tab]:
        ctxs[0].free(b)
    for c in ctxs:
        c.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, steps):
    import torch.distributed as dist

    from tests._oracle import Oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    g = full_matrix()
    n = g.n
    R = n // world
    r0, r1 = rank * R, (rank + 1) * R
    ctx = dpc.Context(0)
    A = dpc.gen_rmat_rows(SCALE, r0, r1, 16, seed=SEED, weights=False, values=True, permute=True)
    dg = dpc.DeviceGraph(ctx, A)
    x_local = ctx.alloc(4 * R)
    flags = ctx.alloc(16 * world)
    ctx.h2d(flags, np.zeros(2 * world, np.uint64))
    ctx.synchronize()
    hs = [None] * world
    dist.all_gather_object(hs, (dpc.ipc_handle(x_local), dpc.ipc_handle(flags)))
    xs, fs, opened = [], [], []
    for q in range(world):
        if q == rank:
            xs.append(x_local)
            fs.append(flags)
        else:
            xp, fp = dpc.ipc_open(ctx, hs[q][0]), dpc.ipc_open(ctx, hs[q][1])
            opened += [xp, fp]
            xs.append(xp)
            fs.append(fp)
    xtab, ftab, yd = ctx.alloc(8 * world), ctx.alloc(8 * world), ctx.alloc(4 * R)
    ctx.h2d(xtab, np.array(xs, np.uint64))
    ctx.h2d(ftab, np.array(fs, np.uint64))
    ok = True
    for s in range(1, steps + 1):
        x = x_vector(n, s)
        ctx.h2d(x_local, x[r0:r1])
        dpc.p2p_barrier(ctx, ftab, world, rank, 2 * s - 1)   # every x slice written
        dg.spmv_fused(xtab, world, R, yd)
        dpc.p2p_barrier(ctx, ftab, world, rank, 2 * s)       # every peer done reading x
        dpc.p2p_check(ctx)
        y = ctx.d2h(yd, R)
        ok = ok and bool(close(y, orc.spmv_f64(g.rowptr, g.col, g.val, x)[r0:r1]))
    flag = [None] * world
    dist.all_gather_object(flag, ok)
    for p in opened:
        dpc.ipc_close(p)
    for b in (x_local, flags, xtab, ftab, yd):
        ctx.free(b)
    dg.close()
    ctx.close()
    dist.destroy_process_group()
    assert all(flag), flag


def test_fused_spmv_two_processes_ipc():
    """Two processes, one GPU: IPC-mapped x slices and barrier flags, the
    handles exchanged over gloo; three SpMV steps with changing x."""
    import torch.multiprocessing as mp
    mp.spawn(_rank, args=(2, _free_port(), 3), nprocs=2, join=True)


def _sssp_parts(world, scale=11):
    n = 1 << scale
    R = n // world
    return n, R, [dpc.gen_rmat_rows(scale, p * R, (p + 1) * R, 16, seed=SEED, weights=True, permute=True)
                  for p in range(world)]


@pytest.mark.parametrize("world", [2, 4])
def test_fused_sssp_partitions_one_process(orc, world):
    """The fused partitioned SSSP with the ranks' steps run in turn in one
    process (peer buffers = the other partitions' device buffers)."""
    n, R, parts = _sssp_parts(world)
    full = dpc.gen_rmat(11, 16, seed=SEED, weights=True, permute=True)
    src = int(np.argmax(full.degrees()))
    want = orc.sssp(full.rowptr, full.col, full.w, src)
    ctx = dpc.Context(0)
    dgs = [dpc.DeviceGraph(ctx, A) for A in parts]
    ps = [dpc.PartitionedSSSP(dg, p, world, n, src) for p, dg in enumerate(dgs)]
    tab = ctx.alloc(8 * 5 * world)
    ctx.h2d(tab, np.array([b for p in ps for b in p.buffers()], np.uint64))
    for p in ps:
        p.set_peers(tab)
    for it in range(n + 1):
        for p in ps:
            cnt = p.relax()
            assert not cnt.any()          # nothing goes through send buffers
        total = sum(p.apply(np.zeros((0, 2), np.uint32)) for p in ps)
        if total == 0:
            break
    got = np.concatenate([dg.get_dist() for dg in dgs])
    np.testing.assert_array_equal(got, want)
    for p in ps:
        p.end()
    ctx.free(tab)
    for dg in dgs:
        dg.close()
    ctx.close()


def _sssp_rank(rank, world, port):
    import torch.distributed as dist

    from tests._oracle import Oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, R, parts = _sssp_parts(world)
    full = dpc.gen_rmat(11, 16, seed=SEED, weights=True, permute=True)
    src = int(np.argmax(full.degrees()))
    want = Oracle().sssp(full.rowptr, full.col, full.w, src)[rank * R:(rank + 1) * R]
    ctx = dpc.Context(0)
    dg = dpc.DeviceGraph(ctx, parts[rank])
    ps = dpc.PartitionedSSSP(dg, rank, world, n, src)
    flags = ctx.alloc(16 * world)
    ctx.h2d(flags, np.zeros(2 * world, np.uint64))
    ctx.synchronize()
    mine = ps.buffers()
    hs = [None] * world
    dist.all_gather_object(hs, ([dpc.ipc_handle(b) for b in mine], dpc.ipc_handle(flags)))
    table, ftab_l, opened = [], [], []
    for q in range(world):
        if q == rank:
            table += mine
            ftab_l.append(flags)
        else:
            ptrs = [dpc.ipc_open(ctx, h) for h in hs[q][0]]
            fp = dpc.ipc_open(ctx, hs[q][1])
            opened += ptrs + [fp]
            table += ptrs
            ftab_l.append(fp)
    tab, ftab = ctx.alloc(8 * 5 * world), ctx.alloc(8 * world)
    ctx.h2d(tab, np.array(table, np.uint64))
    ctx.h2d(ftab, np.array(ftab_l, np.uint64))
    ps.set_peers(tab)
    epoch = 0
    for it in range(n + 1):
        ps.relax()
        epoch += 1
        dpc.p2p_barrier(ctx, ftab, world, rank, epoch)      # every relaxation of the level landed
        nxt = ps.apply(np.zeros((0, 2), np.uint32))
        epoch += 1
        if dpc.p2p_barrier_sum(ctx, ftab, world, rank, epoch, nxt) == 0:
            break
    ps.end()
    ok = bool(np.array_equal(dg.get_dist(), want))
    flag = [None] * world
    dist.all_gather_object(flag, ok)
    for p in opened:
        dpc.ipc_close(p)
    for b in (flags, tab, ftab):
        ctx.free(b)
    dg.close()
    ctx.close()
    dist.destroy_process_group()
    assert all(flag), flag


def test_fused_sssp_two_processes_ipc():
    import torch.multiprocessing as mp
    mp.spawn(_sssp_rank, args=(2, _free_port()), nprocs=2, join=True)
