"""World-size-2 `gloo` test of the multi-GPU partition + exchange logic
(CPU only).  Each rank generates only its row block with dpc_gen_rmat_rows,
all-gathers the x slices (gloo stands in for the ncclAllGather of
dpc_multi_spmv), computes its y block with the CPU oracle, and rank 0 checks
the concatenation against the single-process SpMV of the whole matrix."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1606_08150_b200 as dpc

SCALE = 11


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from tests._oracle import Oracle
    n = 1 << SCALE
    R = n // world
    A = dpc.gen_rmat_rows(SCALE, rank * R, (rank + 1) * R, 16, seed=5, weights=False, values=True,
                          permute=True)
    assert A.n == R and A.ncols == n
    rng = np.random.default_rng(9)
    x_full_ref = (rng.integers(1, 1 << 24, n) / float(1 << 24)).astype(np.float32)
    x_local = torch.from_numpy(x_full_ref[rank * R:(rank + 1) * R].copy())
    parts = [torch.empty(R, dtype=torch.float32) for _ in range(world)]
    dist.all_gather(parts, x_local)                      # the exchange step
    x_full = torch.cat(parts).numpy()
    assert np.array_equal(x_full, x_full_ref)
    y_local = Oracle().spmv_f64(A.rowptr, A.col, A.val, x_full)
    ys = [torch.empty(R, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(ys, torch.from_numpy(y_local))
    nnz = torch.tensor([A.m], dtype=torch.int64)
    dist.all_reduce(nnz)
    if rank == 0:
        np.save(os.path.join(out_dir, "y.npy"), torch.cat(ys).numpy())
        np.save(os.path.join(out_dir, "nnz.npy"), nnz.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_row_partition_spmv_gloo(tmp_path, orc, world):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    y = np.load(tmp_path / "y.npy")
    g = dpc.gen_rmat(SCALE, 16, seed=5, weights=False, values=True, permute=True)
    rng = np.random.default_rng(9)
    x = (rng.integers(1, 1 << 24, g.n) / float(1 << 24)).astype(np.float32)
    assert np.array_equal(y, orc.spmv_f64(g.rowptr, g.col, g.val, x))
    assert int(np.load(tmp_path / "nnz.npy")[0]) == g.m


def test_permuted_blocks_are_balanced():
    g = dpc.gen_rmat(14, 16, seed=1, weights=False, values=True, permute=True)
    nnz = [int(g.rowptr[(p + 1) * g.n // 8] - g.rowptr[p * g.n // 8]) for p in range(8)]
    assert max(nnz) / min(nnz) < 1.6     # vertex permutation balances equal row blocks


def test_partition_rows_equal_nnz():
    g = dpc.gen_rmat(12, 16, seed=2, weights=False)
    b = dpc.partition_rows(g, 4)
    assert b[0] == 0 and b[-1] == g.n and np.all(np.diff(b) >= 0)
    part = np.diff(g.rowptr[b])
    assert part.sum() == g.m and part.max() <= g.m / 4 + g.degrees().max()


def test_row_slice_arguments():
    s = dpc.gen_rmat_rows(8, 0, 64, 8, seed=1)
    assert s.ncols == 256 and s.n == 64
    s.validate()                                  # columns checked against ncols
    with pytest.raises(dpc.DpcError):
        dpc.gen_rmat_rows(8, 10, 5, 8)            # r0 > r1
    with pytest.raises(dpc.DpcError):
        dpc.gen_rmat_rows(8, 0, 300, 8)           # past the last row


def _sssp_worker(rank, world, port, out_dir):
    """Level-synchronous partitioned Bellman-Ford with the dpc_multi_sssp
    exchange pattern (owner-computes, min-filtered remote pairs, all-reduced
    frontier size), ranks talking over gloo."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 1 << SCALE
    R = -(-n // world)
    r0 = rank * R
    A = dpc.gen_rmat_rows(SCALE, r0, min(n, r0 + R), 16, seed=7, permute=True)
    src = int(np.load(os.path.join(out_dir, "src.npy")))
    INF = np.uint64(0xFFFFFFFF)
    d = np.full(A.n, INF, np.uint64)
    rdist = np.full(n, INF, np.uint64)
    front = []
    if r0 <= src < r0 + A.n:
        d[src - r0] = 0
        front = [src - r0]
    while True:
        out = [[] for _ in range(world)]
        nxt = set()
        for u in front:
            for k in range(A.rowptr[u], A.rowptr[u + 1]):
                v, nd = int(A.col[k]), d[u] + np.uint64(A.w[k])
                if r0 <= v < r0 + A.n:
                    if nd < d[v - r0]:
                        d[v - r0] = nd
                        nxt.add(v - r0)
                elif nd < rdist[v]:
                    rdist[v] = nd
                    out[v // R].append((v, int(nd)))
        gathered = [None] * world
        dist.all_gather_object(gathered, out)          # the exchange step
        for p in range(world):
            for v, nd in gathered[p][rank]:
                if nd < d[v - r0]:
                    d[v - r0] = nd
                    nxt.add(v - r0)
        front = sorted(nxt)
        tot = torch.tensor([len(front)], dtype=torch.int64)
        dist.all_reduce(tot)                             # stop test
        if int(tot) == 0:
            break
    parts = [None] * world
    dist.all_gather_object(parts, d.astype(np.uint32))
    if rank == 0:
        np.save(os.path.join(out_dir, "d.npy"), np.concatenate(parts))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_sssp_gloo(tmp_path, orc, world):
    g = dpc.gen_rmat(SCALE, 16, seed=7, permute=True)
    src = int(np.argmax(g.degrees()))
    np.save(tmp_path / "src.npy", np.array(src))
    mp.spawn(_sssp_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    d = np.load(tmp_path / "d.npy")
    assert np.array_equal(d, orc.sssp(g.rowptr, g.col, g.w, src))
