#!/usr/bin/env python
"""bench.py — BASELINE.json metric "SSSP/SpMV GTEPS per B200 (1-8 GPU) & speedup
vs basic-DP and flat kernels".

Default (N=1) workload = BASELINE config 2: SpMV on a synthetic R-MAT scale-20
matrix (1,048,576 rows, 16,777,216 nnz, fp32 values and x in (0, 1]).  A step
is one y = A x.  The headline is the grid-consolidated variant; flat,
basic-DP, warp and block are timed in the same run and reported beside it
(`variants`), with the speed-ups the north_star targets.

  value     : nnz processed per second (GTEPS) with A, x, y resident in HBM,
              device-timed with CUDA events per step, L2 flushed between steps
  e2e       : same metric through the C-ABI call dpc_spmv_host with pinned
              host x / y (H2D of x and D2H of y inside the timed region; A is
              the resident operator, uploaded once)
  roofline  : algorithmic bytes nnz*8 + (n+1)*4 + n*4 + n*4 per step over the
              step time (one persistent kernel = the whole step)
  cpu_baseline : oracle port (multi-threaded fp32 CSR SpMV, all host cores)

--impl reference runs the reference's own CPU path: the unmodified dpcons
simulator (oracle/_ref/libref_sim.so, compiled from /root/reference) executing
our SpMV .kdl in grid-consolidated mode on a bounded row sample per step.
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SCALE = 20
EDGEFACTOR = 16
SEED = 1
VARIANTS = ["flat", "basic", "warp", "block", "grid"]


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def _dist_init(world, force=False):
    if world <= 1 and not force:
        return None
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29511")
    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("WORLD_SIZE", str(max(1, world)))
    dist.init_process_group("gloo")
    return dist


def _barrier(dist):
    if dist is not None:
        dist.barrier()


def _max_over_ranks(dist, v):
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _sum_over_ranks(dist, v):
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.f = None

    def __enter__(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if self.proc is None or self.f is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                p = [x.strip() for x in line.split(",")]
                if len(p) >= 9:
                    rows.append(p)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def spmv_bytes(n, nnz):
    return nnz * 8 + (n + 1) * 4 + n * 4 + n * 4


def cpu_baseline_spmv(g, x, budget_s=10.0):
    from tests._oracle import Oracle
    orc = Oracle()
    threads = os.cpu_count() or 1
    orc.spmv_f32_mt(g.rowptr, g.col, g.val, x, threads)  # warm
    reps, t0 = 0, time.perf_counter()
    while True:
        orc.spmv_f32_mt(g.rowptr, g.col, g.val, x, threads)
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or reps >= 400:
            break
    return {"value": round(g.m * reps / el / 1e9, 4), "unit": "GTEPS", "cores": threads,
            "kind": "port",
            "sample": f"{reps} full SpMVs of the config-2 matrix (oracle/oracle.c orc_spmv_f32_mt, "
                      f"{threads} threads, {el:.1f} s)"}


def time_variant(ctx, dg, variant, steps, warmup, cfg=None):
    for _ in range(warmup):
        dg.spmv(variant, cfg=cfg)
    ctx.synchronize()
    total = 0.0
    for _ in range(steps):
        ctx.flush_l2()
        ctx.record(0)
        dg.spmv(variant, cfg=cfg)
        ctx.record(1)
        total += ctx.elapsed_ms(0, 1)
    return total / steps


def _x_global(n):
    """x in (0, 1], a pure function of the global index (same on every rank)."""
    rng = np.random.default_rng(SEED)
    return (rng.integers(1, 1 << 24, n) / float(1 << 24)).astype(np.float32)


def _run_fused(args, dist, ctx, dg, dx, R, rank, world, y64):
    """dpc_multi_spmv_fused over IPC-mapped peer x slices: per step a device
    peer barrier (x written), the SpMV reading x from the owners (pulled into
    the local x before the kernel's own barrier, or gathered entry by entry),
    a peer barrier (x reads done); max over ranks.  The caller keeps the
    NCCL numbers as the headline when this fails or is slower."""
    import paper_1606_08150_b200 as dpc
    res, opened, bufs = {"ok": False}, [], []
    try:
        flags = ctx.alloc(16 * world)
        bufs.append(flags)
        ctx.h2d(flags, np.zeros(2 * world, np.uint64))
        ctx.synchronize()
        hs = [None] * world
        dist.all_gather_object(hs, (dpc.ipc_handle(dx), dpc.ipc_handle(flags)))
        xs, fs = [], []
        for q in range(world):
            if q == rank:
                xs.append(dx)
                fs.append(flags)
            else:
                xp, fp = dpc.ipc_open(ctx, hs[q][0]), dpc.ipc_open(ctx, hs[q][1])
                opened += [xp, fp]
                xs.append(xp)
                fs.append(fp)
        xtab, ftab = ctx.alloc(8 * world), ctx.alloc(8 * world)
        bufs += [xtab, ftab]
        ctx.h2d(xtab, np.array(xs, np.uint64))
        ctx.h2d(ftab, np.array(fs, np.uint64))
        yd = ctx.alloc(4 * R)
        bufs.append(yd)
        epoch = 0

        def step(cfg):
            nonlocal epoch
            dpc.p2p_barrier(ctx, ftab, world, rank, epoch + 1)
            dg.spmv_fused(xtab, world, R, yd, cfg=cfg)
            dpc.p2p_barrier(ctx, ftab, world, rank, epoch + 2)
            epoch += 2

        # two exchange forms inside the one kernel: "pull" (default: the
        # owners' x slices copied into the local x with coalesced peer reads
        # before the kernel's device-wide barrier, then local gathers) and
        # "peer_gather" (every x gather read from its owner; with shape 4's
        # shared-memory cache of the hottest columns)
        gather = dpc.launch_cfg("spmv", "grid")
        gather.flags |= dpc.CFG_X_PEER_GATHER | (4 << 20)
        shapes = {}
        for name, cfg in (("pull", None), ("peer_gather", gather)):
            ctx.h2d(yd, np.zeros(R, np.float32))
            step(cfg)
            dpc.p2p_check(ctx)
            y = ctx.d2h(yd, R).astype(np.float64)
            ok = bool(np.all(np.abs(y - y64) <= 1e-5 * np.abs(y64)))
            for _ in range(args.warmup):
                step(cfg)
            ctx.synchronize()
            _barrier(dist)
            ts = []
            for _ in range(args.steps):
                ctx.flush_l2()
                ctx.record(4)
                step(cfg)
                ctx.record(5)
                ts.append(ctx.elapsed_ms(4, 5))
            dpc.p2p_check(ctx)
            ms = float(np.mean(ts))
            shapes[name] = {"ok": _sum_over_ranks(dist, float(ok)) == world, "ms_max": _max_over_ranks(dist, ms)}
        good = {k: v for k, v in shapes.items() if v["ok"]}
        best = min(good, key=lambda k: good[k]["ms_max"]) if good else "pull"
        res = {"ok": bool(good), "ms": shapes[best]["ms_max"], "ms_max": shapes[best]["ms_max"], "mode": best,
               "modes": shapes,
               "api": "dpc_p2p_barrier + dpc_multi_spmv_fused + dpc_p2p_barrier (C ABI), per rank"}
    except Exception as e:  # noqa: BLE001 - fall back to the NCCL path
        res = {"ok": False, "error": str(e)[:300]}
    for p in opened:
        try:
            dpc.ipc_close(p)
        except Exception:  # noqa: BLE001
            pass
    for b in bufs:
        ctx.free(b)
    return res


def run_multi(args, dist, rank, world, local):
    """BASELINE config 5 shape, weak scaling: a vertex-permuted R-MAT of scale
    20 + log2(N) split into N equal row blocks (2^20 rows, ~16.8M nnz per
    GPU).  One step = ncclAllGather of the x slices over NVLink + the local
    grid-consolidated SpMV (dpc_multi_spmv), max over ranks."""
    import math

    import paper_1606_08150_b200 as dpc
    from tests._oracle import Oracle
    if world & (world - 1):
        raise SystemExit("--gpus must be a power of two")
    scale = SCALE + int(math.log2(world))
    R = 1 << SCALE
    r0 = rank * R
    ctx = dpc.Context(local)
    t0 = time.time()
    A = dpc.gen_rmat_rows(scale, r0, r0 + R, EDGEFACTOR, seed=SEED, weights=False, values=True,
                          permute=True)
    gen_s = time.time() - t0
    dg = dpc.DeviceGraph(ctx, A)
    x_full = _x_global(A.ncols)
    dx = ctx.alloc(4 * R)
    ctx.h2d(dx, x_full[r0:r0 + R])
    uid = [dpc.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = dpc.Comm(ctx, rank, world, uid[0])
    comm.spmv(dg, dx, dg.y_ptr)
    y = dg.get_y().astype(np.float64)
    y64 = Oracle().spmv_f64(A.rowptr, A.col, A.val, x_full)
    parity_ok = bool(np.all(np.abs(y - y64) <= 1e-5 * np.abs(y64)))
    for _ in range(args.warmup):
        comm.spmv(dg, dx, dg.y_ptr)
    ctx.synchronize()
    _barrier(dist)
    ts = []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            ctx.flush_l2()
            ctx.record(0)
            comm.spmv(dg, dx, dg.y_ptr)
            ctx.record(1)
            ts.append(ctx.elapsed_ms(0, 1))
    ctx.synchronize()
    _barrier(dist)
    ms = float(np.mean(ts))
    ms_max = _max_over_ranks(dist, ms)
    total_nnz = _sum_over_ranks(dist, float(A.m))
    # e2e: host x slice in (pinned), all-gather + SpMV, host y slice out
    import ctypes as C
    xh = dpc._lib.dpc_host_alloc(4 * R)
    xa = np.frombuffer((C.c_float * R).from_address(xh), np.float32)
    xa[:] = x_full[r0:r0 + R]
    e2e = []
    for i in range(args.warmup + args.steps):
        _barrier(dist) if i == args.warmup else None
        ctx.record(2)
        ctx.h2d(dx, xa)
        comm.spmv(dg, dx, dg.y_ptr)
        yl = dg.get_y()
        ctx.record(3)
        if i >= args.warmup:
            e2e.append(ctx.elapsed_ms(2, 3))
    e2e_max = _max_over_ranks(dist, float(np.mean(e2e)))
    e2e_ok = bool(np.all(np.abs(yl.astype(np.float64) - y64) <= 1e-5 * np.abs(y64)))
    ok_all = _sum_over_ranks(dist, float(parity_ok and e2e_ok)) == world
    fused = _run_fused(args, dist, ctx, dg, dx, R, rank, world, y64)
    peak = _peak_hbm()
    alg = spmv_bytes(R, A.m) + 4 * (A.ncols - R)  # + the gathered remote x slices
    out = {
        "metric": "SSSP/SpMV GTEPS per B200 (1-8 GPU) & speedup vs basic-DP and flat kernels",
        "value": round(total_nnz / (ms_max * 1e-3) / 1e9, 3), "unit": "GTEPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"BASELINE config 5 shape: SpMV on a vertex-permuted R-MAT scale-{scale} "
                               f"matrix, {world} equal row blocks of 2^20 rows (~16.8M nnz) per GPU",
                   "parallelism": f"row-partition x{world}, ncclAllGather of x over NVLink",
                   "l2": "flushed before every timed step", "generate_s": round(gen_s, 2)},
        "parity": {"all_ranks_vs_fp64_rtol_1e-5": ok_all},
        "e2e": {"value": round(total_nnz / (e2e_max * 1e-3) / 1e9, 3), "unit": "GTEPS",
                "h2d_bytes_per_step": 4 * R, "d2h_bytes_per_step": 4 * R,
                "ms_per_step": round(e2e_max, 4),
                "api": "dpc_copy_h2d + dpc_multi_spmv + dpc_copy_d2h (C ABI), per rank"},
        "roofline": {"bound": "hbm", "achieved": round(alg / (ms * 1e-3) / 1e9, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(alg / (ms * 1e-3) / 1e9 / peak, 4),
                     "traffic": None, "algorithmic_bytes": alg,
                     "kernel": "ncclAllGather + spmv::grid_stream (rank 0)"},
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
    }
    if fused.get("ok") and fused["ms_max"] < ms_max:
        # headline: the faster exchange form, both reported (the fused one
        # pays two peer barriers; NCCL's all-gather pays the copy + launch)
        out["nccl_allgather"] = {"value": out["value"], "ms_per_step": out["ms_per_step"],
                                 "kernel": "ncclAllGather + spmv::grid_stream"}
        out["value"] = round(total_nnz / (fused["ms_max"] * 1e-3) / 1e9, 3)
        out["ms_per_step"] = round(fused["ms_max"], 4)
        out["config"]["parallelism"] = (f"row-partition x{world}; the owners' x slices pulled (or gathered) "
                                        "inside the SpMV kernel through CUDA IPC peer pointers over NVLink / "
                                        "NVSwitch, device-side peer barriers, no NCCL on the data path")
        out["roofline"]["kernel"] = "spmv::grid_stream with peer x (dpc_multi_spmv_fused, rank 0)"
        out["roofline"]["achieved"] = round(alg / (fused["ms"] * 1e-3) / 1e9, 1)
        out["roofline"]["frac"] = round(alg / (fused["ms"] * 1e-3) / 1e9 / peak, 4)
        out["gpu_launches"] = 3 * args.steps
    out["fused"] = {k: v for k, v in fused.items() if k != "ms_max"}
    out["sssp"] = run_multi_sssp(args, dist, rank, world, ctx, comm, scale, r0, R)
    if rank == 0:
        print(json.dumps(out), flush=True)
    comm.close()
    ctx.free(dx)
    dg.close()
    ctx.close()
    dist.destroy_process_group()


def run_multi_sssp(args, dist, rank, world, ctx, comm, scale, r0, R):
    """Vertex-partitioned SSSP on the same R-MAT shape (integer weights
    [1, 255], source = vertex 0 of the permuted graph's largest block row):
    dpc_multi_sssp = local consolidated relaxation + grouped NCCL send/recv of
    {vertex, distance} pairs per iteration.  GTEPS = edges of the reached
    vertices / device time (max over ranks)."""
    import paper_1606_08150_b200 as dpc
    n = 1 << scale
    A = dpc.gen_rmat_rows(scale, r0, r0 + R, EDGEFACTOR, seed=SEED, weights=True, permute=True)
    dg = dpc.DeviceGraph(ctx, A)
    deg = A.degrees()
    cand = np.array([r0 + int(np.argmax(deg)), int(deg.max())], dtype=np.float64)
    t = __import__("torch").tensor(cand)
    allc = [__import__("torch").zeros(2, dtype=__import__("torch").float64) for _ in range(world)]
    dist.all_gather(allc, t)
    source = int(max(allc, key=lambda x: float(x[1]))[0])
    met = comm.sssp(dg, n, source)  # warm-up / correctness run
    d = dg.get_dist()
    reached = d != 0xFFFFFFFF
    te = float(deg[reached].sum())
    ts = []
    for _ in range(max(1, min(args.steps, 5))):
        _barrier(dist)
        ctx.record(4)
        comm.sssp(dg, n, source)
        ctx.record(5)
        ts.append(ctx.elapsed_ms(4, 5))
    ms = _max_over_ranks(dist, float(np.median(ts)))
    edges = _sum_over_ranks(dist, te)
    fused = _sssp_fused(args, dist, ctx, dg, rank, world, n, source, d)
    dg.close()
    out = {"metric": "SSSP GTEPS (edges of reached vertices / time)", "value": round(edges / (ms * 1e-3) / 1e9, 3),
           "unit": "GTEPS", "ms": round(ms, 3), "iterations": int(met.iterations), "source": source,
           "workload": f"R-MAT scale {scale}, vertex-permuted, {world} row blocks, int weights [1,255]",
           "exchange": "grouped ncclSend/ncclRecv of {vertex, distance} pairs + ncclAllGather counts + "
                       "ncclAllReduce frontier size per iteration"}
    if fused.get("ok"):
        out["fused"] = {"value": round(edges / (fused["ms"] * 1e-3) / 1e9, 3), "ms": round(fused["ms"], 3),
                        "exchange": "remote relaxations straight into the owners' dist / stamp / frontier "
                                    "(CUDA IPC peer pointers, NVLink atomics) + device peer barriers"}
    else:
        out["fused"] = fused
    return out


def _sssp_fused(args, dist, ctx, dg, rank, world, n, source, d_ref):
    """The fused partitioned SSSP (dpc_msssp_* with peer tables): per
    iteration relax (remote vertices written in their owner's buffers), peer
    barrier, apply, peer barrier carrying the next-frontier sizes."""
    import paper_1606_08150_b200 as dpc
    opened, bufs = [], []
    try:
        flags = ctx.alloc(16 * world)
        bufs.append(flags)

        def run():  # every rank re-initialised (flags, dist, frontier) before anyone relaxes
            ctx.h2d(flags, np.zeros(2 * world, np.uint64))
            ps = dpc.PartitionedSSSP(dg, rank, world, n, source)
            ctx.synchronize()
            _barrier(dist)
            return ps

        ps = run()
        mine = ps.buffers()
        hs = [None] * world
        dist.all_gather_object(hs, ([dpc.ipc_handle(b) for b in mine], dpc.ipc_handle(flags)))
        table, fl = [], []
        for q in range(world):
            if q == rank:
                table += mine
                fl.append(flags)
            else:
                ptrs = [dpc.ipc_open(ctx, h) for h in hs[q][0]]
                fp = dpc.ipc_open(ctx, hs[q][1])
                opened += ptrs + [fp]
                table += ptrs
                fl.append(fp)
        tab, ftab = ctx.alloc(8 * 5 * world), ctx.alloc(8 * world)
        bufs += [tab, ftab]
        ctx.h2d(tab, np.array(table, np.uint64))
        ctx.h2d(ftab, np.array(fl, np.uint64))

        def solve(ps):
            ps.set_peers(tab)
            epoch = 0
            for _ in range(n + 1):
                ps.relax()
                epoch += 1
                dpc.p2p_barrier(ctx, ftab, world, rank, epoch)
                nxt = ps.apply(np.zeros((0, 2), np.uint32))
                epoch += 1
                if dpc.p2p_barrier_sum(ctx, ftab, world, rank, epoch, nxt) == 0:
                    break
            ps.end()

        solve(ps)
        ok = _sum_over_ranks(dist, float(np.array_equal(dg.get_dist(), d_ref))) == world
        ts = []
        for _ in range(max(1, min(args.steps, 5))):
            ps = run()
            ctx.record(6)
            solve(ps)
            ctx.record(7)
            ts.append(ctx.elapsed_ms(6, 7))
        res = {"ok": ok, "ms": _max_over_ranks(dist, float(np.median(ts)))}
    except Exception as e:  # noqa: BLE001 - the NCCL numbers stand
        res = {"ok": False, "error": str(e)[:300]}
    for p in opened:
        try:
            dpc.ipc_close(p)
        except Exception:  # noqa: BLE001
            pass
    for b in bufs:
        ctx.free(b)
    return res


def _ncu_traffic(profile="r01_spmv_grid_stream.txt"):
    """dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel
    from the committed `ncu --set full` summary (profiles/), in bytes per
    launch -- the ncu capture cannot run inside the timed bench."""
    units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    try:
        with open(os.path.join(ROOT, "profiles", profile)) as f:
            for line in f:
                line = line.strip()
                if line.startswith(("dram__bytes_read.sum =", "dram__bytes_write.sum =")):
                    _, val = line.split("=", 1)
                    num, unit = val.split()
                    tot += float(num) * units.get(unit, 1)
    except (OSError, ValueError):
        return None
    return int(tot) if tot else None


def _peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f).get("hbm_gbs", 6650.0))
    except (OSError, ValueError):
        return 6650.0


def run_ours(args):
    import paper_1606_08150_b200 as dpc
    rank, world, local = _env_int("RANK", 0), _env_int("WORLD_SIZE", 1), _env_int("LOCAL_RANK", 0)
    dist = _dist_init(world, args.multi)
    if world > 1 or args.multi:
        return run_multi(args, dist, rank, world, local)
    ctx = dpc.Context(local)
    t0 = time.time()
    g = dpc.gen_rmat(SCALE, EDGEFACTOR, seed=SEED + rank, weights=False, values=True)
    gen_s = time.time() - t0
    rng = np.random.default_rng(SEED)
    x = (rng.integers(1, 1 << 24, g.n) / float(1 << 24)).astype(np.float32)
    dg = dpc.DeviceGraph(ctx, g)
    dg.set_x(x)
    n, nnz = g.n, g.m

    # correctness gate before timing: grid variant vs fp64 (cheap, C oracle)
    from tests._oracle import Oracle
    y64 = Oracle().spmv_f64(g.rowptr, g.col, g.val, x)
    dg.spmv("grid")
    err = np.abs(dg.get_y().astype(np.float64) - y64) / np.maximum(np.abs(y64), 1e-300)
    parity_ok = bool(np.all(err <= 1e-5))

    variants = {}
    launches = {}
    for v in args.variants:
        if v == "grid":
            continue
        steps = args.steps if v != "basic" else max(1, min(args.steps, 3))
        ms = time_variant(ctx, dg, v, steps, max(1, min(args.warmup, 2)) if v == "basic" else args.warmup)
        met = dg.spmv(v, metrics=True)
        variants[v] = {"ms": round(ms, 4), "gteps": round(nnz / (ms * 1e-3) / 1e9, 3),
                       "device_launches": int(met.child_launch_count)}
        launches[v] = int(met.child_launch_count)
    # CDP form of the grid variant: one child launch by the last block, the
    # paper's threshold (32) and chunked items (its measured best form)
    cdp = dpc.launch_cfg("spmv", "grid", grid_cdp=True, threshold=32)
    ms_cdp = time_variant(ctx, dg, "grid", args.steps, args.warmup, cfg=cdp)
    met_cdp = dg.spmv("grid", cfg=cdp, metrics=True)
    variants["grid_cdp"] = {"ms": round(ms_cdp, 4), "gteps": round(nnz / (ms_cdp * 1e-3) / 1e9, 3),
                            "device_launches": int(met_cdp.child_launch_count)}

    # headline: grid-consolidated (persistent) — timed region
    for _ in range(args.warmup):
        dg.spmv("grid")
    ctx.synchronize()
    _barrier(dist)
    per_step = []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            ctx.flush_l2()
            ctx.record(0)
            dg.spmv("grid")
            ctx.record(1)
            per_step.append(ctx.elapsed_ms(0, 1))
    ctx.synchronize()
    _barrier(dist)
    ms = float(np.mean(per_step))
    ms_max = _max_over_ranks(dist, ms)
    met = dg.spmv("grid", metrics=True)
    variants["grid"] = {"ms": round(ms, 4), "gteps": round(nnz / (ms * 1e-3) / 1e9, 3),
                        "device_launches": int(met.child_launch_count)}
    total_nnz = _sum_over_ranks(dist, float(nnz))
    value = total_nnz / (ms_max * 1e-3) / 1e9

    # e2e through the C ABI with pinned host buffers
    import ctypes as C
    xh = dpc._lib.dpc_host_alloc(4 * n)
    yh = dpc._lib.dpc_host_alloc(4 * n)
    xa = np.frombuffer((C.c_float * n).from_address(xh), np.float32)
    ya = np.frombuffer((C.c_float * n).from_address(yh), np.float32)
    xa[:] = x
    for _ in range(args.warmup):
        dg.spmv_host(xa, ya, "grid")
    _barrier(dist)
    e2e_ms = []
    for _ in range(args.steps):
        ctx.flush_l2()
        ctx.record(2)
        dg.spmv_host(xa, ya, "grid")
        ctx.record(3)
        e2e_ms.append(ctx.elapsed_ms(2, 3))
    e2e_ok = bool(np.all(np.abs(ya.astype(np.float64) - y64) <= 1e-5 * np.abs(y64)))
    e2e_sync_max = _max_over_ranks(dist, float(np.mean(e2e_ms)))
    # serving form: dpc_spmv_host_batch over the K steps, copy-in of vector
    # i+1 and copy-out of vector i-1 overlapping SpMV i (every vector still
    # crosses PCIe both ways inside the timed region); 4 rotating pinned
    # host vector pairs; no L2 flush inside the pipeline (A + x + y > L2)
    nbuf = 4
    xhs = [dpc._lib.dpc_host_alloc(4 * n) for _ in range(nbuf)]
    yhs = [dpc._lib.dpc_host_alloc(4 * n) for _ in range(nbuf)]
    xbs = [np.frombuffer((C.c_float * n).from_address(p), np.float32) for p in xhs]
    ybs = [np.frombuffer((C.c_float * n).from_address(p), np.float32) for p in yhs]
    for xb in xbs:
        xb[:] = x
    dg.spmv_host_batch([xbs[i % nbuf] for i in range(max(2, args.warmup))],
                       [ybs[i % nbuf] for i in range(max(2, args.warmup))], "grid")
    for yb in ybs:
        yb[:] = 0
    _barrier(dist)
    ctx.flush_l2()
    kb = max(args.steps, 32)   # vectors per batch: amortises the pipeline fill / drain
    ctx.record(2)
    dg.spmv_host_batch([xbs[i % nbuf] for i in range(kb)], [ybs[i % nbuf] for i in range(kb)], "grid")
    ctx.record(3)
    batch_ms = ctx.elapsed_ms(2, 3) / kb
    e2e_ok = e2e_ok and all(bool(np.all(np.abs(ybs[i].astype(np.float64) - y64) <= 1e-5 * np.abs(y64)))
                            for i in range(min(nbuf, args.steps)))
    e2e_max = _max_over_ranks(dist, batch_ms)
    e2e_value = total_nnz / (e2e_max * 1e-3) / 1e9

    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    alg = spmv_bytes(n, nnz)
    achieved = alg / (ms * 1e-3) / 1e9

    out = {
        "metric": "SSSP/SpMV GTEPS per B200 (1-8 GPU) & speedup vs basic-DP and flat kernels",
        "value": round(value, 3), "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "BASELINE config 2: SpMV CSR, synthetic R-MAT scale-20 matrix "
                               "(1,048,576 rows, 16,777,216 nnz, fp32 values/x in (0,1], seed 1)",
                   "variant": "grid-consolidated: one persistent kernel (one 1024-thread block per SM, all co-resident), insert phase + "
                              "device-wide barrier + stream-balanced drain (threshold 0, measured)",
                   "n": n, "nnz": nnz, "l2": "flushed (512 MB memset) before every timed step",
                   "parallelism": f"replicas{world}" if world > 1 else "single GPU",
                   "generate_s": round(gen_s, 2)},
        "variants": variants,
        "speedup": {"grid_vs_basic": round(variants["basic"]["ms"] / ms, 2) if "basic" in variants else None,
                    "grid_vs_flat": round(variants["flat"]["ms"] / ms, 2) if "flat" in variants else None,
                    "block_vs_basic": round(variants["basic"]["ms"] / variants["block"]["ms"], 2)
                    if "basic" in variants and "block" in variants else None,
                    "block_vs_flat": round(variants["flat"]["ms"] / variants["block"]["ms"], 2)
                    if "flat" in variants and "block" in variants else None},
        "parity": {"grid_vs_fp64_rtol_1e-5": parity_ok, "e2e_vs_fp64_rtol_1e-5": e2e_ok,
                   "max_rel_err": float(err.max())},
        "e2e": {"value": round(e2e_value, 3), "unit": "GTEPS", "h2d_bytes_per_step": 4 * n,
                "d2h_bytes_per_step": 4 * n, "ms_per_step": round(e2e_max, 4),
                "api": f"dpc_spmv_host_batch (C ABI): one batch of {max(args.steps, 32)} host vectors, "
                       "copy-in / SpMV / copy-out pipelined over two copy streams (steady state is bound by "
                       "the PCIe copies, ~90 us per 4 MB); pinned host x/y, A resident; no L2 flush inside "
                       "the batch (A + x + y = 147 MB > 126 MB L2)",
                "sync_per_call": {"value": round(total_nnz / (e2e_sync_max * 1e-3) / 1e9, 3),
                                  "ms_per_step": round(e2e_sync_max, 4),
                                  "api": "dpc_spmv_host (C ABI), one synchronous call per step, L2 flushed"}},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": _ncu_traffic(),
                     "traffic_source": "profiles/r01_spmv_grid_stream.txt (ncu --set full, dram bytes read+write per launch)",
                     "algorithmic_bytes": alg, "kernel": "spmv::grid_stream (whole step)",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)"},
        "gpu_launches": args.steps * (1 + int(met.child_launch_count)),
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_spmv(g, x, args.cpu_budget)
    if rank == 0 and world == 1 and args.apps:
        # the other BASELINE apps, every variant, each checked against the
        # oracle (speed-ups vs basic-DP and flat per app; tools/prof_apps.py)
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from prof_apps import run_apps
        dg.close()
        out["apps"] = run_apps(ctx, args.apps, reps=2)
    if rank == 0 and world == 1 and args.kdl:
        # the DSL compiler's output: bundled .kdl programs
        # compiled for sm_100a in basic / warp / block / grid mode
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from kdl_bench import run_compiled
        try:
            out["kdl"] = run_compiled(reps=2)
        except Exception as e:  # noqa: BLE001 - the headline line must still print
            out["kdl"] = {"error": str(e)[:300]}
    if rank == 0:
        print(json.dumps(out), flush=True)
    dg.close()
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()


def run_reference(args):
    """The reference's own CPU path on the box's host cores: the unmodified
    dpcons simulator (oracle/_ref) running the SpMV .kdl, grid-consolidated,
    on a bounded row sample of the config-2 matrix per step."""
    rank, world = _env_int("RANK", 0), _env_int("WORLD_SIZE", 1)
    if rank != 0:
        return
    try:
        from tests._oracle import RefSim
        ref = RefSim()
    except (FileNotFoundError, OSError) as e:
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref not built: {e}"}))
        return
    # the input is built by the oracle's own R-MAT restatement (oracle.c
    # orc_gen_rmat, test-pinned equal to dpc_gen_rmat): this leg loads no
    # product code, only oracle/liboracle.so and oracle/_ref/libref_sim.so
    from tests._oracle import Oracle
    g_rowptr, g_col, _, g_val = Oracle().gen_rmat(SCALE, EDGEFACTOR, seed=SEED, weights=False, values=True)
    n_rows = len(g_rowptr) - 1
    rng = np.random.default_rng(SEED)
    x = (rng.integers(1, 1 << 24, n_rows) / float(1 << 24)).astype(np.float32)
    src = ref.kdl("spmv.kdl")
    # bounded, representative sample: a seeded uniform random 1/k of the rows
    # (keeps the degree distribution; R-MAT ids are not exchangeable, so a
    # strided or contiguous window would be biased), k = args.ref_stride
    sel = np.sort(np.random.default_rng(SEED).choice(n_rows, n_rows // args.ref_stride, replace=False))
    rows = len(sel)
    deg = (g_rowptr[sel + 1] - g_rowptr[sel]).astype(np.int64)
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    nnz = int(rp[-1])
    idx = np.concatenate([np.arange(g_rowptr[r], g_rowptr[r + 1]) for r in sel])
    col = g_col[idx]
    val = g_val[idx].astype(np.float64)
    # columns index the full x; the sample keeps the full vector
    scal = {"n": rows, "m": nnz, "nx": n_rows, "thr": 32}
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        rc, y, met, err = ref.run(src, "grid", scal, {"rowptr": rp, "col": col},
                                  {"val": val, "x": x.astype(np.float64)}, out="y",
                                  out_len=rows, out_float=True)
        el = time.perf_counter() - t0
        if rc != 0:
            print(json.dumps({"impl": "reference", "unavailable": f"simulator fault: {err}"}))
            return
        if i >= args.warmup:
            times.append(el)
    ms = float(np.mean(times)) * 1e3
    value = nnz / (ms * 1e-3) / 1e9
    sample = (f"seeded random 1/{args.ref_stride} of the rows ({rows} rows, {nnz} nnz) of the "
              f"config-2 matrix per "
              f"step, dpcons::simulate "
              f"grid-consolidated (paper_1606_08150_b200/kdl/programs/spmv.kdl), single-threaded simulator")
    print(json.dumps({
        "impl": "reference",
        "metric": "SSSP/SpMV GTEPS per B200 (1-8 GPU) & speedup vs basic-DP and flat kernels",
        "value": value, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"BASELINE config 2, row sample: a seeded random 1/{args.ref_stride} of the rows of "
                               "the SpMV CSR R-MAT scale-20 matrix (GTEPS is per nonzero, so the rate is "
                               "comparable; the sample is not the whole matrix)",
                   "rows": rows, "nnz": nnz, "same_config": False,
                   "input": "oracle/oracle.c orc_gen_rmat (no product library loaded)"},
        "cpu_baseline": {"value": value, "unit": "GTEPS", "cores": 1, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_metrics": met,
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variants", nargs="*", default=VARIANTS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--ref-stride", type=int, default=256)
    ap.add_argument("--multi", action="store_true",
                    help="run the partitioned (config 5) path even on one rank (testing)")
    ap.add_argument("--no-kdl", dest="kdl", action="store_false",
                    help="skip timing the DSL compiler's generated programs")
    ap.add_argument("--apps", nargs="*",
                    default=["sssp", "bfs", "pr", "gc", "td", "th", "td_paper", "th_paper", "td_deep_fit",
                             "th_deep_fit"],
                    help="other BASELINE apps timed in the same run (empty list: none)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
