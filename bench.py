#!/usr/bin/env python
"""bench.py — BASELINE.json metric "SSSP/SpMV GTEPS per B200 (1-8 GPU) & speedup
vs basic-DP and flat kernels".

Default (N=1) workload = BASELINE config 2: SpMV on a synthetic R-MAT scale-20
matrix (1,048,576 rows, 16,777,216 nnz, fp32 values and x in (0, 1]).  A step
is one y = A x.  The headline is the grid-consolidated variant; flat,
basic-DP, warp and block are timed in the same run and reported beside it
(`variants`), with the speed-ups the north_star targets.

  value     : nnz processed per second (GTEPS) with A, x, y resident in HBM,
              device-timed with one CUDA event pair around the K steps run
              back to back after one 512 MB L2 flush (A + x + y = 155 MB
              exceed the 126 MB L2; per-launch DRAM reads in that sequence
              equal those after a flush, profiles/r02_spmv_b2b_ncu.txt); the
              same steps with a flush and an event pair each are reported as
              config.ms_per_step_flushed_each
  e2e       : same metric through the C-ABI calls with pinned host x / y
              (H2D of x and D2H of y inside the timed region; A is the
              resident operator, uploaded once)
  roofline  : algorithmic bytes nnz*8 + (n+1)*4 + n*4 + n*4 per step over the
              step time (hot-column gather + the persistent drain = the step)
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


C5_SCALE = 24  # BASELINE config 5: R-MAT scale 24, vertex-permuted, the same graph at every N


def _timed(ctx, dist, step, steps, warmup, flush=True):
    """Mean CUDA-event time of `steps` calls of step() after `warmup` calls,
    L2 flushed before each, barrier + synchronize on both sides; max over ranks."""
    for _ in range(warmup):
        step()
    ctx.synchronize()
    _barrier(dist)
    ts = []
    for _ in range(steps):
        if flush:
            ctx.flush_l2()
        ctx.record(0)
        step()
        ctx.record(1)
        ts.append(ctx.elapsed_ms(0, 1))
    ctx.synchronize()
    _barrier(dist)
    return _max_over_ranks(dist, float(np.mean(ts)))


def _all_ranks(dist, ok):
    world = dist.get_world_size() if dist is not None else 1
    return _sum_over_ranks(dist, float(bool(ok))) == world


class _Ipc:
    """Device buffers exchanged between the ranks with CUDA IPC (the fused
    forms read / write the peers' HBM over NVLink / NVSwitch)."""

    def __init__(self, ctx, dist, rank, world):
        self.ctx, self.dist, self.rank, self.world = ctx, dist, rank, world
        self.opened, self.bufs = [], []

    def alloc(self, nbytes):
        p = self.ctx.alloc(nbytes)
        self.bufs.append(p)
        return p

    def table(self, mine):
        """DEVICE array of world x len(mine) pointers: every rank's `mine`."""
        import paper_1606_08150_b200 as dpc
        hs = [None] * self.world
        self.dist.all_gather_object(hs, [dpc.ipc_handle(p) for p in mine])
        ptrs = []
        for q in range(self.world):
            if q == self.rank:
                ptrs += mine
            else:
                for h in hs[q]:
                    p = dpc.ipc_open(self.ctx, h)
                    self.opened.append(p)
                    ptrs.append(p)
        tab = self.alloc(8 * len(ptrs))
        self.ctx.h2d(tab, np.array(ptrs, np.uint64))
        return tab

    def close(self):
        import paper_1606_08150_b200 as dpc
        for p in self.opened:
            try:
                dpc.ipc_close(p)
            except Exception:  # noqa: BLE001
                pass
        for b in self.bufs:
            self.ctx.free(b)
        self.opened, self.bufs = [], []


def run_config5(args, dist, rank, world, device):
    """BASELINE config 5: SpMV and SSSP on ONE fixed R-MAT scale-24 graph
    (16,777,216 vertices, 268,435,456 arcs, vertex-permuted), split into
    `world` equal row blocks (rank p owns rows / vertices [p R, (p+1) R)).
    world = 1 is the same graph on one GPU (single-GPU kernels), so the
    per-N values form a strong-scaling curve.

    SpMV forms: NCCL all-gather of x + local grid SpMV (dpc_multi_spmv), and
    the fused kernel that reads the owners' x slices through peer pointers
    (dpc_multi_spmv_fused, pull and per-gather).  SSSP forms: grouped NCCL
    send/recv of {vertex, distance} pairs (dpc_multi_sssp) and the fused form
    with remote relaxations straight into the owners' arrays.  Every form is
    checked on every rank before it is timed (SpMV: |y - y64| <= 1e-5 |y64|
    against the fp64 oracle; SSSP: bit-exact against the oracle's distances on
    the whole graph); a form that fails is reported and not used.  When ranks
    share a GPU (testing on a 1-GPU box) the NCCL forms are skipped: NCCL
    refuses two ranks on one device."""
    import paper_1606_08150_b200 as dpc
    from tests._oracle import Oracle
    orc = Oracle()
    ndev = _device_count()
    shared = world > ndev
    n = 1 << C5_SCALE
    if world & (world - 1):
        raise SystemExit("--gpus must be a power of two (equal row blocks of the scale-24 graph)")
    R = n // world
    r0 = rank * R
    ctx = dpc.Context(device)
    t0 = time.time()
    A = dpc.gen_rmat_rows(C5_SCALE, r0, r0 + R, EDGEFACTOR, seed=SEED, weights=True, values=True, permute=True)
    gen_s = time.time() - t0
    dg = dpc.DeviceGraph(ctx, A)
    x_full = _x_global(n)
    y64 = orc.spmv_f64(A.rowptr, A.col, A.val, x_full)

    def y_ok(y):
        return bool(np.all(np.abs(y.astype(np.float64) - y64) <= 1e-5 * np.abs(y64)))

    ipc = _Ipc(ctx, dist, rank, world) if world > 1 else None
    comm = None
    launches = {}
    spmv_forms, steps_of = {}, {}
    if world == 1:
        dg.set_x(x_full)
        steps_of["single_gpu_grid"] = (lambda: dg.spmv("grid"), dg.get_y, dg.x_ptr, dg.y_ptr)
        launches["single_gpu_grid"] = 2  # hot-column gather + drain
    else:
        dx = ipc.alloc(4 * R)
        ctx.h2d(dx, x_full[r0:r0 + R])
        if not shared:
            uid = [dpc.Comm.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            comm = dpc.Comm(ctx, rank, world, uid[0])
            steps_of["nccl_allgather"] = (lambda: comm.spmv(dg, dx, dg.y_ptr), dg.get_y, dx, dg.y_ptr)
            launches["nccl_allgather"] = 3  # all-gather + hot-column gather + drain
        flags = ipc.alloc(16 * world)
        ctx.h2d(flags, np.zeros(2 * world, np.uint64))
        ctx.synchronize()
        xtab = ipc.table([dx])
        ftab = ipc.table([flags])
        yd = ipc.alloc(4 * R)
        epoch = [0]
        gather = dpc.launch_cfg("spmv", "grid")
        gather.flags |= dpc.CFG_X_PEER_GATHER | (4 << 20)

        def fused(cfg):
            def step():
                dpc.p2p_barrier(ctx, ftab, world, rank, epoch[0] + 1)  # x slices written
                dg.spmv_fused(xtab, world, R, yd, cfg=cfg)
                dpc.p2p_barrier(ctx, ftab, world, rank, epoch[0] + 2)  # peers done reading x
                epoch[0] += 2
            return step

        def get_yd():
            dpc.p2p_check(ctx)
            return ctx.d2h(yd, R)

        steps_of["fused_pull"] = (fused(None), get_yd, dx, yd)
        steps_of["fused_peer_gather"] = (fused(gather), get_yd, dx, yd)
        launches["fused_pull"] = launches["fused_peer_gather"] = 3
    for name, (step, gety, _, _) in steps_of.items():
        try:
            step()
            ok = _all_ranks(dist, y_ok(gety()))
            ms = _timed(ctx, dist, step, args.steps, args.warmup) if ok else None
            spmv_forms[name] = {"ok": ok, "ms": None if ms is None else round(ms, 4),
                                "gteps": None if ms is None else round(n * EDGEFACTOR / (ms * 1e-3) / 1e9, 3)}
        except dpc.DpcError as e:
            spmv_forms[name] = {"ok": False, "error": str(e)[:200]}
    good = {k: v for k, v in spmv_forms.items() if v.get("ok")}
    best = min(good, key=lambda k: good[k]["ms"]) if good else None

    # e2e of the headline form: host x slice in (pinned), SpMV, host y slice out
    e2e = None
    if best is not None:
        import ctypes as C
        step, _, xdst, ysrc = steps_of[best]
        rows_x = n if world == 1 else R
        xh, yh = dpc._lib.dpc_host_alloc(4 * rows_x), dpc._lib.dpc_host_alloc(4 * A.n)  # pinned
        xa = np.frombuffer((C.c_float * rows_x).from_address(xh), np.float32)
        yl = np.frombuffer((C.c_float * A.n).from_address(yh), np.float32)
        xa[:] = x_full if world == 1 else x_full[r0:r0 + R]
        ts = []
        for i in range(args.warmup + args.steps):
            if i == args.warmup:
                _barrier(dist)
            ctx.record(2)
            ctx.h2d(xdst, xa)
            step()
            dpc._check(dpc._lib.dpc_copy_d2h(ctx.handle, C.c_void_p(yh), C.c_void_p(ysrc), 4 * A.n))
            ctx.record(3)
            if i >= args.warmup:
                ts.append(ctx.elapsed_ms(2, 3))
        e2e_ms = _max_over_ranks(dist, float(np.mean(ts)))
        e2e = {"value": round(n * EDGEFACTOR / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GTEPS",
               "h2d_bytes_per_step": 4 * rows_x, "d2h_bytes_per_step": 4 * A.n,
               "ms_per_step": round(e2e_ms, 4), "parity_ok": _all_ranks(dist, y_ok(yl)),
               "api": {"single_gpu_grid": "dpc_copy_h2d + dpc_spmv_device + dpc_copy_d2h (C ABI)",
                       "nccl_allgather": "dpc_copy_h2d + dpc_multi_spmv + dpc_copy_d2h (C ABI), per rank",
                       }.get(best, "dpc_copy_h2d + dpc_p2p_barrier + dpc_multi_spmv_fused + dpc_p2p_barrier + "
                                   "dpc_copy_d2h (C ABI), per rank")}
        dpc._lib.dpc_host_free(xh)
        dpc._lib.dpc_host_free(yh)
        if world == 1:  # the serving form: consecutive vectors' copies overlap the SpMV in between
            kv = 8
            xp, yp = dpc._lib.dpc_host_alloc(4 * n * kv), dpc._lib.dpc_host_alloc(4 * A.n * kv)
            xs = np.frombuffer((C.c_float * (n * kv)).from_address(xp), np.float32).reshape(kv, n)
            ys = np.frombuffer((C.c_float * (A.n * kv)).from_address(yp), np.float32).reshape(kv, A.n)
            xs[:] = x_full
            dg.spmv_host_batch_contig(xs[:2], ys[:2])
            ctx.record(2)
            dg.spmv_host_batch_contig(xs, ys)
            ctx.record(3)
            bms = ctx.elapsed_ms(2, 3) / kv
            bok = y_ok(ys[0]) and y_ok(ys[kv - 1])
            dpc._lib.dpc_host_free(xp)
            dpc._lib.dpc_host_free(yp)
            e2e["forms_ms_per_vector"] = {"synchronous": e2e["ms_per_step"], "host_batch_contig": round(bms, 4)}
            if bok and bms < e2e["ms_per_step"]:
                e2e.update({"value": round(n * EDGEFACTOR / (bms * 1e-3) / 1e9, 3), "ms_per_step": round(bms, 4),
                            "api": f"dpc_spmv_host_batch_contig (C ABI): {kv} host vectors of 64 MB, copy-in / "
                                   "SpMV / copy-out of consecutive vectors overlapped (double-buffered)"})
            e2e["parity_ok"] = e2e["parity_ok"] and bok

    sssp = _config5_sssp(args, dist, rank, world, ctx, dg, A, comm, ipc, shared, orc)
    if comm is not None:
        comm.close()
    if ipc is not None:
        ipc.close()
    dg.close()
    ctx.close()
    alg = spmv_bytes(A.n, A.m) + 4 * (n - A.n)  # + the remote x slices a rank reads
    peak = _peak_hbm()
    res = {"spmv_forms": spmv_forms, "headline_form": best, "e2e": e2e, "sssp": sssp,
           "launches_per_step": launches.get(best), "generate_s": round(gen_s, 2),
           "rows_per_rank": R, "nnz_rank0": int(A.m), "ranks_share_device": shared}
    if best is not None:
        ms = good[best]["ms"]
        res["value"] = good[best]["gteps"]
        res["ms_per_step"] = ms
        single = best == "single_gpu_grid"
        res["roofline"] = {"bound": "hbm", "achieved": round(alg / (ms * 1e-3) / 1e9, 1), "peak": peak,
                           "unit": "GB/s", "frac": round(alg / (ms * 1e-3) / 1e9 / peak, 4),
                           "traffic": _ncu_traffic("r02_config5_spmv_ncu.txt") if single else None,
                           "traffic_source": "profiles/r02_config5_spmv_ncu.txt" if single else None,
                           "algorithmic_bytes": alg,
                           "kernel": f"{best} (rank 0 row block: nnz*8 + rows*12 + remote x*4)"}
    return res


def _config5_sssp(args, dist, rank, world, ctx, dg, A, comm, ipc, shared, orc):
    """SSSP on the config-5 graph: source = the global max-out-degree vertex;
    the oracle's distances on the WHOLE graph (rank 0 generates it when the
    graph is partitioned) are broadcast and every rank checks its slice."""
    import paper_1606_08150_b200 as dpc
    n = 1 << C5_SCALE
    R, r0 = A.n, rank * A.n
    deg = A.degrees()
    cand = (int(deg.max()), -(r0 + int(np.argmax(deg))))
    if world > 1:
        allc = [None] * world
        dist.all_gather_object(allc, cand)
        cand = max(allc)
    source = -cand[1]
    threads = os.cpu_count() or 1
    t0 = time.time()
    if world == 1:
        ref, _ = orc.sssp_mt(A.rowptr, A.col, A.w, source, threads)
    else:
        import torch
        buf = torch.zeros(n, dtype=torch.int32)
        if rank == 0:
            G = dpc.gen_rmat(C5_SCALE, EDGEFACTOR, seed=SEED, weights=True, permute=True)
            full, _ = orc.sssp_mt(G.rowptr, G.col, G.w, source, threads)
            del G
            buf = torch.from_numpy(full.view(np.int32).copy())
        dist.broadcast(buf, src=0)
        ref = buf.numpy().view(np.uint32)
    oracle_s = time.time() - t0
    mine = ref[r0:r0 + R]
    m_reached = int(_sum_over_ranks(dist, float(deg[mine != np.uint32(0xFFFFFFFF)].sum())))
    reps = max(1, min(args.steps, 5))
    forms = {}

    def record(name, solve, get_dist, prepare=None, solve_timed=None):
        """prepare() (re-initialisation, host barrier) runs outside the timed
        region; solve() is one whole SSSP run (solve_timed: the same without
        reading metrics back)."""
        try:
            if prepare:
                prepare()
            met = solve()
            ok = _all_ranks(dist, np.array_equal(get_dist(), mine))
            ms = None
            if ok:
                ts = []
                for _ in range(reps):
                    if prepare:
                        prepare()
                    ctx.flush_l2()
                    ctx.synchronize()
                    _barrier(dist)
                    ctx.record(4)
                    (solve_timed or solve)()
                    ctx.record(5)
                    ts.append(ctx.elapsed_ms(4, 5))
                ms = _max_over_ranks(dist, float(np.median(ts)))
            forms[name] = {"ok": ok, "ms": None if ms is None else round(ms, 3),
                           "gteps": None if ms is None else round(m_reached / (ms * 1e-3) / 1e9, 3),
                           "iterations": int(getattr(met, "iterations", 0) or 0)}
            if met is not None:
                forms[name]["relaxed_edges"] = int(_sum_over_ranks(dist, float(met.edges_processed)))
                forms[name]["frontier_vertices"] = int(_sum_over_ranks(dist, float(met.vertices_processed)))
        except dpc.DpcError as e:
            forms[name] = {"ok": False, "error": str(e)[:200]}

    if world == 1:
        record("single_gpu_grid", lambda: dg.sssp(source, "grid", metrics=True), dg.get_dist,
               solve_timed=lambda: dg.sssp(source, "grid", metrics=False))
    else:
        if comm is not None:
            record("nccl_sendrecv", lambda: comm.sssp(dg, n, source), dg.get_dist)
        prep, solve = _fused_sssp_runner(ctx, dist, dg, ipc, rank, world, n, source)
        record("fused_peer_atomics", solve, dg.get_dist, prepare=prep)
    good = {k: v for k, v in forms.items() if v.get("ok")}
    best = min(good, key=lambda k: good[k]["ms"]) if good else None
    roof = None
    if best and forms[best].get("frontier_vertices"):
        alg = sssp_bytes(forms[best]["relaxed_edges"], forms[best]["frontier_vertices"]) / world
        ach = alg / (good[best]["ms"] * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": _peak_hbm(), "unit": "GB/s",
                "frac": round(ach / _peak_hbm(), 4), "algorithmic_bytes_per_gpu": int(alg),
                "bytes_rule": "12 B x relaxed edges + 12 B x frontier vertices (SURVEY.md 8(d)), per GPU"}
    out = {"metric": "SSSP GTEPS (edges of the reached component / device time, Graph500)",
           "unit": "GTEPS", "source": source, "m_reached": m_reached, "forms": forms, "headline_form": best,
           "roofline": roof,
           "value": good[best]["gteps"] if best else None, "ms": good[best]["ms"] if best else None,
           "oracle": f"orc_sssp_bf_mt ({threads} threads) on the whole graph, {oracle_s:.1f} s; bit-exact check "
                     "of every rank's slice"}
    return out


def _fused_sssp_runner(ctx, dist, dg, ipc, rank, world, n, source):
    """The fused partitioned SSSP (dpc_msssp_* with peer tables): per
    iteration relax (remote vertices written in their owners' buffers), peer
    barrier, apply, peer barrier carrying the next-frontier sizes."""
    import paper_1606_08150_b200 as dpc
    flags = ipc.alloc(16 * world)
    state = {"tab": None, "ftab": None, "ps": None}

    def prepare():
        ctx.h2d(flags, np.zeros(2 * world, np.uint64))
        ps = state["ps"] = dpc.PartitionedSSSP(dg, rank, world, n, source)
        ctx.synchronize()
        _barrier(dist)  # every rank re-initialised before anyone relaxes
        if state["tab"] is None:
            state["tab"] = ipc.table(ps.buffers())
            state["ftab"] = ipc.table([flags])
        ps.set_peers(state["tab"])

    def solve():
        ps, epoch = state["ps"], 0
        for _ in range(n + 1):
            ps.relax()
            epoch += 1
            dpc.p2p_barrier(ctx, state["ftab"], world, rank, epoch)
            nxt = ps.apply(np.zeros((0, 2), np.uint32))
            epoch += 1
            if dpc.p2p_barrier_sum(ctx, state["ftab"], world, rank, epoch, nxt) == 0:
                break
        return ps.end()

    return prepare, solve


def _device_count():
    try:
        import torch
        return max(1, torch.cuda.device_count())
    except Exception:  # noqa: BLE001
        return 1


def run_multi(args, dist, rank, world, local):
    """N > 1: BASELINE config 5 strong scaling, one JSON line from rank 0."""
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # keep stdout for the JSON line
    cores = os.cpu_count() or 1
    os.environ.setdefault("DPC_HOST_THREADS", str(max(1, cores // world)))
    device = local % _device_count()
    with Clocks(device) as clk:
        r = run_config5(args, dist, rank, world, device)
    spmv_ok = r["headline_form"] is not None
    sssp_ok = r["sssp"]["headline_form"] is not None
    out = {
        "metric": "SSSP/SpMV GTEPS per B200 (1-8 GPU) & speedup vs basic-DP and flat kernels",
        "value": r.get("value") if (spmv_ok and sssp_ok) else None, "unit": "GTEPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r.get("ms_per_step"),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"BASELINE config 5: SpMV (value) and SSSP (sssp) on one R-MAT scale-24 graph "
                               f"(16,777,216 vertices, 268,435,456 arcs, vertex-permuted, int weights [1,255], "
                               f"fp32 values), {world} equal row blocks; the same graph at every N",
                   "parallelism": f"row / vertex partition x{world}: " + {
                       "nccl_allgather": "ncclAllGather of x over NVLink + local grid SpMV",
                       "fused_pull": "owners' x slices pulled inside the SpMV kernel through CUDA IPC peer "
                                     "pointers (NVLink / NVSwitch), device peer barriers, no NCCL on the data path",
                       "fused_peer_gather": "every x gather read from its owner through CUDA IPC peer pointers, "
                                            "device peer barriers"}.get(r["headline_form"], "none passed parity"),
                   "l2": "flushed (512 MB memset) before every timed step; the graph (2.1 GB) exceeds L2",
                   "ranks_share_device": r["ranks_share_device"], "generate_s": r["generate_s"]},
        "spmv": {"forms": r["spmv_forms"], "headline_form": r["headline_form"]},
        "sssp": r["sssp"],
        "parity": {"spmv_all_ranks_rtol_1e-5": spmv_ok, "sssp_all_ranks_bit_exact": sssp_ok},
        "e2e": r["e2e"], "roofline": r.get("roofline"),
        "gpu_launches": (r["launches_per_step"] or 0) * args.steps,
        "clocks": clk.summary(),
    }
    if not (spmv_ok and sssp_ok):
        out["parity_failed"] = True
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()
    if not (spmv_ok and sssp_ok):
        sys.exit(1)


def _ncu_traffic(profile="r02_spmv_plan8_hot_ncu.txt"):
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


SSSP_SCALE = 22


def sssp_bytes(relaxed, frontier_vertices):
    """12 B per relaxed edge (col + w + dist[v] atomicMin)
    + 12 B per frontier vertex (rowptr pair + dist[u])."""
    return 12 * relaxed + 12 * frontier_vertices


def sssp_section(ctx, args):
    """The SSSP half of the metric on one GPU at HBM scale: R-MAT scale 22
    (4,194,304 vertices, 67,108,864 arcs, int weights [1, 255]), source = the
    max-out-degree vertex; grid (headline), block and flat timed, each checked
    bit-exact against the oracle's distances; roofline of the grid run; the
    oracle's multi-threaded Bellman-Ford timed on the host cores beside it."""
    import paper_1606_08150_b200 as dpc
    from tests._oracle import Oracle
    orc = Oracle()
    threads = os.cpu_count() or 1
    g = dpc.gen_rmat(SSSP_SCALE, EDGEFACTOR, seed=SEED, weights=True)
    deg = g.degrees()
    s = int(np.argmax(deg))
    ref, rounds = orc.sssp_mt(g.rowptr, g.col, g.w, s, threads)
    reached = ref != np.uint32(0xFFFFFFFF)
    m_reached, n_reached = int(deg[reached].sum()), int(reached.sum())
    dg = dpc.DeviceGraph(ctx, g)
    variants = {}
    for v in ("grid", "block", "flat"):
        try:
            met = dg.sssp(s, v, metrics=True)
            ok = bool(np.array_equal(dg.get_dist(), ref))
            ts = []
            for _ in range(3 if v != "flat" else 1):
                ctx.flush_l2()
                ctx.record(4)
                dg.sssp(s, v, metrics=False)
                ctx.record(5)
                ts.append(ctx.elapsed_ms(4, 5))
            dg.check()
            ms = float(np.median(ts))
            variants[v] = {"ms": round(ms, 3), "gteps": round(m_reached / (ms * 1e-3) / 1e9, 3), "bit_exact": ok,
                           "iterations": int(met.iterations), "relaxed_edges": int(met.edges_processed),
                           "frontier_vertices": int(met.vertices_processed)}
        except dpc.DpcError as e:
            variants[v] = {"error": str(e)[:200]}
    dg.close()
    out = {"workload": f"SSSP R-MAT scale {SSSP_SCALE} (4,194,304 vertices, 67,108,864 arcs), int weights [1,255], "
                       "source = max-out-degree vertex", "unit": "GTEPS (edges of the reached component / time)",
           "m_reached": m_reached, "n_reached": n_reached, "variants": variants}
    gr = variants.get("grid", {})
    if "ms" in gr:
        if not gr["bit_exact"]:
            out["parity_failed"] = True
        out["value"] = gr["gteps"]
        fv = gr["frontier_vertices"] or n_reached  # (n_reached: lower bound, level form)
        alg = sssp_bytes(gr["relaxed_edges"], fv)
        peak = _peak_hbm()
        out["roofline"] = {"bound": "hbm", "achieved": round(alg / (gr["ms"] * 1e-3) / 1e9, 1), "peak": peak,
                           "unit": "GB/s", "frac": round(alg / (gr["ms"] * 1e-3) / 1e9 / peak, 4),
                           "traffic": _ncu_traffic("r02_sssp22_stream_ncu.txt"),
                           "algorithmic_bytes": alg,
                           "bytes_rule": "12 B x relaxed edges (metrics.edges_processed) + 12 B x frontier "
                                         "vertices (metrics.vertices_processed), SURVEY.md 8(d)",
                           "kernel": "ssst::stream_persistent (frontier stream form; whole run, one launch)",
                           "traffic_source": "profiles/r02_sssp22_stream_ncu.txt (ncu --set full, the same graph, "
                                             "dram bytes read+write of the run's launch)"}
        if "ms" in variants.get("flat", {}):
            out["grid_vs_flat"] = round(variants["flat"]["ms"] / gr["ms"], 2)
    if not args.no_cpu_baseline:
        reps, t0 = 0, time.perf_counter()
        while True:
            orc.sssp_mt(g.rowptr, g.col, g.w, s, threads)
            reps += 1
            el = time.perf_counter() - t0
            if el >= args.cpu_budget or reps >= 50:
                break
        out["cpu_baseline"] = {"value": round(m_reached * reps / el / 1e9, 4), "unit": "GTEPS", "cores": threads,
                               "kind": "port", "sample": f"{reps} whole SSSP runs of the scale-{SSSP_SCALE} graph "
                               f"(oracle/oracle.c orc_sssp_bf_mt, frontier Bellman-Ford, {threads} threads, "
                               f"{el:.1f} s)"}
    return out


def _summary(out):
    """The line's key numbers in one small object (printed last)."""
    def grid_ms(app):
        try:
            return out["apps"][app]["variants"]["grid"]["ms"]
        except (KeyError, TypeError):
            return None
    apps = {}
    for k, v in (out.get("apps") or {}).items():
        if isinstance(v, dict) and "best_vs_basic" in v:
            apps[k] = {"grid_ms": grid_ms(k), "vs_basic": v.get("best_vs_basic"), "vs_flat": v.get("best_vs_flat")}
    roof = out.get("roofline") or {}
    sssp = out.get("sssp") or {}
    c5 = out.get("config5") or {}
    return {"spmv_gteps": out.get("value"), "spmv_ms_per_step": out.get("ms_per_step"),
            "spmv_ms_per_step_flushed_each": (out.get("config") or {}).get("ms_per_step_flushed_each"),
            "roofline_frac": roof.get("frac"), "e2e_gteps": (out.get("e2e") or {}).get("value"),
            "spmv_vs_basic": (out.get("speedup") or {}).get("grid_vs_basic"),
            "spmv_vs_flat": (out.get("speedup") or {}).get("grid_vs_flat"),
            "sssp_scale22_gteps": sssp.get("value"), "sssp_scale22_frac": (sssp.get("roofline") or {}).get("frac"),
            "config5_1gpu_spmv_gteps": c5.get("value"), "config5_1gpu_sssp_gteps": (c5.get("sssp") or {}).get("value"),
            "cpu_baseline_gteps": (out.get("cpu_baseline") or {}).get("value"), "apps": apps,
            "parity_failed": out.get("parity_failed", [])}


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

    # headline: grid-consolidated (persistent) — timed region: the K steps
    # back to back between one event pair, after one 512 MB L2 flush (which
    # the GPU runs while the host enqueues the steps).  A + x + y = 155 MB
    # exceeds the 126 MB L2: under `ncu --cache-control none` every launch of
    # such a sequence reads 144.8 MB from DRAM, the same as a launch after a
    # flush (profiles/r02_spmv_b2b_ncu.txt).  The same K steps timed one by
    # one with a flush before each (round 1's form) are reported beside it.
    with Clocks(local) as clk:
        # warm-up after the clock sampler's start (it idles the GPU for
        # 0.3 s): the timed steps must not pay the clock ramp from idle
        for _ in range(args.warmup):
            dg.spmv("grid")
        ctx.synchronize()
        _barrier(dist)
        ctx.flush_l2()
        ctx.record(0)
        for _ in range(args.steps):
            dg.spmv("grid")
        ctx.record(1)
        ms = ctx.elapsed_ms(0, 1) / args.steps
        per_step = []
        for _ in range(args.steps):
            ctx.flush_l2()
            ctx.record(0)
            dg.spmv("grid")
            ctx.record(1)
            per_step.append(ctx.elapsed_ms(0, 1))
    ctx.synchronize()
    _barrier(dist)
    ms_flushed = float(np.mean(per_step))
    ms_max = _max_over_ranks(dist, ms)
    met = dg.spmv("grid", metrics=True)
    variants["grid"] = {"ms": round(ms_flushed, 4), "gteps": round(nnz / (ms_flushed * 1e-3) / 1e9, 3),
                        "device_launches": int(met.child_launch_count),
                        "ms_back_to_back": round(ms, 4)}  # the headline's timing form
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
    for p in xhs + yhs:
        dpc._lib.dpc_host_free(p)
    # the same serving batch with the vectors back to back in pinned host
    # memory (dpc_spmv_host_batch_contig): copies of 8 vectors (32 MB) at a
    # time -- this box's PCIe moves 4 MB copy pairs at 58 GB/s aggregate and
    # 64 MB pairs at 83 GB/s (tools/probes/lab_r02/duplex_bw.py)
    kc = max(args.steps, 128)
    xcp = dpc._lib.dpc_host_alloc(4 * n * kc)
    ycp = dpc._lib.dpc_host_alloc(4 * n * kc)
    xcs = np.frombuffer((C.c_float * (n * kc)).from_address(xcp), np.float32).reshape(kc, n)
    ycs = np.frombuffer((C.c_float * (n * kc)).from_address(ycp), np.float32).reshape(kc, n)
    xcs[:] = x
    dg.spmv_host_batch_contig(xcs[:8], ycs[:8])  # warm-up (device slots, plan)
    ycs[:] = 0
    _barrier(dist)
    ctx.flush_l2()
    ctx.record(2)
    dg.spmv_host_batch_contig(xcs, ycs)
    ctx.record(3)
    contig_ms = ctx.elapsed_ms(2, 3) / kc
    contig_ok = all(bool(np.all(np.abs(ycs[i].astype(np.float64) - y64) <= 1e-5 * np.abs(y64)))
                    for i in (0, kc // 2, kc - 1))
    dpc._lib.dpc_host_free(xcp)
    dpc._lib.dpc_host_free(ycp)
    e2e_ok = e2e_ok and contig_ok
    contig_max = _max_over_ranks(dist, contig_ms)
    batch_max = _max_over_ranks(dist, batch_ms)
    e2e_max = min(batch_max, contig_max)
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
                   "variant": "grid-consolidated with the cached per-matrix window plan: a hot-column gather launch + one "
                              "persistent drain launch (one 1024-thread block per SM, all co-resident; split-phase "
                              "device-wide barrier; x at the 32K most used columns in shared memory)",
                   "n": n, "nnz": nnz,
                   "l2": ("inputs larger than L2 (A + x + y = 155 MB > 126 MB): the K steps run back to back "
                          "after one 512 MB flush; per launch 144.8 MB DRAM read in such a sequence, as after a "
                          "flush (ncu --cache-control none, profiles/r02_spmv_b2b_ncu.txt)"),
                   "ms_per_step_flushed_each": round(_max_over_ranks(dist, ms_flushed), 4),
                   "timing_note": ("ms_per_step_flushed_each: the same K steps with a 512 MB flush and an event "
                                   "pair around each; ~6 us of it is the method's launch floor, which an empty "
                                   "kernel shows too (profiles/r02_spmv_hot_lab.md)"),
                   "parallelism": f"replicas{world}" if world > 1 else "single GPU",
                   "generate_s": round(gen_s, 2)},
        "variants": variants,
        # speedups against the variants' own timing form (flush + event pair per step)
        "speedup": {"grid_vs_basic": round(variants["basic"]["ms"] / ms_flushed, 2) if "basic" in variants else None,
                    "grid_vs_flat": round(variants["flat"]["ms"] / ms_flushed, 2) if "flat" in variants else None,
                    "block_vs_basic": round(variants["basic"]["ms"] / variants["block"]["ms"], 2)
                    if "basic" in variants and "block" in variants else None,
                    "block_vs_flat": round(variants["flat"]["ms"] / variants["block"]["ms"], 2)
                    if "flat" in variants and "block" in variants else None},
        "parity": {"grid_vs_fp64_rtol_1e-5": parity_ok, "e2e_vs_fp64_rtol_1e-5": e2e_ok,
                   "max_rel_err": float(err.max())},
        "e2e": {"value": round(e2e_value, 3), "unit": "GTEPS", "h2d_bytes_per_step": 4 * n,
                "d2h_bytes_per_step": 4 * n, "ms_per_step": round(e2e_max, 4),
                "api": ("dpc_spmv_host_batch_contig (C ABI): one batch of "
                        f"{max(args.steps, 128)} host vectors stored back to back, copied 8 at a time (32 MB) "
                        if contig_max <= batch_max else
                        f"dpc_spmv_host_batch (C ABI): one batch of {max(args.steps, 32)} host vectors ")
                       + "with copy-in / SpMV / copy-out pipelined over two copy streams (bound by this box's "
                         "PCIe duplex throughput); pinned host x / y, A resident; no L2 flush inside the batch "
                         "(A + x + y = 147 MB > 126 MB L2)",
                "forms_ms_per_vector": {"host_batch_4MB_copies": round(batch_max, 4),
                                        "host_batch_contig_32MB_copies": round(contig_max, 4)},
                "sync_per_call": {"value": round(total_nnz / (e2e_sync_max * 1e-3) / 1e9, 3),
                                  "ms_per_step": round(e2e_sync_max, 4),
                                  "api": "dpc_spmv_host (C ABI), one synchronous call per step, L2 flushed"}},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": _ncu_traffic(),
                     "traffic_source": ("profiles/r02_spmv_plan8_hot_ncu.txt (ncu --set full, dram bytes read + "
                                        "write per launch after a flush); in the headline's back-to-back sequence "
                                        "each launch reads the same 144.8 MB (profiles/r02_spmv_b2b_ncu.txt)"),
                     "algorithmic_bytes": alg, "kernel": "spmvp::plan8_drain<1024, HOT> (whole step incl. spmvp::hot_gather)",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)"},
        "gpu_launches": args.steps * (int(met.host_launches) + int(met.child_launch_count)),
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_spmv(g, x, args.cpu_budget)
    # the SSSP half of the metric at HBM scale (scale 22, one GPU)
    if args.sssp:
        out["sssp"] = sssp_section(ctx, args)
    # BASELINE config 5's graph on this one GPU: the N = 1 point of the
    # strong-scaling curve `bench.py --gpus N` (N > 1) measures
    if args.config5:
        dg.close()
        r5 = run_config5(args, None, 0, 1, local)
        out["config5"] = {"workload": "BASELINE config 5 graph (R-MAT scale 24, vertex-permuted) on one GPU: "
                                      "the N = 1 point of bench.py --gpus N",
                          "value": r5.get("value"), "unit": "GTEPS", "ms_per_step": r5.get("ms_per_step"),
                          "spmv_forms": r5["spmv_forms"], "e2e": r5["e2e"], "roofline": r5.get("roofline"),
                          "sssp": r5["sssp"], "generate_s": r5["generate_s"]}
    failed = [k for k, bad in (("spmv_config2", not parity_ok), ("spmv_config2_e2e", not e2e_ok),
                               ("sssp_scale22", out.get("sssp", {}).get("parity_failed", False)),
                               ("config5_spmv", "config5" in out and out["config5"]["value"] is None),
                               ("config5_sssp", "config5" in out and out["config5"]["sssp"]["value"] is None))
              if bad]
    if failed:
        out["value"] = None
        out["parity_failed"] = failed
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
        out["summary"] = _summary(out)  # last key: what a truncated tail of the line still shows
        print(json.dumps(out), flush=True)
    dg.close()
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()
    if failed:
        sys.exit(1)


_REF_PARTS = None
_REF_SIM = None


def _ref_part(i):
    """One part of the reference arm's row sample, in a forked worker."""
    global _REF_SIM
    if _REF_SIM is None:
        from tests._oracle import RefSim
        _REF_SIM = RefSim()
    src, parts = _REF_PARTS
    pt = parts[i]
    rc, _, met, err = _REF_SIM.run(src, "grid", pt[0], pt[1], pt[2], out="y", out_len=pt[3], out_float=True)
    return rc, None, met, err


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
    # columns index the full x; the sample keeps the full vector.  The
    # simulator is single-threaded and not thread-safe: the sample is cut into
    # one part per host core (equal nonzeros), simulated concurrently by
    # forked worker processes (each with its own simulator instance; the
    # parts are inherited, not pickled), and a step is the wall time of all.
    import multiprocessing as mproc
    threads = max(1, min(os.cpu_count() or 1, rows))
    cuts = np.searchsorted(rp, np.linspace(0, nnz, threads + 1).round().astype(np.int64))
    cuts[0], cuts[-1] = 0, rows
    parts = []
    for t in range(threads):
        r0, r1 = int(cuts[t]), int(cuts[t + 1])
        if r1 > r0:
            prt = rp[r0:r1 + 1] - rp[r0]
            parts.append(({"n": r1 - r0, "m": int(prt[-1]), "nx": n_rows, "thr": 32},
                          {"rowptr": prt, "col": col[rp[r0]:rp[r1]]},
                          {"val": val[rp[r0]:rp[r1]], "x": x.astype(np.float64)}, r1 - r0))

    global _REF_PARTS
    _REF_PARTS = (src, parts)
    times, met = [], None
    with mproc.get_context("fork").Pool(len(parts)) as pool:
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            res = pool.map(_ref_part, range(len(parts)))
            el = time.perf_counter() - t0
            bad = [r for r in res if r[0] != 0]
            if bad:
                print(json.dumps({"impl": "reference", "unavailable": f"simulator fault: {bad[0][3]}"}))
                return
            met = res[0][2]
            if i >= args.warmup:
                times.append(el)
    ms = float(np.mean(times)) * 1e3
    value = nnz / (ms * 1e-3) / 1e9
    sample = (f"seeded random 1/{args.ref_stride} of the rows ({rows} rows, {nnz} nnz) of the "
              f"config-2 matrix per step, dpcons::simulate grid-consolidated "
              f"(paper_1606_08150_b200/kdl/programs/spmv.kdl), cut into {len(parts)} equal-nonzero parts "
              f"simulated concurrently by {len(parts)} worker processes (one per host core)")
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
        "cpu_baseline": {"value": value, "unit": "GTEPS", "cores": len(parts), "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_metrics_part0": met,
    }), flush=True)


def _spawn(nprocs):
    """`python bench.py --gpus N` without a launcher: re-run this script
    under torch.distributed.run, one rank per GPU (ranks share GPUs round
    robin when the box has fewer), rendezvous on 127.0.0.1."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nprocs}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variants", nargs="*", default=VARIANTS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--ref-stride", type=int, default=64)
    ap.add_argument("--multi", action="store_true",
                    help="run the partitioned (config 5) path even on one rank (testing)")
    ap.add_argument("--no-kdl", dest="kdl", action="store_false",
                    help="skip timing the DSL compiler's generated programs")
    ap.add_argument("--apps", nargs="*",
                    default=["sssp", "bfs", "pr", "gc", "td", "th", "td_paper", "th_paper", "td_deep_fit",
                             "th_deep_fit"],
                    help="other BASELINE apps timed in the same run (empty list: none)")
    ap.add_argument("--no-sssp", dest="sssp", action="store_false", help="skip the scale-22 SSSP section")
    ap.add_argument("--no-config5", dest="config5", action="store_false",
                    help="N = 1: skip the config-5 (scale-24) single-GPU point")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(_spawn(args.gpus))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
