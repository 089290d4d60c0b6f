"""SpMV parity on the B200: every variant against the fp64 CPU oracle.

Tolerance (BASELINE.json north_star): per row |y - y64| <= 1e-5 * |y64|
(values and x are positive, so there is no cancellation; empty rows must be 0).
"""
import numpy as np
import pytest

import paper_1606_08150_b200 as dpc

pytestmark = pytest.mark.gpu

VARIANTS = ["flat", "basic", "warp", "block", "grid"]
RTOL = 1e-5


def _x(n, seed=7):
    rng = np.random.default_rng(seed)
    return (rng.integers(1, 1 << 24, n) / float(1 << 24)).astype(np.float32)


def _check(orc, g, x, y):
    y64 = orc.spmv_f64(g.rowptr, g.col, g.val, x)
    err = np.abs(y.astype(np.float64) - y64)
    bad = err > RTOL * np.abs(y64)
    assert not bad.any(), f"{bad.sum()} rows off; worst rel {np.max(err / np.maximum(np.abs(y64), 1e-300))}"


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("scale", [8, 12, 14])
def test_spmv_rmat(ctx, orc, variant, scale):
    g = dpc.gen_rmat(scale, 16, seed=scale, weights=False, values=True)
    x = _x(g.n)
    y, met = dpc.run_spmv(g, x, variant, ctx=ctx)
    _check(orc, g, x, y)
    heavy = int((g.degrees() > 32).sum())
    if variant == "flat":
        assert met.child_launch_count == 0
    elif variant == "basic":
        assert met.child_launch_count == heavy
    elif variant == "grid":
        assert met.child_launch_count == 0  # persistent default: one cooperative kernel


@pytest.mark.parametrize("variant", ["warp", "block", "grid"])
def test_spmv_launch_laws(ctx, variant):
    """Launch-count law (corrected per SURVEY §4): warp <= #warps
    with a heavy row, block <= #blocks with one, grid == 1."""
    g = dpc.gen_rmat(13, 16, seed=3, weights=False, values=True)
    deg = g.degrees()
    heavy = deg > 32
    cfg = dpc.launch_cfg("spmv", variant, grid_cdp=True, threshold=32)
    y, met = dpc.run_spmv(g, _x(g.n), variant, cfg=cfg, ctx=ctx)
    pad = np.zeros((-len(heavy)) % 256, bool)
    h = np.concatenate([heavy, pad])
    if variant == "warp":
        assert met.child_launch_count == int(h.reshape(-1, 32).any(1).sum())
    elif variant == "block":
        assert met.child_launch_count == int(h.reshape(-1, 256).any(1).sum())
    else:
        assert met.child_launch_count == 1


def test_spmv_grid_cdp(ctx, orc):
    g = dpc.gen_rmat(14, 16, seed=5, weights=False, values=True)
    x = _x(g.n)
    y, met = dpc.run_spmv(g, x, "grid", cfg=dpc.launch_cfg("spmv", "grid", grid_cdp=True), ctx=ctx)
    _check(orc, g, x, y)
    assert met.child_launch_count == 1


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("chunk,threshold", [(32, 0), (64, 32), (1000, 5), (4096, 32)])
def test_spmv_cfg_sweep(ctx, orc, variant, chunk, threshold):
    """Moldability: results independent of the configuration."""
    g = dpc.gen_graph(3000, powerlaw=(1.6, 2500), seed=11, weights=False, values=True)
    x = _x(g.n)
    cfg = dpc.launch_cfg("spmv", variant, chunk=chunk, threshold=threshold)
    y, _ = dpc.run_spmv(g, x, variant, cfg=cfg, ctx=ctx)
    _check(orc, g, x, y)


@pytest.mark.parametrize("variant", VARIANTS)
def test_spmv_edge_cases(ctx, orc, variant):
    # empty matrix, single empty row
    g = dpc.csr_from_arrays([0], [], val=[])
    assert g.n == 0
    g = dpc.csr_from_arrays([0, 0], [], val=[])
    y, _ = dpc.run_spmv(g, np.ones(1, np.float32), variant, ctx=ctx)
    assert y.tolist() == [0.0]
    # SPEC.md:459 identity example
    g = dpc.csr_from_arrays([0, 1, 2], [0, 1], val=[1.0, 1.0])
    y, _ = dpc.run_spmv(g, np.array([3, 7], np.float32), variant, ctx=ctx)
    assert y.tolist() == [3.0, 7.0]
    # ragged: rows of every length 0..300 (unaligned starts), plus one hub row
    lens = np.concatenate([np.arange(0, 301), [100_003]])
    rowptr = np.concatenate([[0], np.cumsum(lens)])
    n = len(lens)
    rng = np.random.default_rng(1)
    col = rng.integers(0, n, rowptr[-1]).astype(np.int32)
    val = (rng.integers(1, 1 << 24, rowptr[-1]) / float(1 << 24)).astype(np.float32)
    g = dpc.csr_from_arrays(rowptr, col, val=val)
    x = _x(n)
    y, _ = dpc.run_spmv(g, x, variant, ctx=ctx)
    _check(orc, g, x, y)


def test_spmv_config2_full_size(ctx, orc):
    """BASELINE config 2 at full size (R-MAT scale 20, 16.8M nnz), grid variant
    via the device-resident path, plus the end-to-end host path."""
    g = dpc.gen_rmat(20, 16, seed=1, weights=False, values=True)
    x = _x(g.n)
    dg = dpc.DeviceGraph(ctx, g)
    dg.set_x(x)
    for variant in ["flat", "basic", "warp", "block", "grid"]:
        met = dg.spmv(variant, metrics=True)
        _check(orc, g, x, dg.get_y())
    y = np.empty(g.n, np.float32)
    dg.spmv_host(x, y, "grid")
    _check(orc, g, x, y)
    dg.close()


def _ragged(seed=1, hub=100_003):
    lens = np.concatenate([np.arange(0, 301), [hub], np.arange(300, -1, -7), [4] * 500, [1] * 777])
    rowptr = np.concatenate([[0], np.cumsum(lens)])
    n = len(lens)
    rng = np.random.default_rng(seed)
    col = rng.integers(0, n, rowptr[-1]).astype(np.int32)
    val = (rng.integers(1, 1 << 24, rowptr[-1]) / float(1 << 24)).astype(np.float32)
    return dpc.csr_from_arrays(rowptr, col, val=val)


@pytest.mark.parametrize("shape", [0, 1, 2, 3, 4, 5, 6, 7])
@pytest.mark.parametrize("threshold", [0, 3, 7, 31, 32, 100])
def test_spmv_grid_stream_forms(ctx, orc, shape, threshold):
    """Stream-balanced grid drain: every kernel shape x consolidation
    threshold on ragged rows (unaligned starts, window-boundary items, a hub)
    and on an R-MAT matrix."""
    for g in (_ragged(), dpc.gen_rmat(13, 16, seed=4, weights=False, values=True)):
        x = _x(g.n)
        cfg = dpc.launch_cfg("spmv", "grid", threshold=threshold, spmv_stream=True)
        cfg.flags |= shape << 20
        y, met = dpc.run_spmv(g, x, "grid", cfg=cfg, ctx=ctx)
        _check(orc, g, x, y)
        assert met.child_launch_count == 0


@pytest.mark.parametrize("threshold", [0, 32])
def test_spmv_grid_chunked_form(ctx, orc, threshold):
    g = _ragged(seed=3)
    x = _x(g.n)
    cfg = dpc.launch_cfg("spmv", "grid", grid_chunked=True, threshold=threshold)
    y, _ = dpc.run_spmv(g, x, "grid", cfg=cfg, ctx=ctx)
    _check(orc, g, x, y)


@pytest.mark.parametrize("variant", ["warp", "block"])
def test_spmv_device_heap_allocator(ctx, orc, variant):
    """Allocator study form (DPC_CFG_ALLOC_MALLOC): same results as the pool."""
    g = _ragged(seed=5)
    x = _x(g.n)
    cfg = dpc.launch_cfg("spmv", variant)
    cfg.flags |= 16
    y, met = dpc.run_spmv(g, x, variant, cfg=cfg, ctx=ctx)
    _check(orc, g, x, y)
    assert met.child_launch_count > 0


@pytest.mark.gpu
@pytest.mark.parametrize("count", [1, 2, 5])
def test_spmv_host_batch_pipelined(ctx, orc, count):
    """dpc_spmv_host_batch: distinct host vectors through the pipelined
    copy-in / SpMV / copy-out path, each y checked against the oracle."""
    g = dpc.gen_rmat(14, 16, seed=9, weights=False, values=True)
    dg = dpc.DeviceGraph(ctx, g)
    xs = [((np.arange(g.n) * (i + 3)) % 101 + 1).astype(np.float32) / 101.0 for i in range(count)]
    ys = [np.zeros(g.n, np.float32) for _ in range(count)]
    dg.spmv_host_batch(xs, ys, "grid")
    for x, y in zip(xs, ys):
        y64 = orc.spmv_f64(g.rowptr, g.col, g.val, x)
        assert np.all(np.abs(y - y64) <= 1e-5 * np.abs(y64) + 1e-30)
    dg.close()


# ---- the default grid form: drain with the cached per-matrix window plan
PLAN_FORMS = {"w256": 0, "w128_reg": 1 << 9, "w128_tma": 1 << 12}


def _plan_cases():
    yield _ragged()
    yield _ragged(seed=5, hub=3 * 256 * 32 + 17)        # a hub spanning several chunks
    yield dpc.gen_rmat(13, 16, seed=4, weights=False, values=True)
    yield dpc.gen_rmat(12, 8, seed=6, weights=False, values=True, permute=True)
    # rows of exactly 256 / 128 / 512 nonzeros on window boundaries, then empty rows
    lens = np.array([256, 128, 128, 512, 0, 0, 256, 1, 255, 0, 7, 0], np.int64)
    rowptr = np.concatenate([[0], np.cumsum(lens)])
    rng = np.random.default_rng(2)
    col = rng.integers(0, len(lens), rowptr[-1]).astype(np.int32)
    val = (rng.integers(1, 1 << 24, rowptr[-1]) / float(1 << 24)).astype(np.float32)
    yield dpc.csr_from_arrays(rowptr, col, val=val)
    # all rows empty except the last; a single nonzero; no nonzeros
    yield dpc.csr_from_arrays(np.concatenate([np.zeros(1000, np.int64), [3]]), [5, 6, 7], val=[0.5, 0.25, 1.0])
    yield dpc.csr_from_arrays([0, 1], [0], val=[2.0])
    yield dpc.csr_from_arrays([0, 0, 0, 0], [], val=[])


@pytest.mark.parametrize("form", list(PLAN_FORMS))
def test_spmv_grid_plan_forms(ctx, orc, form):
    """Cached-plan drain (default grid form) and its W = 128 variants on ragged
    rows, window-boundary rows, chunk-spanning hubs, empty rows, R-MAT
    (plain and permuted); repeated calls reuse the plan and the self-resetting
    barrier; results independent of the previous y contents."""
    for g in _plan_cases():
        x = _x(g.ncols if g.ncols else g.n)
        cfg = dpc.launch_cfg("spmv", "grid")
        cfg.flags |= PLAN_FORMS[form]
        dg = dpc.DeviceGraph(ctx, g)
        dg.set_x(x)
        for rep in range(3):
            if g.n:
                ctx.h2d(dg.y_ptr, np.full(g.n, 123.0, np.float32))  # stale y must not leak
            met = dg.spmv("grid", cfg=cfg, metrics=rep == 0)
            if met is not None:
                assert met.child_launch_count == 0
            if g.n:
                _check(orc, g, x, dg.get_y())
        dg.close()


def test_spmv_grid_plan_unaligned_y_and_row_slice(ctx, orc):
    """dpc_spmv_device with a y pointer that is not 16-byte aligned, and the
    plan on a row slice of a larger matrix (global column ids, as the
    partitioned path uploads it)."""
    import ctypes as C
    g = _ragged(seed=9)
    x = _x(g.n)
    dg = dpc.DeviceGraph(ctx, g)
    dg.set_x(x)
    buf = ctx.alloc(4 * (g.n + 1))
    dpc._check(dpc._lib.dpc_spmv_device(ctx.handle, dg._h, C.c_void_p(dg.x_ptr), C.c_void_p(buf + 4),
                                        C.byref(dpc.launch_cfg("spmv", "grid")), None))
    ctx.synchronize()
    dg.check()
    _check(orc, g, x, ctx.d2h(buf + 4, g.n))
    ctx.free(buf)
    dg.close()
    full = dpc.gen_rmat(12, 16, seed=3, weights=False, values=True, permute=True)
    part = dpc.gen_rmat_rows(12, 1024, 2048, 16, seed=3, weights=False, values=True, permute=True)
    xf = _x(full.n)
    dg = dpc.DeviceGraph(ctx, part)
    dg.set_x(xf)
    dg.spmv("grid")
    y64 = orc.spmv_f64(full.rowptr, full.col, full.val, xf)[1024:2048]
    y = dg.get_y().astype(np.float64)
    assert np.all(np.abs(y - y64) <= RTOL * np.abs(y64))
    dg.close()


@pytest.mark.parametrize("cap", ["0", "4", "1000", "32768", "57344"])
def test_spmv_grid_hot_column_cache(ctx, orc, cap, monkeypatch):
    """Default grid form with the hot-column x cache at several slot
    capacities (DPC_SPMV_HOT_CAP; 0 = no cache, 4 = fewer slots than hot
    columns, 57344 = the one-1024-thread-block shape with 224 KB of slots), on
    the plan cases and R-MAT; x changes between calls (the slot table is
    re-gathered every call), and the same matrix switches capacity (the plan
    is rebuilt)."""
    monkeypatch.setenv("DPC_SPMV_HOT_CAP", cap)
    cases = list(_plan_cases()) + [dpc.gen_rmat(14, 16, seed=5, weights=False, values=True)]
    for g in cases:
        if not g.n:
            continue
        dg = dpc.DeviceGraph(ctx, g)
        for rep in range(2):
            x = _x(g.ncols if g.ncols else g.n) * (1.0 + rep)
            dg.set_x(x)
            dg.spmv("grid")
            _check(orc, g, x, dg.get_y())
        monkeypatch.setenv("DPC_SPMV_HOT_CAP", "16")
        dg.spmv("grid")
        _check(orc, g, x, dg.get_y())
        monkeypatch.setenv("DPC_SPMV_HOT_CAP", cap)
        dg.close()


def test_spmv_grid_nohot_shape_bit(ctx, orc):
    """Shape bit 13 drops the x cache (2 x 512-thread blocks, plain gathers)."""
    g = dpc.gen_rmat(13, 16, seed=6, weights=False, values=True, permute=True)
    x = _x(g.n)
    cfg = dpc.launch_cfg("spmv", "grid")
    cfg.flags |= 1 << 13
    y, _ = dpc.run_spmv(g, x, cfg=cfg, ctx=ctx)
    _check(orc, g, x, y)


@pytest.mark.parametrize("count,group", [(1, 0), (5, 2), (33, 0), (7, 7), (9, 16)])
def test_spmv_host_batch_contig(ctx, orc, count, group):
    """dpc_spmv_host_batch_contig: vectors back to back in (pinned) host
    memory, copied `group` at a time, double-buffered; every y exact vs the
    fp64 oracle, ragged last group included."""
    import ctypes as C
    g = dpc.gen_rmat(12, 16, seed=11, weights=False, values=True)
    n = g.n
    xp = dpc._lib.dpc_host_alloc(4 * n * count)
    yp = dpc._lib.dpc_host_alloc(4 * n * count)
    try:
        xs = np.frombuffer((C.c_float * (n * count)).from_address(xp), np.float32).reshape(count, n)
        ys = np.frombuffer((C.c_float * (n * count)).from_address(yp), np.float32).reshape(count, n)
        for i in range(count):
            xs[i] = _x(n, seed=100 + i)
        ys[:] = -1.0
        dg = dpc.DeviceGraph(ctx, g)
        dg.spmv_host_batch_contig(xs, ys, group=group)
        for i in range(count):
            _check(orc, g, xs[i], ys[i])
        dg.close()
    finally:
        dpc._lib.dpc_host_free(xp)
        dpc._lib.dpc_host_free(yp)


@pytest.mark.parametrize("scale", [12, 20])
def test_spmv_back_to_back_chain(ctx, orc, scale):
    """The bench's back-to-back form with data flowing between calls: three
    independent products, then a power-iteration chain that reads the previous
    call's y as its x, all enqueued without a host synchronisation (the
    hot-column gather of call i+1 must see call i's y)."""
    g = dpc.gen_rmat(scale, 16, seed=3, weights=False, values=True)
    dg = dpc.DeviceGraph(ctx, g)
    n = g.n
    xs = [_x(n, seed=s) for s in (1, 2, 3)]
    bx = [ctx.alloc(4 * n) for _ in range(3)]
    by = [ctx.alloc(4 * n) for _ in range(6)]
    for p, x in zip(bx, xs):
        ctx.h2d(p, x)
    ctx.synchronize()
    cfg = dpc._cfg_arg("spmv", "grid", None)
    for i in range(3):
        dpc._check(dpc._lib.dpc_spmv_device(ctx.handle, dg._h, bx[i], by[i], cfg, None))
    chain = [by[0]] + by[3:]
    for i in range(3):  # y3 = A y0, y4 = A y3, y5 = A y4
        dpc._check(dpc._lib.dpc_spmv_device(ctx.handle, dg._h, chain[i], chain[i + 1], cfg, None))
    ctx.synchronize()
    ys = [ctx.d2h(p, n) for p in by]
    dg.check()
    for i in range(3):
        _check(orc, g, xs[i], ys[i])
    _check(orc, g, ys[0], ys[3])
    _check(orc, g, ys[3], ys[4])
    _check(orc, g, ys[4], ys[5])
    for p in bx + by:
        ctx.free(p)
    dg.close()
