"""B200-native workload consolidation (arXiv 1606.08150) — Python host mirror.

Thin ctypes layer over ``libdpc.so`` (C ABI in ``include/dpc.h``).  It mirrors
the reference's application layer, which the reference specifies but does not
ship (``/root/reference/SPEC.md:406-478``, module ``workloads``):

    CsrGraph / Tree
    gen_graph / gen_rmat
    gen_tree
    load_csr / save_csr        SPEC.md:446-450, text format SPEC.md:473
    benchmark(name)            SPEC.md:451-459 (apps only; oracles live in tests)

and one run function per hot-path app (SSSP, SpMV, GC, TD, TH) in the five
variants ``flat | basic | warp | block | grid`` (the SPEC cli modes,
SPEC.md:500-506).  Errors raise :class:`DpcError` carrying the status kind that
mirrors ``SimFault.kind`` (sim.hpp:49-52).

There is no CPU fallback: if ``libdpc.so`` is missing the import fails, and
run calls on a machine without an sm_100 GPU raise ``DpcError('cuda', ...)``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

__all__ = [
    "DpcError", "VARIANTS", "APPS", "LaunchCfg", "Metrics", "CsrGraph", "Tree",
    "gen_rmat", "gen_rmat_rows", "partition_rows", "Comm", "gen_graph", "gen_tree", "csr_from_arrays", "tree_from_parent",
    "load_csr", "save_csr", "load_tree", "save_tree", "Context", "DeviceGraph",
    "DeviceTree", "default_context", "run_spmv", "run_sssp", "run_color",
    "run_tree_desc", "run_tree_height", "benchmark", "lib_path",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# DPC_LIB_PATH: load another build of the library (timing-probe builds, tools/probes)
_LIB_PATH = os.environ.get("DPC_LIB_PATH") or os.path.join(_HERE, "libdpc.so")


def lib_path() -> str:
    return _LIB_PATH


if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(or `make -C paper_1606_08150_b200/csrc`). There is no CPU fallback.")

_lib = C.CDLL(_LIB_PATH)

STATUS = {0: "ok", 1: "invalid", 2: "overflow", 3: "nesting", 4: "cuda", 5: "nccl",
          6: "oom", 7: "io", 8: "deadlock"}
VARIANTS = {"flat": 0, "basic": 1, "warp": 2, "block": 3, "grid": 4}
APPS = {"sssp": 0, "spmv": 1, "color": 2, "tree_desc": 3, "tree_height": 4}
GEN_WEIGHTS, GEN_VALUES, GEN_PERMUTE, GEN_SYMMETRIC = 1, 2, 4, 8
CFG_GRID_CDP = 1
CFG_GRID_CHUNKED = 2
CFG_GRID_ASYNC = 8
CFG_X_PEER_GATHER = 32
CFG_GRID_STREAM = 64
CFG_GRID_LEVEL = 128
CFG_SPMV_STREAM = 256
CFG_GC_HASH = 1 << 28
CFG_GC_LLF = 1 << 29
GC_ORDERS = {"canonical": 0, "hash": CFG_GC_HASH, "llf": CFG_GC_LLF}


class DpcError(RuntimeError):
    """A failed dpc_* call; ``kind`` mirrors SimFault.kind (sim.hpp:49-52)."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.kind = STATUS.get(status, str(status))
        super().__init__(f"[{self.kind}] {message}")


class _Csr(C.Structure):
    _fields_ = [("n", C.c_int64), ("m", C.c_int64), ("rowptr", C.POINTER(C.c_int64)),
                ("col", C.POINTER(C.c_int32)), ("w", C.POINTER(C.c_int32)),
                ("val", C.POINTER(C.c_float)), ("ncols", C.c_int64)]


class _Tree(C.Structure):
    _fields_ = [("n", C.c_int64), ("root", C.c_int32), ("depth", C.c_int32),
                ("parent", C.POINTER(C.c_int32)), ("cstart", C.POINTER(C.c_int64)),
                ("clist", C.POINTER(C.c_int32))]


class LaunchCfg(C.Structure):
    """dpc_launch_cfg (include/dpc.h) — the Directive / KC_X policy surface
    (ast.hpp:90-111, config.hpp:68-84)."""
    _fields_ = [("variant", C.c_int32), ("threshold", C.c_int32), ("parent_threads", C.c_int32),
                ("child_threads", C.c_int32), ("child_blocks", C.c_int32), ("kc_x", C.c_int32),
                ("chunk", C.c_int32), ("flags", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Metrics(C.Structure):
    """dpc_metrics — the B200 counterpart of Metrics (sim.hpp:34-47)."""
    _fields_ = [("child_launch_count", C.c_int64), ("buffer_items_inserted", C.c_int64),
                ("pool_peak", C.c_int64), ("iterations", C.c_int64),
                ("edges_processed", C.c_int64), ("host_launches", C.c_int64),
                ("device_ms", C.c_double), ("overflow", C.c_int32), ("result_count", C.c_int32),
                ("vertices_processed", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_P = C.c_void_p
_i32, _i64, _u32, _u64, _f64 = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double
_CsrP, _TreeP = C.POINTER(_Csr), C.POINTER(_Tree)

_SIGS = {
    "dpc_last_error": (C.c_char_p, []),
    "dpc_abi_version": (C.c_int, []),
    "dpc_gen_rmat": (C.c_int, [C.c_int, C.c_int, _f64, _f64, _f64, _i32, _i32, _u64, _u32,
                               C.POINTER(_CsrP)]),
    "dpc_gen_rmat_rows": (C.c_int, [C.c_int, C.c_int, _f64, _f64, _f64, _i32, _i32, _u64, _u32,
                                    _i64, _i64, C.POINTER(_CsrP)]),
    "dpc_gen_graph_uniform": (C.c_int, [_i64, _i32, _i32, _i32, _i32, _u64, _u32, C.POINTER(_CsrP)]),
    "dpc_gen_graph_powerlaw": (C.c_int, [_i64, _f64, _i32, _i32, _i32, _u64, _u32, C.POINTER(_CsrP)]),
    "dpc_gen_tree": (C.c_int, [_i32, _i32, _i32, _f64, _u64, C.POINTER(_TreeP)]),
    "dpc_csr_create": (C.c_int, [_i64, _i64, _P, _P, _P, _P, C.POINTER(_CsrP)]),
    "dpc_csr_create_rows": (C.c_int, [_i64, _i64, _i64, _P, _P, _P, _P, C.POINTER(_CsrP)]),
    "dpc_csr_validate": (C.c_int, [_CsrP]),
    "dpc_csr_free": (None, [_CsrP]),
    "dpc_tree_create": (C.c_int, [_i64, _P, C.POINTER(_TreeP)]),
    "dpc_tree_free": (None, [_TreeP]),
    "dpc_load_csr": (C.c_int, [C.c_char_p, C.POINTER(_CsrP)]),
    "dpc_load_dimacs": (C.c_int, [C.c_char_p, C.POINTER(_CsrP)]),
    "dpc_save_csr": (C.c_int, [_CsrP, C.c_char_p]),
    "dpc_load_tree": (C.c_int, [C.c_char_p, C.POINTER(_TreeP)]),
    "dpc_save_tree": (C.c_int, [_TreeP, C.c_char_p]),
    "dpc_launch_cfg_default": (C.c_int, [_i32, _i32, C.POINTER(LaunchCfg)]),
    "dpc_ctx_create": (C.c_int, [_i32, C.POINTER(_P)]),
    "dpc_ctx_destroy": (None, [_P]),
    "dpc_ctx_stream": (_P, [_P]),
    "dpc_ctx_sm_count": (_i32, [_P]),
    "dpc_ctx_event_record": (C.c_int, [_P, _i32]),
    "dpc_ctx_event_elapsed": (C.c_int, [_P, _i32, _i32, C.POINTER(C.c_float)]),
    "dpc_ctx_synchronize": (C.c_int, [_P]),
    "dpc_ctx_flush_l2": (C.c_int, [_P]),
    "dpc_run_spmv": (C.c_int, [_P, _CsrP, _P, _P, C.POINTER(LaunchCfg), C.POINTER(Metrics)]),
    "dpc_run_sssp": (C.c_int, [_P, _CsrP, _i32, _P, C.POINTER(LaunchCfg), C.POINTER(Metrics)]),
    "dpc_run_color": (C.c_int, [_P, _CsrP, _u64, _P, C.POINTER(_i32), C.POINTER(LaunchCfg),
                                C.POINTER(Metrics)]),
    "dpc_run_tree_desc": (C.c_int, [_P, _TreeP, _P, C.POINTER(LaunchCfg), C.POINTER(Metrics)]),
    "dpc_run_tree_height": (C.c_int, [_P, _TreeP, _P, C.POINTER(LaunchCfg), C.POINTER(Metrics)]),
    "dpc_dgraph_upload": (C.c_int, [_P, _CsrP, C.POINTER(_P)]),
    "dpc_dgraph_free": (None, [_P]),
    "dpc_dgraph_x": (_P, [_P]),
    "dpc_dgraph_y": (_P, [_P]),
    "dpc_dgraph_dist": (_P, [_P]),
    "dpc_dgraph_color": (_P, [_P]),
    "dpc_dgraph_phase_ns": (C.c_int, [_P, _P]),
    "dpc_dgraph_trace": (C.c_int, [_P, _P, _i64]),
    "dpc_spmv_device": (C.c_int, [_P, _P, _P, _P, C.POINTER(LaunchCfg), C.POINTER(Metrics)]),
    "dpc_spmv_host": (C.c_int, [_P, _P, _P, _P, C.POINTER(LaunchCfg), C.POINTER(Metrics)]),
    "dpc_spmv_host_batch": (C.c_int, [_P, _P, _P, _P, C.c_int64, C.POINTER(LaunchCfg), C.POINTER(Metrics)]),
    "dpc_spmv_host_batch_contig": (C.c_int, [_P, _P, _P, _P, C.c_int64, C.c_int64, C.POINTER(LaunchCfg),
                                             C.POINTER(Metrics)]),
    "dpc_dtree_phase_ns": (C.c_int, [_P, _P]),
    "dpc_dgraph_check": (C.c_int, [_P, _P]),
    "dpc_dtree_check": (C.c_int, [_P, _P]),
    "dpc_ipc_handle": (C.c_int, [_P, _P]),
    "dpc_ipc_open": (C.c_int, [_P, _P, C.POINTER(_P)]),
    "dpc_ipc_close": (C.c_int, [_P]),
    "dpc_p2p_barrier": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_uint64]),
    "dpc_p2p_check": (C.c_int, [_P]),
    "dpc_p2p_barrier_sum": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_uint64, C.c_uint32,
                                      C.POINTER(C.c_uint64)]),
    "dpc_msssp_buffers": (C.c_int, [_P, _P]),
    "dpc_msssp_set_peers": (C.c_int, [_P, _P]),
    "dpc_multi_spmv_fused": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int64, _P, C.POINTER(LaunchCfg),
                                       C.POINTER(Metrics)]),
    "dpc_sssp_device": (C.c_int, [_P, _P, _i32, C.POINTER(LaunchCfg), C.POINTER(Metrics)]),
    "dpc_bfs_device": (C.c_int, [_P, _P, _i32, C.POINTER(LaunchCfg), C.POINTER(Metrics)]),
    "dpc_run_bfs": (C.c_int, [_P, _CsrP, _i32, _P, C.POINTER(LaunchCfg), C.POINTER(Metrics)]),
    "dpc_pr_upload": (C.c_int, [_P, _CsrP, C.POINTER(_P)]),
    "dpc_pr_free": (None, [_P]),
    "dpc_pr_device": (C.c_int, [_P, _P, _i32, C.c_double, C.POINTER(LaunchCfg), C.POINTER(Metrics)]),
    "dpc_pr_rank": (_P, [_P]),
    "dpc_run_pagerank": (C.c_int, [_P, _CsrP, _i32, C.c_double, _P, C.POINTER(LaunchCfg), C.POINTER(Metrics)]),
    "dpc_color_device": (C.c_int, [_P, _P, _u64, C.POINTER(LaunchCfg), C.POINTER(Metrics)]),
    "dpc_dtree_upload": (C.c_int, [_P, _TreeP, C.POINTER(_P)]),
    "dpc_dtree_free": (None, [_P]),
    "dpc_tree_device": (C.c_int, [_P, _P, _i32, C.POINTER(LaunchCfg), C.POINTER(Metrics)]),
    "dpc_dtree_result": (_P, [_P]),
    "dpc_dev_alloc": (_P, [_P, C.c_size_t]),
    "dpc_dev_free": (None, [_P, _P]),
    "dpc_host_alloc": (_P, [C.c_size_t]),
    "dpc_host_free": (None, [_P]),
    "dpc_copy_h2d": (C.c_int, [_P, _P, _P, C.c_size_t]),
    "dpc_dev_memset": (C.c_int, [_P, _P, C.c_int32, C.c_size_t]),
    "dpc_copy_d2h": (C.c_int, [_P, _P, _P, C.c_size_t]),
    "dpc_comm_unique_id": (C.c_int, [_P]),
    "dpc_comm_init": (C.c_int, [_P, _i32, _i32, _P, C.POINTER(_P)]),
    "dpc_comm_destroy": (None, [_P]),
    "dpc_comm_rank": (_i32, [_P]),
    "dpc_comm_world": (_i32, [_P]),
    "dpc_partition_rows": (C.c_int, [_CsrP, _i32, _P]),
    "dpc_multi_spmv": (C.c_int, [_P, _P, _P, _P, _P, C.POINTER(LaunchCfg), C.POINTER(Metrics)]),
    "dpc_multi_sssp": (C.c_int, [_P, _P, _P, _i64, _i64, C.POINTER(LaunchCfg), C.POINTER(Metrics)]),
    "dpc_msssp_begin": (C.c_int, [_P, _P, _i64, _i64, _i64, _i32, _i64, C.POINTER(LaunchCfg)]),
    "dpc_msssp_relax": (C.c_int, [_P, _P, _P]),
    "dpc_msssp_send_buffer": (_P, [_P, _i32]),
    "dpc_msssp_recv_buffer": (_P, [_P]),
    "dpc_msssp_recv_capacity": (C.c_uint64, [_P]),
    "dpc_msssp_recv_reserve": (C.c_int, [_P, _P, C.c_uint64, C.POINTER(C.c_void_p)]),
    "dpc_msssp_send_counts": (_P, [_P]),
    "dpc_msssp_apply": (C.c_int, [_P, _P, _P, _u64, C.POINTER(_u32)]),
    "dpc_msssp_end": (C.c_int, [_P, _P, C.POINTER(Metrics)]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

if _lib.dpc_abi_version() != 1:
    raise ImportError("libdpc.so ABI version mismatch; rebuild it")


def exported_symbols():
    """Names the binding expects libdpc.so to export (tests check include/dpc.h)."""
    return sorted(_SIGS)


def _check(st: int):
    if st != 0:
        raise DpcError(st, _lib.dpc_last_error().decode(errors="replace"))


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _view(ptr, count, ctype, dtype):
    if not ptr or count == 0:
        return np.zeros(0, dtype=dtype)
    buf = (ctype * count).from_address(C.addressof(ptr.contents))
    return np.frombuffer(buf, dtype=dtype, count=count)


# ---------------------------------------------------------------- data layer
class CsrGraph:
    """CsrGraph: library-owned CSR; arrays are zero-copy numpy
    views that stay valid while the object lives."""

    def __init__(self, handle):
        self._h = handle
        c = handle.contents
        self.n = int(c.n)
        self.m = int(c.m)
        self.ncols = int(c.ncols) or self.n
        self.rowptr = _view(c.rowptr, self.n + 1, C.c_int64, np.int64)
        self.col = _view(c.col, self.m, C.c_int32, np.int32)
        self.w = _view(c.w, self.m, C.c_int32, np.int32) if c.w else None
        self.val = _view(c.val, self.m, C.c_float, np.float32) if c.val else None

    node_count = property(lambda self: self.n)
    edge_count = property(lambda self: self.m)

    def degrees(self) -> np.ndarray:
        return np.diff(self.rowptr)

    def validate(self):
        _check(_lib.dpc_csr_validate(self._h))

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None:  # interpreter shutdown clears module globals
            _lib.dpc_csr_free(h)


class Tree:
    """Tree: parent[] with root = -1, children lists, depth."""

    def __init__(self, handle):
        self._h = handle
        c = handle.contents
        self.n = int(c.n)
        self.root = int(c.root)
        self.depth = int(c.depth)
        self.parent = _view(c.parent, self.n, C.c_int32, np.int32)
        self.cstart = _view(c.cstart, self.n + 1, C.c_int64, np.int64)
        self.clist = _view(c.clist, self.n, C.c_int32, np.int32)

    def children(self, v: int) -> np.ndarray:
        return self.clist[self.cstart[v]:self.cstart[v + 1]]

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None:  # interpreter shutdown clears module globals
            _lib.dpc_tree_free(h)


def _gen_flags(weights, values, permute, symmetric):
    return ((GEN_WEIGHTS if weights else 0) | (GEN_VALUES if values else 0)
            | (GEN_PERMUTE if permute else 0) | (GEN_SYMMETRIC if symmetric else 0))


def gen_rmat(scale: int, edgefactor: int = 16, a: float = 0.57, b: float = 0.19, c: float = 0.19,
             wmin: int = 1, wmax: int = 255, seed: int = 1, weights: bool = True,
             values: bool = False, permute: bool = False, symmetric: bool = False) -> CsrGraph:
    """Seeded R-MAT graph with 2**scale vertices and edgefactor * 2**scale arcs."""
    h = _CsrP()
    _check(_lib.dpc_gen_rmat(scale, edgefactor, a, b, c, wmin, wmax, seed & (2**64 - 1),
                             _gen_flags(weights, values, permute, symmetric), C.byref(h)))
    return CsrGraph(h)


def gen_rmat_rows(scale: int, r0: int, r1: int, edgefactor: int = 16, a: float = 0.57,
                  b: float = 0.19, c: float = 0.19, wmin: int = 1, wmax: int = 255, seed: int = 1,
                  weights: bool = True, values: bool = False, permute: bool = False) -> CsrGraph:
    """Rows [r0, r1) of gen_rmat(scale, ...) with global column ids (ncols = 2**scale)."""
    h = _CsrP()
    _check(_lib.dpc_gen_rmat_rows(scale, edgefactor, a, b, c, wmin, wmax, seed & (2**64 - 1),
                                  _gen_flags(weights, values, permute, False), r0, r1, C.byref(h)))
    return CsrGraph(h)


def partition_rows(g: CsrGraph, world: int) -> np.ndarray:
    """Equal-nnz row split: bounds[0..world]."""
    b = np.zeros(world + 1, np.int64)
    _check(_lib.dpc_partition_rows(g._h, world, _ptr(b)))
    return b


def gen_graph(node_count: int, uniform: tuple | None = None, powerlaw: tuple | None = None,
              seed: int = 1, wmin: int = 1, wmax: int = 255, weights: bool = True,
              values: bool = False, symmetric: bool = False) -> CsrGraph:
    """SPEC.md:435-444 gen_graph(nodeCount, uniform(min,max) | powerlaw(alpha,maxDeg), seed)."""
    h = _CsrP()
    flags = _gen_flags(weights, values, False, symmetric)
    if (uniform is None) == (powerlaw is None):
        raise DpcError(1, "give exactly one of uniform=(min,max) or powerlaw=(alpha,maxDeg)")
    if uniform is not None:
        _check(_lib.dpc_gen_graph_uniform(node_count, uniform[0], uniform[1], wmin, wmax,
                                          seed & (2**64 - 1), flags, C.byref(h)))
    else:
        _check(_lib.dpc_gen_graph_powerlaw(node_count, float(powerlaw[0]), int(powerlaw[1]), wmin,
                                           wmax, seed & (2**64 - 1), flags, C.byref(h)))
    return CsrGraph(h)


def gen_tree(depth: int, min_children: int, max_children: int, fill: float,
             seed: int = 1) -> Tree:
    """SPEC.md:425-433 gen_tree(depth, minChildren, maxChildren, nonLeafFillFraction, seed)."""
    h = _TreeP()
    _check(_lib.dpc_gen_tree(depth, min_children, max_children, fill, seed & (2**64 - 1),
                             C.byref(h)))
    return Tree(h)


def csr_from_arrays(rowptr, col, w=None, val=None) -> CsrGraph:
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    w = None if w is None else np.ascontiguousarray(w, dtype=np.int32)
    val = None if val is None else np.ascontiguousarray(val, dtype=np.float32)
    h = _CsrP()
    _check(_lib.dpc_csr_create(len(rowptr) - 1, len(col), _ptr(rowptr), _ptr(col), _ptr(w),
                               _ptr(val), C.byref(h)))
    return CsrGraph(h)


def csr_rows_from_arrays(rowptr, col, ncols, w=None, val=None) -> CsrGraph:
    """A row slice of a larger matrix: col holds global column ids < ncols
    (dpc_csr_create_rows; the partitioned multi-GPU paths take such slices)."""
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    w = None if w is None else np.ascontiguousarray(w, dtype=np.int32)
    val = None if val is None else np.ascontiguousarray(val, dtype=np.float32)
    h = _CsrP()
    _check(_lib.dpc_csr_create_rows(len(rowptr) - 1, ncols, len(col), _ptr(rowptr), _ptr(col), _ptr(w),
                                    _ptr(val), C.byref(h)))
    return CsrGraph(h)


def tree_from_parent(parent) -> Tree:
    parent = np.ascontiguousarray(parent, dtype=np.int32)
    h = _TreeP()
    _check(_lib.dpc_tree_create(len(parent), _ptr(parent), C.byref(h)))
    return Tree(h)


def load_csr(path: str) -> CsrGraph:
    h = _CsrP()
    _check(_lib.dpc_load_csr(os.fsencode(path), C.byref(h)))
    return CsrGraph(h)


def load_dimacs(path: str) -> CsrGraph:
    """DIMACS 9th-challenge .gr (weighted arcs) or 10th-challenge / METIS
    graph file (dpc_load_dimacs)."""
    h = _CsrP()
    _check(_lib.dpc_load_dimacs(os.fsencode(path), C.byref(h)))
    return CsrGraph(h)


def save_csr(g: CsrGraph, path: str):
    _check(_lib.dpc_save_csr(g._h, os.fsencode(path)))


def load_tree(path: str) -> Tree:
    h = _TreeP()
    _check(_lib.dpc_load_tree(os.fsencode(path), C.byref(h)))
    return Tree(h)


def save_tree(t: Tree, path: str):
    _check(_lib.dpc_save_tree(t._h, os.fsencode(path)))


def ipc_handle(d_ptr: int) -> bytes:
    """CUDA IPC handle (64 bytes) of a device buffer from dpc_dev_alloc."""
    buf = (C.c_uint8 * 64)()
    _check(_lib.dpc_ipc_handle(C.c_void_p(d_ptr), buf))
    return bytes(buf)


def ipc_open(ctx, handle: bytes) -> int:
    """Maps a peer's buffer (its 64-byte IPC handle) into this process."""
    out = C.c_void_p()
    _check(_lib.dpc_ipc_open(ctx.handle, (C.c_uint8 * 64).from_buffer_copy(handle), C.byref(out)))
    return int(out.value)


def ipc_close(d_ptr: int):
    _check(_lib.dpc_ipc_close(C.c_void_p(d_ptr)))


def p2p_barrier(ctx, d_flag_table: int, world: int, me: int, epoch: int):
    """Device-side barrier over peer memory (enqueued on ctx's stream)."""
    _check(_lib.dpc_p2p_barrier(ctx.handle, C.c_void_p(d_flag_table), world, me, epoch))


def p2p_check(ctx):
    _check(_lib.dpc_p2p_check(ctx.handle))


def p2p_barrier_sum(ctx, d_flag_table: int, world: int, me: int, epoch: int, value: int) -> int:
    """Peer barrier carrying one u32 per rank; returns the sum over ranks."""
    out = C.c_uint64()
    _check(_lib.dpc_p2p_barrier_sum(ctx.handle, C.c_void_p(d_flag_table), world, me, epoch, value, C.byref(out)))
    return int(out.value)


def launch_cfg(app: str, variant: str, **overrides) -> LaunchCfg:
    """Measured default dpc_launch_cfg for (app, variant), with overrides."""
    cfg = LaunchCfg()
    _check(_lib.dpc_launch_cfg_default(APPS[app], VARIANTS[variant], C.byref(cfg)))
    for k, v in overrides.items():
        if k == "grid_cdp":
            cfg.flags = (cfg.flags | CFG_GRID_CDP) if v else (cfg.flags & ~CFG_GRID_CDP)
        elif k == "grid_chunked":
            cfg.flags = (cfg.flags | CFG_GRID_CHUNKED) if v else (cfg.flags & ~CFG_GRID_CHUNKED)
        elif k == "grid_async":
            cfg.flags = (cfg.flags | CFG_GRID_ASYNC) if v else (cfg.flags & ~CFG_GRID_ASYNC)
        elif k == "grid_stream":
            cfg.flags = (cfg.flags | CFG_GRID_STREAM) if v else (cfg.flags & ~CFG_GRID_STREAM)
        elif k == "spmv_stream":
            cfg.flags = (cfg.flags | CFG_SPMV_STREAM) if v else (cfg.flags & ~CFG_SPMV_STREAM)
        elif k == "grid_level":
            cfg.flags = (cfg.flags | CFG_GRID_LEVEL) if v else (cfg.flags & ~CFG_GRID_LEVEL)
        elif k == "gc_order":  # "hash" | "canonical" | "llf"
            cfg.flags = (cfg.flags & ~(CFG_GC_HASH | CFG_GC_LLF)) | GC_ORDERS[v]
        else:
            setattr(cfg, k, int(v))
    return cfg


# ---------------------------------------------------------------- device side
class Context:
    """dpc_ctx: one CUDA device + stream.  Raises DpcError('cuda') without an
    sm_100 GPU — there is no CPU path."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(_lib.dpc_ctx_create(device, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return _lib.dpc_ctx_stream(self._h) or 0

    @property
    def sm_count(self) -> int:
        return _lib.dpc_ctx_sm_count(self._h)

    def record(self, slot: int):
        _check(_lib.dpc_ctx_event_record(self._h, slot))

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_float()
        _check(_lib.dpc_ctx_event_elapsed(self._h, a, b, C.byref(ms)))
        return float(ms.value)

    def synchronize(self):
        _check(_lib.dpc_ctx_synchronize(self._h))

    def alloc(self, nbytes: int) -> int:
        """Device buffer on this context's GPU (free with free())."""
        p = _lib.dpc_dev_alloc(self._h, nbytes)
        if not p:
            raise DpcError(6, f"device allocation of {nbytes} bytes failed")
        return p

    def free(self, p: int):
        _lib.dpc_dev_free(self._h, p)

    def memset(self, dst: int, value: int, nbytes: int):
        """Byte fill of device memory on the context stream (asynchronous)."""
        _check(_lib.dpc_dev_memset(self._h, dst, value, nbytes))

    def h2d(self, dst: int, a: np.ndarray):
        a = np.ascontiguousarray(a)
        _check(_lib.dpc_copy_h2d(self._h, dst, _ptr(a), a.nbytes))

    def d2h(self, src: int, count: int, dtype=np.float32) -> np.ndarray:
        out = np.empty(count, dtype)
        _check(_lib.dpc_copy_d2h(self._h, _ptr(out), src, out.nbytes))
        return out

    def flush_l2(self):
        _check(_lib.dpc_ctx_flush_l2(self._h))

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None:  # interpreter shutdown clears module globals
            _lib.dpc_ctx_destroy(h)

    __del__ = close


def _cfg_arg(app, variant, cfg):
    if cfg is None:
        cfg = launch_cfg(app, variant)
    elif isinstance(cfg, dict):
        cfg = launch_cfg(app, variant, **cfg)
    return C.byref(cfg)


class DeviceGraph:
    """dpc_dgraph: a graph resident in HBM with all app buffers."""

    def __init__(self, ctx: Context, g: CsrGraph):
        h = C.c_void_p()
        _check(_lib.dpc_dgraph_upload(ctx.handle, g._h, C.byref(h)))
        self._h, self.ctx, self.n, self.m = h, ctx, g.n, g.m

    @property
    def x_ptr(self):
        return _lib.dpc_dgraph_x(self._h)

    @property
    def y_ptr(self):
        return _lib.dpc_dgraph_y(self._h)

    def set_x(self, x: np.ndarray):
        x = np.ascontiguousarray(x, dtype=np.float32)
        _check(_lib.dpc_copy_h2d(self.ctx.handle, self.x_ptr, _ptr(x), x.nbytes))

    def get_y(self) -> np.ndarray:
        y = np.empty(self.n, dtype=np.float32)
        _check(_lib.dpc_copy_d2h(self.ctx.handle, _ptr(y), self.y_ptr, y.nbytes))
        return y

    def check(self):
        """Fault check of the last run made without metrics (dpc_dgraph_check)."""
        _check(_lib.dpc_dgraph_check(self.ctx.handle, self._h))

    def get_dist(self) -> np.ndarray:
        self.check()
        d = np.empty(self.n, dtype=np.uint32)
        _check(_lib.dpc_copy_d2h(self.ctx.handle, _ptr(d), _lib.dpc_dgraph_dist(self._h), d.nbytes))
        return d

    def trace(self, words: int = 0) -> np.ndarray:
        """Per-vertex timestamps (ns) of the last DPC_TRACE=1 run (see dpc.h)."""
        t = np.empty(words or self.n, dtype=np.uint64)
        _check(_lib.dpc_dgraph_trace(self._h, _ptr(t), len(t)))
        return t

    def get_color(self) -> np.ndarray:
        d = np.empty(self.n, dtype=np.int32)
        _check(_lib.dpc_copy_d2h(self.ctx.handle, _ptr(d), _lib.dpc_dgraph_color(self._h), d.nbytes))
        return d

    def phase_ns(self):
        """(start, barrier, end) %globaltimer stamps of the last persistent run read with metrics."""
        t = np.zeros(3, np.uint64)
        _check(_lib.dpc_dgraph_phase_ns(self._h, _ptr(t)))
        return [int(v) for v in t]

    def spmv(self, variant="grid", cfg=None, metrics: bool = False):
        """y = A x on the resident vectors (asynchronous unless metrics)."""
        met = Metrics() if metrics else None
        _check(_lib.dpc_spmv_device(self.ctx.handle, self._h, self.x_ptr, self.y_ptr,
                                    _cfg_arg("spmv", variant, cfg),
                                    C.byref(met) if met is not None else None))
        return met

    def spmv_host(self, x: np.ndarray, y: np.ndarray, variant="grid", cfg=None):
        """End-to-end: host x in, host y out, through the C ABI."""
        _check(_lib.dpc_spmv_host(self.ctx.handle, self._h, x.ctypes.data_as(C.c_void_p),
                                  y.ctypes.data_as(C.c_void_p), _cfg_arg("spmv", variant, cfg),
                                  None))

    def spmv_host_batch(self, xs, ys, variant="grid", cfg=None):
        """Pipelined end-to-end SpMV over len(xs) host vectors (pinned for
        overlap): copy-in / kernel / copy-out of consecutive vectors overlap."""
        if len(xs) != len(ys):
            raise ValueError("xs and ys must have the same length")
        k = len(xs)
        xp = (C.c_void_p * max(1, k))(*[x.ctypes.data for x in xs])
        yp = (C.c_void_p * max(1, k))(*[y.ctypes.data for y in ys])
        _check(_lib.dpc_spmv_host_batch(self.ctx.handle, self._h, xp, yp, k, _cfg_arg("spmv", variant, cfg),
                                        None))

    def spmv_host_batch_contig(self, xs: np.ndarray, ys: np.ndarray, group: int = 0, variant="grid", cfg=None):
        """Pipelined end-to-end SpMV over the rows of xs (count x ncols,
        float32, C-contiguous, pinned for overlap) into ys (count x n):
        copies move `group` vectors at a time (0 = about 32 MB)."""
        if xs.dtype != np.float32 or ys.dtype != np.float32 or not xs.flags.c_contiguous or not ys.flags.c_contiguous:
            raise ValueError("xs / ys must be C-contiguous float32")
        if xs.shape[0] != ys.shape[0]:
            raise ValueError("xs and ys must hold the same number of vectors")
        _check(_lib.dpc_spmv_host_batch_contig(self.ctx.handle, self._h, xs.ctypes.data, ys.ctypes.data, xs.shape[0],
                                               group, _cfg_arg("spmv", variant, cfg), None))

    def spmv_fused(self, d_xpeer_table: int, world: int, rows_per_rank: int, d_y: int, variant="grid", cfg=None):
        """Fused multi-GPU SpMV of this row block: x gathered from the owners
        through a DEVICE table of `world` peer pointers (dpc_multi_spmv_fused)."""
        _check(_lib.dpc_multi_spmv_fused(self.ctx.handle, self._h, C.c_void_p(d_xpeer_table), world, rows_per_rank,
                                         C.c_void_p(d_y), _cfg_arg("spmv", variant, cfg), None))

    def sssp(self, source: int, variant="grid", cfg=None, metrics: bool = True):
        met = Metrics() if metrics else None
        _check(_lib.dpc_sssp_device(self.ctx.handle, self._h, source,
                                    _cfg_arg("sssp", variant, cfg),
                                    C.byref(met) if met is not None else None))
        return met

    def bfs(self, source: int, variant="grid", cfg=None, metrics: bool = True):
        """BFS levels into the handle's dist buffer (get_dist())."""
        met = Metrics() if metrics else None
        _check(_lib.dpc_bfs_device(self.ctx.handle, self._h, source, _cfg_arg("sssp", variant, cfg),
                                   C.byref(met) if met is not None else None))
        return met

    def color(self, seed: int, variant="grid", cfg=None, metrics: bool = True):
        met = Metrics() if metrics else None
        _check(_lib.dpc_color_device(self.ctx.handle, self._h, seed & (2**64 - 1),
                                     _cfg_arg("color", variant, cfg),
                                     C.byref(met) if met is not None else None))
        return met

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None:  # interpreter shutdown clears module globals
            _lib.dpc_dgraph_free(h)

    __del__ = close


class Comm:
    """dpc_comm: an NCCL communicator for one rank (one process per GPU)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(_lib.dpc_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, ctx: Context, rank: int, world: int, uid: bytes):
        h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(_lib.dpc_comm_init(ctx.handle, rank, world, buf, C.byref(h)))
        self._h, self.ctx, self.rank, self.world = h, ctx, rank, world

    def spmv(self, local: "DeviceGraph", d_x_local: int, d_y_local: int, variant="grid", cfg=None):
        """AllGather x slices over NCCL, then y_local = A_local x (async)."""
        _check(_lib.dpc_multi_spmv(self.ctx.handle, self._h, local._h, d_x_local, d_y_local,
                                   _cfg_arg("spmv", variant, cfg), None))

    def sssp(self, local: "DeviceGraph", n_global: int, source: int, variant="grid", cfg=None):
        """Vertex-partitioned SSSP over NCCL; local distances stay in `local`."""
        met = Metrics()
        _check(_lib.dpc_multi_sssp(self.ctx.handle, self._h, local._h, n_global, source,
                                   _cfg_arg("sssp", variant, cfg), C.byref(met)))
        return met

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None:  # interpreter shutdown clears module globals
            _lib.dpc_comm_destroy(h)

    __del__ = close


class PartitionedSSSP:
    """The dpc_msssp_* steps of one rank's block (transport left to the
    caller): begin -> [relax -> exchange -> apply]* -> end."""

    def __init__(self, local: "DeviceGraph", rank: int, world: int, n_global: int, source: int,
                 variant="grid", cfg=None):
        self.g, self.ctx, self.world = local, local.ctx, world
        R = -(-n_global // world)
        _check(_lib.dpc_msssp_begin(self.ctx.handle, local._h, rank * R, R, n_global, world, source,
                                    _cfg_arg("sssp", variant, cfg)))

    def relax(self) -> np.ndarray:
        cnt = np.zeros(self.world, np.uint32)
        _check(_lib.dpc_msssp_relax(self.ctx.handle, self.g._h, _ptr(cnt)))
        return cnt

    def outgoing(self, owner: int, count: int) -> np.ndarray:
        """The {vertex, distance} pairs queued for `owner` (host copy, (count, 2) uint32)."""
        out = np.empty((count, 2), np.uint32)
        if count:
            _check(_lib.dpc_copy_d2h(self.ctx.handle, _ptr(out), _lib.dpc_msssp_send_buffer(self.g._h, owner),
                                     out.nbytes))
        return out

    def apply(self, pairs: np.ndarray) -> int:
        pairs = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
        pbuf = C.c_void_p()
        _check(_lib.dpc_msssp_recv_reserve(self.ctx.handle, self.g._h, len(pairs), C.byref(pbuf)))
        buf = pbuf.value
        if len(pairs):
            _check(_lib.dpc_copy_h2d(self.ctx.handle, buf, _ptr(pairs), pairs.nbytes))
        nxt = _u32()
        _check(_lib.dpc_msssp_apply(self.ctx.handle, self.g._h, buf, len(pairs), C.byref(nxt)))
        return int(nxt.value)

    def end(self):
        met = Metrics()
        _check(_lib.dpc_msssp_end(self.ctx.handle, self.g._h, C.byref(met)))
        return met

    # ---- fused form: remote relaxations straight into the owners' buffers
    def buffers(self):
        """The 5 device buffers this rank exports (dist, stamp, front0,
        front1, counters) for the fused form."""
        out = (C.c_void_p * 5)()
        _check(_lib.dpc_msssp_buffers(self.g._h, out))
        return [int(p) for p in out]

    def set_peers(self, d_peer_table: int):
        """DEVICE array of world x 5 pointers (every rank's buffers()), own and mapped."""
        _check(_lib.dpc_msssp_set_peers(self.g._h, C.c_void_p(d_peer_table)))


class DeviceTree:
    """dpc_dtree: a tree resident in HBM."""

    def __init__(self, ctx: Context, t: Tree):
        h = C.c_void_p()
        _check(_lib.dpc_dtree_upload(ctx.handle, t._h, C.byref(h)))
        self._h, self.ctx, self.n = h, ctx, t.n

    def run(self, which: str, variant="grid", cfg=None, metrics: bool = True):
        met = Metrics() if metrics else None
        _check(_lib.dpc_tree_device(self.ctx.handle, self._h, APPS[which],
                                    _cfg_arg(which, variant, cfg),
                                    C.byref(met) if met is not None else None))
        return met

    def phase_ns(self):
        out = (C.c_uint64 * 3)()
        _check(_lib.dpc_dtree_phase_ns(self._h, out))
        return [int(v) for v in out]

    def result(self) -> np.ndarray:
        _check(_lib.dpc_dtree_check(self.ctx.handle, self._h))
        r = np.empty(self.n, dtype=np.int32)
        _check(_lib.dpc_copy_d2h(self.ctx.handle, _ptr(r), _lib.dpc_dtree_result(self._h), r.nbytes))
        return r

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None:  # interpreter shutdown clears module globals
            _lib.dpc_dtree_free(h)

    __del__ = close


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ------------------------------------------------ host-buffer run functions
def run_spmv(A: CsrGraph, x, variant="grid", cfg=None, ctx: Context | None = None):
    """y = A x (fp32).  Returns (y, Metrics)."""
    ctx = ctx or default_context()
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.empty(A.n, dtype=np.float32)
    met = Metrics()
    _check(_lib.dpc_run_spmv(ctx.handle, A._h, _ptr(x), _ptr(y), _cfg_arg("spmv", variant, cfg),
                             C.byref(met)))
    return y, met


def run_sssp(G: CsrGraph, source: int, variant="grid", cfg=None, ctx: Context | None = None):
    """Shortest distances (uint32, UINT32_MAX = unreachable).  Returns (dist, Metrics)."""
    ctx = ctx or default_context()
    dist = np.empty(G.n, dtype=np.uint32)
    met = Metrics()
    _check(_lib.dpc_run_sssp(ctx.handle, G._h, source, _ptr(dist), _cfg_arg("sssp", variant, cfg),
                             C.byref(met)))
    return dist, met


def run_bfs(G: CsrGraph, source: int, variant="grid", cfg=None, ctx: Context | None = None):
    """BFS levels (uint32 hops, UINT32_MAX = unreachable) -- the paper's BFS-Rec
    benchmark as the SSSP consolidation with unit weights.  Returns (level, Metrics)."""
    ctx = ctx or default_context()
    level = np.empty(G.n, dtype=np.uint32)
    met = Metrics()
    _check(_lib.dpc_run_bfs(ctx.handle, G._h, source, _ptr(level), _cfg_arg("sssp", variant, cfg),
                            C.byref(met)))
    return level, met


def run_pagerank(G: CsrGraph, iters: int = 20, damping: float = 0.85, variant="grid", cfg=None,
                 ctx: Context | None = None):
    """PageRank ranks (float32): `iters` power iterations, each one SpMV of the
    transposed graph with the SpMV consolidation `variant`.  Returns (rank, Metrics)."""
    ctx = ctx or default_context()
    rank = np.empty(G.n, dtype=np.float32)
    met = Metrics()
    _check(_lib.dpc_run_pagerank(ctx.handle, G._h, iters, damping, _ptr(rank), _cfg_arg("spmv", variant, cfg),
                                 C.byref(met)))
    return rank, met


class PageRankGraph:
    """dpc_prgraph: the transposed graph resident in HBM for repeated PR runs."""

    def __init__(self, ctx: Context, g: CsrGraph):
        h = C.c_void_p()
        _check(_lib.dpc_pr_upload(ctx.handle, g._h, C.byref(h)))
        self._h, self.ctx, self.n = h, ctx, g.n

    def run(self, iters=20, damping=0.85, variant="grid", cfg=None, metrics: bool = True):
        met = Metrics() if metrics else None
        _check(_lib.dpc_pr_device(self.ctx.handle, self._h, iters, damping, _cfg_arg("spmv", variant, cfg),
                                  C.byref(met) if met is not None else None))
        return met

    def rank(self) -> np.ndarray:
        r = np.empty(self.n, dtype=np.float32)
        _check(_lib.dpc_copy_d2h(self.ctx.handle, _ptr(r), _lib.dpc_pr_rank(self._h), r.nbytes))
        return r

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None:  # interpreter shutdown clears module globals
            _lib.dpc_pr_free(h)

    __del__ = close


def run_color(G: CsrGraph, seed: int = 1, variant="grid", cfg=None, ctx: Context | None = None):
    """Greedy first-fit coloring in canonical node order, or the
    order cfg selects (launch_cfg(..., gc_order="hash" | "llf")).  Returns
    (color, ncolors, Metrics)."""
    ctx = ctx or default_context()
    color = np.empty(G.n, dtype=np.int32)
    nc = C.c_int32()
    met = Metrics()
    _check(_lib.dpc_run_color(ctx.handle, G._h, seed & (2**64 - 1), _ptr(color), C.byref(nc),
                              _cfg_arg("color", variant, cfg), C.byref(met)))
    return color, int(nc.value), met


def run_tree_desc(T: Tree, variant="grid", cfg=None, ctx: Context | None = None):
    ctx = ctx or default_context()
    out = np.empty(T.n, dtype=np.int32)
    met = Metrics()
    _check(_lib.dpc_run_tree_desc(ctx.handle, T._h, _ptr(out), _cfg_arg("tree_desc", variant, cfg),
                                  C.byref(met)))
    return out, met


def run_tree_height(T: Tree, variant="grid", cfg=None, ctx: Context | None = None):
    ctx = ctx or default_context()
    out = np.empty(T.n, dtype=np.int32)
    met = Metrics()
    _check(_lib.dpc_run_tree_height(ctx.handle, T._h, _ptr(out),
                                    _cfg_arg("tree_height", variant, cfg), C.byref(met)))
    return out, met


# ---------------------------------------------------------------- benchmarks
@dataclass
class BenchmarkCase:
    """SPEC.md:420-423 BenchmarkCase, restricted to the hot-path apps.  The
    sequential oracles are test infrastructure (oracle/), not product code."""
    name: str
    app: str
    make_input: object
    run: object


def benchmark(name: str) -> BenchmarkCase:
    name_l = name.lower()
    if name_l == "sssp":
        return BenchmarkCase("SSSP", "sssp",
                             lambda scale=16, seed=1: gen_rmat(scale, 16, seed=seed),
                             lambda g, variant="grid", source=0: run_sssp(g, source, variant))
    if name_l == "spmv":
        return BenchmarkCase("SpMV", "spmv",
                             lambda scale=20, seed=1: gen_rmat(scale, 16, seed=seed, weights=False,
                                                               values=True),
                             lambda g, x, variant="grid": run_spmv(g, x, variant))
    if name_l == "gc":
        return BenchmarkCase("GC", "color",
                             lambda scale=20, seed=1: gen_rmat(scale, 16, seed=seed, weights=False,
                                                               symmetric=True),
                             lambda g, variant="grid", seed=1: run_color(g, seed, variant))
    if name_l == "td":
        return BenchmarkCase("TD", "tree_desc",
                             lambda depth=24, lo=1, hi=4, fill=0.76, seed=1: gen_tree(depth, lo, hi, fill, seed),
                             lambda t, variant="grid": run_tree_desc(t, variant))
    if name_l == "th":
        return BenchmarkCase("TH", "tree_height",
                             lambda depth=24, lo=1, hi=4, fill=0.76, seed=1: gen_tree(depth, lo, hi, fill, seed),
                             lambda t, variant="grid": run_tree_height(t, variant))
    raise DpcError(1, f"unknown benchmark '{name}' (SSSP, SpMV, GC, TD, TH)")
