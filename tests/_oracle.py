"""ctypes access to the CPU checkers (TEST INFRASTRUCTURE).

- oracle/liboracle.so : our C restatement of the reference's sequential oracles
- oracle/_ref/libref_sim.so : the unmodified reference simulator (dpcons)
  compiled in place from /root/reference (absent on the GPU box unless built
  here first; it travels with the snapshot because it is not gpurun-ignored).
"""
import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
LIB = os.path.join(ORACLE_DIR, "liboracle.so")
REF = os.path.join(ORACLE_DIR, "_ref", "libref_sim.so")
KDL_DIR = os.path.join(ROOT, "paper_1606_08150_b200", "kdl", "programs")


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def build():
    subprocess.run(["make", "-s", "-C", ORACLE_DIR, "liboracle.so"], check=True)


class Oracle:
    def __init__(self):
        if not os.path.exists(LIB):
            build()
        L = self.L = C.CDLL(LIB)
        P, i64, i32, u64 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64
        L.orc_mix64.restype, L.orc_mix64.argtypes = u64, [u64]
        L.orc_spmv_f64.restype, L.orc_spmv_f64.argtypes = None, [i64, P, P, P, P, P]
        L.orc_spmv_f32_mt.restype, L.orc_spmv_f32_mt.argtypes = None, [i64, P, P, P, P, P, C.c_int]
        L.orc_sssp_dijkstra.restype, L.orc_sssp_dijkstra.argtypes = C.c_int, [i64, P, P, P, i32, P]
        L.orc_bfs.restype, L.orc_bfs.argtypes = C.c_int, [i64, P, P, i32, P]
        L.orc_pagerank.restype, L.orc_pagerank.argtypes = C.c_int, [i64, P, P, i32, C.c_double, P]
        L.orc_sssp_bf_mt.restype, L.orc_sssp_bf_mt.argtypes = i64, [i64, P, P, P, i32, P, C.c_int]
        L.orc_color_greedy.restype, L.orc_color_greedy.argtypes = i32, [i64, P, P, u64, P]
        L.orc_color_greedy_order.restype = i32
        L.orc_color_greedy_order.argtypes = [i64, P, P, u64, C.c_int, P]
        L.orc_color_valid.restype, L.orc_color_valid.argtypes = C.c_int, [i64, P, P, P, i32]
        L.orc_tree_desc.restype, L.orc_tree_desc.argtypes = C.c_int, [i64, P, P]
        L.orc_tree_height.restype, L.orc_tree_height.argtypes = C.c_int, [i64, P, P]
        L.orc_gen_rmat.restype = C.c_int
        L.orc_gen_rmat.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, i32, i32, u64,
                                   C.c_int, P, P, P, P]

    def mix64(self, z):
        return self.L.orc_mix64(z & (2**64 - 1))

    def spmv_f64(self, rowptr, col, val, x):
        rowptr = np.ascontiguousarray(rowptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        val = np.ascontiguousarray(val, np.float32)
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty(len(rowptr) - 1, np.float64)
        self.L.orc_spmv_f64(len(y), _p(rowptr), _p(col), _p(val), _p(x), _p(y))
        return y

    def spmv_f32_mt(self, rowptr, col, val, x, threads):
        y = np.empty(len(rowptr) - 1, np.float32)
        self.L.orc_spmv_f32_mt(len(y), _p(rowptr), _p(col), _p(val), _p(x), _p(y), threads)
        return y

    def pagerank(self, rowptr, col, iters, damping=0.85):
        rowptr = np.ascontiguousarray(rowptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        r = np.empty(len(rowptr) - 1, np.float64)
        assert self.L.orc_pagerank(len(r), _p(rowptr), _p(col), iters, damping, _p(r)) == 0
        return r

    def bfs(self, rowptr, col, source):
        rowptr = np.ascontiguousarray(rowptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        d = np.empty(len(rowptr) - 1, np.uint32)
        assert self.L.orc_bfs(len(d), _p(rowptr), _p(col), source, _p(d)) == 0
        return d

    def sssp(self, rowptr, col, w, source):
        rowptr = np.ascontiguousarray(rowptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        w = np.ascontiguousarray(w, np.int32)
        d = np.empty(len(rowptr) - 1, np.uint32)
        assert self.L.orc_sssp_dijkstra(len(d), _p(rowptr), _p(col), _p(w), source, _p(d)) == 0
        return d

    def sssp_mt(self, rowptr, col, w, source, threads):
        d = np.empty(len(rowptr) - 1, np.uint32)
        r = self.L.orc_sssp_bf_mt(len(d), _p(rowptr), _p(col), _p(w), source, _p(d), threads)
        return d, r

    def color(self, rowptr, col, seed, order=1):
        """order: 1 canonical node order (the product default), 0 hash priority,
        2 largest-log-degree-first."""
        rowptr = np.ascontiguousarray(rowptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        c = np.empty(len(rowptr) - 1, np.int32)
        k = self.L.orc_color_greedy_order(len(c), _p(rowptr), _p(col), seed & (2**64 - 1), order, _p(c))
        return c, k

    def color_valid(self, rowptr, col, color, ncolors):
        rowptr = np.ascontiguousarray(rowptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        color = np.ascontiguousarray(color, np.int32)
        return bool(self.L.orc_color_valid(len(color), _p(rowptr), _p(col), _p(color), ncolors))

    def tree_desc(self, parent):
        parent = np.ascontiguousarray(parent, np.int32)
        out = np.empty(len(parent), np.int32)
        assert self.L.orc_tree_desc(len(parent), _p(parent), _p(out)) == 0
        return out

    def tree_height(self, parent):
        parent = np.ascontiguousarray(parent, np.int32)
        out = np.empty(len(parent), np.int32)
        assert self.L.orc_tree_height(len(parent), _p(parent), _p(out)) == 0
        return out

    def gen_rmat(self, scale, edgefactor=16, a=0.57, b=0.19, c=0.19, wmin=1, wmax=255, seed=1,
                 weights=True, values=False, permute=False):
        """Directed R-MAT graph, the oracle's own restatement (oracle.c
        orc_gen_rmat): same graph as dpc_gen_rmat for the same arguments.
        Returns (rowptr int64, col int32, w int32 | None, val float32 | None)."""
        n = 1 << scale
        m = n * edgefactor
        rowptr = np.empty(n + 1, np.int64)
        col = np.empty(m, np.int32)
        w = np.empty(m, np.int32) if weights else None
        val = np.empty(m, np.float32) if values else None
        rc = self.L.orc_gen_rmat(scale, edgefactor, a, b, c, wmin, wmax, seed & (2**64 - 1), int(permute),
                                 _p(rowptr), _p(col), _p(w), _p(val))
        if rc != 0:
            raise MemoryError("orc_gen_rmat: allocation failed")
        return rowptr, col, w, val


MODES = {"basic": 0, "flat": 0, "warp": 1, "block": 2, "grid": 3}


class RefSim:
    """The reference's own CPU path: parse -> consolidate -> simulate."""

    def __init__(self):
        if not os.path.exists(REF):
            raise FileNotFoundError(REF)
        L = self.L = C.CDLL(REF)
        P, i64 = C.c_void_p, C.c_int64
        L.ref_run.restype = C.c_int
        L.ref_run.argtypes = [C.c_char_p, C.c_int, C.c_int, P, P, C.c_int, P, P, P, C.c_int, P, P, P,
                              C.c_char_p, P, i64, P, C.c_char_p, C.c_int]
        L.ref_kc_config.restype = None
        L.ref_kc_config.argtypes = [i64, i64, i64, C.POINTER(i64), C.POINTER(i64)]
        L.ref_per_buffer_size.restype = i64
        L.ref_per_buffer_size.argtypes = [i64, i64, i64]
        L.ref_consolidate_text.restype = C.c_int
        L.ref_consolidate_text.argtypes = [C.c_char_p, C.c_int, C.c_char_p, C.c_int]

    @staticmethod
    def kdl(name):
        with open(os.path.join(KDL_DIR, name)) as f:
            return f.read()

    def run(self, src, mode, scalars=None, int_arrays=None, float_arrays=None, out=None,
            out_len=0, out_float=False):
        scalars = scalars or {}
        int_arrays = int_arrays or {}
        float_arrays = float_arrays or {}
        keep = []

        def names(keys):
            arr = (C.c_char_p * max(1, len(keys)))(*[k.encode() for k in keys])
            keep.append(arr)
            return C.cast(arr, C.c_void_p)

        sk = list(scalars)
        sv = np.array([scalars[k] for k in sk] or [0], np.int64)
        ik = list(int_arrays)
        iarrs = [np.ascontiguousarray(int_arrays[k], np.int64) for k in ik]
        iptr = (C.c_void_p * max(1, len(ik)))(*[a.ctypes.data for a in iarrs])
        ilen = np.array([len(a) for a in iarrs] or [0], np.int64)
        fk = list(float_arrays)
        farrs = [np.ascontiguousarray(float_arrays[k], np.float64) for k in fk]
        fptr = (C.c_void_p * max(1, len(fk)))(*[a.ctypes.data for a in farrs])
        flen = np.array([len(a) for a in farrs] or [0], np.int64)
        res = np.zeros(out_len, np.float64 if out_float else np.int64)
        met = np.zeros(12, np.int64)
        err = C.create_string_buffer(4096)
        rc = self.L.ref_run(src.encode(), MODES.get(mode, mode) if isinstance(mode, str) else mode,
                            len(sk), names(sk), _p(sv), len(ik), names(ik),
                            C.cast(iptr, C.c_void_p), _p(ilen), len(fk), names(fk),
                            C.cast(fptr, C.c_void_p), _p(flen),
                            out.encode() if out else None, _p(res) if out else None, out_len,
                            _p(met), err, 4096)
        keys = ["childLaunchCount", "fixedPoolPeak", "virtualPoolPeak", "simulatedCycles",
                "parentSwapEvents", "maxConcurrentObserved", "bufferItemsInserted",
                "allocCyclesCharged", "dramTransactions", "deadlockDetected",
                "warpExecEfficiency_1e6", "smOccupancyAchieved_1e6"]
        return rc, res, dict(zip(keys, met.tolist())), err.value.decode()

    def kc_config(self, b, t, x):
        ob, ot = C.c_int64(), C.c_int64()
        self.L.ref_kc_config(b, t, x, C.byref(ob), C.byref(ot))
        return ob.value, ot.value

    def per_buffer_size(self, threads, nvars, k):
        return self.L.ref_per_buffer_size(threads, nvars, k)

    def consolidate_text(self, src, mode):
        buf = C.create_string_buffer(1 << 20)
        rc = self.L.ref_consolidate_text(src.encode(), MODES[mode], buf, 1 << 20)
        return rc, buf.value.decode()
