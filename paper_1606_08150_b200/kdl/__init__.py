"""B200 consolidation compiler for the reference's kernel DSL (.kdl):
parse -> consolidate (warp / block / grid, the paper's directive compiler)
-> sm_100a CUDA (kdl_rt.cuh runtime) -> nvcc -> a loadable module that runs
the program on the GPU with CDP2 device launches.

    import paper_1606_08150_b200.kdl as kdl
    mod = kdl.compile(open("spmv.kdl").read(), mode="grid")
    res = mod.run({"n": n, "m": m, "nx": n, "thr": 32},
                  {"rowptr": rowptr, "col": col, "val": val, "x": x})
    y = res.arrays["y"]

`mode` is "basic" (the program as written: one device launch per annotated
site execution, Fig. 1), "warp" / "block" / "grid" (consolidated at that
granularity, the reference's granularityOverride) or "directive" (each
site's own consltdt clause).  `consolidated=True` takes an already
consolidated program (e.g. the reference's consolidate() text) as is.

This mirrors the reference's compiler pipeline (parse_program,
parser.hpp:783 -> consolidate, transform.hpp:971) with the simulator
(simulate, sim.hpp:1746) replaced by real execution on a B200.  There is no
CPU fallback: running a module needs the CUDA device.
"""
import ctypes as C
import glob
import hashlib
import os
import subprocess

import numpy as np

from . import ast
from .transform import Config, consolidate, k20c_occupancy, lower_kc
from .cuda import generate
from .parse import KdlError, parse_program
from .unparse import unparse

__all__ = ["compile", "compile_program", "Module", "KdlError", "KdlFault", "Config", "parse_program",
           "consolidate", "lower_kc", "k20c_occupancy", "generate", "build_programs", "autotune", "unparse", "PROGRAMS"]

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "_build")
PROGRAMS = os.path.join(HERE, "programs")
INCLUDE = os.path.join(os.path.dirname(os.path.dirname(HERE)), "include")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-rdc=true", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]
NVCC_LIBS = ["-lcudadevrt", "-lcudart_static", "-lpthread", "-ldl", "-lrt"]
MODES = ("basic", "warp", "block", "grid", "directive")

FAULTS = {1: ("overflow", "consolidation buffer overflow"), 2: ("overflow", "pre-allocated pool exhausted"),
          4: ("runtime", "array index out of bounds"), 8: ("runtime", "integer division or modulo by zero"),
          16: ("config", "launch extents outside [1, 2^31) x [1, 1024]"),
          32: ("oom", "device launch refused (pending-launch pool)"), 64: ("oom", "launch-record arena exhausted"),
          128: ("runtime", "dp_buf_get / dp_buf_cfg index out of range")}


class KdlFault(RuntimeError):
    """A fault raised by the running program (the simulator's SimFault kinds,
    sim.hpp:49-52)."""

    def __init__(self, bits):
        self.bits = bits
        self.kinds = sorted({FAULTS[b][0] for b in FAULTS if bits & b})
        super().__init__("; ".join(f"{FAULTS[b][0]}: {FAULTS[b][1]}" for b in FAULTS if bits & b))


def read_program(name):
    with open(os.path.join(PROGRAMS, name)) as f:
        return f.read()


def _nvcc():
    return os.environ.get("NVCC") or ("/usr/local/cuda/bin/nvcc" if os.path.exists("/usr/local/cuda/bin/nvcc")
                                      else "nvcc")


def build_so(cu_src, tag):
    """Compile one generated unit into paper_1606_08150_b200/kdl/_build/
    (cached by content hash; the .so travels with the repo snapshot)."""
    rt = ""
    for hdr in (os.path.join(HERE, "kdl_rt.cuh"), os.path.join(INCLUDE, "dpc_kdl.h")):
        with open(hdr) as f:
            rt += f.read()
    h = hashlib.sha1((cu_src + rt + " ".join(NVCC_FLAGS)).encode()).hexdigest()[:16]
    so = os.path.join(BUILD, f"{tag}_{h}.so")
    if os.path.exists(so):
        return so
    os.makedirs(BUILD, exist_ok=True)
    cu = so[:-3] + ".cu"
    with open(cu, "w") as f:
        f.write(cu_src)
    tmp = so + f".tmp{os.getpid()}"
    cmd = [_nvcc(), *NVCC_FLAGS, "-I", HERE, "-I", INCLUDE, cu, "-o", tmp, *NVCC_LIBS]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise KdlError("cuda.nvcc", f"nvcc failed for {cu}:\n{r.stderr[-4000:]}")
    os.replace(tmp, so)
    # keep one build per (program, mode): drop units of older sources
    for old in glob.glob(os.path.join(BUILD, f"{glob.escape(tag)}_" + "[0-9a-f]" * 16 + ".*")):
        if not old.startswith(so[:-3]):
            try:
                os.remove(old)
            except OSError:
                pass
    return so


def eval_host(e, scalars):
    """Evaluate a host-side expression (array lengths, entry launch) over the
    workload scalars, with the DSL's int64 / float rules."""
    k = e.kind
    if k == "int":
        return int(e.ival)
    if k == "float":
        return float(e.fval)
    if k == "name":
        if e.name not in scalars:
            raise KdlError("run.scalar", f"workload scalar {e.name!r} is not given")
        return scalars[e.name]
    if k == "unary":
        v = eval_host(e.args[0], scalars)
        return int(v == 0) if e.name == "!" else -v
    if k == "minmax":
        a, b = (eval_host(x, scalars) for x in e.args)
        return min(a, b) if e.name == "min" else max(a, b)
    if k == "binary":
        a, b = (eval_host(x, scalars) for x in e.args)
        op = e.name
        flt = isinstance(a, float) or isinstance(b, float)
        if op == "/":
            if flt:
                return a / b
            q = abs(a) // abs(b)
            return q if (a >= 0) == (b >= 0) else -q
        if op == "%":
            return a - b * (abs(a) // abs(b) * (1 if (a >= 0) == (b >= 0) else -1))
        return {"+": lambda: a + b, "-": lambda: a - b, "*": lambda: a * b,
                "<": lambda: int(a < b), "<=": lambda: int(a <= b), ">": lambda: int(a > b),
                ">=": lambda: int(a >= b), "==": lambda: int(a == b), "!=": lambda: int(a != b),
                "&&": lambda: int(bool(a) and bool(b)), "||": lambda: int(bool(a) or bool(b))}[op]()
    raise KdlError("run.expr", f"{k!r} is not allowed in a host-side expression")


class _Rt(C.Structure):
    _fields_ = [("arr", C.c_void_p * 64), ("len", C.c_int64 * 64), ("ctr", C.c_void_p),
                ("arena", C.c_void_p), ("arena_words", C.c_uint64), ("inst", C.c_void_p),
                ("inst_cap", C.c_uint64), ("region", C.c_void_p * 2), ("region_words", C.c_uint64),
                ("narr", C.c_int64)]


class Result:
    def __init__(self, arrays, launches, runs, kc, ms):
        self.arrays, self.launches, self.runs, self.kc, self.ms = arrays, launches, runs, kc, ms


_CTX = {}


def _context(device):
    """The library context (device + stream) the modules run on: device
    memory, copies, events and the launch stream all come from libdpc.so
    (no torch on this path).  Raises DpcError('cuda') without an sm_100 GPU
    -- there is no CPU fallback."""
    from .. import Context
    if device not in _CTX:
        _CTX[device] = Context(device)
    return _CTX[device]


class Module:
    """A compiled program.  run() owns device memory through the library
    context (dpc_dev_alloc / dpc_copy_* / dpc_dev_memset); every kernel that
    executes is generated code from this module's .so."""

    def __init__(self, prog, so, kc, mode, width=64):
        self.prog, self.so, self.kc_rows, self.mode, self.width = prog, so, kc, mode, width
        self.lib = None
        self._dev = None
        self.grid_total = max([s.total_bytes for k in prog.kernels for s in k.body
                               if s.kind == "buf_decl" and s.gran == "grid"] or [0])

    def _load(self, device, pending):
        ctx = _context(device)
        if self.lib is None:
            L = C.CDLL(self.so)
            L.dk_error.restype = C.c_char_p
            L.dk_init.argtypes = [C.c_int, C.c_longlong]
            L.dk_set_rt.argtypes = [C.c_void_p]
            L.dk_kc_values.argtypes = [C.c_void_p]
            L.dk_launch_entry.argtypes = [C.c_longlong, C.c_longlong, C.c_void_p, C.c_void_p, C.c_void_p]
            if L.dk_sizeof_rt() != C.sizeof(_Rt):
                raise RuntimeError("kdl runtime struct layout mismatch")
            self.lib = L
        if self._dev != device:
            ctx.synchronize()
            if self.lib.dk_init(device, pending) != 0:
                raise RuntimeError("dk_init: " + self.lib.dk_error().decode())
            self._dev = device
        kc = (C.c_longlong * max(1, len(self.kc_rows)))()
        self.lib.dk_kc_values(kc)
        return ctx, {f"{k}/KC_{x}/T{t}": int(kc[i]) for i, (k, x, t) in enumerate(self.kc_rows)}

    def run(self, scalars, arrays=None, *, until_stable=None, max_runs=10000, device=0,
            pool_bytes=1 << 30, inst_cap=1 << 20, pending=1 << 17, timed=False):
        """Run the entry launch once, or — with `until_stable=<array>` —
        repeat it until that array stops changing (the host sweep loop the
        SSSP / TH formulations need).  Returns Result(arrays as numpy,
        device launches, entry runs, KC block counts, device ms)."""
        ctx, kc = self._load(device, pending)
        arrays = arrays or {}
        for n in arrays:
            if self.prog.global_(n) is None:
                raise KdlError("run.array", f"{n!r} is not a global array of the program")
        rt = _Rt()
        bufs = []  # every device allocation of this run (freed at the end)

        def alloc(nbytes):
            p = ctx.alloc(max(int(nbytes), 8))
            bufs.append(p)
            return p

        try:
            devarr = {}  # name -> (device pointer, length, numpy dtype)
            for i, g in enumerate(self.prog.globals):
                ln = int(eval_host(g.length, scalars))
                if ln < 0:
                    raise KdlError("run.array", f"array {g.name!r} has negative length {ln}")
                w32 = self.width == 32
                npt = (np.float32 if w32 else np.float64) if g.type == ast.FLOAT else (np.int32 if w32 else np.int64)
                ptr = 0
                if ln > 0:
                    ptr = alloc(ln * np.dtype(npt).itemsize)
                    if g.name in arrays:
                        src = np.asarray(arrays[g.name])
                        if w32 and g.type != ast.FLOAT and src.size and (src.min() < -2**31 or src.max() >= 2**31):
                            raise KdlError("run.array", f"array {g.name!r} does not fit the 32-bit width")
                        a = src.astype(npt)
                        if a.shape != (ln,):
                            raise KdlError("run.array", f"array {g.name!r} must have {ln} elements, got {a.shape}")
                        ctx.h2d(ptr, a)
                    else:
                        ctx.memset(ptr, 0, ln * np.dtype(npt).itemsize)
                elif g.name in arrays and np.asarray(arrays[g.name]).size:
                    raise KdlError("run.array", f"array {g.name!r} must have 0 elements")
                devarr[g.name] = (ptr, ln, npt)
                rt.arr[i] = ptr
                rt.len[i] = ln
            rt.narr = len(self.prog.globals)
            ctr = alloc(8 * 8)
            arena_words = max(1, pool_bytes // 8)
            arena = alloc(8 * arena_words)
            inst = alloc(8 * 3 * inst_cap)
            ctx.memset(inst, 0, 8 * 3 * inst_cap)
            region_words = max(1, self.grid_total // 8) if self.grid_total else 1
            regions = [alloc(8 * region_words) for _ in range(2)]
            rt.ctr, rt.arena, rt.arena_words = ctr, arena, arena_words
            rt.inst, rt.inst_cap = inst, inst_cap
            rt.region[0], rt.region[1] = regions[0], regions[1]
            rt.region_words = region_words
            if self.lib.dk_set_rt(C.byref(rt)) != 0:
                raise RuntimeError("dk_set_rt: " + self.lib.dk_error().decode())

            e = self.prog.entry
            ek = self.prog.kernel(e.kernel)
            gdim = int(eval_host(e.grid, scalars))
            bdim = int(eval_host(e.block, scalars))
            if len(e.args) != len(ek.params):
                raise KdlError("run.entry", f"entry passes {len(e.args)} arguments, kernel takes {len(ek.params)}")
            args = (C.c_longlong * max(1, len(e.args)))()
            for j, (a, p) in enumerate(zip(e.args, ek.params)):
                if p.is_array:
                    args[j] = [x.name for x in self.prog.globals].index(a.name)
                elif p.type == ast.FLOAT:
                    args[j] = int(np.array([float(eval_host(a, scalars))], np.float64).view(np.int64)[0])
                else:
                    v = eval_host(a, scalars)
                    if isinstance(v, float):
                        raise KdlError("run.entry", f"float argument for int parameter {p.name!r}")
                    args[j] = int(v)
            stream = C.c_void_p(ctx.stream)
            launches, runs, ms = 0, 0, 0.0
            if until_stable and until_stable not in devarr:
                raise KdlError("run.array", f"until_stable names unknown array {until_stable!r}")

            def fetch(name):
                ptr, ln, npt = devarr[name]
                return ctx.d2h(ptr, ln, npt) if ln > 0 else np.zeros(0, npt)

            ctr_init = np.array([0, 0, 0, 1, 0, 0, 0, 0], np.int64)
            while True:
                ctx.h2d(ctr, ctr_init)
                ctx.memset(inst, 0, 8 * 3)
                before = fetch(until_stable) if until_stable else None
                if timed:
                    ctx.record(60)
                rc = self.lib.dk_launch_entry(gdim, bdim, args, C.c_void_p(inst), stream)
                if rc != 0:
                    raise RuntimeError("entry launch: " + self.lib.dk_error().decode())
                if timed:
                    ctx.record(61)
                ctx.synchronize()
                if timed:
                    ms += ctx.elapsed_ms(60, 61)
                c = ctx.d2h(ctr, 8, np.int64).tolist()
                runs += 1
                launches += c[1]
                if c[0]:
                    raise KdlFault(c[0])
                if not until_stable or np.array_equal(before, fetch(until_stable)) or runs >= max_runs:
                    break
            out = {n: fetch(n) for n in devarr}
        finally:
            ctx.synchronize()
            for p in bufs:
                ctx.free(p)
        return Result(out, launches, runs, kc, ms)


def compile_program(prog, mode="basic", config=None, name="kdl", consolidated=False, schedule="block",
                    width=64):
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}")
    if not consolidated and mode != "basic":
        prog = consolidate(prog, granularity=None if mode == "directive" else mode, config=config,
                           schedule=schedule)
    src, kc = generate(prog, name, width)
    tag = f"{name}_{mode}" + ("" if schedule == "block" or consolidated or mode == "basic" else f"_{schedule}")
    tag += "" if width == 64 else "_w32"
    so = build_so(src, tag)
    return Module(prog, so, kc, mode, width)


def compile(source, mode="basic", config=None, name="kdl", consolidated=False, schedule="block",  # noqa: A001
            width=64):
    """.kdl text -> Module (compiled for sm_100a; cached under kdl/_build).
    schedule="block" (default) drains multi-block children one item per
    block; "reference" keeps the reference's drain loop.  width=64 keeps the
    simulator's int64 / fp64 values; width=32 runs the program on int32 /
    fp32 arrays and scalars (integer literals must fit)."""
    return compile_program(parse_program(source), mode, config, name, consolidated, schedule, width)


def autotune(source, scalars, arrays=None, *, until_stable=None, modes=("warp", "block", "grid"),
             kc=(None, 4, 16, 64), reps=3, name="kdl", device=0):
    """Pick the consolidation granularity and the KC_X concurrency of a
    program by measurement on the device (the reference picks them from its
    cost model: directive + KC_X defaults, config.hpp:77-86).  Every
    candidate runs `reps` times on the same inputs (device time of the entry
    launch tree); candidates whose output differs from the first one's are
    rejected.  Returns (best, table) with rows {mode, kc_x, ms, launches}."""
    from .transform import default_concurrency
    table, ref_out = [], None
    for mode in modes:
        for x in kc:
            if mode == "grid" and x not in (None, 1):
                continue  # KC_1: the grid form's single consolidated launch fills the device
            cfg = Config("kc", x=x) if x else None
            mod = compile(source, mode, config=cfg, name=f"{name}_x{x or 0}")
            runs = [mod.run(scalars, arrays, until_stable=until_stable, device=device, timed=True)
                    for _ in range(reps)]
            outs = runs[-1].arrays
            if ref_out is None:
                ref_out = outs
            same = all(np.array_equal(outs[k], ref_out[k]) if outs[k].dtype.kind != "f"
                       else np.allclose(outs[k], ref_out[k], rtol=1e-9, atol=1e-12) for k in outs)
            table.append({"mode": mode, "kc_x": x or default_concurrency(mode), "ms": min(r.ms for r in runs),
                          "launches": runs[-1].launches, "same_result": bool(same)})
    ok = [r for r in table if r["same_result"]]
    return min(ok, key=lambda r: r["ms"]), table


def build_programs(jobs=8):
    """Pre-compile the bundled programs in every mode (called by build())."""
    from concurrent.futures import ThreadPoolExecutor
    work = [(f, m, "block") for f in sorted(os.listdir(PROGRAMS)) if f.endswith(".kdl")
            for m in ("basic", "warp", "block", "grid")]
    with ThreadPoolExecutor(jobs) as ex:
        list(ex.map(lambda w: compile(read_program(w[0]), w[1], name=w[0][:-4], schedule=w[2]), work))
    return len(work)
