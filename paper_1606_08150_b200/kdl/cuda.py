"""CUDA builder of the B200 consolidation compiler: ast.Program (as written,
or after consolidate()) -> one sm_100a CUDA translation unit.

Mapping (the reference's dp_* builtins, ast.hpp:25-33 / 63-65, onto the
device runtime in kdl_rt.cuh):

  kernel k(params)            __global__ k_k(params..., dk::Inh dk_inh, dk::Inst* dk_inst)
  int / float                 long long / double (the simulator's Value, sim.hpp:72-80)
  global T a[len]             device array, checked access through dk_rt.arr[id]
  k<<<g, b>>>(args)           CDP2 fire-and-forget launch by the executing thread
  sync_device; k<<<..>>>      the launch becomes a tail launch (CDP2 has no device sync)
  barrier_block               __syncthreads()
  dp_buffers(warp|block, ...) shared-memory owner record per warp / block
  dp_buffers(grid, ...)       the launch's Inst record (+ region[level & 1])
  dp_insert(g, b, w...)       warp-aggregated slot reservation, item = {g, b, w...}
  dp_buf_pending()            this thread's owner count (clamped to capacity)
  dp_buf_count / get / cfg_*  the inherited buffer (dk_inh), range-checked
  dp_grid_last()              last-block ticket on the launch's Inst record
  kc_blocks(k, X, T)          max(1, occupancy(k, T) * SMs / X), resolved at load
  &&, ||                      both operands evaluated (the simulator does not
                              short-circuit, sim.hpp:1598-1599)

Entry point of the generated unit (extern "C"): dk_init(device, pending),
dk_sizeof_rt(), dk_set_rt(rt), dk_kc_values(out), dk_launch_entry(g, b,
args, inst0, stream), dk_error().
"""
from . import ast as A
from .parse import KdlError

_ARITH = {"+", "-", "*", "/", "%"}
_CMP = {"<", "<=", ">", ">=", "==", "!="}


def _ctype(t):
    return "dk_flt" if t == A.FLOAT else "dk_int"


def _float_lit(v, width=64):
    s = repr(float(v))
    if "inf" in s or "nan" in s:
        raise KdlError("cuda.literal", f"non-finite float literal {s}")
    s = s if ("." in s or "e" in s) else s + ".0"
    return s + "f" if width == 32 else s


class _KInfo:
    def __init__(self, k):
        self.k = k
        self.decl = None          # buf_decl statement
        self.insert_types = None  # slot types of this kernel's inserts
        self.slot_types = None    # slot types of the buffer it drains
        self.uses_grid_last = False
        self.targets = []
        # top-level sync_device splits the kernel into tail-launched phases
        self.phases = [[]]
        for st in k.body:
            if st.kind == "sync":
                self.phases.append([])
            else:
                self.phases[-1].append(st)
        for s in A.walk_stmts(k.body):
            if s.kind == "buf_decl":
                if self.decl is not None:
                    raise KdlError("cuda.bufdecl", f"kernel {k.name!r} declares buffers twice")
                if s not in k.body:
                    raise KdlError("cuda.bufdecl", f"kernel {k.name!r}: dp_buffers must be a top-level statement")
                self.decl = s
            if s.kind == "launch":
                self.targets.append(s.name)
            for e in s.exprs:
                if any(n.kind == "grid_last" for n in A.walk_expr(e)):
                    self.uses_grid_last = True

    @property
    def split(self):
        return len(self.phases) > 1

    @property
    def needs_inst(self):
        return self.uses_grid_last or self.split or (self.decl is not None and self.decl.gran == "grid")


class Builder:
    def __init__(self, prog, name="kdl", width=64):
        if width not in (32, 64):
            raise KdlError("cuda.width", "width must be 32 or 64")
        self.prog = prog
        self.name = name
        self.width = width
        if len(prog.globals) > 64:
            raise KdlError("cuda.arrays", "at most 64 global arrays")
        self.arr = {g.name: (i, g.type) for i, g in enumerate(prog.globals)}
        self.info = {k.name: _KInfo(k) for k in prog.kernels}
        if prog.entry is None or prog.entry.kernel not in self.info:
            raise KdlError("cuda.entry", "entry kernel is not defined")
        for ki in self.info.values():
            for t in ki.targets:
                if t not in self.info:
                    raise KdlError("cuda.target", f"launch of unknown kernel {t!r}")
        self.kc = []
        self.hoist = False      # top-level lets of a split kernel are hoisted
        self.ret_label = None   # return -> jump to the split point
        self._analyse()

    # ---------------- analysis ----------------
    def _analyse(self):
        # two passes: insert types may depend on drained slot types
        for _ in range(3):
            for ki in self.info.values():
                self.cur = ki
                self.env = [{p.name: ("array" if p.is_array else p.type, p.is_array) for p in ki.k.params}]
                ins = []
                self._scan(ki.k.body, ins)
                if ins:
                    ref = ins[0]
                    for t in ins[1:]:
                        if t != ref:
                            raise KdlError("cuda.insert", f"kernel {ki.k.name!r}: dp_insert sites disagree on types")
                    ki.insert_types = ref
            changed = True
            while changed:
                changed = False
                for ki in self.info.values():
                    src = ki.insert_types if ki.decl is not None else ki.slot_types
                    if src is None:
                        continue
                    for t in ki.targets:
                        tk = self.info[t]
                        if tk.slot_types is None:
                            tk.slot_types = src
                            changed = True
                        elif tk.slot_types != src:
                            raise KdlError("cuda.inherit", f"kernel {t!r} drains buffers of different shapes")

    def _scan(self, body, ins):
        self.env.append({})
        for s in body:
            if s.kind == "let":
                self.env[-1][s.name] = (s.scalar, False)
            elif s.kind == "for":
                self.env.append({s.name: (A.INT, False)})
                self._scan(s.body, ins)
                self.env.pop()
            elif s.kind == "insert":
                ins.append(tuple(self.etype(e) for e in s.exprs[2:]))
            elif s.kind == "if":
                self._scan(s.body, ins)
                self._scan(s.else_body, ins)
        self.env.pop()

    def lookup(self, n):
        for scope in reversed(self.env):
            if n in scope:
                return scope[n]
        return None

    def etype(self, e):
        k = e.kind
        if k in ("int", "intrinsic", "buf_count", "buf_pending", "buf_cfg_grid", "buf_cfg_block",
                 "grid_last", "kc_blocks"):
            return A.INT
        if k == "float":
            return A.FLOAT
        if k == "name":
            v = self.lookup(e.name)
            if v is None:
                if e.name in self.arr:
                    return "array"
                raise KdlError("cuda.name", f"kernel {self.cur.k.name!r}: unknown name {e.name!r}")
            return v[0]
        if k in ("index", "atomic"):
            return self.array_of(e.name)[1]
        if k == "unary":
            return A.INT if e.name == "!" else self.etype(e.args[0])
        if k == "binary":
            if e.name in _ARITH:
                ts = {self.etype(a) for a in e.args}
                return A.FLOAT if A.FLOAT in ts else A.INT
            return A.INT
        if k == "minmax":
            ts = {self.etype(a) for a in e.args}
            return A.FLOAT if A.FLOAT in ts else A.INT
        if k == "buf_get":
            st = self.cur.slot_types
            slot = e.args[1].ival
            if st is None or slot >= len(st):
                return A.INT
            return st[slot]
        raise KdlError("cuda.expr", f"unknown expression kind {k!r}")

    def array_of(self, n):
        """-> (code for the array id, element type)."""
        v = self.lookup(n)
        if v is not None:
            if not v[1]:
                raise KdlError("cuda.array", f"{n!r} is not an array")
            # array parameters carry the id of a global; element type declared
            return f"v_{n}", self._param_elem(n)
        if n in self.arr:
            i, t = self.arr[n]
            return str(i), t
        raise KdlError("cuda.array", f"unknown array {n!r}")

    def _param_elem(self, n):
        for p in self.cur.k.params:
            if p.name == n:
                return p.type
        raise KdlError("cuda.array", f"unknown array parameter {n!r}")

    # ---------------- expressions ----------------
    def ex(self, e):
        k = e.kind
        if k == "int":
            if self.width == 32:
                if not -2**31 <= e.ival < 2**31:
                    raise KdlError("cuda.literal", f"integer literal {e.ival} does not fit the 32-bit width")
                return f"({e.ival})"
            return f"{e.ival}LL"
        if k == "float":
            return _float_lit(e.fval, self.width)
        if k == "name":
            t = self.etype(e)
            if t == "array":
                raise KdlError("cuda.name", f"array {e.name!r} used as a scalar")
            return f"v_{e.name}"
        if k == "intrinsic":
            return {"threadIdx": "((dk_int)threadIdx.x)", "blockIdx": "((dk_int)blockIdx.x)",
                    "blockDim": "((dk_int)blockDim.x)", "gridDim": "((dk_int)gridDim.x)"}[e.name]
        if k == "index":
            aid, t = self.array_of(e.name)
            return f"(*dk_{'f' if t == A.FLOAT else 'i'}p({aid}, {self.int_ex(e.args[0])}))"
        if k == "atomic":
            aid, t = self.array_of(e.name)
            return self.atomic(aid, t, e.args[0], e.args[1])
        if k == "unary":
            a = self.ex(e.args[0])
            return f"((dk_int)(({a}) == 0))" if e.name == "!" else f"(-({a}))"
        if k == "binary":
            op = e.name
            l, r = e.args
            if op in ("&&", "||"):
                return f"((dk_int)((({self.ex(l)}) != 0) {'&' if op == '&&' else '|'} (({self.ex(r)}) != 0)))"
            if op in _CMP:
                return f"((dk_int)(({self.ex(l)}) {op} ({self.ex(r)})))"
            if self.etype(e) == A.FLOAT:
                if op == "%":
                    raise KdlError("cuda.type", "modulo requires integer operands")
                return f"((dk_flt)({self.ex(l)}) {op} (dk_flt)({self.ex(r)}))"
            if op == "/":
                return f"dk_idiv({self.ex(l)}, {self.ex(r)})"
            if op == "%":
                return f"dk_imod({self.ex(l)}, {self.ex(r)})"
            return f"(({self.ex(l)}) {op} ({self.ex(r)}))"
        if k == "minmax":
            ct = _ctype(self.etype(e))
            return f"dk_{e.name}<{ct}>(({ct})({self.ex(e.args[0])}), ({ct})({self.ex(e.args[1])}))"
        if k == "buf_count":
            return "dk_inh.n"
        if k == "buf_pending":
            return self.pending()
        if k == "buf_get":
            w = f"dk_buf_word(dk_inh, {self.int_ex(e.args[0])}, {2 + e.args[1].ival}LL)"
            return f"dk_word_flt({w})" if self.etype(e) == A.FLOAT else f"((dk_int)({w}))"
        if k in ("buf_cfg_grid", "buf_cfg_block"):
            return f"((dk_int)dk_buf_word(dk_inh, {self.int_ex(e.args[0])}, {0 if k == 'buf_cfg_grid' else 1}LL))"
        if k == "grid_last":
            return "((dk_int)dk_grid_last(dk_inst, &dk_gl))"
        if k == "kc_blocks":
            key = (e.name, e.ival, e.args[0].ival)
            if e.name not in self.info:
                raise KdlError("cuda.kc", f"kc_blocks names unknown kernel {e.name!r}")
            if key not in self.kc:
                self.kc.append(key)
            return f"((dk_int)dk_kc[{self.kc.index(key)}])"
        raise KdlError("cuda.expr", f"unknown expression kind {k!r}")

    def int_ex(self, e):
        if self.etype(e) != A.INT:
            raise KdlError("cuda.type", "array index / launch extent / buffer index must be an integer")
        return self.ex(e)

    def atomic(self, aid, t, i, v):
        if t == A.INT and self.etype(v) == A.FLOAT:
            raise KdlError("cuda.type", "atomicAdd of a float value on an int array")
        if t == A.FLOAT:
            return f"dk_atomic_f(dk_fp({aid}, {self.int_ex(i)}), (dk_flt)({self.ex(v)}))"
        return f"dk_atomic_i(dk_ip({aid}, {self.int_ex(i)}), (dk_int)({self.ex(v)}))"

    # ---------------- owner helpers ----------------
    def _own(self):
        d = self.cur.decl
        return "&dk_wown[threadIdx.x >> 5]" if d.gran == "warp" else "&dk_bown"

    def _stride(self):
        return 2 + self.cur.decl.nvars

    def _grid_cap(self):
        d = self.cur.decl
        return f"dk_grid_cap({d.total_bytes}LL, {d.nvars}LL, {self._stride()}LL)"

    def pending(self):
        d = self.cur.decl
        if d is None:
            return "((dk_int)0)"
        if d.gran == "grid":
            return f"((dk_int)dk_pending_grid(dk_inst, {self._grid_cap()}))"
        return f"((dk_int)dk_pending_own({self._own()}))"

    # ---------------- statements ----------------
    def emit_body(self, body, ind):
        self.env.append({})
        out = []
        tail = False
        for s in body:
            if tail and s.kind != "launch":
                raise KdlError("cuda.sync", "only launches may follow sync_device on CDP2 (they become tail "
                               "launches); other postwork after a device sync is unsupported")
            if s.kind == "sync":
                tail = True
                out.append(f"{ind}// sync_device: the launches below are tail launches")
                continue
            out += self.emit(s, ind, tail)
        self.env.pop()
        return out

    def emit(self, s, ind, tail=False):
        k = s.kind
        if k == "let":
            t = self.etype(s.exprs[0])
            if s.scalar == A.INT and t != A.INT:
                raise KdlError("cuda.type", f"assigning float value to int variable {s.name!r}")
            code = f"{ind}{_ctype(s.scalar)} v_{s.name} = {self.ex(s.exprs[0])};"
            if self.hoist and len(self.env) == 2:
                code = f"{ind}v_{s.name} = {self.ex(s.exprs[0])};"
            self.env[-1][s.name] = (s.scalar, False)
            return [code]
        if k == "assign":
            v = self.lookup(s.name)
            if v is None or v[1]:
                raise KdlError("cuda.name", f"assignment to unknown scalar {s.name!r}")
            if v[0] == A.INT and self.etype(s.exprs[0]) != A.INT:
                raise KdlError("cuda.type", f"assigning float value to int variable {s.name!r}")
            return [f"{ind}v_{s.name} = {self.ex(s.exprs[0])};"]
        if k == "store":
            aid, t = self.array_of(s.name)
            if t == A.INT and self.etype(s.exprs[1]) != A.INT:
                raise KdlError("cuda.type", f"storing float value into int array {s.name!r}")
            p = f"dk_{'f' if t == A.FLOAT else 'i'}p({aid}, {self.int_ex(s.exprs[0])})"
            return [f"{ind}*{p} = {self.ex(s.exprs[1])};"]
        if k == "atomic":
            aid, t = self.array_of(s.name)
            code = self.atomic(aid, t, s.exprs[0], s.exprs[1])
            return [f"{ind}{code.replace('dk_atomic_', 'dk_add_', 1)};"]
        if k == "if":
            out = [f"{ind}if (({self.ex(s.exprs[0])}) != 0) {{"]
            out += self.emit_body(s.body, ind + "  ")
            if s.else_body:
                out.append(f"{ind}}} else {{")
                out += self.emit_body(s.else_body, ind + "  ")
            out.append(f"{ind}}}")
            return out
        if k == "for":
            a, b, c = s.exprs
            if self.etype(a) != A.INT or self.etype(c) != A.INT:
                raise KdlError("cuda.type", "for loop start and step must be integers")
            self.env.append({s.name: (A.INT, False)})
            hdr = f"{ind}for (dk_int v_{s.name} = {self.ex(a)}; v_{s.name} < {self.ex(b)}; v_{s.name} += {self.ex(c)}) {{"
            out = [hdr] + self.emit_body(s.body, ind + "  ") + [f"{ind}}}"]
            self.env.pop()
            return out
        if k == "barrier":
            return [f"{ind}__syncthreads();"]
        if k == "return":
            if self.ret_label:
                return [f"{ind}{{ dk_alive = 0; goto {self.ret_label}; }}"]
            return [f"{ind}return;"]
        if k == "grid_barrier":
            raise KdlError("cuda.gridbarrier", "dp_grid_barrier (the naive spin barrier) deadlocks when the grid "
                           "is not co-resident; use the counter/exit protocol (dp_grid_last)")
        if k == "buf_decl":
            return self.emit_decl(s, ind)
        if k == "insert":
            return self.emit_insert(s, ind)
        if k == "launch":
            return self.emit_launch(s, ind, tail)
        raise KdlError("cuda.stmt", f"unsupported statement {k!r}")

    def emit_decl(self, s, ind):
        if s.gran == "grid":
            return [f"{ind}// dp_buffers(grid): the launch's Inst record, region[level & 1]"]
        per = s.exprs[0]
        names = [n.name for n in A.walk_expr(per) if n.kind == "name"]
        if any(self.lookup(n) is None for n in names):
            raise KdlError("cuda.bufdecl", "perBufferSize must be a literal or a kernel parameter")
        cap = self.int_ex(per)
        if s.gran == "warp":
            return [f"{ind}{{",
                    f"{ind}  const long long dk_cap = {cap};",
                    f"{ind}  if ((threadIdx.x & 31u) == 0) dk_own_init(&dk_wown[threadIdx.x >> 5], dk_cap);",
                    f"{ind}  __syncwarp(__activemask());",
                    f"{ind}}}"]
        return [f"{ind}{{",
                f"{ind}  const long long dk_cap = {cap};",
                f"{ind}  if (threadIdx.x == 0) dk_own_init(&dk_bown, dk_cap);",
                f"{ind}  __syncthreads();",
                f"{ind}}}"]

    def emit_insert(self, s, ind):
        d = self.cur.decl
        if d is None:
            raise KdlError("cuda.insert", f"kernel {self.cur.k.name!r}: dp_insert without dp_buffers")
        vals = s.exprs[2:]
        if len(vals) != d.nvars:
            raise KdlError("cuda.insert", f"dp_insert carries {len(vals)} values, dp_buffers declares {d.nvars}")
        out = [f"{ind}{{",
               f"{ind}  const long long dk_w0 = {self.int_ex(s.exprs[0])};",
               f"{ind}  const long long dk_w1 = {self.int_ex(s.exprs[1])};"]
        for j, v in enumerate(vals):
            c = self.ex(v)
            if self.etype(v) == A.FLOAT:
                c = f"dk_flt_word({c})"
            out.append(f"{ind}  const long long dk_w{j + 2} = {c};")
        st = self._stride()
        if d.gran == "grid":
            out.append(f"{ind}  long long* dk_p = dk_reserve_grid(dk_inst, {st}LL, {self._grid_cap()});")
        else:
            out.append(f"{ind}  long long* dk_p = dk_reserve_own({self._own()}, {st}LL);")
        stores = " ".join(f"dk_p[{j}] = dk_w{j};" for j in range(st))
        out += [f"{ind}  if (dk_p) {{ {stores} __threadfence(); }}", f"{ind}}}"]
        return out

    def emit_launch(self, s, ind, tail):
        tgt = self.info[s.name]
        params = tgt.k.params
        args = s.exprs[2:]
        if len(args) != len(params):
            raise KdlError("cuda.launch", f"launch of {s.name!r} passes {len(args)} arguments, kernel takes {len(params)}")
        out = [f"{ind}{{",
               f"{ind}  const long long dk_g = {self.int_ex(s.exprs[0])};",
               f"{ind}  const long long dk_b = {self.int_ex(s.exprs[1])};"]
        names = []
        for j, (a, p) in enumerate(zip(args, params)):
            if p.is_array:
                if a.kind != "name":
                    raise KdlError("cuda.launch", f"array argument {j + 1} of {s.name!r} must be an array name")
                aid, t = self.array_of(a.name)
                if t != p.type:
                    raise KdlError("cuda.type", f"array argument {j + 1} of {s.name!r} has the wrong element type")
                out.append(f"{ind}  const long long dk_a{j} = {aid};")
            else:
                t = self.etype(a)
                if p.type == A.INT and t != A.INT:
                    raise KdlError("cuda.type", f"float argument {j + 1} for int parameter {p.name!r}")
                out.append(f"{ind}  const {_ctype(p.type)} dk_a{j} = {self.ex(a)};")
            names.append(f"dk_a{j}")
        d = self.cur.decl
        if d is None:
            inh = "dk_inh"
        elif d.gran == "grid":
            inh = f"dk_inherit_grid(dk_inst, {self._stride()}LL, {self._grid_cap()})"
        else:
            inh = f"dk_inherit_own({self._own()}, {self._stride()}LL)"
        stream = "cudaStreamTailLaunch" if tail else "cudaStreamFireAndForget"
        call = f"k_{s.name}<<<(unsigned)dk_g, (unsigned)dk_b, 0, {stream}>>>({', '.join(names + ['dk_ci', 'dk_cn'])});"
        out += [f"{ind}  if (dk_launch_ok(dk_g, dk_b)) {{",
                f"{ind}    const dk::Inh dk_ci = {inh};",
                f"{ind}    dk::Inst* dk_cn = {'dk_new_inst(dk_inst)' if tgt.needs_inst else 'nullptr'};"]
        if tgt.needs_inst:
            out.append(f"{ind}    if (dk_cn) {{ {call} dk_launched(cudaGetLastError()); }}")
        else:
            out.append(f"{ind}    {call}")
            out.append(f"{ind}    dk_launched(cudaGetLastError());")
        out += [f"{ind}  }}", f"{ind}}}"]
        return out

    # ---------------- kernels / unit ----------------
    def _sig(self, k):
        ps = [f"{'long long' if p.is_array else _ctype(p.type)} v_{p.name}" for p in k.params]
        return ", ".join(ps + ["dk::Inh dk_inh", "dk::Inst* dk_inst"])

    def _prologue(self, ki, phase0=True):
        out = []
        if ki.uses_grid_last or ki.split:
            out += ["  __shared__ int dk_gl;", "  if (threadIdx.x == 0) dk_gl = -1;"]
        if phase0 and ki.decl is not None and ki.decl.gran == "warp":
            out.append("  __shared__ dk::Own dk_wown[32];")
        if phase0 and ki.decl is not None and ki.decl.gran == "block":
            out.append("  __shared__ dk::Own dk_bown;")
        return out

    def emit_kernel(self, ki):
        self.cur = ki
        k = ki.k
        if ki.split:
            return self.emit_split_kernel(ki)
        self.env = [{p.name: ("array" if p.is_array else p.type, p.is_array) for p in k.params}]
        out = [f"__global__ void k_{k.name}({self._sig(k)}) {{"] + self._prologue(ki)
        out += self.emit_body(k.body, "  ")
        out.append("}")
        return out

    @staticmethod
    def phase_name(k, j):
        return k.name if j == 0 else f"{k.name}__c{j}"

    def emit_split_kernel(self, ki):
        """Top-level sync_device on CDP2 (no device-side join): the kernel is
        split at each top-level sync into phases.  Phase j saves its live
        scalars (parameters + top-level locals) and an alive flag per thread,
        and the last block to finish (dp_grid_last protocol) tail-launches
        phase j+1 with the same geometry: a tail launch runs after the whole
        grid and everything it launched, i.e. after every child the sync
        waited for.  Threads that returned in phase j stay dead."""
        k = ki.k
        live = [(p.name, "array" if p.is_array else p.type, p.is_array) for p in k.params]
        out = []
        for j, ph in enumerate(ki.phases):
            last = j == len(ki.phases) - 1
            if j > 0:
                for s in A.walk_stmts(ph):
                    if s.kind in ("insert", "buf_decl") or any(
                            n.kind == "buf_pending" for e in s.exprs for n in A.walk_expr(e)):
                        raise KdlError("cuda.sync", f"kernel {k.name!r}: consolidation buffers cannot be used "
                                       "after sync_device (owner state does not survive the split)")
            sig = self._sig(k) if j == 0 else "const long long* dk_state, dk::Inh dk_inh, dk::Inst* dk_inst"
            out.append(f"__global__ void k_{self.phase_name(k, j)}({sig}) {{")
            out += self._prologue(ki, j == 0)
            scope = {}
            if j == 0:
                scope = {p.name: ("array" if p.is_array else p.type, p.is_array) for p in k.params}
            else:
                W = 1 + len(live)
                out += [f"  const long long* dk_sl = dk_state + ((long long)blockIdx.x * blockDim.x + threadIdx.x) * {W}LL;",
                        "  if (dk_sl[0] == 0) return;"]
                for i, (n, t, arr) in enumerate(live):
                    w = f"dk_sl[{1 + i}]"
                    out.append(f"  {_ctype(t) if t != 'array' else 'long long'} v_{n} = "
                               f"{'dk_word_flt(' + w + ')' if t == A.FLOAT else '(' + (_ctype(t) if t != 'array' else 'long long') + ')' + w};")
                    scope[n] = (t, arr)
            self.env = [scope, {}]
            new = []
            for s in ph:
                if s.kind == "let" and s.name not in scope and s.name not in [x[0] for x in new]:
                    new.append((s.name, s.scalar, False))
            for n, t, _ in new:
                out.append(f"  {_ctype(t)} v_{n} = 0;")
            self.hoist = True
            self.ret_label = None if last else f"dk_split{j}"
            if not last:
                out.append("  long long dk_alive = 1;")
            for s in ph:
                out += self.emit(s, "  ")
            self.hoist = False
            self.ret_label = None
            if not last:
                live = live + new
                W = 1 + len(live)
                saves = " ".join(f"dk_so[{1 + i}] = {'dk_flt_word(v_' + n + ')' if t == A.FLOAT else '(long long)v_' + n};"
                                 for i, (n, t, _) in enumerate(live))
                nxt = self.phase_name(k, j + 1)
                out += [f"dk_split{j}:",
                        "  __syncthreads();",
                        "  {",
                        "    __shared__ long long* dk_stb;",
                        f"    if (threadIdx.x == 0) dk_stb = dk_state_base(dk_inst, (long long)gridDim.x * blockDim.x * {W}LL);",
                        "    __syncthreads();",
                        "    if (dk_stb) {",
                        f"      long long* dk_so = dk_stb + ((long long)blockIdx.x * blockDim.x + threadIdx.x) * {W}LL;",
                        f"      dk_so[0] = dk_alive; {saves}",
                        "    }",
                        "    if (dk_grid_last(dk_inst, &dk_gl) != 0 && threadIdx.x == 0 && dk_stb) {",
                        "      dk::Inst* dk_cn = dk_new_inst(dk_inst);",
                        f"      if (dk_cn) {{ k_{nxt}<<<gridDim.x, blockDim.x, 0, cudaStreamTailLaunch>>>(dk_stb, dk_inh, dk_cn); "
                        "dk_launched(cudaGetLastError()); }",
                        "    }",
                        "  }"]
            out += ["}", ""]
        return out

    def generate(self):
        lines = [f"// Generated by paper_1606_08150_b200.kdl from program {self.name!r}; do not edit.",
                 f"#define DK_WIDTH {self.width}", '#include "kdl_rt.cuh"', ""]
        for g in self.prog.globals:
            i, t = self.arr[g.name]
            lines.append(f"// array {i}: {t} {g.name}")
        lines.append("")
        for ki in self.info.values():
            lines.append(f"__global__ void k_{ki.k.name}({self._sig(ki.k)});")
            for j in range(1, len(ki.phases)):
                lines.append(f"__global__ void k_{self.phase_name(ki.k, j)}(const long long* dk_state, "
                             "dk::Inh dk_inh, dk::Inst* dk_inst);")
        body = []
        for ki in self.info.values():
            body += self.emit_kernel(ki) + [""]
        nkc = max(1, len(self.kc))
        lines += ["", f"__device__ long long dk_kc[{nkc}];", ""] + body
        lines += self.host_part()
        return "\n".join(lines) + "\n"

    def host_part(self):
        e = self.prog.entry
        ek = self.info[e.kernel].k
        unpack = []
        for j, p in enumerate(ek.params):
            if p.type == A.FLOAT and not p.is_array:
                unpack.append(f"(dk_flt)dk_bits(a[{j}])")
            elif p.is_array:
                unpack.append(f"a[{j}]")
            else:
                unpack.append(f"(dk_int)a[{j}]")
        kc_rows = ", ".join(f"{{(const void*)k_{k}, {x}, {t}}}" for (k, x, t) in self.kc) or "{nullptr, 1, 1}"
        nkc = len(self.kc)
        return [
            "static thread_local char dk_msg[256];",
            "static long long dk_kc_host[%d];" % max(1, nkc),
            "struct DkKc { const void* fn; int x; int t; };",
            f"static const DkKc dk_kc_rows[{max(1, nkc)}] = {{{kc_rows}}};",
            "static int dk_fail(cudaError_t e) { snprintf(dk_msg, sizeof dk_msg, \"%s\", cudaGetErrorString(e)); return 1; }",
            "static double dk_bits(long long v) { double d; memcpy(&d, &v, 8); return d; }",
            'extern "C" const char* dk_error() { return dk_msg; }',
            'extern "C" int dk_sizeof_rt() { return (int)sizeof(dk::Rt); }',
            f'extern "C" int dk_kc_count() {{ return {nkc}; }}',
            'extern "C" int dk_kc_values(long long* out) {',
            f"  for (int i = 0; i < {nkc}; i++) out[i] = dk_kc_host[i];",
            "  return 0;",
            "}",
            'extern "C" int dk_init(int device, long long pending) {',
            "  cudaError_t e = cudaSetDevice(device);",
            "  if (e != cudaSuccess) return dk_fail(e);",
            "  if (pending > 0) {",
            "    e = cudaDeviceSetLimit(cudaLimitDevRuntimePendingLaunchCount, (size_t)pending);",
            "    if (e != cudaSuccess) return dk_fail(e);",
            "  }",
            "  int sms = 0;",
            "  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);",
            "  if (e != cudaSuccess) return dk_fail(e);",
            f"  for (int i = 0; i < {nkc}; i++) {{",
            "    int bps = 0;",
            "    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, dk_kc_rows[i].fn, dk_kc_rows[i].t, 0);",
            "    if (e != cudaSuccess) return dk_fail(e);",
            "    long long b = (long long)bps * sms / dk_kc_rows[i].x;",
            "    dk_kc_host[i] = b < 1 ? 1 : b;",
            "  }",
            f"  if ({nkc} > 0) {{",
            f"    e = cudaMemcpyToSymbol(dk_kc, dk_kc_host, sizeof(long long) * {max(1, nkc)});",
            "    if (e != cudaSuccess) return dk_fail(e);",
            "  }",
            "  return 0;",
            "}",
            'extern "C" int dk_set_rt(const void* rt) {',
            "  cudaError_t e = cudaMemcpyToSymbol(dk_rt, rt, sizeof(dk::Rt));",
            "  return e == cudaSuccess ? 0 : dk_fail(e);",
            "}",
            'extern "C" int dk_launch_entry(long long g, long long b, const long long* a, void* inst0, void* stream) {',
            "  (void)a;",
            "  if (g < 1 || g > 0x7fffffffLL || b < 1 || b > 1024) { snprintf(dk_msg, sizeof dk_msg, \"entry launch extents\"); return 2; }",
            f"  k_{ek.name}<<<(unsigned)g, (unsigned)b, 0, (cudaStream_t)stream>>>("
            + ", ".join(unpack + ["dk::Inh{nullptr, nullptr, 0, 0, 0}", "(dk::Inst*)inst0"]) + ");",
            "  cudaError_t e = cudaGetLastError();",
            "  return e == cudaSuccess ? 0 : dk_fail(e);",
            "}",
        ]


def generate(prog, name="kdl", width=64):
    """-> (CUDA source, list of (kernel, X, T) KC launch rows)."""
    b = Builder(prog, name, width)
    src = b.generate()
    return src, list(b.kc)
