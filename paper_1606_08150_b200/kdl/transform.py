"""Workload-consolidation rewrite of a .kdl program (the paper's directive
compiler), restating the reference's consolidate()
(transform.hpp:971) on this package's AST:

* the annotated launch becomes `dp_insert(grid, block, work...)` into a
  warp / block / grid buffer declared by `dp_buffers(...)` at the top of the
  parent (transform.hpp:588-610, 455-480);
* the child becomes `<child>_cons`, a drain loop over the inherited buffer
  whose per-item body is the original child with its launch geometry
  rebound: solo-thread, solo-block or multi-block (moldable or through a
  virtual-thread loop), classified as in transform.hpp:196-217 and drained as
  in transform.hpp:484-566;
* a selected thread per warp / block / grid launches the consolidated child
  (transform.hpp:570-600); at grid level the last block to finish (the
  counter/exit protocol, `dp_grid_last()`) launches it, and postwork moves
  into `<parent>_post` with the prework it needs re-run per virtual thread
  (transform.hpp:805-867);
* a self-recursive site becomes `<k>_cons` (pop + re-insert + relaunch
  itself) plus a `<k>_boot` kernel that seeds the entry item
  (transform.hpp:870-964).

Diagnostics carry the reference's codes (tf.target, tf.chain, tf.workarray,
val.workarg, tf.nonmoldable, tf.arg, tf.childreturn, tf.postdep, tf.recsync,
tf.multiparent, tf.dangling).

B200 difference: the KC_X block count of a consolidated launch is emitted as
a `kc_blocks` node (consolidated kernel, X, T) that the CUDA builder resolves
from the compiled kernel's real occupancy on the device; `lower_kc()` turns
it into the literal the reference would print for a given device model so the
two rewrites can be compared node for node.
"""
import copy

from . import ast as A
from .parse import KdlError

DEFAULT_SIZE_CONST = 4      # memplan.hpp:18, work items per thread estimate
WARP = 32


def default_concurrency(gran):
    """KC_X default per granularity (config.hpp:79-86)."""
    return {"grid": 1, "block": 16, "warp": 32}[gran]


class Config:
    """How consolidated launches are sized (config.hpp:89-125): scheme is
    'kc' (KC_X with X = default_concurrency or `x`), 'one_to_one', or
    'explicit' (blocks, threads)."""

    def __init__(self, scheme="kc", x=None, blocks=None, threads=None):
        self.scheme, self.x, self.blocks, self.threads = scheme, x, blocks, threads


def _is_one(e):
    return e.kind == "int" and e.ival == 1


def _is_canonical_gts(e):
    """`blockIdx * blockDim + threadIdx` or `gridDim * blockDim` (transform.hpp:44-63)."""
    if e.kind != "binary":
        return False
    if e.name == "+":
        l, r = e.args
        return (l.kind == "binary" and l.name == "*" and l.args[0] == A.intr("blockIdx")
                and l.args[1] == A.intr("blockDim") and r == A.intr("threadIdx"))
    if e.name == "*":
        return e.args[0] == A.intr("gridDim") and e.args[1] == A.intr("blockDim")
    return False


def _only_canonical_dims(e):
    if _is_canonical_gts(e):
        return True
    if e.kind == "intrinsic" and e.name in ("gridDim", "blockDim"):
        return False
    return all(_only_canonical_dims(a) for a in e.args)


def _body_canonical(body):
    return all(all(_only_canonical_dims(e) for e in s.exprs) for s in A.walk_stmts(body))


def classify_child(site, child):
    """-> (shape, moldable) with shape in solo_thread | solo_block | multi_block."""
    g, b = site.exprs[0], site.exprs[1]
    if _is_one(g) and _is_one(b):
        return "solo_thread", True
    if _is_one(g):
        return "solo_block", True
    return "multi_block", _body_canonical(child.body)


def subst(x, table):
    """Replace intrinsic nodes by the expressions in `table` (deep copy)."""
    if isinstance(x, list):
        return [subst(s, table) for s in x]
    if isinstance(x, A.Stmt):
        s = copy.copy(x)
        s.exprs = [subst(e, table) for e in x.exprs]
        s.body = subst(x.body, table)
        s.else_body = subst(x.else_body, table)
        return s
    if x.kind == "intrinsic" and x.name in table:
        return copy.deepcopy(table[x.name])
    e = copy.copy(x)
    e.args = [subst(a, table) for a in x.args]
    return e


def find_site(body):
    for s in A.walk_stmts(body):
        if s.kind == "launch" and s.directive is not None:
            return s
    return None


def _replace_site(body, repl):
    for i, s in enumerate(body):
        if s.kind == "launch" and s.directive is not None:
            body[i:i + 1] = repl
            return True
        if _replace_site(s.body, repl) or _replace_site(s.else_body, repl):
            return True
    return False


def _contains(body, kind):
    return any(s.kind == kind for s in A.walk_stmts(body))


class _RW:
    def __init__(self):
        self.sr, self.sw, self.ar, self.aw = set(), set(), set(), set()


def _expr_names(e, rw):
    for n in A.walk_expr(e):
        if n.kind == "name":
            rw.sr.add(n.name)
        if n.kind in ("index", "atomic"):
            rw.ar.add(n.name)


def _stmt_rw(s, rw):
    """Name-level read / write sets of one statement (transform.hpp:148-193)."""
    for e in s.exprs:
        _expr_names(e, rw)
    if s.kind in ("let", "assign", "for"):
        rw.sw.add(s.name)
    if s.kind in ("store", "atomic"):
        rw.aw.add(s.name)
        rw.ar.add(s.name)
    for t in s.body + s.else_body:
        _stmt_rw(t, rw)


def _body_rw(body):
    rw = _RW()
    for s in body:
        _stmt_rw(s, rw)
    return rw


class _Site:
    pass


class _Consolidator:
    def __init__(self, prog, gran_override, config, default_threads, schedule="reference"):
        if schedule not in ("reference", "block"):
            raise ValueError("schedule must be 'reference' or 'block'")
        self.schedule = schedule
        self.prog = prog
        self.gran_override = gran_override
        self.config = config or Config()
        self.default_threads = default_threads

    def run(self):
        annotated = [k for k in self.prog.kernels if find_site(k.body)]
        out = copy.deepcopy(self.prog)
        if not annotated:
            return out
        done = set()
        for parent in annotated:
            p = self.plan(parent)
            if p.child in done:
                raise KdlError("tf.multiparent", f"kernel {p.child!r} is consolidated from more than one site")
            done.add(p.child)
            self.apply(out, p)
        for k in out.kernels:
            for s in A.walk_stmts(k.body):
                if s.kind == "launch" and out.kernel(s.name) is None:
                    raise KdlError("tf.dangling", f"launch targets consolidated-away kernel {s.name!r}")
        return out

    # -- planning (transform.hpp:320-383) --
    def plan(self, parent):
        site = find_site(parent.body)
        p = _Site()
        p.parent, p.child, p.dir = parent.name, site.name, site.directive
        p.gran = self.gran_override or p.dir.granularity
        p.launch = copy.deepcopy(site)
        p.recursive = site.name == parent.name
        child = self.prog.kernel(site.name)
        if child is None:
            raise KdlError("tf.target", f"annotated launch targets unknown kernel {site.name!r}")
        if not p.recursive and find_site(child.body):
            raise KdlError("tf.chain", f"kernel {p.child!r} is both a consolidation target and an "
                           "annotated parent; chained consolidation is unsupported")
        p.shape, p.moldable = classify_child(site, child)
        p.work = []   # (name, type, param index, slot)
        for slot, w in enumerate(p.dir.work):
            for i, a in enumerate(site.exprs[2:]):
                if a.kind == "name" and a.name == w:
                    prm = child.params[i]
                    if prm.is_array:
                        raise KdlError("tf.workarray", f"work variable {w!r} binds an array parameter; "
                                       "only scalar indices can be buffered")
                    p.work.append((prm.name, prm.type, i, slot))
                    break
            else:
                raise KdlError("val.workarg", f"work variable {w!r} must be passed as a launch argument")
        if p.shape == "multi_block" and not p.moldable:
            if p.dir.threads or p.dir.blocks or self.config.scheme in ("explicit", "one_to_one"):
                raise KdlError("tf.nonmoldable", "non-moldable child cannot be reconfigured")
        return p

    @staticmethod
    def is_work(p, i):
        return any(w[2] == i for w in p.work)

    def uniform(self, parent, e):
        if e.kind in ("int", "float"):
            return True
        if e.kind == "name":
            return any(q.name == e.name for q in parent.params) or self.prog.global_(e.name) is not None
        return False

    # -- launch geometry (transform.hpp:385-452) --
    def resolve(self, p, cons):
        c = self.config
        T = self.default_threads
        if c.scheme == "explicit":
            T = c.threads
        if p.dir.threads:
            T = p.dir.threads
        pending = A.call0("buf_pending")
        if c.scheme == "one_to_one" and not p.dir.blocks:
            clamped = A.Expr("minmax", name="max", args=[pending, A.lit(1)])
            if p.shape == "solo_thread":
                blk = A.Expr("minmax", name="min", args=[copy.deepcopy(clamped), A.lit(T)])
                grid = A.binop("/", A.binop("+", copy.deepcopy(clamped), A.lit(T - 1)), A.lit(T))
                return grid, blk
            return clamped, A.lit(T)
        if p.dir.blocks:
            return A.lit(p.dir.blocks), A.lit(T)
        if c.scheme == "explicit":
            return A.lit(c.blocks), A.lit(T)
        x = c.x if c.scheme == "kc" and c.x else default_concurrency(p.gran)
        return A.Expr("kc_blocks", name=cons, ival=x, args=[A.lit(T)]), A.lit(T)

    def per_buffer(self, p):
        nv = len(p.dir.work)
        if p.gran == "grid":
            return A.lit(0)
        if p.dir.per_buffer_lit:
            return A.lit(p.dir.per_buffer_lit)
        if p.dir.per_buffer_var:
            return A.ref(p.dir.per_buffer_var)
        if p.gran == "warp":
            return A.lit(WARP * nv * DEFAULT_SIZE_CONST)
        return A.binop("*", A.intr("blockDim"), A.lit(nv * DEFAULT_SIZE_CONST))

    def buf_decl(self, p):
        alloc = {"default": "default", "halloc": "halloc", "custom": "prealloc"}[p.dir.buffer]
        return A.Stmt("buf_decl", gran=p.gran, alloc=alloc, nvars=len(p.dir.work),
                      total_bytes=p.dir.total_bytes, exprs=[self.per_buffer(p)])

    @staticmethod
    def insert(p):
        return A.Stmt("insert", exprs=[copy.deepcopy(p.launch.exprs[0]), copy.deepcopy(p.launch.exprs[1])]
                      + [A.ref(w) for w in p.dir.work])

    # -- drain loop (transform.hpp:484-566) --
    def drain(self, p, body):
        out = [A.let(A.INT, "__n", A.call0("buf_count"))]
        item = [A.let(t, n, A.Expr("buf_get", args=[A.ref("__i"), A.lit(slot)])) for (n, t, _, slot) in p.work]
        gts = A.binop("+", A.binop("*", A.intr("blockIdx"), A.intr("blockDim")), A.intr("threadIdx"))
        stride = A.binop("*", A.intr("gridDim"), A.intr("blockDim"))
        if p.shape == "solo_thread":
            item += subst(body, {"threadIdx": A.lit(0), "blockIdx": A.lit(0),
                                 "blockDim": A.lit(1), "gridDim": A.lit(1)})
            out.append(A.for_("__i", gts, A.ref("__n"), stride, item))
        elif p.shape == "solo_block":
            item.append(A.let(A.INT, "__ob", A.Expr("buf_cfg_block", args=[A.ref("__i")])))
            item.append(A.for_("__vt", A.intr("threadIdx"), A.ref("__ob"), A.intr("blockDim"),
                               subst(body, {"threadIdx": A.ref("__vt"), "blockIdx": A.lit(0),
                                            "blockDim": A.ref("__ob"), "gridDim": A.lit(1)})))
            out.append(A.for_("__i", A.intr("blockIdx"), A.ref("__n"), A.intr("gridDim"), item))
        elif self.schedule == "block":
            # B200 schedule: one item per block; the block walks the item's
            # virtual blocks in turn and strides each one's virtual threads.
            # Rebinding the four intrinsics to the item's own geometry is
            # valid for every multi-block child (moldable or not); it removes
            # the reference form's O(#items) loop that every thread of the
            # grid runs, and the 2-D loop needs no per-thread division.
            item.append(A.let(A.INT, "__og", A.Expr("buf_cfg_grid", args=[A.ref("__i")])))
            item.append(A.let(A.INT, "__ob", A.Expr("buf_cfg_block", args=[A.ref("__i")])))
            tbl = {"threadIdx": A.ref("__vt"), "blockIdx": A.ref("__vb"),
                   "blockDim": A.ref("__ob"), "gridDim": A.ref("__og")}
            inner = A.for_("__vt", A.intr("threadIdx"), A.ref("__ob"), A.intr("blockDim"), subst(body, tbl))
            item.append(A.for_("__vb", A.lit(0), A.ref("__og"), A.lit(1), [inner]))
            out.append(A.for_("__i", A.intr("blockIdx"), A.ref("__n"), A.intr("gridDim"), item))
        else:
            if p.moldable:
                item += copy.deepcopy(body)
            else:
                item.append(A.let(A.INT, "__og", A.Expr("buf_cfg_grid", args=[A.ref("__i")])))
                item.append(A.let(A.INT, "__ob", A.Expr("buf_cfg_block", args=[A.ref("__i")])))
                tbl = {"threadIdx": A.binop("%", A.ref("__vt"), A.ref("__ob")),
                       "blockIdx": A.binop("/", A.ref("__vt"), A.ref("__ob")),
                       "blockDim": A.ref("__ob"), "gridDim": A.ref("__og")}
                item.append(A.for_("__vt", gts, A.binop("*", A.ref("__og"), A.ref("__ob")), stride,
                                   subst(body, tbl)))
            out.append(A.for_("__i", A.lit(0), A.ref("__n"), A.lit(1), item))
        return out

    @staticmethod
    def tail(p, target, args, grid, block, guard):
        """The selected thread launches the consolidated kernel (transform.hpp:570-600)."""
        ln = A.launch(target, copy.deepcopy(grid), copy.deepcopy(block), copy.deepcopy(args))
        if p.gran == "warp":
            sel = A.if_(A.binop("==", A.binop("%", A.intr("threadIdx"), A.lit(WARP)), A.lit(0)), [ln])
        else:
            sel = A.if_(A.binop("==", A.intr("threadIdx"), A.lit(0)), [ln])
        if not guard:
            return [sel]
        return [A.if_(A.binop(">", A.call0("buf_pending"), A.lit(0)), [sel])]

    # -- application --
    def apply(self, out, p):
        if p.recursive:
            return self.apply_recursive(out, p)
        child = out.kernel(p.child)
        if _contains(child.body, "return"):
            raise KdlError("tf.childreturn", f"child kernel {child.name!r} uses return; the drain loop "
                           "cannot keep its early-exit semantics")
        cons = A.Kernel(child.name + "_cons",
                        [q for i, q in enumerate(child.params) if not self.is_work(p, i)],
                        self.drain(p, child.body))
        post = self.rewrite_parent(p, out.kernel(p.parent), cons.name)
        out.kernels[out.kernels.index(child)] = cons
        if post is not None:
            out.kernels.append(post)

    def rewrite_parent(self, p, parent, cons):
        site = next(i for i, s in enumerate(parent.body) if find_site([s]))
        orig_sync = site + 1 < len(parent.body) and parent.body[site + 1].kind == "sync"
        post_i = site + 2 if orig_sync else site + 1
        prework = parent.body[:site]
        site_stmt = [copy.deepcopy(parent.body[site])]
        postwork = parent.body[post_i:]
        args = []
        for i, a in enumerate(p.launch.exprs[2:]):
            if self.is_work(p, i):
                continue
            if not self.uniform(parent, a):
                raise KdlError("tf.arg", f"launch argument {i + 1} is not uniform across consolidated items "
                               "(must be a literal, parameter or array name)")
            args.append(a)
        grid, block = self.resolve(p, cons)
        post_kernel = None
        body = [self.buf_decl(p)] + prework
        _replace_site(site_stmt, [self.insert(p)])
        body += site_stmt
        if p.gran == "warp":
            body += self.tail(p, cons, args, grid, block, True)
            if orig_sync:
                body.append(A.bare("sync"))
            body += postwork
        elif p.gran == "block":
            body.append(A.bare("barrier"))
            body += self.tail(p, cons, args, grid, block, True)
            if orig_sync:
                body.append(A.bare("sync"))
            elif postwork:
                body.append(A.bare("barrier"))
            body += postwork
        else:
            if postwork:
                post_kernel = self.postwork_kernel(p, parent, prework, site_stmt, postwork)
            body.append(A.bare("barrier"))
            body.append(A.if_(A.binop("==", A.call0("grid_last"), A.lit(0)), [A.bare("return")]))
            last = [A.launch(cons, copy.deepcopy(grid), copy.deepcopy(block), copy.deepcopy(args))]
            if postwork:
                last.append(A.bare("sync"))
                pargs = [A.ref(q.name) for q in parent.params] + [A.intr("gridDim"), A.intr("blockDim")]
                last.append(A.launch(parent.name + "_post", copy.deepcopy(grid), copy.deepcopy(block), pargs))
            body.append(A.if_(A.binop("==", A.intr("threadIdx"), A.lit(0)), last))
        parent.body = body
        return post_kernel

    def postwork_kernel(self, p, parent, prework, site_stmt, postwork):
        """Grid-level postwork extraction (transform.hpp:805-867)."""
        post_rw, pre_rw, site_rw = _body_rw(postwork), _body_rw(prework), _body_rw(site_stmt)
        pre_reads = pre_rw.ar | site_rw.ar
        for a in sorted(post_rw.aw):
            if a in pre_reads:
                raise KdlError("tf.postdep", f"irreducible prework/postwork dependence: postwork writes {a!r} "
                               "which the prework phase reads")
        params = {q.name for q in parent.params}
        needed = {n for n in post_rw.sr if n not in params}
        keep = [False] * len(prework)
        for i in range(len(prework) - 1, -1, -1):
            rw = _RW()
            _stmt_rw(prework[i], rw)
            if not (rw.sw & needed):
                continue
            keep[i] = True
            needed |= {n for n in rw.sr if n not in params}
        dup = [copy.deepcopy(s) for s, k in zip(prework, keep) if k] + copy.deepcopy(postwork)
        tbl = {"threadIdx": A.binop("%", A.ref("__v"), A.ref("__ob")),
               "blockIdx": A.binop("/", A.ref("__v"), A.ref("__ob")),
               "blockDim": A.ref("__ob"), "gridDim": A.ref("__og")}
        gts = A.binop("+", A.binop("*", A.intr("blockIdx"), A.intr("blockDim")), A.intr("threadIdx"))
        body = [A.for_("__v", gts, A.binop("*", A.ref("__og"), A.ref("__ob")),
                       A.binop("*", A.intr("gridDim"), A.intr("blockDim")), subst(dup, tbl))]
        return A.Kernel(parent.name + "_post",
                        copy.deepcopy(parent.params) + [A.Param("__og"), A.Param("__ob")], body)

    def apply_recursive(self, out, p):
        parent = copy.deepcopy(out.kernel(p.parent))
        if _contains(parent.body, "sync"):
            raise KdlError("tf.recsync", "device synchronization inside a recursive consolidation target "
                           "is unsupported")
        if _contains(parent.body, "return"):
            raise KdlError("tf.childreturn", f"kernel {parent.name!r} uses return; the drain loop cannot keep "
                           "its early-exit semantics")
        cons = parent.name + "_cons"
        inner = copy.deepcopy(parent.body)
        _replace_site(inner, [self.insert(p)])
        grid, block = self.resolve(p, cons)
        self_args = [A.ref(q.name) for i, q in enumerate(parent.params) if not self.is_work(p, i)]
        ck = A.Kernel(cons, [copy.deepcopy(q) for i, q in enumerate(parent.params) if not self.is_work(p, i)])
        ck.body = [self.buf_decl(p)] + self.drain(p, inner) + self.recursive_tail(p, cons, self_args, grid, block)
        boot = A.Kernel(parent.name + "_boot", copy.deepcopy(parent.params) + [A.Param("__og"), A.Param("__ob")])
        boot.body = [self.buf_decl(p),
                     A.Stmt("insert", exprs=[A.ref("__og"), A.ref("__ob")] + [A.ref(w[0]) for w in p.work])]
        boot.body += self.recursive_tail(p, cons, self_args, grid, block)
        if out.entry.kernel == parent.name:
            e = out.entry
            e.kernel = boot.name
            e.args = e.args + [e.grid, e.block]
            e.grid, e.block = A.lit(1), A.lit(1)
        i = [k.name for k in out.kernels].index(p.parent)
        out.kernels[i] = ck
        out.kernels.append(boot)

    def recursive_tail(self, p, cons, args, grid, block):
        if p.gran == "warp":
            return self.tail(p, cons, args, grid, block, True)
        body = [A.bare("barrier")]
        if p.gran == "grid":
            body.append(A.if_(A.binop("==", A.call0("grid_last"), A.lit(0)), [A.bare("return")]))
        return body + self.tail(p, cons, args, grid, block, True)


def consolidate(prog, granularity=None, config=None, default_threads=256, schedule="reference"):
    """Rewrite every annotated site of `prog` (ast.Program, not modified).
    `granularity` overrides the directives' consltdt clause (the reference's
    TransformOptions.granularityOverride, transform.hpp:219-225).
    `schedule` picks the multi-block drain: "reference" (transform.hpp:
    538-566: the whole grid walks every item) or "block" (one item per
    block; the B200 default of kdl.compile)."""
    if granularity not in (None, "warp", "block", "grid"):
        raise ValueError(f"granularity must be warp, block or grid, not {granularity!r}")
    return _Consolidator(prog, granularity, config, default_threads, schedule).run()


def kc_blocks(occupancy_blocks, x):
    """KC_X block count: max(1, B_occ / X) (config.hpp:63-72)."""
    return max(1, occupancy_blocks // max(1, x))


def lower_kc(prog, occupancy_blocks):
    """Replace every kc_blocks node by its literal for a device model:
    `occupancy_blocks(T)` -> resident blocks of T threads on the whole device."""
    out = copy.deepcopy(prog)

    def fix(e):
        if e.kind == "kc_blocks":
            T = e.args[0].ival
            return A.lit(kc_blocks(occupancy_blocks(T), e.ival))
        e.args = [fix(a) for a in e.args]
        return e

    for k in out.kernels:
        for s in A.walk_stmts(k.body):
            s.exprs = [fix(e) for e in s.exprs]
    return out


def k20c_occupancy(T, sms=13, max_blocks=16, max_warps=64):
    """Resident blocks of T threads on the reference's default device model
    (device.hpp: 13 SMs, 16 blocks / 64 warps per SM, no register or shared
    memory stubs), for comparing against the reference's printed literals."""
    return sms * min(max_blocks, max_warps // ((T + WARP - 1) // WARP))
