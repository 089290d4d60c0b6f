"""AST of the kernel DSL (.kdl) accepted by the B200 consolidation compiler.

The node set is the reference DSL's (ast.hpp:17-34 expression kinds,
ast.hpp:52-66 statement kinds, ast.hpp:92-114 directive clauses), restated
as plain Python dataclasses so the front end, the consolidation rewrite and
the CUDA builder can share it.  Nodes compare structurally, which the parity
tests use to check this compiler's rewrite against the reference's
consolidate() output (transform.hpp:971).

Expression kinds: int, float, name, index, unary, binary, intrinsic, minmax,
atomic, buf_count, buf_pending, buf_get, buf_cfg_grid, buf_cfg_block,
grid_last, and kc_blocks (B200 extension: the KC_X block count of a
consolidated launch, resolved from the real occupancy at module load).
Statement kinds: let, assign, store, atomic, if, for, barrier, sync, launch,
return, buf_decl, insert, grid_barrier.
"""
from dataclasses import dataclass, field
from typing import List, Optional

INT, FLOAT = "int", "float"
INTRINSICS = ("threadIdx", "blockIdx", "blockDim", "gridDim")


@dataclass(eq=True)
class Expr:
    kind: str
    ival: int = 0
    fval: float = 0.0
    name: str = ""
    args: List["Expr"] = field(default_factory=list)


@dataclass(eq=True)
class Directive:
    granularity: str = "warp"          # warp | block | grid
    buffer: str = "custom"             # default | halloc | custom
    per_buffer_lit: Optional[int] = None
    per_buffer_var: Optional[str] = None
    total_bytes: int = 500 * 1024 * 1024
    work: List[str] = field(default_factory=list)
    threads: Optional[int] = None
    blocks: Optional[int] = None


@dataclass(eq=True)
class Stmt:
    kind: str
    name: str = ""
    scalar: str = INT                  # let type
    exprs: List[Expr] = field(default_factory=list)
    body: List["Stmt"] = field(default_factory=list)
    else_body: List["Stmt"] = field(default_factory=list)
    directive: Optional[Directive] = None
    gran: str = "warp"                 # buf_decl
    alloc: str = "prealloc"            # buf_decl: default | halloc | prealloc
    nvars: int = 0                     # buf_decl
    total_bytes: int = 0               # buf_decl


@dataclass(eq=True)
class Param:
    name: str
    type: str = INT
    is_array: bool = False


@dataclass(eq=True)
class Kernel:
    name: str
    params: List[Param] = field(default_factory=list)
    body: List[Stmt] = field(default_factory=list)


@dataclass(eq=True)
class Global:
    name: str
    type: str
    length: Expr


@dataclass(eq=True)
class Entry:
    kernel: str
    grid: Expr
    block: Expr
    args: List[Expr] = field(default_factory=list)


@dataclass(eq=True)
class Program:
    globals: List[Global] = field(default_factory=list)
    kernels: List[Kernel] = field(default_factory=list)
    entry: Optional[Entry] = None

    def kernel(self, name):
        for k in self.kernels:
            if k.name == name:
                return k
        return None

    def global_(self, name):
        for g in self.globals:
            if g.name == name:
                return g
        return None


# ---- constructors used by the rewrite ----

def lit(v):
    return Expr("int", ival=int(v))


def ref(n):
    return Expr("name", name=n)


def intr(n):
    return Expr("intrinsic", name=n)


def binop(op, a, b):
    return Expr("binary", name=op, args=[a, b])


def call0(kind):
    return Expr(kind)


def let(t, n, e):
    return Stmt("let", name=n, scalar=t, exprs=[e])


def if_(c, body, else_body=None):
    return Stmt("if", exprs=[c], body=list(body), else_body=list(else_body or []))


def for_(v, a, b, c, body):
    return Stmt("for", name=v, exprs=[a, b, c], body=list(body))


def launch(k, g, b, args, directive=None):
    return Stmt("launch", name=k, exprs=[g, b] + list(args), directive=directive)


def bare(kind):
    return Stmt(kind)


def walk_stmts(body):
    """Pre-order over every statement of a body, nested ones included."""
    for s in body:
        yield s
        yield from walk_stmts(s.body)
        yield from walk_stmts(s.else_body)


def walk_expr(e):
    yield e
    for a in e.args:
        yield from walk_expr(a)
