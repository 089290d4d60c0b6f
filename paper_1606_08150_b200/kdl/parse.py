"""Front end of the B200 consolidation compiler: .kdl text -> ast.Program.

Accepts the reference DSL (SPEC.md's grammar as implemented by lexer.hpp
and parser.hpp): `global T name[len];`, `kernel name(params) { ... }`,
`entry k<<<g, b>>>(args);`, statements let / assign / store / atomicAdd /
if-else / for (`for (int v = a; v < b; v += c)`) / barrier_block /
sync_device / return / launches with an optional preceding
`#pragma dp consltdt(...) buffer(...) work(...) threads(...) blocks(...)`
(parser.hpp:638-779), and the consolidated-program builtins the rewrite
emits (dp_buffers, dp_insert, dp_buf_count / pending / get / cfg_grid /
cfg_block, dp_grid_last, dp_grid_barrier; parser.hpp:250-280, 553-581) —
so the CUDA builder can take either this compiler's rewrite or the
reference's own consolidate() text as input.  Operator precedence follows
parser.hpp:413-495 (|| < && < == != < relational < + - < * / % < unary).
"""
import re

from . import ast as A


class KdlError(Exception):
    def __init__(self, code, msg, line=0):
        super().__init__(f"{code}: {msg}" + (f" (line {line})" if line else ""))
        self.code = code
        self.line = line


_TOK = re.compile(r"""
    (?P<ws>[ \t\r\n]+|//[^\n]*)
  | (?P<pragma>\#[^\n]*)
  | (?P<num>\d+(\.\d*)?([eE][+-]?\d+)?)
  | (?P<id>[A-Za-z_][A-Za-z_0-9]*)
  | (?P<sym><<<|>>>|<=|>=|==|!=|&&|\|\||\+=|[(){}\[\],;=+\-*/%<>!])
""", re.X)


def tokenize(src):
    out, pos, line = [], 0, 1
    while pos < len(src):
        m = _TOK.match(src, pos)
        if not m:
            raise KdlError("lex.char", f"unexpected character {src[pos]!r}", line)
        kind = m.lastgroup
        text = m.group(kind)
        if kind == "num":
            isf = ("." in text) or ("e" in text) or ("E" in text)
            out.append(("float" if isf else "int", float(text) if isf else int(text), line))
        elif kind != "ws":
            out.append((kind, text, line))
        line += text.count("\n")
        pos = m.end()
    out.append(("eof", None, line))
    return out


_BINOPS = [("||",), ("&&",), ("==", "!="), ("<", "<=", ">", ">="), ("+", "-"), ("*", "/", "%")]


class _Parser:
    def __init__(self, src):
        self.t = tokenize(src)
        self.i = 0

    # -- token helpers --
    def peek(self, k=0):
        return self.t[min(self.i + k, len(self.t) - 1)]

    def line(self):
        return self.peek()[2]

    def at(self, text):
        tk = self.peek()
        return tk[0] in ("id", "sym") and tk[1] == text

    def take(self, text=None, kind=None):
        tk = self.peek()
        if (text is not None and not (tk[0] in ("id", "sym") and tk[1] == text)) or \
           (kind is not None and tk[0] != kind):
            want = repr(text) if text is not None else kind
            raise KdlError("parse.syntax", f"expected {want}, got {tk[1]!r}", tk[2])
        self.i += 1
        return tk[1]

    def ident(self):
        return self.take(kind="id")

    # -- top level --
    def program(self):
        p = A.Program()
        while self.peek()[0] != "eof":
            if self.at("global"):
                self.take("global")
                t = self.type_kw()
                name = self.ident()
                self.take("[")
                ln = self.expr()
                self.take("]")
                self.take(";")
                p.globals.append(A.Global(name, t, ln))
            elif self.at("kernel"):
                p.kernels.append(self.kernel())
            elif self.at("entry"):
                if p.entry is not None:
                    raise KdlError("parse.entry", "more than one entry declaration", self.line())
                self.take("entry")
                k = self.ident()
                g, b, args = self.launch_tail()
                self.take(";")
                p.entry = A.Entry(k, g, b, args)
            else:
                raise KdlError("parse.syntax", "expected 'kernel', 'global' or 'entry'", self.line())
        if p.entry is None:
            raise KdlError("parse.entry", "program has no entry declaration")
        return p

    def type_kw(self):
        tk = self.peek()
        if tk[0] == "id" and tk[1] in (A.INT, A.FLOAT):
            self.i += 1
            return tk[1]
        raise KdlError("parse.syntax", "expected 'int' or 'float'", tk[2])

    def kernel(self):
        self.take("kernel")
        k = A.Kernel(self.ident())
        self.take("(")
        while not self.at(")"):
            t = self.type_kw()
            n = self.ident()
            arr = False
            if self.at("["):
                self.take("[")
                self.take("]")
                arr = True
            k.params.append(A.Param(n, t, arr))
            if not self.at(")"):
                self.take(",")
        self.take(")")
        k.body = self.block()
        return k

    def launch_tail(self):
        self.take("<<<")
        g = self.expr()
        self.take(",")
        b = self.expr()
        self.take(">>>")
        self.take("(")
        args = []
        while not self.at(")"):
            args.append(self.expr())
            if not self.at(")"):
                self.take(",")
        self.take(")")
        return g, b, args

    def block(self):
        self.take("{")
        out = []
        while not self.at("}"):
            if self.peek()[0] == "eof":
                raise KdlError("parse.syntax", "unterminated block", self.line())
            out.append(self.stmt())
        self.take("}")
        return out

    # -- statements --
    def stmt(self):
        tk = self.peek()
        if tk[0] == "pragma":
            self.i += 1
            d = parse_directive(tk[1], tk[2])
            s = self.stmt()
            if s.kind != "launch":
                raise KdlError("parse.pragma", "#pragma dp must precede a launch statement", tk[2])
            s.directive = d
            return s
        if tk[0] != "id":
            raise KdlError("parse.syntax", f"unexpected {tk[1]!r}", tk[2])
        w = tk[1]
        if w == "if":
            self.take("if")
            self.take("(")
            c = self.expr()
            self.take(")")
            body = self.block()
            els = []
            if self.at("else"):
                self.take("else")
                els = [self.stmt()] if self.at("if") else self.block()
            return A.if_(c, body, els)
        if w == "for":
            self.take("for")
            self.take("(")
            if not self.at("int"):
                raise KdlError("parse.for", "for loop variable must be 'int'", self.line())
            self.take("int")
            v = self.ident()
            self.take("=")
            a = self.expr()
            self.take(";")
            if self.ident() != v:
                raise KdlError("parse.for", "for condition must test the loop variable", self.line())
            self.take("<")
            b = self.expr()
            self.take(";")
            if self.ident() != v:
                raise KdlError("parse.for", "for step must update the loop variable", self.line())
            self.take("+=")
            c = self.expr()
            self.take(")")
            return A.for_(v, a, b, c, self.block())
        simple = {"return": "return", "barrier_block": "barrier", "sync_device": "sync",
                  "dp_grid_barrier": "grid_barrier"}
        if w in simple:
            self.i += 1
            self.take(";")
            return A.bare(simple[w])
        if w == "atomicAdd":
            self.take("atomicAdd")
            self.take("(")
            arr = self.ident()
            self.take(",")
            i = self.expr()
            self.take(",")
            v = self.expr()
            self.take(")")
            self.take(";")
            return A.Stmt("atomic", name=arr, exprs=[i, v])
        if w == "dp_buffers":
            self.take("dp_buffers")
            self.take("(")
            gran = self.ident()
            if gran not in ("warp", "block", "grid"):
                raise KdlError("parse.bufdecl", f"unknown granularity {gran!r}", self.line())
            self.take(",")
            alloc = self.ident()
            alloc = {"custom": "prealloc"}.get(alloc, alloc)
            if alloc not in ("default", "halloc", "prealloc"):
                raise KdlError("parse.bufdecl", f"unknown allocator {alloc!r}", self.line())
            self.take(",")
            nv = self.take(kind="int")
            self.take(",")
            per = self.expr()
            self.take(",")
            tot = self.take(kind="int")
            self.take(")")
            self.take(";")
            return A.Stmt("buf_decl", gran=gran, alloc=alloc, nvars=nv, total_bytes=tot, exprs=[per])
        if w == "dp_insert":
            self.take("dp_insert")
            self.take("(")
            args = [self.expr()]
            while self.at(","):
                self.take(",")
                args.append(self.expr())
            self.take(")")
            self.take(";")
            if len(args) < 3:
                raise KdlError("parse.insert", "dp_insert takes (grid, block, value...)", self.line())
            return A.Stmt("insert", exprs=args)
        if w in (A.INT, A.FLOAT):
            t = self.type_kw()
            n = self.ident()
            self.take("=")
            e = self.expr()
            self.take(";")
            return A.let(t, n, e)
        n = self.ident()
        if self.at("="):
            self.take("=")
            e = self.expr()
            self.take(";")
            return A.Stmt("assign", name=n, exprs=[e])
        if self.at("["):
            self.take("[")
            i = self.expr()
            self.take("]")
            self.take("=")
            v = self.expr()
            self.take(";")
            return A.Stmt("store", name=n, exprs=[i, v])
        if self.at("<<<"):
            g, b, args = self.launch_tail()
            self.take(";")
            return A.launch(n, g, b, args)
        raise KdlError("parse.syntax", "expected '=', '[' or '<<<' after identifier", self.line())

    # -- expressions --
    def expr(self, level=0):
        if level == len(_BINOPS):
            return self.unary()
        e = self.expr(level + 1)
        while self.peek()[0] == "sym" and self.peek()[1] in _BINOPS[level]:
            op = self.take()
            e = A.binop(op, e, self.expr(level + 1))
        return e

    def unary(self):
        if self.at("-") or self.at("!"):
            op = self.take()
            return A.Expr("unary", name=op, args=[self.unary()])
        return self.primary()

    def primary(self):
        tk = self.peek()
        if tk[0] == "int":
            self.i += 1
            return A.lit(tk[1])
        if tk[0] == "float":
            self.i += 1
            return A.Expr("float", fval=tk[1])
        if self.at("("):
            self.take("(")
            e = self.expr()
            self.take(")")
            return e
        n = self.ident()
        if n in A.INTRINSICS:
            return A.intr(n)
        if n in ("min", "max"):
            self.take("(")
            a = self.expr()
            self.take(",")
            b = self.expr()
            self.take(")")
            return A.Expr("minmax", name=n, args=[a, b])
        if n == "atomicAdd":
            self.take("(")
            arr = self.ident()
            self.take(",")
            i = self.expr()
            self.take(",")
            v = self.expr()
            self.take(")")
            return A.Expr("atomic", name=arr, args=[i, v])
        zero = {"dp_buf_count": "buf_count", "dp_buf_pending": "buf_pending", "dp_grid_last": "grid_last"}
        if n in zero:
            self.take("(")
            self.take(")")
            return A.call0(zero[n])
        if n == "dp_buf_get":
            self.take("(")
            i = self.expr()
            self.take(",")
            slot = self.take(kind="int")
            self.take(")")
            return A.Expr("buf_get", args=[i, A.lit(slot)])
        if n == "dp_kc_blocks":  # B200 extension (unparse.py): KC_X launch size resolved at load
            self.take("(")
            k = self.ident()
            self.take(",")
            x = self.take(kind="int")
            self.take(",")
            t = self.expr()
            self.take(")")
            return A.Expr("kc_blocks", name=k, ival=x, args=[t])
        if n in ("dp_buf_cfg_grid", "dp_buf_cfg_block"):
            self.take("(")
            i = self.expr()
            self.take(")")
            return A.Expr("buf_cfg_grid" if n.endswith("grid") else "buf_cfg_block", args=[i])
        if self.at("["):
            self.take("[")
            i = self.expr()
            self.take("]")
            return A.Expr("index", name=n, args=[i])
        return A.ref(n)


def parse_directive(text, line=0):
    """`#pragma dp clause(args) ...` -> ast.Directive (parser.hpp:638-779)."""
    toks = tokenize(text.lstrip("#"))
    words = [t[1] for t in toks if t[0] != "eof"]
    if words[:2] != ["pragma", "dp"]:
        raise KdlError("dir.syntax", "directive must start with '#pragma dp'", line)
    d = A.Directive()
    have_gran = have_work = False
    i = 2
    while i < len(words):
        clause = words[i]
        if i + 1 >= len(words) or words[i + 1] != "(":
            raise KdlError("dir.syntax", f"expected '(' after clause {clause!r}", line)
        j = i + 2
        args = []
        while j < len(words) and words[j] != ")":
            if words[j] != ",":
                args.append(words[j])
            j += 1
        if j >= len(words):
            raise KdlError("dir.syntax", f"unterminated clause {clause!r}", line)
        i = j + 1
        if clause == "consltdt":
            if len(args) != 1 or args[0] not in ("warp", "block", "grid"):
                raise KdlError("dir.arg", "consltdt takes one of warp|block|grid", line)
            d.granularity = args[0]
            have_gran = True
        elif clause == "buffer":
            if not args or args[0] not in ("default", "halloc", "custom"):
                raise KdlError("dir.arg", "buffer takes (default|halloc|custom[, perBufferSize[, totalSize]])", line)
            if len(args) > 3:
                raise KdlError("dir.arg", "too many buffer arguments", line)
            d.buffer = args[0]
            if len(args) >= 2:
                if isinstance(args[1], int):
                    if args[1] != 0:
                        d.per_buffer_lit = args[1]
                elif isinstance(args[1], str):
                    d.per_buffer_var = args[1]
                else:
                    raise KdlError("dir.arg", "perBufferSize must be an integer or a variable name", line)
            if len(args) == 3:
                if not isinstance(args[2], int):
                    raise KdlError("dir.arg", "totalSize must be an integer byte count", line)
                d.total_bytes = args[2]
        elif clause == "work":
            if not args or not all(isinstance(a, str) for a in args):
                raise KdlError("dir.arg", "work takes a nonempty identifier list", line)
            d.work = list(args)
            have_work = True
        elif clause in ("threads", "blocks"):
            if len(args) != 1 or not isinstance(args[0], int) or args[0] < 1:
                raise KdlError("dir.arg", f"{clause} takes one positive integer", line)
            setattr(d, clause, args[0])
        else:
            raise KdlError("dir.clause", f"unknown clause {clause!r}", line)
    if not have_gran:
        raise KdlError("dir.missing", "missing mandatory consltdt clause", line)
    if not have_work:
        raise KdlError("dir.missing", "missing mandatory work clause", line)
    return d


def parse_program(src):
    return _Parser(src).program()
