"""Printer for ast.Program in the reference's text layout (unparse.hpp:37-340:
two-space indentation, minimal parentheses by binary precedence, `%.17g`
float literals), so a program this package rewrote prints character for
character like the reference's consolidate() output (tests/test_kdl.py).
The B200-only `kc_blocks` node prints as `dp_kc_blocks(kernel, X, T)`, which
parse.py reads back; lower_kc() replaces it by the literal the reference
would print."""
from . import ast as A

_PREC = {"*": 6, "/": 6, "%": 6, "+": 5, "-": 5, "<": 4, "<=": 4, ">": 4, ">=": 4, "==": 3, "!=": 3,
         "&&": 2, "||": 1}


def _float(v):
    s = "%.17g" % v
    return s if ("." in s or "e" in s or "E" in s) else s + ".0"


def expr(e, parent=0):
    k = e.kind
    if k == "int":
        return str(e.ival)
    if k == "float":
        return _float(e.fval)
    if k in ("name", "intrinsic"):
        return e.name
    if k == "index":
        return f"{e.name}[{expr(e.args[0])}]"
    if k == "unary":
        a = e.args[0]
        return e.name + (f"({expr(a)})" if a.kind in ("binary", "unary") else expr(a, 7))
    if k == "binary":
        p = _PREC[e.name]
        s = f"{expr(e.args[0], p)} {e.name} {expr(e.args[1], p + 1)}"
        return f"({s})" if p < parent else s
    if k == "minmax":
        return f"{e.name}({expr(e.args[0])}, {expr(e.args[1])})"
    if k == "atomic":
        return f"atomicAdd({e.name}, {expr(e.args[0])}, {expr(e.args[1])})"
    if k == "buf_count":
        return "dp_buf_count()"
    if k == "buf_pending":
        return "dp_buf_pending()"
    if k == "grid_last":
        return "dp_grid_last()"
    if k == "buf_get":
        return f"dp_buf_get({expr(e.args[0])}, {e.args[1].ival})"
    if k == "buf_cfg_grid":
        return f"dp_buf_cfg_grid({expr(e.args[0])})"
    if k == "buf_cfg_block":
        return f"dp_buf_cfg_block({expr(e.args[0])})"
    if k == "kc_blocks":
        return f"dp_kc_blocks({e.name}, {e.ival}, {expr(e.args[0])})"
    raise ValueError(f"unknown expression kind {k!r}")


def _directive(d):
    s = f"#pragma dp consltdt({d.granularity}) buffer({d.buffer}"
    if d.per_buffer_lit:
        s += f", {d.per_buffer_lit}"
    elif d.per_buffer_var:
        s += f", {d.per_buffer_var}"
    if d.total_bytes != A.Directive().total_bytes:
        if not d.per_buffer_lit and not d.per_buffer_var:
            s += ", 0"
        s += f", {d.total_bytes}"
    s += ") work(" + ", ".join(d.work) + ")"
    if d.threads:
        s += f" threads({d.threads})"
    if d.blocks:
        s += f" blocks({d.blocks})"
    return s


def _stmts(body, depth, out):
    for s in body:
        _stmt(s, depth, out)


def _stmt(s, depth, out):
    ind = "  " * depth
    k = s.kind
    if k == "let":
        out.append(f"{ind}{s.scalar} {s.name} = {expr(s.exprs[0])};")
    elif k == "assign":
        out.append(f"{ind}{s.name} = {expr(s.exprs[0])};")
    elif k == "store":
        out.append(f"{ind}{s.name}[{expr(s.exprs[0])}] = {expr(s.exprs[1])};")
    elif k == "atomic":
        out.append(f"{ind}atomicAdd({s.name}, {expr(s.exprs[0])}, {expr(s.exprs[1])});")
    elif k == "if":
        out.append(f"{ind}if ({expr(s.exprs[0])}) {{")
        _stmts(s.body, depth + 1, out)
        if s.else_body:
            out.append(f"{ind}}} else {{")
            _stmts(s.else_body, depth + 1, out)
        out.append(f"{ind}}}")
    elif k == "for":
        a, b, c = s.exprs
        out.append(f"{ind}for (int {s.name} = {expr(a)}; {s.name} < {expr(b)}; {s.name} += {expr(c)}) {{")
        _stmts(s.body, depth + 1, out)
        out.append(f"{ind}}}")
    elif k in ("barrier", "sync", "grid_barrier", "return"):
        out.append(ind + {"barrier": "barrier_block;", "sync": "sync_device;", "grid_barrier": "dp_grid_barrier;",
                          "return": "return;"}[k])
    elif k == "launch":
        if s.directive is not None:
            out.append(ind + _directive(s.directive))
        args = ", ".join(expr(e) for e in s.exprs[2:])
        out.append(f"{ind}{s.name}<<<{expr(s.exprs[0])}, {expr(s.exprs[1])}>>>({args});")
    elif k == "buf_decl":
        out.append(f"{ind}dp_buffers({s.gran}, {s.alloc}, {s.nvars}, {expr(s.exprs[0])}, {s.total_bytes});")
    elif k == "insert":
        out.append(f"{ind}dp_insert({', '.join(expr(e) for e in s.exprs)});")
    else:
        raise ValueError(f"unknown statement kind {k!r}")


def unparse(prog):
    out = []
    for g in prog.globals:
        out.append(f"global {g.type} {g.name}[{expr(g.length)}];")
    if prog.globals:
        out.append("")
    for k in prog.kernels:
        params = ", ".join(f"{p.type} {p.name}" + ("[]" if p.is_array else "") for p in k.params)
        out.append(f"kernel {k.name}({params}) {{")
        _stmts(k.body, 1, out)
        out.append("}")
        out.append("")
    e = prog.entry
    out.append(f"entry {e.kernel}<<<{expr(e.grid)}, {expr(e.block)}>>>({', '.join(expr(a) for a in e.args)});")
    return "\n".join(out) + "\n"
