"""CPU tests of the .kdl -> CUDA compiler: front end,
consolidation rewrite parity with the reference's consolidate() output
(committed fixtures from tests/golden/make_kdl_golden.py), diagnostics,
CUDA generation and the nvcc build (cross-compiles here, no GPU needed)."""
import copy
import json
import os

import pytest

import paper_1606_08150_b200.kdl as kdl
from paper_1606_08150_b200.kdl import ast as A
from paper_1606_08150_b200.kdl import transform as T

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "kdl_reference.json")))


def src_of(name):
    p = os.path.join(kdl.PROGRAMS, name)
    if not os.path.exists(p):
        p = os.path.join(HERE, "kdl", name)
    return open(p).read()


CASES = [(n, m) for n in sorted(GOLD["consolidated"]) for m in ("warp", "block", "grid")]


@pytest.mark.parametrize("name,mode", CASES)
def test_rewrite_matches_reference_consolidate(name, mode):
    """Our rewrite == the reference's consolidate() output, node for node,
    with the KC_X launch sizes lowered for the reference's device model."""
    ref_txt = GOLD["consolidated"][name][mode]
    assert isinstance(ref_txt, str), ref_txt
    ref = kdl.parse_program(ref_txt)
    ours = T.lower_kc(kdl.consolidate(kdl.parse_program(src_of(name)), mode), T.k20c_occupancy)
    if (name, mode) == ("post.kdl", "grid"):
        # Reference bug: rewrite_parent moves the prework statements into the
        # new body before build_postwork_kernel reads them (transform.hpp:
        # 728-729 then 792-795), so the def-use closure sees empty statements
        # and <parent>_post uses `v` without its definition (the simulator then
        # reads 0 and produces wrong output; see tests/test_kdl_gpu.py).  Our
        # rewrite keeps the defining statement; apart from it, identical.
        post = ours.kernel("parent_post")
        loop = post.body[0]
        assert loop.body[0] == A.let(A.INT, "v", T.subst(
            A.binop("+", A.binop("*", A.intr("blockIdx"), A.intr("blockDim")), A.intr("threadIdx")),
            {"threadIdx": A.binop("%", A.ref("__v"), A.ref("__ob")),
             "blockIdx": A.binop("/", A.ref("__v"), A.ref("__ob")),
             "blockDim": A.ref("__ob"), "gridDim": A.ref("__og")}))
        ours = copy.deepcopy(ours)
        del ours.kernel("parent_post").body[0].body[0]
    assert ours == ref


def test_reference_consolidated_text_parses_and_generates():
    """The CUDA builder accepts the reference's own consolidate() text."""
    for name in sorted(GOLD["consolidated"]):
        for mode in ("warp", "block", "grid"):
            prog = kdl.parse_program(GOLD["consolidated"][name][mode])
            if (name, mode) == ("post.kdl", "grid"):
                # the reference's postwork kernel uses `v` undeclared (see above)
                with pytest.raises(kdl.KdlError) as ei:
                    kdl.generate(prog, name[:-4])
                assert ei.value.code == "cuda.name"
                continue
            src, kc = kdl.generate(prog, name[:-4])
            assert "cudaStreamFireAndForget" in src
            assert kc == []  # literal launch sizes: nothing to resolve at load


def test_kc_blocks_resolved_per_granularity():
    prog = kdl.consolidate(kdl.parse_program(src_of("td.kdl")), "warp")
    src, kc = kdl.generate(prog, "td")
    assert kc == [("td_cons", 32, 256)]
    assert "dk_kc[0]" in src
    # KC_X = max(1, B_occ / X) (config.hpp:63-72): B200 with 8 x 256-thread blocks per SM
    assert T.kc_blocks(148 * 8, 32) == 37 and T.kc_blocks(148 * 8, 16) == 74 and T.kc_blocks(148 * 8, 1) == 1184


def test_directive_parsing_and_errors():
    d = kdl.parse.parse_directive("#pragma dp consltdt(block) buffer(custom, 64, 4096) work(a, b) threads(128)")
    assert (d.granularity, d.buffer, d.per_buffer_lit, d.total_bytes, d.work, d.threads) == \
        ("block", "custom", 64, 4096, ["a", "b"], 128)
    d = kdl.parse.parse_directive("#pragma dp consltdt(warp) buffer(default, cap) work(x)")
    assert d.per_buffer_var == "cap" and d.per_buffer_lit is None
    for bad, code in [("#pragma dp work(a)", "dir.missing"), ("#pragma dp consltdt(grid)", "dir.missing"),
                      ("#pragma dp consltdt(team) work(a)", "dir.arg"),
                      ("#pragma dp consltdt(grid) work(a) bogus(1)", "dir.clause"),
                      ("#pragma dp consltdt(grid) threads(0) work(a)", "dir.arg")]:
        with pytest.raises(kdl.KdlError) as ei:
            kdl.parse.parse_directive(bad)
        assert ei.value.code == code


def test_parser_precedence_and_float_literals():
    p = kdl.parse_program("global int a[n];\nkernel k(int x) { int y = 1 + 2 * x - -3 % 2 < 4 || !x && x == 1; "
                          "float z = 1.5e2; a[0] = y; }\nentry k<<<1, 1>>>(7);")
    y = p.kernels[0].body[0].exprs[0]
    assert y.name == "||" and y.args[1].name == "&&"
    lt = y.args[0]
    assert lt.name == "<" and lt.args[0].name == "-" and lt.args[0].args[0].name == "+"
    assert p.kernels[0].body[1].exprs[0] == A.Expr("float", fval=150.0)


BAD_PROGRAMS = [
    # annotated launch of an annotated parent (chained consolidation)
    ("kernel c(int v) { #pragma dp consltdt(warp) work(v)\n d<<<1, 1>>>(v); }\n"
     "kernel d(int v) { }\nkernel p(int v) { #pragma dp consltdt(warp) work(v)\n c<<<1, 1>>>(v); }\n"
     "entry p<<<1, 1>>>(0);", "tf.chain"),
    ("global int a[4];\nkernel c(int h[]) { }\nkernel p() { #pragma dp consltdt(warp) work(a)\n c<<<1, 1>>>(a); }\n"
     "entry p<<<1, 1>>>();", "tf.workarray"),
    ("kernel c(int v) { }\nkernel p(int v) { int w = v; #pragma dp consltdt(warp) work(w)\n c<<<1, 1>>>(v); }\n"
     "entry p<<<1, 1>>>(0);", "val.workarg"),
    ("kernel c(int v) { return; }\nkernel p(int v) { #pragma dp consltdt(block) work(v)\n c<<<1, 1>>>(v); }\n"
     "entry p<<<1, 1>>>(0);", "tf.childreturn"),
    ("kernel c(int v, int u) { }\nkernel p(int v) { int u = v + 1; #pragma dp consltdt(block) work(v)\n"
     " c<<<1, 1>>>(v, u); }\nentry p<<<1, 1>>>(0);", "tf.arg"),
    ("kernel p(int v) { if (v > 0) { #pragma dp consltdt(grid) work(v)\n p<<<1, 1>>>(v - 1); } sync_device; }\n"
     "entry p<<<1, 1>>>(3);", "val.workarg"),
    ("kernel p(int v) { int w = v - 1; if (v > 0) { #pragma dp consltdt(grid) work(w)\n p<<<1, 1>>>(w); } "
     "sync_device; }\nentry p<<<1, 1>>>(3);", "tf.recsync"),
    ("kernel c(int s) { int k = blockIdx * 7; }\nkernel p(int v) { #pragma dp consltdt(warp) threads(64) work(v)\n"
     " c<<<v, 32>>>(v); }\nentry p<<<1, 1>>>(3);", None),   # moldable? no: gridDim-free -> legal
    ("kernel c(int s) { int k = s + blockDim; }\nkernel p(int v) { #pragma dp consltdt(warp) threads(64) work(v)\n"
     " c<<<v, 32>>>(v); }\nentry p<<<1, 1>>>(3);", "tf.nonmoldable"),
]


@pytest.mark.parametrize("src,code", BAD_PROGRAMS)
def test_rewrite_diagnostics(src, code):
    prog = kdl.parse_program(src)
    if code is None:
        kdl.consolidate(prog, None)
        return
    with pytest.raises(kdl.KdlError) as ei:
        kdl.consolidate(prog, None)
    assert ei.value.code == code


@pytest.mark.parametrize("src,code", [
    ("global int a[4];\nkernel k() { int x = 1.5; }\nentry k<<<1, 1>>>();", "cuda.type"),
    ("global int a[4];\nkernel k() { a[0] = 0.5; }\nentry k<<<1, 1>>>();", "cuda.type"),
    ("global int a[4];\nkernel k() { dp_insert(1, 1, 2); }\nentry k<<<1, 1>>>();", "cuda.insert"),
    ("global int a[4];\nkernel c() { }\nkernel k() { if (1) { c<<<1, 1>>>(); sync_device; a[0] = 1; } }\n"
     "entry k<<<1, 1>>>();", "cuda.sync"),
    ("global int a[4];\nkernel c() { }\nkernel k() { dp_buffers(warp, prealloc, 1, 8, 4096); c<<<1, 1>>>(); "
     "sync_device; dp_insert(1, 1, 3); }\nentry k<<<1, 1>>>();", "cuda.sync"),
    ("kernel k() { dp_grid_barrier; }\nentry k<<<1, 1>>>();", "cuda.gridbarrier"),
    ("kernel k() { int x = y; }\nentry k<<<1, 1>>>();", "cuda.name"),
])
def test_builder_diagnostics(src, code):
    with pytest.raises(kdl.KdlError) as ei:
        kdl.generate(kdl.parse_program(src))
    assert ei.value.code == code


def test_recursive_rewrite_shape():
    prog = kdl.consolidate(kdl.parse_program(src_of("td.kdl")), "grid")
    names = [k.name for k in prog.kernels]
    assert names == ["td_cons", "td_boot"]
    assert prog.entry.kernel == "td_boot" and prog.entry.grid == A.lit(1)
    assert [a.kind for a in prog.entry.args] == ["name", "int", "name"]   # root, 1, rootnc


def test_host_expression_semantics():
    e = kdl.parse_program("global int a[(n + 255) / 256 - -7 / 2 + -7 % 3];\nkernel k() { }\nentry k<<<1,1>>>();")
    # C truncation: -7 / 2 = -3, -7 % 3 = -1
    assert kdl.eval_host(e.globals[0].length, {"n": 1000}) == 4 + 3 - 1


def test_generated_unit_builds_for_sm100a(tmp_path, monkeypatch):
    """nvcc cross-compiles the generated unit (CDP2, rdc) for sm_100a."""
    mod = kdl.compile(src_of("spmv.kdl"), "grid", name="spmv")
    assert os.path.exists(mod.so)
    import subprocess
    out = subprocess.run(["nm", "-D", mod.so], capture_output=True, text=True).stdout
    import re
    hdr = open(os.path.join(os.path.dirname(HERE), "include", "dpc_kdl.h")).read()
    syms = re.findall(r"^(?:int|const char\*) (dk_\w+)\(", hdr, re.M)
    assert len(syms) == 7
    for sym in syms:   # every entry point include/dpc_kdl.h declares
        assert f" T {sym}" in out, sym


@pytest.mark.parametrize("name,mode", CASES)
def test_rewrite_prints_like_reference(name, mode):
    """Character for character: our rewrite, printed in the reference's
    layout, equals the reference's consolidate() text."""
    if (name, mode) == ("post.kdl", "grid"):
        pytest.skip("reference bug, see test_rewrite_matches_reference_consolidate")
    ours = T.lower_kc(kdl.consolidate(kdl.parse_program(src_of(name)), mode), T.k20c_occupancy)
    assert kdl.unparse(ours) == GOLD["consolidated"][name][mode]


@pytest.mark.parametrize("name", sorted(GOLD["consolidated"]))
def test_unparse_parse_round_trip(name):
    p = kdl.parse_program(src_of(name))
    assert kdl.parse_program(kdl.unparse(p)) == p
    for mode in ("warp", "block", "grid"):
        c = kdl.consolidate(p, mode)   # kc_blocks nodes print as dp_kc_blocks(...)
        assert kdl.parse_program(kdl.unparse(c)) == c


def test_expression_round_trip_random():
    from hypothesis import given, settings
    from hypothesis import strategies as st

    from paper_1606_08150_b200.kdl.unparse import expr as print_expr

    leaves = st.one_of(st.integers(0, 10**12).map(A.lit), st.sampled_from(["a", "b"]).map(A.ref),
                       st.sampled_from(A.INTRINSICS).map(A.intr),
                       st.floats(0, 1e6, allow_nan=False).map(lambda v: A.Expr("float", fval=v)))
    ops = ["+", "-", "*", "/", "%", "<", "<=", ">", ">=", "==", "!=", "&&", "||"]

    def extend(children):
        return st.one_of(
            st.tuples(st.sampled_from(ops), children, children).map(lambda t: A.binop(*t)),
            st.tuples(st.sampled_from(["-", "!"]), children).map(lambda t: A.Expr("unary", name=t[0], args=[t[1]])),
            st.tuples(st.sampled_from(["min", "max"]), children, children).map(
                lambda t: A.Expr("minmax", name=t[0], args=[t[1], t[2]])),
            children.map(lambda c: A.Expr("index", name="arr", args=[c])))

    @settings(max_examples=300, deadline=None)
    @given(st.recursive(leaves, extend, max_leaves=12))
    def check(e):
        src = ("global int arr[n];\nkernel k(int a, int b) { int z = " + print_expr(e) +
               "; }\nentry k<<<1, 1>>>(0, 0);")
        assert kdl.parse_program(src).kernels[0].body[0].exprs[0] == e

    check()
