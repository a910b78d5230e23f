"""BASELINE-shaped motif SDFGs built with the REFERENCE builder API.

Test infrastructure only: this module imports the reference package
(``sdfg`` from /root/reference/pkg/src) and therefore only runs in the build
container.  ``make_golden.py`` uses it to serialise the graphs with the
reference's own canonical JSON writer (serialization.py:106-160) and to
record interpreter / reference-generated-C outputs as fixtures, so the GPU
box (which has no /root/reference) can replay them.

Recipes follow SURVEY.md §8(c):
  * histogram  -- binned two-tasklet form; ``bi = v * 256 // 1`` into an
                  int64 transient, ``h[k] = 1`` subscript write with WCR sum
                  (gallery.py:354-386 is the integer-image variant).
  * query      -- gallery.query (gallery.py:300-347) with predicate ``v < limit``.
  * spmv       -- gallery.spmv as is (gallery.py:152-213).
  * jacobi2d   -- the laplace pattern (gallery.py:59-100) lifted to 2-D,
                  5-point ``o = 0.2 * (c + n + s + w + e)``.
  * matmul     -- gallery.matmul (gallery.py:107-144) after MapReduceFusion
                  (library.py:461-554); optionally MapTiling -> LocalStorage.
"""

from __future__ import annotations

import os
import sys

REF_SRC = os.environ.get("SDFG_REF_SRC", "/root/reference/pkg/src")
if REF_SRC not in sys.path:
    sys.path.insert(0, REF_SRC)

from sdfg import gallery  # noqa: E402
from sdfg.ir import Memlet, Sdfg  # noqa: E402
from sdfg.rewriting import apply_transformation, find_matches  # noqa: E402


def histogram(bins: int = 256, name: str = "histogram") -> Sdfg:
    g = Sdfg(name)
    g.add_symbol("H")
    g.add_symbol("W")
    g.add_array("img", ["H", "W"], "float64")
    g.add_array("hist", [str(bins)], "int64")
    g.add_array("bin", ["1"], "int64", transient=True)
    st = g.add_state("binning", is_start=True)
    img = st.add_access("img")
    hist = st.add_access("hist")
    me, mx = st.add_map(["i", "j"], ["0:H - 1", "0:W - 1"])
    binner = st.add_tasklet("binner", ["v"], ["bi"], f"bi = v * {bins} // 1")
    st.add_memlet_path(img, me, binner, dst_conn="v",
                       memlet=Memlet.simple("img", "[i, j]"))
    b = st.add_access("bin")
    st.add_edge(binner, "bi", b, None, Memlet.simple("bin", "[0]"))
    bump = st.add_tasklet("bump", ["k"], ["h"], "h[k] = 1")
    st.add_edge(b, None, bump, "k", Memlet.simple("bin", "[0]"))
    st.add_memlet_path(bump, mx, hist, src_conn="h",
                       memlet=Memlet.simple("hist", f"[0:{bins - 1}]", wcr="sum",
                                            accesses=1))
    g.finalize()
    return g


def _wrap_in_loop(g: Sdfg, first: str, last: str, reps: str) -> None:
    """Put the straight-line states ``first .. last`` in a guard loop of
    ``reps`` trips (the motif then runs several times: ADVICE r1)."""
    init = g.add_state("loop_init", is_start=True)
    guard = g.add_state("loop_guard")
    g.add_transition(init, guard, assignments=[("r", "0")])
    g.add_transition(guard, g.state(first), condition=f"r < {reps}")
    g.add_transition(g.state(last), guard, assignments=[("r", "r + 1")])


def histogram_looped(reps: int = 3) -> Sdfg:
    """The binned histogram inside a ``reps``-trip guard loop: the counts
    accumulate ``reps`` times (hist_out = hist_in + reps * counts)."""
    g = histogram(name="histogram_looped")
    _wrap_in_loop(g, "binning", "binning", str(reps))
    g.finalize()
    return g


def query_cond() -> Sdfg:
    """The query behind a condition on a symbol: it runs only when N > 8."""
    g = query("<", name="query_cond")
    pre = g.add_state("pre", is_start=True)
    g.add_transition(pre, g.state("filter"), condition="N > 8")
    g.finalize()
    return g


def histogram_int() -> Sdfg:
    """The gallery's integer-image variant (gallery.py:354-386)."""
    return gallery.fixture("histogram").sdfg


def query(op: str = "<", name: str = "query") -> Sdfg:
    g = Sdfg(name)
    g.add_symbol("N")
    g.add_array("col", ["N"], "float64")
    g.add_array("thr", ["1"], "float64")
    g.add_array("out_vals", ["N"], "float64")
    g.add_array("count", ["1"], "int64")
    g.add_stream("S", "float64")
    st = g.add_state("filter", is_start=True)
    col = st.add_access("col")
    thr = st.add_access("thr")
    me, mx = st.add_map("i", "0:N - 1")
    t = st.add_tasklet("pred", ["v", "limit"], ["sv", "c"],
                       f"if v {op} limit:\n    sv = v\n    c = 1")
    st.add_memlet_path(col, me, t, dst_conn="v", memlet=Memlet.simple("col", "[i]"))
    st.add_memlet_path(thr, me, t, dst_conn="limit",
                       memlet=Memlet.simple("thr", "[0]"))
    s_acc = st.add_access("S")
    st.add_memlet_path(t, mx, s_acc, src_conn="sv", dst_conn="push",
                       memlet=Memlet.simple("S", "[0]", dynamic=True))
    cnt = st.add_access("count")
    st.add_memlet_path(t, mx, cnt, src_conn="c",
                       memlet=Memlet.simple("count", "[0]", wcr="sum", dynamic=True))
    vals = st.add_access("out_vals")
    st.add_edge(s_acc, "pop", vals, None, Memlet.simple("S", "[0]", dynamic=True))
    g.finalize()
    return g


def query_gallery() -> Sdfg:
    """gallery.query as is: predicate ``v > limit`` (gallery.py:314-315)."""
    return gallery.fixture("query").sdfg


def spmv() -> Sdfg:
    return gallery.fixture("spmv").sdfg


def jacobi2d(coef: str = "0.2", name: str = "jacobi2d") -> Sdfg:
    g = Sdfg(name)
    g.add_symbol("N")
    g.add_symbol("T")
    g.add_array("A", ["2", "N", "N"], "float64")
    init = g.add_state("init", is_start=True)
    guard = g.add_state("guard")
    body = g.add_state("body")
    g.add_transition(init, guard, assignments=[("t", "0")])
    g.add_transition(guard, body, condition="t < T")
    g.add_transition(body, guard, assignments=[("t", "t + 1")])
    rd = body.add_access("A")
    wr = body.add_access("A")
    me, mx = body.add_map(["i", "j"], ["1:N - 2", "1:N - 2"])
    t = body.add_tasklet("stencil", ["c", "n", "s", "w", "e"], ["o"],
                         f"o = {coef} * (c + n + s + w + e)")
    for conn, idx in (("c", "i, j"), ("n", "i - 1, j"), ("s", "i + 1, j"),
                      ("w", "i, j - 1"), ("e", "i, j + 1")):
        body.add_memlet_path(rd, me, t, dst_conn=conn,
                             memlet=Memlet.simple("A", f"[t % 2, {idx}]"))
    body.add_memlet_path(t, mx, wr, src_conn="o",
                         memlet=Memlet.simple("A", "[(t + 1) % 2, i, j]"))
    g.finalize()
    return g


def laplace1d() -> Sdfg:
    return gallery.fixture("laplace").sdfg


def axpy(n: int = 64) -> Sdfg:
    """Element-wise ``y[i] = a * x[i] + y[i]`` over a constant-length map --
    the shape the reference's Vectorization rule applies to
    (library.py:763-840)."""
    g = Sdfg("axpy")
    g.add_array("x", [str(n)], "float64")
    g.add_array("y", [str(n)], "float64")
    g.add_array("a", ["1"], "float64")
    st = g.add_state("main", is_start=True)
    xr, yr, ar, yw = st.add_access("x"), st.add_access("y"), st.add_access("a"), st.add_access("y")
    me, mx = st.add_map("i", f"0:{n - 1}")
    t = st.add_tasklet("fma", ["xi", "yi", "av"], ["o"], "o = av * xi + yi")
    st.add_memlet_path(xr, me, t, dst_conn="xi", memlet=Memlet.simple("x", "[i]"))
    st.add_memlet_path(yr, me, t, dst_conn="yi", memlet=Memlet.simple("y", "[i]"))
    st.add_memlet_path(ar, me, t, dst_conn="av", memlet=Memlet.simple("a", "[0]"))
    st.add_memlet_path(t, mx, yw, src_conn="o", memlet=Memlet.simple("y", "[i]"))
    g.finalize()
    return g


def maxabs(n: int = 200, bins: int = 7) -> Sdfg:
    """``out[i % B] = x[i]`` under a custom WCR keeping the smallest
    magnitude (ir.py:100-121 custom WcrFunc with its own identity)."""
    from sdfg.ir import WcrFunc
    from sdfg.tasklets import parse_tasklet
    g = Sdfg("maxabs")
    g.add_array("x", [str(n)], "float64")
    g.add_array("out", [str(bins)], "float64")
    st = g.add_state("main", is_start=True)
    me, mx = st.add_map("i", f"0:{n - 1}")
    t = st.add_tasklet("pick", ["v"], ["o"], "o = v")
    # the reference applies WCR on blocks (interpreter.py:300-303), so the
    # function must be branch-free: smallest magnitude seen so far
    keep = WcrFunc("custom", custom=parse_tasklet("out = min(old, abs(new))", ["old", "new"], ["out"]),
                   custom_identity=1e300)
    st.add_memlet_path(st.add_access("x"), me, t, dst_conn="v", memlet=Memlet.simple("x", "[i]"))
    st.add_memlet_path(t, mx, st.add_access("out"), src_conn="o",
                       memlet=Memlet.simple("out", f"[i % {bins}]", wcr=keep))
    g.finalize()
    return g


def matmul_raw() -> Sdfg:
    return gallery.fixture("matmul").sdfg


def matmul(chain: tuple = ()) -> Sdfg:
    """gallery.matmul -> MapReduceFusion, then the optional paper §5.2 chain.

    ``chain`` items: ("MapTiling", {"tile": 32}) / ("LocalStorage", {"data": "B"}).
    """
    g = matmul_raw()
    g, _ = apply_transformation(g, find_matches(g, "MapReduceFusion")[0])
    for name, params in chain:
        ms = find_matches(g, name)
        if name == "MapTiling":
            # tile the multiplication map (the one in state 'mult')
            ms = [m for m in ms if m.state == "mult"]
        g, _ = apply_transformation(g, ms[0], params)
    return g


BUILDERS = {
    "histogram": histogram,
    "histogram_int": histogram_int,
    "query": query,
    "query_gallery": query_gallery,
    "spmv": spmv,
    "jacobi2d": jacobi2d,
    "laplace1d": laplace1d,
    "matmul": matmul,
    "matmul_tiled": lambda: matmul((("MapTiling", {"tile": 4}),)),
    "matmul_chain": lambda: matmul((("MapTiling", {"tile": 4}),
                                    ("LocalStorage", {"data": "B"}))),
}
