"""Generate the golden fixtures from the REFERENCE (run in the build container).

    python tests/golden/make_golden.py

Outputs (committed):
  tests/golden/graphs/<motif>.sdfg.json   reference canonical JSON (serialization.to_json)
  tests/golden/cases/<motif>__<case>.npz  inputs, symbols, interpreter outputs
                                          (or the reference's error class name)

Every output comes from ``sdfg.interpreter.run`` (interpreter.py:767-832), the
reference's ground-truth executor; the reference's KATs
(test_interpreter.py:45-82, test_acceptance.py:87-96) are reproduced as named
cases.  Nothing here is imported by the product.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import motifs_ref as M  # noqa: E402
from sdfg.interpreter import run  # noqa: E402
from sdfg.serialization import to_json  # noqa: E402

GRAPHS = os.path.join(HERE, "graphs")
CASES = os.path.join(HERE, "cases")

F32 = np.float32


def f32(a):
    """fp32-representable float64 data (BASELINE inputs are fp32)."""
    return np.asarray(a, dtype=F32).astype(np.float64)


def save_graph(name, g):
    os.makedirs(GRAPHS, exist_ok=True)
    with open(os.path.join(GRAPHS, f"{name}.sdfg.json"), "w") as f:
        json.dump(to_json(g), f, sort_keys=True, indent=1)


def save_case(motif, case, g, arrays, symbols):
    os.makedirs(CASES, exist_ok=True)
    payload = {f"in__{k}": np.asarray(v) for k, v in arrays.items()}
    payload["symbols"] = np.array(json.dumps({k: int(v) for k, v in symbols.items()}))
    try:
        rep = run(g, arrays, symbols)
        for k, v in rep.outputs.items():
            payload[f"out__{k}"] = v
        payload["states"] = np.array(json.dumps(rep.states_visited))
        payload["moved"] = np.array(json.dumps(rep.elements_moved))
        payload["tasklets"] = np.array(int(rep.tasklet_invocations))
        payload["error"] = np.array("")
    except Exception as exc:  # the reference's error class is part of the contract
        payload["error"] = np.array(type(exc).__name__)
        payload["error_msg"] = np.array(str(exc))
    np.savez_compressed(os.path.join(CASES, f"{motif}__{case}.npz"), **payload)
    print(f"{motif}__{case}: error={payload['error']}")


def histogram_cases():
    g = M.histogram()
    save_graph("histogram", g)
    rng = np.random.default_rng(0)
    for case, (H, W) in {"16x16": (16, 16), "64x64": (64, 64), "1x1": (1, 1),
                         "3x37": (3, 37)}.items():
        img = f32(rng.random((H, W), dtype=F32))
        save_case("histogram", case, g, {"img": img, "hist": np.zeros(256, np.int64)},
                  {"H": H, "W": W})
    # accumulate into existing contents (gallery.py:374-377 semantics)
    img = f32(rng.random((8, 8), dtype=F32))
    save_case("histogram", "accumulate", g,
              {"img": img, "hist": rng.integers(0, 1000, 256).astype(np.int64)},
              {"H": 8, "W": 8})
    # exact bin boundaries k/256 and the largest fp32 below 1
    edges = np.concatenate([np.arange(256) / 256.0,
                            [np.nextafter(F32(1), F32(0))], [0.0]]).astype(F32)
    save_case("histogram", "boundaries", g,
              {"img": f32(edges.reshape(1, -1)), "hist": np.zeros(256, np.int64)},
              {"H": 1, "W": edges.size})
    # out-of-range bin -> reference raises OutOfBoundsError (interpreter.py:265-268)
    bad = f32(np.array([[0.5, 1.0]], dtype=F32))
    save_case("histogram", "oob_high", g, {"img": bad, "hist": np.zeros(256, np.int64)},
              {"H": 1, "W": 2})
    bad = f32(np.array([[-0.25, 0.5]], dtype=F32))
    save_case("histogram", "oob_low", g, {"img": bad, "hist": np.zeros(256, np.int64)},
              {"H": 1, "W": 2})

    gi = M.histogram_int()
    save_graph("histogram_int", gi)
    from sdfg.gallery import fixture
    fx = fixture("histogram")
    for seed in range(3):
        arrays, symbols = fx.make_inputs(np.random.default_rng(seed))
        save_case("histogram_int", f"seed{seed}", gi, arrays, symbols)


def query_cases():
    g = M.query("<")
    save_graph("query", g)
    rng = np.random.default_rng(1)
    for case, N in {"n4096": 4096, "n1": 1, "n1000": 1000, "n33": 33}.items():
        col = f32(rng.random(N, dtype=F32))
        save_case("query", case, g,
                  {"col": col, "thr": np.array([0.5]), "out_vals": np.zeros(N),
                   "count": np.zeros(1, np.int64)}, {"N": N})
    N = 64
    col = f32(rng.random(N, dtype=F32))
    col[::7] = 0.5  # ties with the threshold are rejected by '<'
    save_case("query", "ties_accumulate", g,
              {"col": col, "thr": np.array([0.5]),
               "out_vals": f32(rng.random(N, dtype=F32)),  # tail must stay untouched
               "count": np.array([7], np.int64)}, {"N": N})
    save_case("query", "none_pass", g,
              {"col": np.ones(40), "thr": np.array([0.5]), "out_vals": np.full(40, 3.0),
               "count": np.zeros(1, np.int64)}, {"N": 40})
    save_case("query", "all_pass", g,
              {"col": np.zeros(40), "thr": np.array([0.5]), "out_vals": np.zeros(40),
               "count": np.zeros(1, np.int64)}, {"N": 40})
    save_case("query", "n0", g,
              {"col": np.zeros(0), "thr": np.array([0.5]), "out_vals": np.zeros(0),
               "count": np.zeros(1, np.int64)}, {"N": 0})

    gq = M.query_gallery()
    save_graph("query_gallery", gq)
    # KAT test_interpreter.py:76-82
    save_case("query_gallery", "kat", gq,
              {"col": np.array([1.0, 6.0, 3.0, 8.0]), "thr": np.array([5.0]),
               "out_vals": np.zeros(4), "count": np.zeros(1, np.int64)}, {"N": 4})
    from sdfg.gallery import fixture
    fx = fixture("query")
    for seed in range(3):
        arrays, symbols = fx.make_inputs(np.random.default_rng(seed))
        save_case("query_gallery", f"seed{seed}", gq, arrays, symbols)


def spmv_inputs(rng, H, W, nnz_row, y_in=False):
    cols = np.sort(rng.integers(0, W, size=(H, nnz_row)), axis=1).reshape(-1)
    return ({"A_row": (np.arange(H + 1) * nnz_row).astype(np.int64),
             "A_col": cols.astype(np.int64),
             "A_val": f32(rng.random(H * nnz_row, dtype=F32)),
             "x": f32(rng.random(W, dtype=F32)),
             "b": f32(rng.random(H, dtype=F32)) if y_in else np.zeros(H)},
            {"H": H, "W": W, "nnz": H * nnz_row})


def spmv_cases():
    g = M.spmv()
    save_graph("spmv", g)
    # KAT test_interpreter.py:56-67
    save_case("spmv", "kat", g,
              {"A_row": np.array([0, 1, 3], np.int64), "A_col": np.array([1, 0, 2], np.int64),
               "A_val": np.array([2.0, 3.0, 4.0]), "x": np.array([1.0, 2.0, 3.0]),
               "b": np.zeros(2)}, {"H": 2, "W": 3, "nnz": 3})
    rng = np.random.default_rng(3)
    a, s = spmv_inputs(rng, 128, 128, 16)
    save_case("spmv", "h128_nnz16", g, a, s)
    a, s = spmv_inputs(rng, 64, 200, 64, y_in=True)
    save_case("spmv", "h64_nnz64_accumulate", g, a, s)
    # ragged rows incl. empty rows
    lens = np.array([0, 3, 0, 1, 7, 33, 0, 2])
    rowptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    nnz = int(rowptr[-1])
    save_case("spmv", "ragged", g,
              {"A_row": rowptr, "A_col": rng.integers(0, 50, nnz).astype(np.int64),
               "A_val": f32(rng.random(nnz, dtype=F32)), "x": f32(rng.random(50, dtype=F32)),
               "b": np.zeros(8)}, {"H": 8, "W": 50, "nnz": nnz})
    from sdfg.gallery import fixture
    fx = fixture("spmv")
    for seed in range(3):
        arrays, symbols = fx.make_inputs(np.random.default_rng(seed))
        save_case("spmv", f"gallery_seed{seed}", g, arrays, symbols)


def jacobi_inputs(rng, N, border=False, distinct=False):
    A = np.zeros((2, N, N), dtype=F32)
    A[0, 1:N - 1, 1:N - 1] = rng.random((N - 2, N - 2), dtype=F32) if N > 2 else 0
    if border:
        A[0, 0, :] = rng.random(N, dtype=F32)
        A[0, :, -1] = rng.random(N, dtype=F32)
    A[1] = A[0]
    if distinct:
        A[1] = rng.random((N, N), dtype=F32)
    return f32(A)


def jacobi_cases():
    g = M.jacobi2d()
    save_graph("jacobi2d", g)
    rng = np.random.default_rng(2)
    for case, (N, T, kw) in {"n16_t3": (16, 3, {}), "n5_t1": (5, 1, {}),
                             "n3_t2": (3, 2, {}), "n12_t0": (12, 0, {}),
                             "n13_t4_border": (13, 4, {"border": True}),
                             "n9_t3_distinct": (9, 3, {"distinct": True}),
                             "n24_t6": (24, 6, {})}.items():
        save_case("jacobi2d", case, g, {"A": jacobi_inputs(rng, N, **kw)}, {"N": N, "T": T})

    gl = M.laplace1d()
    save_graph("laplace1d", gl)
    # KAT test_interpreter.py:45-49
    save_case("laplace1d", "ramp", gl,
              {"A": np.array([[0, 1, 2, 3, 4], [0, 0, 0, 0, 0]], dtype=float)}, {"N": 5, "T": 1})


def matmul_cases():
    for name, b in (("matmul", M.matmul), ("matmul_raw", M.matmul_raw),
                    ("matmul_tiled", M.BUILDERS["matmul_tiled"]),
                    ("matmul_chain", M.BUILDERS["matmul_chain"])):
        g = b()
        save_graph(name, g)
    g = M.matmul()
    rng = np.random.default_rng(4)
    for case, (m, n, k) in {"16x16x16": (16, 16, 16), "5x7x3": (5, 7, 3),
                            "1x1x1": (1, 1, 1), "24x8x40": (24, 8, 40)}.items():
        save_case("matmul", case, g,
                  {"A": f32(rng.random((m, k), dtype=F32)), "B": f32(rng.random((k, n), dtype=F32)),
                   "C": f32(rng.random((m, n), dtype=F32))}, {"M": m, "N": n, "K": k})
    # KAT test_interpreter.py:69-74 (identity operand)
    save_case("matmul", "identity", g,
              {"A": np.eye(2), "B": np.array([[1.0, 2.0], [3.0, 4.0]]), "C": np.zeros((2, 2))},
              {"M": 2, "N": 2, "K": 2})
    for name in ("matmul_raw", "matmul_tiled", "matmul_chain"):
        gg = {"matmul_raw": M.matmul_raw, "matmul_tiled": M.BUILDERS["matmul_tiled"],
              "matmul_chain": M.BUILDERS["matmul_chain"]}[name]()
        save_case(name, "6x9x5", gg,
                  {"A": f32(rng.random((6, 5), dtype=F32)), "B": f32(rng.random((5, 9), dtype=F32)),
                   "C": np.zeros((6, 9))}, {"M": 6, "N": 9, "K": 5})


def gallery_cases():
    """The reference gallery (gallery.py:55-545) for the generic lowering:
    graphs gal_<name>, inputs from each fixture's own make_inputs plus a
    few larger / edge cases, outputs from the interpreter."""
    from sdfg import gallery
    for name in gallery.fixture_names():
        fx = gallery.fixture(name)
        save_graph(f"gal_{name}", fx.sdfg)
        for seed in (0, 1, 2):
            arrays, symbols = fx.make_inputs(np.random.default_rng(100 + seed))
            save_case(f"gal_{name}", f"seed{seed}", fx.sdfg, arrays, symbols)
    rng = np.random.default_rng(7)
    g = gallery.fixture("laplace").sdfg
    save_case("gal_laplace", "n300_t9", g, {"A": rng.random((2, 300))}, {"N": 300, "T": 9})
    g = gallery.fixture("mandelbrot").sdfg
    save_case("gal_mandelbrot", "12x9_k40", g,
              {"CR": rng.uniform(-2, 0.5, 12), "CI": rng.uniform(-1.2, 1.2, 9),
               "IT": np.zeros((9, 12), dtype=np.int64)}, {"W": 12, "H": 9, "K": 40})
    g = gallery.fixture("indirection").sdfg
    save_case("gal_indirection", "w50_m200", g,
              {"x": rng.random(50), "ind": rng.integers(0, 50, 200), "y": np.zeros(200)}, {"W": 50, "M": 200})
    save_case("gal_indirection", "oob", g,
              {"x": rng.random(5), "ind": np.array([0, 7, 2]), "y": np.zeros(3)}, {"W": 5, "M": 3})
    g = gallery.fixture("histogram").sdfg
    fx = gallery.fixture("histogram")
    arrays, symbols = fx.make_inputs(np.random.default_rng(11))
    save_case("gal_histogram", "again", g, arrays, symbols)
    save_case("gal_fibonacci", "n20_p4", gallery.fixture("fibonacci").sdfg,
              {"n_in": np.array([20], dtype=np.int64), "out": np.zeros(1, dtype=np.int64)}, {"P": 4})
    for a in (0, 3, -1):
        save_case("gal_branching", f"a{a}".replace("-", "m"), gallery.fixture("branching").sdfg,
                  {"a": np.array([a], dtype=np.int64), "out": np.zeros(1, dtype=np.int64)}, {})


def transformed_cases():
    """Each motif graph after each reference transformation that matches it
    (the dispatcher must accept these unchanged in result):
    graphs x_<motif>_<transformation>, interpreter outputs on small inputs."""
    from sdfg.rewriting import apply_transformation, find_matches, registry
    rng = np.random.default_rng(21)
    col = f32(rng.random(300, dtype=F32))
    inputs = {
        "histogram": ({"img": f32(rng.random((12, 17), dtype=F32)), "hist": np.zeros(256, np.int64)},
                      {"H": 12, "W": 17}),
        "query": ({"col": col, "thr": np.array([0.5]), "out_vals": np.zeros(300),
                   "count": np.array([4], np.int64)}, {"N": 300}),
        "spmv": spmv_inputs(rng, 40, 60, 9),
        "jacobi2d": ({"A": jacobi_inputs(rng, 19, border=True, distinct=True)}, {"N": 19, "T": 5}),
        "matmul": ({"A": f32(rng.random((7, 11), dtype=F32)), "B": f32(rng.random((11, 6), dtype=F32)),
                    "C": np.zeros((7, 6))}, {"M": 7, "N": 6, "K": 11}),
    }
    builders = {"histogram": M.histogram, "query": lambda: M.query("<"), "spmv": M.spmv,
                "jacobi2d": M.jacobi2d, "matmul": M.matmul}
    from sdfg import gallery
    for name in gallery.fixture_names():
        fx = gallery.fixture(name)
        builders[f"gal_{name}"] = (lambda fx=fx: gallery.fixture(fx.name).sdfg)
        inputs[f"gal_{name}"] = fx.make_inputs(np.random.default_rng(300))
    for motif, build in builders.items():
        g = build()
        for tname in sorted(registry):
            try:
                ms = find_matches(g, tname)
            except Exception:
                continue
            if not ms:
                continue
            try:
                g2, _ = apply_transformation(g, ms[0], {})
            except Exception:
                continue
            name = f"x_{motif}_{tname}"
            save_graph(name, g2)
            arrays, symbols = inputs[motif]
            save_case(name, "small", g2, {k: np.array(v, copy=True) for k, v in arrays.items()}, symbols)


def xform_fixture_cases():
    """The reference's transformation micro-programs (tests/xform_fixtures.py:
    nested_scale, flat_scale_2d, two_stage_pipeline, scale_1d,
    looped_pipeline, two_states, nested_invoke, copy_chain, tiled_matmul)
    as graphs xf_<name>, and each after every registered transformation that
    matches it as x_xf_<name>_<rule> -- interpreter outputs on the fixture's
    own input generator."""
    import importlib.util
    from sdfg.rewriting import apply_transformation, find_matches, registry
    spec = importlib.util.spec_from_file_location(
        "xform_fixtures", os.path.join(os.path.dirname(M.REF_SRC), "tests", "xform_fixtures.py"))
    xf = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(xf)
    names = ["nested_scale", "flat_scale_2d", "two_stage_pipeline", "scale_1d", "looped_pipeline", "two_states",
             "nested_invoke", "copy_chain", "tiled_matmul"]
    for k, name in enumerate(names):
        fx = getattr(xf, name)()
        arrays, symbols = fx.make_inputs(np.random.default_rng(400 + k))
        base = f"xf_{name}"
        save_graph(base, fx.sdfg)
        save_case(base, "fx", fx.sdfg, {a: np.array(v, copy=True) for a, v in arrays.items()}, symbols)
        for tname in sorted(registry):
            try:
                ms = find_matches(fx.sdfg, tname)
            except Exception:
                continue
            if not ms:
                continue
            try:
                g2, _ = apply_transformation(fx.sdfg, ms[0], {})
            except Exception:
                continue
            gname = f"x_xf_{name}_{tname}"
            save_graph(gname, g2)
            save_case(gname, "fx", g2, {a: np.array(v, copy=True) for a, v in arrays.items()}, symbols)
    # the acceptance suite's own parameterisations (test_acceptance.py:125-138)
    accept = {"MapExpansion": ("flat_scale_2d", {"split": 1}), "MapTiling": ("scale_1d", {"tile": 4}),
              "LocalStorage": ("tiled_matmul", {"data": "B"}), "Vectorization": ("scale_1d", {"width": 4})}
    for tname, (name, params) in accept.items():
        fx = getattr(xf, name)()
        arrays, symbols = fx.make_inputs(np.random.default_rng(500 + len(tname)))
        g2, _ = apply_transformation(fx.sdfg, find_matches(fx.sdfg, tname)[0], params)
        gname = f"x_xf_{name}_{tname}_acc"
        save_graph(gname, g2)
        save_case(gname, "acc", g2, {a: np.array(v, copy=True) for a, v in arrays.items()}, symbols)


def vector_cases():
    """Vectorization (library.py:763-840): an element-wise map widened to 4-
    and 8-lane tiles; the same inputs through the plain graph."""
    from sdfg.rewriting import apply_transformation, find_matches
    rng = np.random.default_rng(31)
    arrays = {"x": rng.random(64), "y": rng.random(64), "a": np.array([1.75])}
    g = M.axpy(64)
    save_graph("axpy", g)
    save_case("axpy", "n64", g, dict(arrays), {})
    for w in (4, 8):
        gv, _ = apply_transformation(g, find_matches(g, "Vectorization")[0], {"width": w})
        save_graph(f"x_axpy_Vectorization{w}", gv)
        save_case(f"x_axpy_Vectorization{w}", "n64", gv, {k: v.copy() for k, v in arrays.items()}, {})


def oob_cases():
    """test_interpreter.py:176-189: a static memlet read past the container
    raises (InterpreterError naming the memlet)."""
    from sdfg.ir import Memlet as Mm, Sdfg as Sg
    g = Sg("oob")
    g.add_array("x", ["4"], "float64")
    g.add_array("y", ["4"], "float64")
    st = g.add_state("s", is_start=True)
    t = st.add_tasklet("t", ["a"], ["b"], "b = a")
    st.add_edge(st.add_access("x"), None, t, "a", Mm.simple("x", "[7]"))
    st.add_edge(t, "b", st.add_access("y"), None, Mm.simple("y", "[0]"))
    g.finalize()
    save_graph("oob", g)
    save_case("oob", "read7", g, {"x": np.zeros(4), "y": np.zeros(4)}, {})


def custom_wcr_cases():
    g = M.maxabs(200, 7)
    save_graph("maxabs", g)
    rng = np.random.default_rng(41)
    save_case("maxabs", "n200", g, {"x": rng.uniform(-1, 1, 200), "out": np.full(7, 0.5)}, {})


def control_flow_cases():
    """Motifs under non-trivial control flow: a histogram run
    three times by a guard loop, a query behind a symbol condition.  The
    motif kernels run a state once, so these must take the generic
    lowering, whose state machine follows the interpreter's."""
    g = M.histogram_looped(3)
    save_graph("histogram_looped", g)
    rng = np.random.default_rng(5)
    img = f32(rng.random((4, 4), dtype=F32))
    save_case("histogram_looped", "r3", g, {"img": img, "hist": np.zeros(256, np.int64)}, {"H": 4, "W": 4})
    q = M.query_cond()
    save_graph("query_cond", q)
    for case, N in {"n16": 16, "n8": 8}.items():
        col = f32(rng.random(N, dtype=F32))
        save_case("query_cond", case, q,
                  {"col": col, "thr": np.array([0.5]), "out_vals": np.zeros(N),
                   "count": np.zeros(1, np.int64)}, {"N": N})


if __name__ == "__main__" and len(sys.argv) > 1:
    for fn in sys.argv[1:]:
        globals()[fn]()
elif __name__ == "__main__":
    control_flow_cases()
    xform_fixture_cases()
    oob_cases()
    custom_wcr_cases()
    vector_cases()
    transformed_cases()
    gallery_cases()
    histogram_cases()
    query_cases()
    spmv_cases()
    jacobi_cases()
    matmul_cases()
