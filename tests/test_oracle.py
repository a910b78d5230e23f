"""Pin the C oracle to the reference: every golden fixture (reference
interpreter outputs, tests/golden/make_golden.py) must be reproduced exactly
(integers) or to the reference's own 1e-9 (floats, test_interpreter.py:16-24)."""

import json
import os
import subprocess

import numpy as np
import pytest

import oracle
from conftest import REPO, load_cases

ORC = os.path.join(REPO, "oracle")


@pytest.fixture(scope="session", autouse=True)
def _built():
    if not os.path.exists(oracle.LIB_PATH):
        subprocess.check_call(["make", "-s", "-C", ORC])


@pytest.mark.parametrize("c", load_cases("histogram") + load_cases("histogram_int"), ids=repr)
def test_histogram(c):
    integer = c.motif == "histogram_int"
    hist, oob = oracle.histogram(c.inputs["img"], c.inputs["hist"], integer=integer)
    if c.error:
        assert c.error == "OutOfBoundsError" and oob > 0
        return
    assert oob == 0
    np.testing.assert_array_equal(hist, c.outputs["hist"])


@pytest.mark.parametrize("c", load_cases("query") + load_cases("query_gallery"), ids=repr)
def test_query(c):
    op = ">" if c.motif == "query_gallery" else "<"
    out, cnt = oracle.query(c.inputs["col"], c.inputs["thr"][0], c.inputs["out_vals"],
                            c.inputs["count"], op=op)
    np.testing.assert_array_equal(out, c.outputs["out_vals"])
    np.testing.assert_array_equal(cnt, c.outputs["count"])


@pytest.mark.parametrize("c", load_cases("spmv"), ids=repr)
def test_spmv(c):
    i = c.inputs
    b = oracle.spmv(i["A_row"], i["A_col"], i["A_val"], i["x"], i["b"])
    # same j-sequential order as the interpreter -> bit-identical
    np.testing.assert_array_equal(b, c.outputs["b"])


@pytest.mark.parametrize("c", load_cases("jacobi2d"), ids=repr)
def test_jacobi2d(c):
    A = oracle.jacobi2d(c.inputs["A"], c.symbols["T"])
    np.testing.assert_array_equal(A, c.outputs["A"])


@pytest.mark.parametrize("c", [x for m in ("matmul", "matmul_raw", "matmul_tiled",
                                            "matmul_chain") for x in load_cases(m)], ids=repr)
def test_matmul(c):
    C = oracle.matmul(c.inputs["A"], c.inputs["B"])
    if c.motif == "matmul_raw":
        # the raw graph reduces with np.add.reduce (interpreter.py:617-619):
        # pairwise order, so only rounding-level agreement
        np.testing.assert_allclose(C, c.outputs["C"], rtol=1e-12)
    else:
        np.testing.assert_array_equal(C, c.outputs["C"])


def test_fp32_jacobi_restatement_close_to_f64():
    rng = np.random.default_rng(0)
    A = np.zeros((2, 40, 40), np.float32)
    A[0, 1:-1, 1:-1] = rng.random((38, 38), dtype=np.float32)
    A[1] = A[0]
    a64 = oracle.jacobi2d(A.astype(np.float64), 30)
    a32 = oracle.jacobi2d(A, 30, fp32=True)
    err = np.linalg.norm(a32 - a64) / np.linalg.norm(a64)
    assert err < 1e-5


@pytest.mark.skipif(not os.path.exists(os.path.join(ORC, "_ref", "manifest.json")),
                    reason="oracle/_ref not built (python oracle/make_ref.py)")
def test_oracle_matches_reference_generated_c():
    """Cross-check the restatement against the reference's own generated C
    (oracle/_ref, codegen.py:802-913) at a size the interpreter cannot reach."""
    import ctypes
    man = json.load(open(os.path.join(ORC, "_ref", "manifest.json")))
    rng = np.random.default_rng(5)

    def call(key, arrays, syms):
        m = man[key]
        L = ctypes.CDLL(os.path.join(ORC, "_ref", m["lib"]))
        fn = getattr(L, m["entry"])
        fn.restype = None
        bufs = []
        for name, bt in m["pointer_args"]:
            bufs.append(np.ascontiguousarray(arrays[name],
                                             dtype=np.int64 if bt == "int64" else np.float64).copy())
        fn(*[ctypes.c_void_p(b.ctypes.data) for b in bufs],
           *[ctypes.c_int64(syms[s]) for s in m["symbol_args"]])
        return {n: b for (n, _), b in zip(m["pointer_args"], bufs)}

    img = rng.random((300, 301), dtype=np.float32).astype(np.float64)
    r = call("histogram", {"img": img, "hist": np.zeros(256, np.int64)}, {"H": 300, "W": 301})
    np.testing.assert_array_equal(r["hist"], oracle.histogram(img, np.zeros(256, np.int64))[0])

    col = rng.random(100000, dtype=np.float32).astype(np.float64)
    r = call("query", {"col": col, "thr": np.array([0.5]), "out_vals": np.zeros(col.size),
                       "count": np.zeros(1, np.int64)}, {"N": col.size})
    out, cnt = oracle.query(col, 0.5, np.zeros(col.size), np.zeros(1, np.int64))
    np.testing.assert_array_equal(r["out_vals"], out)
    np.testing.assert_array_equal(r["count"], cnt)

    A = np.zeros((2, 70, 70))
    A[0, 1:-1, 1:-1] = rng.random((68, 68))
    A[1] = A[0]
    r = call("jacobi2d", {"A": A}, {"N": 70, "T": 9})
    np.testing.assert_array_equal(r["A"].reshape(A.shape), oracle.jacobi2d(A, 9))

    H, W, k = 500, 700, 9
    cols = np.sort(rng.integers(0, W, (H, k)), axis=1).reshape(-1)
    arr = {"A_row": np.arange(H + 1) * k, "A_col": cols, "A_val": rng.random(H * k),
           "x": rng.random(W), "b": rng.random(H)}
    r = call("spmv", arr, {"H": H, "W": W, "nnz": H * k})
    np.testing.assert_array_equal(r["b"], oracle.spmv(arr["A_row"], cols, arr["A_val"],
                                                      arr["x"], arr["b"]))

    Am, Bm = rng.random((33, 65)), rng.random((65, 47))
    for key in ("matmul", "matmul_chain32"):
        r = call(key, {"A": Am, "B": Bm, "C": np.zeros((33, 47))}, {"M": 33, "N": 47, "K": 65})
        np.testing.assert_array_equal(r["C"].reshape(33, 47), oracle.matmul(Am, Bm))
