"""numpy front of the C oracle (TEST INFRASTRUCTURE -- never the product path).

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline leg
may import this module.  It loads ``oracle/_build/liboracle.so`` (built by
``__graft_entry__.build()`` / ``make -C oracle``) and exposes one function per
motif with the reference's semantics; see oracle.c for the file:line
citations into the reference.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_F64 = ctypes.c_double
_F32 = ctypes.c_float

CMP_OPS = {"<": 0, "<=": 1, ">": 2, ">=": 3, "==": 4, "!=": 5}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"oracle library missing: {LIB_PATH} (run make -C oracle)")
        L = ctypes.CDLL(LIB_PATH)
        sig = {
            "orc_histogram_f64": (_I64, [_P, _I64, _P, _I64, _F64, _F64]),
            "orc_histogram_f32": (_I64, [_P, _I64, _P, _I64, _F64, _F64]),
            "orc_histogram_i64": (_I64, [_P, _I64, _P, _I64]),
            "orc_query_f64": (_I64, [_P, _I64, ctypes.c_int, _F64, _P, _P]),
            "orc_query_f32": (_I64, [_P, _I64, ctypes.c_int, _F64, _P, _P]),
            "orc_spmv_f64": (None, [_P, _P, _P, _P, _P, _I64]),
            "orc_spmv_f32": (None, [_P, _P, _P, _P, _P, _I64]),
            "orc_jacobi2d_f64": (None, [_P, _I64, _I64, _F64, _P, _P, _I32]),
            "orc_jacobi2d_f32": (None, [_P, _I64, _I64, _F32, _P, _P, _I32]),
            "orc_matmul_f64": (None, [_P, _P, _P, _I64, _I64, _I64, _I64, _I64]),
            "orc_matmul_f32in_f64acc": (None, [_P, _P, _P, _I64, _I64, _I64, _I64, _I64]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a):
    return a.ctypes.data


JACOBI5 = ((0, 0), (-1, 0), (1, 0), (0, -1), (0, 1))  # c, n, s, w, e


def histogram(img, hist_in, scale=256.0, div=1.0, integer=False):
    """Returns (hist, n_out_of_bounds)."""
    hist = _c(hist_in, np.int64).copy()
    if integer:
        x = _c(img, np.int64).reshape(-1)
        oob = lib().orc_histogram_i64(_p(x), x.size, _p(hist), hist.size)
    elif np.asarray(img).dtype == np.float32:
        x = _c(img, np.float32).reshape(-1)
        oob = lib().orc_histogram_f32(_p(x), x.size, _p(hist), hist.size, scale, div)
    else:
        x = _c(img, np.float64).reshape(-1)
        oob = lib().orc_histogram_f64(_p(x), x.size, _p(hist), hist.size, scale, div)
    return hist, int(oob)


def query(col, thr, out_vals_in, count_in, op="<"):
    """Returns (out_vals, count); out_vals dtype follows col."""
    f32 = np.asarray(col).dtype == np.float32
    dt = np.float32 if f32 else np.float64
    x = _c(col, dt).reshape(-1)
    out = _c(out_vals_in, dt).reshape(-1).copy()
    cnt = _c(count_in, np.int64).reshape(-1).copy()
    fn = lib().orc_query_f32 if f32 else lib().orc_query_f64
    fn(_p(x), x.size, CMP_OPS[op], float(thr), _p(out), _p(cnt))
    return out, cnt


def spmv(rowptr, col, val, x, b_in, fp32=False):
    if fp32:
        rp, ci = _c(rowptr, np.int32), _c(col, np.int32)
        v, xx = _c(val, np.float32), _c(x, np.float32)
        b = _c(b_in, np.float32).copy()
        lib().orc_spmv_f32(_p(rp), _p(ci), _p(v), _p(xx), _p(b), b.size)
    else:
        rp, ci = _c(rowptr, np.int64), _c(col, np.int64)
        v, xx = _c(val, np.float64), _c(x, np.float64)
        b = _c(b_in, np.float64).copy()
        lib().orc_spmv_f64(_p(rp), _p(ci), _p(v), _p(xx), _p(b), b.size)
    return b


def jacobi2d(A_in, T, coef=0.2, terms=JACOBI5, fp32=False):
    dt = np.float32 if fp32 else np.float64
    A = _c(A_in, dt).copy()
    N = A.shape[-1]
    di = np.array([t[0] for t in terms], np.int32)
    dj = np.array([t[1] for t in terms], np.int32)
    fn = lib().orc_jacobi2d_f32 if fp32 else lib().orc_jacobi2d_f64
    fn(_p(A), N, int(T), coef, _p(di), _p(dj), len(terms))
    return A


def matmul(A, B, rows=None):
    """C = A @ B with k-sequential accumulation; ``rows`` = (r0, r1) sample."""
    M, K = np.shape(A)
    N = np.shape(B)[1]
    r0, r1 = rows if rows is not None else (0, M)
    if np.asarray(A).dtype == np.float32 and np.asarray(B).dtype == np.float32:
        a, b = _c(A, np.float32), _c(B, np.float32)
        C = np.zeros((r1 - r0, N), np.float64)
        lib().orc_matmul_f32in_f64acc(_p(a), _p(b), _p(C), M, N, K, r0, r1)
        return C
    a, b = _c(A, np.float64), _c(B, np.float64)
    C = np.zeros((M, N), np.float64)
    lib().orc_matmul_f64(_p(a), _p(b), _p(C), M, N, K, r0, r1)
    return C[r0:r1]


# ------------------------------------------------ the reference's own C

REF_DIR = os.path.join(HERE, "_ref")


def ref_available(key: str = None) -> bool:
    man = os.path.join(REF_DIR, "manifest.json")
    if not os.path.exists(man):
        return False
    if key is None:
        return True
    import json
    return key in json.load(open(man))


def ref_call(key: str, arrays: dict, syms: dict) -> dict:
    """Call the reference's own generated C (oracle/_ref, built by
    make_ref.py from codegen.generate + invoke_toolchain) the way
    CompiledSdfg.run does (codegen.py:875-887); returns the buffers."""
    import json
    m = json.load(open(os.path.join(REF_DIR, "manifest.json")))[key]
    L = ctypes.CDLL(os.path.join(REF_DIR, m["lib"]))
    fn = getattr(L, m["entry"])
    fn.restype = None
    bufs = []
    for name, bt in m["pointer_args"]:
        bufs.append(np.ascontiguousarray(arrays[name], dtype=np.int64 if bt == "int64" else np.float64).copy())
    fn(*[ctypes.c_void_p(b.ctypes.data) for b in bufs], *[ctypes.c_int64(syms[s]) for s in m["symbol_args"]])
    return {n: b for (n, _), b in zip(m["pointer_args"], bufs)}
