"""Device-resident entry points over torch CUDA tensors (the timed path).

PyTorch supplies device memory and streams only; every call goes through
the C ABI of libsdfgb200.so (include/sdfgb200.h) on the caller's current
stream.  Used by bench.py, the multi-GPU runners and the GPU parity tests.
"""

from __future__ import annotations

import ctypes

from . import _lib

_KIND = {}


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _require(t, dtype, name):
    import torch
    if not t.is_cuda or t.dtype != dtype or not t.is_contiguous():
        raise TypeError(f"{name}: expected a contiguous CUDA {dtype} tensor, got {t.dtype} on {t.device}")


def hist(img, hist_, oob, scale=256.0, div=1.0, stream=None):
    """hist_[floor(v*scale/div)] += 1 (int64 hist_), oob[0] += #out of range."""
    import torch
    L = _lib.load()
    _require(hist_, torch.int64, "hist")
    _require(oob, torch.int64, "oob")
    n = img.numel()
    if img.dtype == torch.float32:
        rc = L.sdfgb_hist_f32(_p(img), n, scale, div, _p(hist_), hist_.numel(), _p(oob), _stream(stream))
    elif img.dtype == torch.float64:
        rc = L.sdfgb_hist_f64(_p(img), n, scale, div, _p(hist_), hist_.numel(), _p(oob), _stream(stream))
    elif img.dtype == torch.int64:
        rc = L.sdfgb_hist_i64(_p(img), n, _p(hist_), hist_.numel(), _p(oob), _stream(stream))
    else:
        raise TypeError(f"hist: unsupported image dtype {img.dtype}")
    _lib.check(rc)


def query_workspace(n, elem_bytes=4, device=None):
    import torch
    nb = _lib.load().sdfgb_query_workspace_bytes(n, elem_bytes)
    return torch.zeros(nb, dtype=torch.uint8, device=device or "cuda")


def query(col, thr, out, count, ws, op="<", stream=None, ordered=False):
    """out[0:k) = survivors of ``col OP thr``; count[0] += k.  The survivors'
    order is unspecified (concurrent pushes) unless ``ordered``, which keeps
    the input order of the reference's FIFO drain."""
    import torch
    L = _lib.load()
    _require(count, torch.int64, "count")
    fn = {torch.float32: L.sdfgb_query_f32, torch.float64: L.sdfgb_query_f64}.get(col.dtype)
    if fn is None or out.dtype != col.dtype:
        raise TypeError("query: col/out must both be float32 or float64")
    opf = _lib.CMP[op] | (_lib.QUERY_ORDERED if ordered else 0)
    _lib.check(fn(_p(col), col.numel(), opf, float(thr), _p(out), _p(count), _p(ws),
                  ws.numel(), _stream(stream)))


def spmv(rowptr, col, val, x, b, stream=None):
    """b[i] += sum_j val[j] * x[col[j]]."""
    import torch
    L = _lib.load()
    H = b.numel()
    if val.dtype == torch.float32:
        _require(rowptr, torch.int32, "rowptr")
        _require(col, torch.int32, "col")
        rc = L.sdfgb_spmv_csr_f32(_p(rowptr), _p(col), _p(val), _p(x), _p(b), H, _stream(stream))
    else:
        _require(rowptr, torch.int64, "rowptr")
        _require(col, torch.int64, "col")
        rc = L.sdfgb_spmv_csr_f64(_p(rowptr), _p(col), _p(val), _p(x), _p(b), H, _stream(stream))
    _lib.check(rc)


JACOBI5 = ((0, 0), (-1, 0), (1, 0), (0, -1), (0, 1))


def _terms(terms):
    di = (ctypes.c_int32 * len(terms))(*[t[0] for t in terms])
    dj = (ctypes.c_int32 * len(terms))(*[t[1] for t in terms])
    return di, dj


def jacobi2d(A, T, coef=0.2, terms=JACOBI5, stream=None):
    """T steps on A[2, N, N]; result in A[T % 2]."""
    import torch
    L = _lib.load()
    N = A.shape[-1]
    di, dj = _terms(terms)
    fn = {torch.float32: L.sdfgb_jacobi2d_f32, torch.float64: L.sdfgb_jacobi2d_f64}[A.dtype]
    _lib.check(fn(_p(A), N, int(T), float(coef), di, dj, len(terms), _stream(stream)))


def jacobi2d_rect(A, T, coef=0.2, terms=JACOBI5, stream=None):
    """T steps on fp32 A[2, M, N] whose border is the plane edge."""
    L = _lib.load()
    M, N = A.shape[-2], A.shape[-1]
    di, dj = _terms(terms)
    _lib.check(L.sdfgb_jacobi2d_rect_f32(_p(A), M, N, int(T), float(coef), di, dj, len(terms), _stream(stream)))


def jacobi2d_block(src, dst, k, coef=0.2, stream=None):
    """One temporal-blocking launch: k in {1,3,5,7} steps, plane src (state
    t) -> plane dst (state t+k), canonical 5-point order."""
    L = _lib.load()
    M, N = src.shape[-2], src.shape[-1]
    _lib.check(L.sdfgb_jacobi2d_block_f32(_p(src), _p(dst), M, N, int(k), float(coef), _stream(stream)))


def jacobi2d_band(src, dst, k, r0, r1, coef=0.2, stream=None):
    """Rows [r0, r1) of one k-step launch src -> dst (banded
    jacobi2d_block; k > 1 needs N >= 128 and >= 16 rows)."""
    L = _lib.load()
    M, N = src.shape[-2], src.shape[-1]
    _lib.check(L.sdfgb_jacobi2d_band_f32(_p(src), _p(dst), M, N, int(k), int(r0), int(r1), float(coef),
                                         _stream(stream)))


def jacobi2d_band_mirror(src, dst, k, r0, r1, mirror_ptr, m0, m1, coef=0.2, stream=None):
    """jacobi2d_band, its output rows r in [m0, m1) also stored at
    mirror_ptr + (r - m0) rows (a raw device address: a neighbour's ghost
    rows in peer memory)."""
    L = _lib.load()
    M, N = src.shape[-2], src.shape[-1]
    _lib.check(L.sdfgb_jacobi2d_band_mirror_f32(_p(src), _p(dst), M, N, int(k), int(r0), int(r1), float(coef),
                                                ctypes.c_void_p(int(mirror_ptr)), int(m0), int(m1),
                                                _stream(stream)))


def flag_signal(flag_ptr, value, stream=None):
    """Stream-ordered: store ``value`` into the int32 flag at ``flag_ptr``
    (system-scope release) after the work queued before it."""
    _lib.check(_lib.load().sdfgb_flag_signal(ctypes.c_void_p(int(flag_ptr)), int(value), _stream(stream)))


def flag_wait(flag_ptr, value, stream=None):
    """Stream-ordered: hold the stream until the int32 flag at ``flag_ptr``
    reaches ``value``."""
    _lib.check(_lib.load().sdfgb_flag_wait(ctypes.c_void_p(int(flag_ptr)), int(value), _stream(stream)))


def jacobi2d_step(src, dst, N, rows, g0, r0, r1, coef=0.2, terms=JACOBI5, stream=None):
    L = _lib.load()
    di, dj = _terms(terms)
    _lib.check(L.sdfgb_jacobi2d_step_f32(_p(src), _p(dst), N, rows, g0, r0, r1, float(coef), di, dj,
                                         len(terms), _stream(stream)))


def gemm_workspace(M, N, K, device=None):
    import torch
    nb = _lib.load().sdfgb_gemm_workspace_bytes(M, N, K)
    return torch.empty(nb, dtype=torch.uint8, device=device or "cuda")


def gemm(A, B, C, ws, stream=None, b_split=False):
    """C = A @ B (fp32, 3xTF32 tcgen05).  ``b_split``: B's split operands
    are already in ``ws`` from an earlier call with this B (row pieces of
    one product split B once)."""
    import torch
    L = _lib.load()
    for t, n in ((A, "A"), (B, "B"), (C, "C")):
        _require(t, torch.float32, n)
    M, K = A.shape
    N = B.shape[1]
    _lib.check(L.sdfgb_gemm_f32_ex(_p(A), _p(B), _p(C), M, N, K, _p(ws), ws.numel(),
                                   _lib.GEMM_B_SPLIT if b_split else 0, _stream(stream)))


def gemm_f64(A, B, C, stream=None):
    """C = A @ B in float64, each element summed in k order with separately
    rounded multiply and add (the reference's MapReduceFusion loop)."""
    import torch
    L = _lib.load()
    for t, n in ((A, "A"), (B, "B"), (C, "C")):
        _require(t, torch.float64, n)
    M, K = A.shape
    N = B.shape[1]
    _lib.check(L.sdfgb_gemm_f64(_p(A), _p(B), _p(C), M, N, K, _stream(stream)))


def gemm_simt(A, B, C, stream=None):
    L = _lib.load()
    M, K = A.shape
    N = B.shape[1]
    _lib.check(L.sdfgb_gemm_f32_simt(_p(A), _p(B), _p(C), M, N, K, _stream(stream)))
