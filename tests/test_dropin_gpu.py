"""The drop-in boundary on the GPU (round 2): the per-graph shims with the
reference's exact ``void <name>(...)`` signature, the host entries' staging
(lossless narrowing in native precision, declared rounding in fp32), their
error paths, and the BASELINE configurations at full size through them.

Rules as in test_gpu_parity.py: histogram and query bit-exact (query as a
sorted set unless FIFO), Jacobi bit-exact against the fp32 restatement and
<= 1e-4 normwise against the reference's own float64 C, SpMV 1e-5 rel.
"""

import ctypes
import json

import numpy as np
import pytest

import oracle
from conftest import graph_path, load_cases

import paper_1902_10345_b200 as b200
from paper_1902_10345_b200 import _lib

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def marked(name, precision, order="any"):
    doc = json.load(open(graph_path(name)))
    for d in doc["data"]:
        if not d["transient"]:
            d["storage"] = f"GPU_Global:{precision}" + (":fifo" if order == "fifo" else "")
    return doc


def _vp(a):
    return ctypes.c_void_p(a.ctypes.data)


# ----------------------------------------------------- the reference's call

@pytest.mark.parametrize("name", ["histogram", "query", "spmv", "jacobi2d", "matmul", "histogram_int"])
def test_shim_called_exactly_like_compiled_sdfg_run(name):
    """CompiledSdfg.run (codegen.py:875-887) verbatim against the B200 shim:
    ctypes.CDLL, getattr(lib, code.name), restype None, contiguous copies
    passed as typed pointers, then the int64 symbols.  Results equal the
    reference interpreter's fixtures."""
    code = b200.generate(marked(name, "native", "fifo"))
    lib = ctypes.CDLL(b200.dispatch.build_shim(code))
    fn = getattr(lib, code.name)
    fn.restype = None
    case = [c for c in load_cases(name) if not c.error][0]
    buffers, args = {}, []
    for cname, bt in code.pointer_args:
        dt = np.int64 if bt == "int64" else np.float64
        buf = np.ascontiguousarray(np.asarray(case.inputs[cname], dtype=dt)).copy()
        buffers[cname] = buf
        args.append(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_int64 if bt == "int64" else ctypes.c_double)))
    for sym in code.symbol_args:
        args.append(ctypes.c_int64(int(case.symbols[sym])))
    fn(*args)
    assert _lib.load().sdfgb_last_status() == _lib.OK, _lib.load().sdfgb_last_error()
    for k, exp in case.outputs.items():
        got = buffers[k].reshape(exp.shape)
        if name == "spmv" and exp.dtype.kind == "f":
            np.testing.assert_allclose(got, exp, rtol=1e-12, atol=1e-12 * np.abs(exp).max())
        else:
            np.testing.assert_array_equal(got, exp, err_msg=k)


def test_shim_reports_out_of_bounds_through_the_status():
    case = [c for c in load_cases("histogram") if c.error][0]
    prog = b200.invoke_toolchain(b200.generate(marked("histogram", "native")))
    with pytest.raises(b200.OutOfBoundsError):
        prog.run(case.inputs, case.symbols)
    assert _lib.load().sdfgb_last_status() == _lib.ERR_OOB


# ------------------------------------------- native precision stays exact

def test_native_histogram_bins_values_rounding_would_move():
    """v in [1 - 2^-25, 1) rounds to 1.0f: fp32 would bin it to 256 (out of
    bounds).  Native precision narrows toward -inf, so it lands in bin 255
    like the reference's float64 binning; likewise just below every edge."""
    rng = np.random.default_rng(1)
    H, W = 1500, 3001  # > one staging slot, ragged
    img = rng.random((H, W))
    edges = (np.arange(1, 257) / 256.0)
    img.flat[: 256 * 40] = np.repeat(np.nextafter(edges, 0), 40)
    img.flat[-5:] = 1 - 2.0 ** -25
    hist = rng.integers(0, 9, 256).astype(np.int64)
    ref, bad = oracle.histogram(img, hist)
    assert bad == 0
    got = hist.copy()
    _lib.check(_lib.load().sdfgb_host_histogram(_vp(img), _vp(got), H, W, 256, 256.0, 1.0, _lib.PREC_NATIVE))
    np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("scale,div", [(100.0, 1.0), (256.0, 3.0)])
def test_native_histogram_general_binning_keeps_float64(scale, div):
    rng = np.random.default_rng(2)
    img = rng.random((700, 900)) * 2.55
    bins = 256
    ref, bad = oracle.histogram(img, np.zeros(bins, np.int64), scale, div)
    got = np.zeros(bins, np.int64)
    rc = _lib.load().sdfgb_host_histogram(_vp(img), _vp(got), 700, 900, bins, scale, div, _lib.PREC_NATIVE)
    if bad:
        assert rc == _lib.ERR_OOB
    else:
        _lib.check(rc)
        np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("ordered", [False, True])
def test_native_query_mixed_exact_and_inexact_chunks(ordered):
    """Chunks whose values all round-trip ship as fp32, the others as
    float64; survivors are the reference's either way (FIFO: same order)."""
    rng = np.random.default_rng(3)
    N = 5_000_003  # several staging chunks
    col = rng.random(N, dtype=np.float32).astype(np.float64)
    col[1_500_000] = 0.5 - 2.0 ** -40  # not an fp32 value: that chunk keeps float64
    col[1_500_001] = np.nextafter(0.5, 0)
    col[4_999_000] = np.nan
    out = np.full(N, -1.0)
    cnt = np.array([5], np.int64)
    ref_out, ref_cnt = oracle.query(col, 0.5, out.copy(), cnt.copy())
    thr = np.array([0.5])
    op = _lib.CMP["<"] | (_lib.QUERY_ORDERED if ordered else 0)
    _lib.check(_lib.load().sdfgb_host_query(_vp(col), _vp(thr), _vp(out), _vp(cnt), N, op, _lib.PREC_NATIVE))
    k = int(ref_cnt[0] - 5)
    assert cnt[0] == ref_cnt[0]
    assert (out[:k] == 0.5 - 2.0 ** -40).sum() == 1
    if ordered:
        np.testing.assert_array_equal(out, ref_out)
    else:
        np.testing.assert_array_equal(np.sort(out[:k]), np.sort(ref_out[:k]))
        np.testing.assert_array_equal(out[k:], ref_out[k:])


def _pinned(a):
    t = torch.empty(a.shape, dtype={np.float64: torch.float64, np.int64: torch.int64}[a.dtype.type],
                    pin_memory=True)
    t.numpy()[...] = a
    return t  # keep the tensor alive; t.numpy() shares its page-locked memory


@pytest.mark.parametrize("prec", ["native", "fp32"])
@pytest.mark.parametrize("ordered", [False, True])
@pytest.mark.parametrize("pinned_out", [False, True])
def test_query_page_locked_buffers(prec, ordered, pinned_out):
    """Page-locked (pinned) caller buffers, as the bench passes them: the
    column still goes through the narrowing ring (chunks holding non-fp32
    values keep float64), a pinned out_vals takes the survivors widened on
    the device and DMA'd straight in.  Survivors are the oracle's either
    way, in FIFO order when asked."""
    rng = np.random.default_rng(11)
    N = 9_000_001  # many staging chunks, ragged tail
    col = rng.random(N, dtype=np.float32).astype(np.float64)
    for i in (3, 2_000_003, 4_500_000, N - 2):  # non-fp32 values in narrowed and direct chunks
        col[i] = 0.5 - 2.0 ** -40
    col[7_000_000] = 0.5 + 2.0 ** -30
    tcol = _pinned(col)
    tout = _pinned(np.full(N, -1.0)) if pinned_out else None
    out = tout.numpy() if pinned_out else np.full(N, -1.0)
    cnt = np.array([2], np.int64)
    p = _lib.PREC_NATIVE if prec == "native" else _lib.PREC_FP32
    src = col if prec == "native" else col.astype(np.float32).astype(np.float64)
    ref_out, ref_cnt = oracle.query(src, 0.5, np.full(N, -1.0), cnt.copy())
    op = _lib.CMP["<"] | (_lib.QUERY_ORDERED if ordered else 0)
    thr = np.array([0.5])
    _lib.check(_lib.load().sdfgb_host_query(ctypes.c_void_p(tcol.data_ptr()), _vp(thr), _vp(out), _vp(cnt), N, op,
                                            p))
    k = int(ref_cnt[0] - 2)
    assert cnt[0] == ref_cnt[0]
    if ordered:
        np.testing.assert_array_equal(out[:k], ref_out[:k])
    else:
        np.testing.assert_array_equal(np.sort(out[:k]), np.sort(ref_out[:k]))
    np.testing.assert_array_equal(out[k:], -1.0)


# ------------------------------------------------------------- error paths

def test_failed_calls_leave_the_entries_clean():
    """A failure in the middle of a pipelined call (an out-of-range column in
    a later SpMV row chunk, after earlier chunks' kernels were queued; an
    out-of-range bin) must leave nothing behind: the next calls of every
    entry, sharing the device pool and the query workspace, match the oracle
    bit for bit.  (events leaked and copies were still in flight
    on early returns; the query workspace was cleared only once.)"""
    L = _lib.load()
    rng = np.random.default_rng(4)
    H, W, k = 600_000, 50_000, 8
    rp = np.arange(H + 1, dtype=np.int64) * k
    ci = np.sort(rng.integers(0, W, (H, k)), axis=1).reshape(-1)
    v, x, b = rng.random(H * k), rng.random(W), rng.random(H)
    bad = ci.copy()
    bad[-100] = W  # last row chunk
    bb = b.copy()
    assert L.sdfgb_host_spmv(_vp(rp), _vp(bad), _vp(v), _vp(x), _vp(bb), H, W, H * k, _lib.PREC_FP32) == _lib.ERR_OOB
    np.testing.assert_array_equal(bb, b)  # b is written back only after every chunk validated
    bad_rp = rp.copy()
    bad_rp[7] = bad_rp[8] + 1
    assert L.sdfgb_host_spmv(_vp(bad_rp), _vp(ci), _vp(v), _vp(x), _vp(bb), H, W, H * k,
                             _lib.PREC_FP32) == _lib.ERR_INVALID
    img = rng.random((100, 100))
    img[50, 50] = 1.5
    h = np.zeros(256, np.int64)
    assert L.sdfgb_host_histogram(_vp(img), _vp(h), 100, 100, 256, 256.0, 1.0, _lib.PREC_NATIVE) == _lib.ERR_OOB
    assert not h.any()
    # clean calls afterwards
    for prec in (_lib.PREC_FP32, _lib.PREC_NATIVE):
        got = b.copy()
        _lib.check(L.sdfgb_host_spmv(_vp(rp), _vp(ci), _vp(v), _vp(x), _vp(got), H, W, H * k, prec))
        ref = oracle.spmv(rp, ci, v, x, b)
        tol = 1e-5 if prec == _lib.PREC_FP32 else 1e-12
        np.testing.assert_allclose(got, ref, rtol=tol, atol=tol * np.abs(ref).max())
    col = rng.random(3_000_000, dtype=np.float32).astype(np.float64)
    out, cnt, thr = np.zeros(col.size), np.zeros(1, np.int64), np.array([0.25])
    _lib.check(L.sdfgb_host_query(_vp(col), _vp(thr), _vp(out), _vp(cnt), col.size,
                                  _lib.CMP[">="] | _lib.QUERY_ORDERED, _lib.PREC_NATIVE))
    ro, rc_ = oracle.query(col, 0.25, np.zeros(col.size), np.zeros(1, np.int64), ">=")
    np.testing.assert_array_equal(out, ro)
    np.testing.assert_array_equal(cnt, rc_)
    img[50, 50] = 0.5
    _lib.check(L.sdfgb_host_histogram(_vp(img), _vp(h), 100, 100, 256, 256.0, 1.0, _lib.PREC_NATIVE))
    np.testing.assert_array_equal(h, oracle.histogram(img, np.zeros(256, np.int64))[0])


# ---------------------------------------------- BASELINE configs, full size

@pytest.mark.slow
def test_j1_baseline_config_8192_t1000():
    """J1 exactly as configured (BASELINE.json configs[2]; SURVEY §8d inputs):
    8192^2, T = 1000, through the drop-in (fp32 precision).  Bit-exact against
    the fp32 same-order restatement (oracle.c, OpenMP over rows), and within
    1e-4 normwise of the reference's OWN generated float64 C (oracle/_ref,
    cpu_parallel schedule) -- the reference pins its stencil the same way at
    a smaller size (test_codegen.py:110-118)."""
    N, T = 8192, 1000
    rng = np.random.default_rng(2)
    A = np.zeros((2, N, N), np.float32)
    A[0, 1:-1, 1:-1] = rng.random((N - 2, N - 2), dtype=np.float32)
    A[1] = A[0]
    prog = b200.invoke_toolchain(b200.generate(marked("jacobi2d", "fp32")))
    got = prog.run({"A": A.astype(np.float64)}, {"N": N, "T": T})["A"].reshape(2, N, N)
    ref32 = oracle.jacobi2d(A, T, fp32=True)
    np.testing.assert_array_equal(got, ref32.astype(np.float64))
    if not oracle.ref_available("jacobi2d_omp"):
        pytest.skip("oracle/_ref not built")
    ref64 = oracle.ref_call("jacobi2d_omp", {"A": A.astype(np.float64)}, {"N": N, "T": T})["A"].reshape(2, N, N)
    for p in (0, 1):
        err = np.linalg.norm(got[p] - ref64[p]) / np.linalg.norm(ref64[p])
        assert err <= 1e-4, (p, err)


@pytest.mark.slow
def test_s1_baseline_config_all_rows():
    """S1 as configured (2^22 x 2^22, 64 nnz/row, SURVEY §8d recipe): every
    row of the device entry and of the drop-in host entry against the
    oracle's j-sequential float64 sum, at 1e-5 relative."""
    from paper_1902_10345_b200 import device
    H = W = 1 << 22
    rng = np.random.default_rng(3)
    col = np.sort(rng.integers(0, W, (H, 64), dtype=np.int32), axis=1).reshape(-1)
    val = rng.random(H * 64, dtype=np.float32)
    x = rng.random(W, dtype=np.float32)
    rowptr = (np.arange(H + 1, dtype=np.int64) * 64)
    ref = oracle.spmv(rowptr, col, val.astype(np.float64), x.astype(np.float64), np.zeros(H))
    b = torch.zeros(H, dtype=torch.float32, device="cuda")
    device.spmv(*(torch.from_numpy(a).cuda() for a in (rowptr.astype(np.int32), col, val, x)), b)
    np.testing.assert_allclose(b.cpu().numpy(), ref, rtol=1e-5, atol=1e-5 * np.abs(ref).max())
    got = np.zeros(H)
    col64, val64, x64 = col.astype(np.int64), val.astype(np.float64), x.astype(np.float64)  # kept alive
    _lib.check(_lib.load().sdfgb_host_spmv(_vp(rowptr), _vp(col64), _vp(val64), _vp(x64), _vp(got), H, W, H * 64,
                                           _lib.PREC_FP32))
    np.testing.assert_allclose(got, ref, rtol=1e-5, atol=1e-5 * np.abs(ref).max())


def test_q1_and_h1_baseline_configs_native_are_the_reference():
    """Q1 (2^26, x < 0.5) and H1 (4096^2, 256 bins) with the SURVEY §8d
    inputs through the drop-in in NATIVE precision: the lossless fp32
    staging must give exactly the reference's float64 results."""
    L = _lib.load()
    col = np.random.default_rng(1).random(1 << 26, dtype=np.float32).astype(np.float64)
    out, cnt, thr = np.zeros(col.size), np.zeros(1, np.int64), np.array([0.5])
    _lib.check(L.sdfgb_host_query(_vp(col), _vp(thr), _vp(out), _vp(cnt), col.size,
                                  _lib.CMP["<"] | _lib.QUERY_ORDERED, _lib.PREC_NATIVE))
    ro, rc_ = oracle.query(col, 0.5, np.zeros(col.size), np.zeros(1, np.int64))
    np.testing.assert_array_equal(cnt, rc_)
    np.testing.assert_array_equal(out, ro)
    img = np.random.default_rng(0).random((4096, 4096), dtype=np.float32).astype(np.float64)
    h = np.zeros(256, np.int64)
    _lib.check(L.sdfgb_host_histogram(_vp(img), _vp(h), 4096, 4096, 256, 256.0, 1.0, _lib.PREC_NATIVE))
    np.testing.assert_array_equal(h, oracle.histogram(img, np.zeros(256, np.int64))[0])
