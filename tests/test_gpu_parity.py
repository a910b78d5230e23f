"""GPU parity: the sm_100a kernels against the reference (golden fixtures from
its interpreter) and against the C oracle, through the C ABI.

Tolerances: histogram counts and query survivors bit-exact
(query compared as a sorted set by default -- concurrent pushes have no
order -- and in input order with stream_order "fifo" / ordered=True); Jacobi
bit-exact against the same-op-order restatement (fp32) or the reference
itself (native f64); SpMV 1e-5 rel (fp32) / 1e-12 (native); GEMM 1e-4 rel.
"""

import json

import numpy as np
import pytest

import oracle
from conftest import graph_path, load_cases

import paper_1902_10345_b200 as b200

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


DEV = "cuda"


def marked(name, precision, order="any"):
    doc = json.load(open(graph_path(name)))
    for d in doc["data"]:
        if not d["transient"]:
            d["storage"] = f"GPU_Global:{precision}" + (":fifo" if order == "fifo" else "")
    return doc


def _as_set(out_vals, count, count0):
    """survivors sorted (a stream's push order is unspecified), tail as is"""
    k = int(count[0] - count0[0])
    o = np.array(out_vals, copy=True)
    o[:k] = np.sort(o[:k])
    return o


SUPPORTED = ["histogram", "histogram_int", "query", "query_gallery", "spmv", "jacobi2d", "matmul",
             "matmul_raw", "matmul_tiled", "matmul_chain"]
CASES = [c for m in SUPPORTED for c in load_cases(m)]


# ------------------------------------------------ drop-in vs reference fixtures

def _f32_exact(a):
    a = np.asarray(a, np.float64)
    return np.array_equal(a, a.astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("order", ["any", "fifo"])
@pytest.mark.parametrize("precision", ["native", "fp32"])
@pytest.mark.parametrize("c", CASES, ids=repr)
def test_dropin_matches_reference_interpreter(c, precision, order):
    if order == "fifo" and not c.motif.startswith("query"):
        pytest.skip("stream order only applies to the query motif")
    prog = b200.invoke_toolchain(b200.generate(marked(c.motif, precision, order)))
    if c.error:
        with pytest.raises(b200.OutOfBoundsError):
            prog.run(c.inputs, c.symbols)
        return
    got = prog.run(c.inputs, c.symbols)
    outputs = dict(c.outputs)
    if precision == "fp32" and not all(_f32_exact(v) for v in c.inputs.values() if v.dtype.kind == "f"):
        # fp32 precision rounds the inputs on the device (declared semantics):
        # the expectation is the oracle on the rounded inputs
        if c.motif == "histogram":
            outputs["hist"] = oracle.histogram(c.inputs["img"].astype(np.float32), c.inputs["hist"])[0]
        elif c.motif.startswith("query"):
            op = ">" if c.motif == "query_gallery" else "<"
            o, n = oracle.query(c.inputs["col"].astype(np.float32), c.inputs["thr"][0],
                                np.zeros(c.inputs["col"].size, np.float32), c.inputs["count"], op)
            k = int(n[0] - c.inputs["count"][0])
            full = np.array(c.inputs["out_vals"], np.float64)
            full[:k] = o[:k]
            outputs["out_vals"], outputs["count"] = full, n
    if c.motif.startswith("query") and order == "any":
        got = dict(got)
        got["out_vals"] = _as_set(got["out_vals"], got["count"], c.inputs["count"])
        outputs["out_vals"] = _as_set(outputs["out_vals"], outputs["count"], c.inputs["count"])
    for name, exp in outputs.items():
        g = got[name].reshape(exp.shape)
        if exp.dtype.kind == "i" or c.motif.startswith(("histogram", "query")):
            np.testing.assert_array_equal(g, exp, err_msg=name)
        elif c.motif == "jacobi2d":
            if precision == "native":
                np.testing.assert_array_equal(g, exp, err_msg=name)
            else:
                ref32 = oracle.jacobi2d(c.inputs["A"].astype(np.float32), c.symbols["T"], fp32=True)
                np.testing.assert_array_equal(g, ref32.astype(np.float64), err_msg=name)
                nrm = np.linalg.norm(exp) or 1.0
                assert np.linalg.norm(g - exp) / nrm < 1e-5
        elif c.motif == "spmv":
            rtol = 1e-12 if precision == "native" else 1e-5
            np.testing.assert_allclose(g, exp, rtol=rtol, atol=rtol * (np.abs(exp).max() + 1e-30))
        elif precision == "native":  # matmul, float64 k-ordered multiply + add
            if c.motif == "matmul":
                # MapReduceFusion form: the interpreter accumulates WCR sums in k order
                np.testing.assert_array_equal(g, exp, err_msg=name)
            else:
                # Reduce node form: numpy's pairwise add.reduce order (interpreter.py:619)
                np.testing.assert_allclose(g, exp, rtol=1e-12, atol=1e-12 * (np.abs(exp).max() + 1e-30))
        else:  # matmul, 3xTF32
            scale = np.abs(exp).max() + 1e-30
            assert np.abs(g - exp).max() / scale < 1e-4, name


# ------------------------------------------------ device entries vs oracle

def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.mark.parametrize("offset", [0, 1, 2, 3])
@pytest.mark.parametrize("shape", [(1000, 1003), (1, 5), (7, 33), (64, 4096)])
def test_hist_f32_random_and_misaligned(shape, offset):
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(sum(shape) + offset)
    img = rng.random(shape, dtype=np.float32)
    base = t(np.concatenate([np.zeros(offset, np.float32), img.reshape(-1)]))
    view = base[offset:]
    h = torch.full((256,), 5, dtype=torch.int64, device=DEV)
    oob = torch.zeros(1, dtype=torch.int64, device=DEV)
    device.hist(view, h, oob)
    ref, bad = oracle.histogram(img, np.full(256, 5, np.int64))
    assert oob.item() == bad == 0
    np.testing.assert_array_equal(h.cpu().numpy(), ref)


@pytest.mark.parametrize("kind", ["zeros", "half_one_bin", "boundaries", "oob", "nan"])
def test_hist_f32_skewed_and_edge_values(kind):
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(1)
    img = rng.random(300007, dtype=np.float32)
    if kind == "zeros":
        img[:] = 0
    elif kind == "half_one_bin":
        img[::2] = 0.5
    elif kind == "boundaries":
        img[:257] = np.concatenate([np.arange(256) / 256.0, [np.nextafter(np.float32(1), np.float32(0))]])
    elif kind == "oob":
        img[::1001] = 1.0
        img[5::999] = -0.25
    else:
        img[3::777] = np.nan
    h = torch.zeros(256, dtype=torch.int64, device=DEV)
    oob = torch.zeros(1, dtype=torch.int64, device=DEV)
    device.hist(t(img), h, oob)
    ref, bad = oracle.histogram(img, np.zeros(256, np.int64))
    assert oob.item() == bad
    np.testing.assert_array_equal(h.cpu().numpy(), ref)


@pytest.mark.parametrize("bins,scale,div", [(100, 100.0, 1.0), (1000, 3000.0, 3.0), (20000, 20000.0, 1.0),
                                            (7, 7.0, 1.0)])
def test_hist_general_binning(bins, scale, div):
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(bins)
    for dt in (np.float32, np.float64):
        img = rng.random(123457).astype(dt)
        h = torch.zeros(bins, dtype=torch.int64, device=DEV)
        oob = torch.zeros(1, dtype=torch.int64, device=DEV)
        device.hist(t(img), h, oob, scale, div)
        ref, bad = oracle.histogram(img, np.zeros(bins, np.int64), scale, div)
        assert oob.item() == bad
        np.testing.assert_array_equal(h.cpu().numpy(), ref)


def test_hist_i64():
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(2)
    img = rng.integers(-3, 70, 99991).astype(np.int64)
    h = torch.zeros(64, dtype=torch.int64, device=DEV)
    oob = torch.zeros(1, dtype=torch.int64, device=DEV)
    device.hist(t(img), h, oob)
    ref, bad = oracle.histogram(img, np.zeros(64, np.int64), integer=True)
    assert oob.item() == bad
    np.testing.assert_array_equal(h.cpu().numpy(), ref)


@pytest.mark.parametrize("ordered", [False, True])
@pytest.mark.parametrize("op", ["<", "<=", ">", ">=", "==", "!="])
@pytest.mark.parametrize("n,offset", [(1, 0), (31, 1), (4096, 0), (4097, 3), (1000003, 2), (65536 * 3, 0)])
def test_query(n, offset, op, ordered):
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(n + offset)
    col = rng.random(n, dtype=np.float32)
    col[::5] = 0.5
    base = t(np.concatenate([np.zeros(offset, np.float32), col]))
    view = base[offset:]
    out = torch.full((n,), -1.0, dtype=torch.float32, device=DEV)
    cnt = torch.full((1,), 11, dtype=torch.int64, device=DEV)
    ws = device.query_workspace(n, 4, DEV)
    for rep in range(3):  # workspace reuse across launches (epoch + self-reset)
        out.fill_(-1.0)
        cnt.fill_(11)
        device.query(view, 0.5, out, cnt, ws, op, ordered=ordered)
        rout, rcnt = oracle.query(col, 0.5, np.full(n, -1.0, np.float32), np.array([11]), op)
        np.testing.assert_array_equal(cnt.cpu().numpy(), rcnt)
        got = out.cpu().numpy()
        if not ordered:
            got, rout = _as_set(got, rcnt, [11]), _as_set(rout, rcnt, [11])
        np.testing.assert_array_equal(got, rout)


@pytest.mark.parametrize("ordered", [False, True])
@pytest.mark.parametrize("n", [100003, 3 * 4096 * 16])
def test_query_misaligned_output(n, ordered):
    """an output view that is not 16 B aligned (the register-path kernel
    for FIFO order; scalar stores for the push kernel)"""
    from paper_1902_10345_b200 import device
    col = np.random.default_rng(n).random(n, dtype=np.float32)
    base = torch.full((n + 1,), -1.0, dtype=torch.float32, device=DEV)
    out = base[1:]
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    device.query(t(col), 0.5, out, cnt, device.query_workspace(n, 4, DEV), "<", ordered=ordered)
    rout, rcnt = oracle.query(col, 0.5, np.full(n, -1.0, np.float32), np.zeros(1, np.int64), "<")
    k = int(rcnt[0])
    assert cnt.item() == k and base[0].item() == -1.0
    got = out.cpu().numpy()
    np.testing.assert_array_equal(got[k:], rout[k:])
    if ordered:
        np.testing.assert_array_equal(got[:k], rout[:k])
    else:
        np.testing.assert_array_equal(np.sort(got[:k]), np.sort(rout[:k]))


@pytest.mark.parametrize("ordered", [False, True])
def test_query_f64(ordered):
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(9)
    col = rng.random(777777)
    out = torch.zeros(col.size, dtype=torch.float64, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    ws = device.query_workspace(col.size, 8, DEV)
    device.query(t(col), 0.3, out, cnt, ws, ">=", ordered=ordered)
    rout, rcnt = oracle.query(col, 0.3, np.zeros(col.size), np.zeros(1, np.int64), ">=")
    assert cnt.item() == rcnt[0]
    got = out.cpu().numpy()
    if not ordered:
        got, rout = _as_set(got, rcnt, [0]), _as_set(rout, rcnt, [0])
    np.testing.assert_array_equal(got, rout)


@pytest.mark.parametrize("dtype,thr", [(np.float32, 0.0), (np.float32, 0.03), (np.float32, 0.5),
                                       (np.float32, 1.0), (np.float64, 0.5)])
def test_query_ordered_many_pieces(dtype, thr):
    """FIFO order across several 64 MB pieces (the piece kernel's counts of
    piece p+1 are published while piece p is compacted); a ragged tail and
    0 / 3 / 50 / 100 % selectivity exercise the per-warp stage carry"""
    from paper_1902_10345_b200 import device
    n = (160 << 20) // np.dtype(dtype).itemsize + 12345
    col = np.random.default_rng(int(thr * 100) + n).random(n).astype(dtype)
    out = torch.full((n,), -1.0, dtype=torch.from_numpy(col[:1]).dtype, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    ws = device.query_workspace(n, col.itemsize, DEV)
    for rep in range(2):
        out.fill_(-1.0)
        cnt.zero_()
        device.query(t(col), thr, out, cnt, ws, "<", ordered=True)
        rout, rcnt = oracle.query(col, thr, np.full(n, -1.0, dtype), np.zeros(1, np.int64), "<")
        assert cnt.item() == rcnt[0]
        np.testing.assert_array_equal(out.cpu().numpy(), rout)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("pieces,delta", [(1, -1), (1, 1), (2, 0), (2, 129), (3, -517)])
def test_query_ordered_piece_boundaries(dtype, pieces, delta):
    """sizes at and around whole multiples of the FIFO kernel's 32 MB piece:
    equalised pieces, the last CTA's short range and the column's ragged
    tail all meet the per-piece count words"""
    from paper_1902_10345_b200 import device
    n = pieces * (32 << 20) // np.dtype(dtype).itemsize + delta
    col = np.random.default_rng(n).random(n).astype(dtype)
    out = torch.full((n,), -1.0, dtype=torch.from_numpy(col[:1]).dtype, device=DEV)
    cnt = torch.full((1,), 3, dtype=torch.int64, device=DEV)
    device.query(t(col), 0.7, out, cnt, device.query_workspace(n, col.itemsize, DEV), ">=", ordered=True)
    rout, rcnt = oracle.query(col, 0.7, np.full(n, -1.0, dtype), np.array([3], np.int64), ">=")
    assert cnt.item() == rcnt[0]
    np.testing.assert_array_equal(out.cpu().numpy(), rout)


@pytest.mark.parametrize("ordered", [False, True])
def test_query_beyond_int32_elements(ordered):
    """2^31 + 12345 elements (8.6 GB in, up to 8.6 GB out): element counts,
    offsets and chunk indices past 32 bits.  Checked through properties
    (the count; the survivors equal the masked column, in FIFO order or as
    a sorted multiset)"""
    from paper_1902_10345_b200 import device
    n = (1 << 31) + 12345
    g = torch.Generator(device=DEV).manual_seed(7)
    col = torch.rand(n, device=DEV, generator=g)
    out = torch.empty(n, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    device.query(col, 0.25, out, cnt, device.query_workspace(n, 4, DEV), "<", ordered=ordered)
    sel = col[col < 0.25]
    k = sel.numel()
    assert cnt.item() == k
    if ordered:
        assert torch.equal(out[:k], sel)
    else:
        assert torch.equal(torch.sort(out[:k]).values, torch.sort(sel).values)


def test_query_mixed_modes_share_workspace():
    """ordered and unordered launches alternate on one workspace; the
    unordered kernel's counter/ticket must be left zeroed every time"""
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(12)
    col = rng.random(300001, dtype=np.float32)
    ws = device.query_workspace(col.size, 4, DEV)
    sel = col[col < 0.25]
    for rep in range(6):
        out = torch.zeros(col.size, dtype=torch.float32, device=DEV)
        cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
        device.query(t(col), 0.25, out, cnt, ws, "<", ordered=bool(rep % 2))
        assert cnt.item() == sel.size
        got = out[:sel.size].cpu().numpy()
        if rep % 2:
            np.testing.assert_array_equal(got, sel)
        else:
            np.testing.assert_array_equal(np.sort(got), np.sort(sel))


def random_csr(rng, H, W, max_len):
    lens = rng.integers(0, max_len + 1, H)
    rowptr = np.concatenate([[0], np.cumsum(lens)])
    nnz = int(rowptr[-1])
    col = np.concatenate([np.sort(rng.integers(0, W, l)) for l in lens]) if nnz else np.zeros(0, np.int64)
    return rowptr, col, rng.random(nnz, dtype=np.float32), rng.random(W, dtype=np.float32)


@pytest.mark.parametrize("H,W,max_len", [(1, 1, 1), (1000, 2000, 200), (50001, 4000, 10), (8, 5, 0)])
def test_spmv(H, W, max_len):
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(H)
    rowptr, col, val, x = random_csr(rng, H, W, max_len)
    b0 = rng.random(H, dtype=np.float32)
    ref = oracle.spmv(rowptr, col, val.astype(np.float64), x.astype(np.float64), b0.astype(np.float64))
    b = t(b0)
    device.spmv(t(rowptr.astype(np.int32)), t(col.astype(np.int32)), t(val), t(x), b)
    np.testing.assert_allclose(b.cpu().numpy(), ref, rtol=1e-5, atol=1e-6)
    b64 = t(b0.astype(np.float64))
    device.spmv(t(rowptr.astype(np.int64)), t(col.astype(np.int64)), t(val.astype(np.float64)),
                t(x.astype(np.float64)), b64)
    np.testing.assert_allclose(b64.cpu().numpy(), ref, rtol=1e-12, atol=1e-13)


NINE = [(1, 1), (0, 0), (-1, 0), (1, 0), (0, -1), (0, 1), (-1, -1), (-1, 1), (1, -1)]


@pytest.mark.parametrize("N,T", [(3, 2), (4, 3), (5, 1), (67, 5), (130, 4), (515, 3), (1024, 2)])
@pytest.mark.parametrize("terms", ["canon", "nine"])
def test_jacobi_bit_exact(N, T, terms):
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(N * 10 + T)
    A = rng.random((2, N, N), dtype=np.float32)  # non-zero borders, distinct planes
    tm = oracle.JACOBI5 if terms == "canon" else NINE
    coef = 0.2 if terms == "canon" else 1.0 / 9.0
    ref = oracle.jacobi2d(A, T, coef=np.float32(coef), terms=tm, fp32=True)
    At = t(A)
    device.jacobi2d(At, T, coef=float(np.float32(coef)), terms=tm)
    np.testing.assert_array_equal(At.cpu().numpy(), ref)
    A64 = A.astype(np.float64)
    ref64 = oracle.jacobi2d(A64, T, coef=coef, terms=tm)
    At64 = t(A64)
    device.jacobi2d(At64, T, coef=coef, terms=tm)
    np.testing.assert_array_equal(At64.cpu().numpy(), ref64)


@pytest.mark.parametrize("N,T", [(16, 4), (20, 5), (124, 9), (132, 6), (240, 8), (256, 7), (1000, 11), (1024, 12),
                                 (520, 1003)])
def test_jacobi_temporal_blocking_bit_exact(N, T):
    """fp32 canonical order with N % 4 == 0 and T >= 4 runs the TMA temporal-
    blocking kernel (odd step blocks + a final single step): both planes must
    equal the one-step-at-a-time fp32 restatement bit for bit."""
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(N + T)
    A = rng.random((2, N, N), dtype=np.float32)
    ref = oracle.jacobi2d(A, T, fp32=True)
    At = t(A)
    device.jacobi2d(At, T)
    got = At.cpu().numpy()
    np.testing.assert_array_equal(got[T % 2], ref[T % 2])
    np.testing.assert_array_equal(got[(T + 1) % 2], ref[(T + 1) % 2])


@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (256, 384, 128), (1000, 777, 300), (64, 200, 4),
                                   (129, 130, 36), (512, 512, 4096)])
def test_gemm_3xtf32(M, N, K):
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(M + N + K)
    a = rng.random((M, K), dtype=np.float32) - 0.5
    b = rng.random((K, N), dtype=np.float32) - 0.5
    ref = oracle.matmul(a, b)
    C = torch.full((M, N), 7.0, dtype=torch.float32, device=DEV)
    device.gemm(t(a), t(b), C, device.gemm_workspace(M, N, K, DEV))
    got = C.cpu().numpy().astype(np.float64)
    scale = np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64)
    err = np.abs(got - ref) / scale
    assert err.max() < 1e-5, f"max rel (to |A||B|) err {err.max():.3e}"
    C2 = torch.zeros((M, N), dtype=torch.float32, device=DEV)
    device.gemm_simt(t(a), t(b), C2)
    assert (np.abs(C2.cpu().numpy() - ref) / scale).max() < 1e-5


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (5, 7, 3), (65, 130, 47), (256, 128, 300), (3, 2, 0)])
def test_gemm_f64_native_is_k_ordered(M, N, K):
    """native precision: bit-identical to the k-ordered WCR sum (0 + p0 + p1 + ...)"""
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(M * N + K)
    a = rng.random((M, K)) - 0.5
    b = rng.random((K, N)) - 0.5
    ref = np.zeros((M, N))
    for k in range(K):
        ref = ref + a[:, k:k + 1] * b[k:k + 1, :]
    C = torch.full((M, N), 7.0, dtype=torch.float64, device=DEV)
    device.gemm_f64(t(a), t(b), C)
    np.testing.assert_array_equal(C.cpu().numpy(), ref)


# ------------------------------------------------ BASELINE shapes (properties)

def test_full_histogram_4096():
    from paper_1902_10345_b200 import device
    img = np.random.default_rng(0).random((4096, 4096), dtype=np.float32)
    h = torch.zeros(256, dtype=torch.int64, device=DEV)
    oob = torch.zeros(1, dtype=torch.int64, device=DEV)
    device.hist(t(img), h, oob)
    ref, _ = oracle.histogram(img, np.zeros(256, np.int64))
    np.testing.assert_array_equal(h.cpu().numpy(), ref)
    assert int(h.sum()) == img.size


def test_histogram_beyond_int32_elements():
    """2^31 + 999 pixels (8.6 GB): per-bin counts past 32 bits of element
    index, checked against torch.bincount of the same binning"""
    from paper_1902_10345_b200 import device
    n = (1 << 31) + 999
    g = torch.Generator(device=DEV).manual_seed(3)
    img = torch.rand(n, device=DEV, generator=g)
    h = torch.zeros(256, dtype=torch.int64, device=DEV)
    oob = torch.zeros(1, dtype=torch.int64, device=DEV)
    device.hist(img, h, oob)
    ref = torch.bincount((img * 256.0).to(torch.int64), minlength=256)
    assert torch.equal(h, ref) and oob.item() == 0 and int(h.sum()) == n


def test_full_query_2pow26():
    from paper_1902_10345_b200 import device
    col = np.random.default_rng(1).random(1 << 26, dtype=np.float32)
    out = torch.zeros(col.size, dtype=torch.float32, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    ws = device.query_workspace(col.size, 4, DEV)
    sel = col[col < 0.5]
    for ordered in (False, True):
        cnt.zero_()
        device.query(t(col), 0.5, out, cnt, ws, "<", ordered=ordered)
        k = int(cnt.item())
        assert k == sel.size
        got = out[:k].cpu().numpy()
        if ordered:
            np.testing.assert_array_equal(got, sel)
        else:
            np.testing.assert_array_equal(np.sort(got), np.sort(sel))


def test_full_jacobi_8192_three_steps():
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(2)
    A = np.zeros((2, 8192, 8192), np.float32)
    A[0, 1:-1, 1:-1] = rng.random((8190, 8190), dtype=np.float32)
    A[1] = A[0]
    ref = oracle.jacobi2d(A, 3, fp32=True)
    At = t(A)
    device.jacobi2d(At, 3)
    np.testing.assert_array_equal(At.cpu().numpy(), ref)


def test_full_jacobi_8192_nine_steps_temporal_blocking():
    """BASELINE size through the temporal-blocking path (one 7-step launch
    with fused two-step sweeps, a 1-step launch, then the final step)"""
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(5)
    A = rng.random((2, 8192, 8192), dtype=np.float32)
    ref = oracle.jacobi2d(A, 9, fp32=True)
    At = t(A)
    device.jacobi2d(At, 9)
    np.testing.assert_array_equal(At.cpu().numpy(), ref)


@pytest.mark.parametrize("M,N,K", [(256, 384, 40000), (130, 200, 16388)])
def test_gemm_long_k_register_flush(M, N, K):
    """K > 16384 takes the kernel that folds accumulator chunks into fp32
    registers: error independent of K (1e-5 here, where one accumulation
    per TMEM accumulator would drift past 1e-4)."""
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(K)
    A = rng.random((M, K), dtype=np.float32)
    B = rng.random((K, N), dtype=np.float32)
    C = torch.empty((M, N), dtype=torch.float32, device=DEV)
    device.gemm(t(A), t(B), C, device.gemm_workspace(M, N, K, DEV))
    ref = A.astype(np.float64) @ B.astype(np.float64)
    assert np.abs(C.cpu().numpy() - ref).max() / np.abs(ref).max() < 1e-5


def _jacobi_rect_ref(A, T):
    ref = A.copy()
    for t in range(T):
        s, d = ref[t % 2], ref[(t + 1) % 2]
        acc = s[1:-1, 1:-1] + s[0:-2, 1:-1]
        acc = acc + s[2:, 1:-1]
        acc = acc + s[1:-1, 0:-2]
        acc = acc + s[1:-1, 2:]
        d[1:-1, 1:-1] = np.float32(0.2) * acc
    return ref


@pytest.mark.parametrize("M,N,T", [(16, 132, 9), (300, 144, 15), (1000, 256, 11), (129, 512, 8), (17, 248, 7),
                                   (2000, 128, 8), (33, 1000, 14)])
def test_jacobi_rect_temporal_blocking_bit_exact(M, N, T):
    from paper_1902_10345_b200 import device
    A = np.random.default_rng(M + N).random((2, M, N), dtype=np.float32)
    At = t(A)
    device.jacobi2d_rect(At, T)
    np.testing.assert_array_equal(At.cpu().numpy(), _jacobi_rect_ref(A, T))


@pytest.mark.parametrize("ranks", [2, 3])
def test_jacobi_ghost_zone_slabs_on_one_device(ranks):
    """The multi-GPU decomposition (multigpu.jacobi: 7-row ghost zones, one
    exchange per temporal block) with its device kernels, ranks run one after
    another on this GPU with the exchanges done by copies: equals the
    single-domain restatement bit for bit."""
    from paper_1902_10345_b200 import multigpu as MG
    from paper_1902_10345_b200 import device
    rows, N, T = 300, 256, 23
    Ng = rows * ranks
    A = np.random.default_rng(ranks).random((2, Ng, N), dtype=np.float32)
    ref = _jacobi_rect_ref(A, T)
    slabs = [MG.jacobi_slab(t(A[:, r * rows:(r + 1) * rows].copy()), r * rows, Ng) for r in range(ranks)]

    def exchange(p):
        for r in range(ranks - 1):
            lo, hi = slabs[r], slabs[r + 1]
            hi.A[p, 0:hi.top] = lo.A[p, lo.top + rows - lo.bot:lo.top + rows]
            lo.A[p, lo.top + rows:lo.top + rows + lo.bot] = hi.A[p, hi.top:2 * hi.top]
    exchange(1)
    step = 0
    while step < T:
        k = 1 if T - step <= 1 else min(MG.GHOST, T - 1 - step)
        if T - step > 1 and k % 2 == 0:
            k -= 1
        p = step % 2
        exchange(p)
        for sl in slabs:
            device.jacobi2d_block(sl.A[p], sl.A[1 - p], k)
        step += k
    for r, sl in enumerate(slabs):
        np.testing.assert_array_equal(sl.A[:, sl.top:sl.top + rows].cpu().numpy(),
                                      ref[:, r * rows:(r + 1) * rows])


from paper_1902_10345_b200.errors import CodegenError  # noqa: E402


@pytest.mark.parametrize("k", [1, 3, 5, 7])
@pytest.mark.parametrize("M,N,cuts", [(200, 256, (16, 184)), (129, 512, (40, 57)), (96, 132, (1, 95)),
                                      (300, 1000, (23, 151))])
def test_jacobi_band_composition(k, M, N, cuts):
    """sdfgb_jacobi2d_band_f32: the edge bands and the interior band of one
    k-step launch (as multigpu.jacobi computes them around the in-flight
    ghost exchange) write exactly the rows the whole-plane launch writes,
    with the same bits, and nothing else."""
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(M + N + k)
    P = rng.random((2, M, N), dtype=np.float32)
    whole = t(P)
    device.jacobi2d_block(whole[0], whole[1], k)
    banded = t(P)
    e0, e1 = cuts
    for r0, r1 in ((0, e0), (e1, M), (e0, e1)):
        if k > 1 and 0 < min(r1, M - 1) - max(r0, 1) < 8:
            with pytest.raises(CodegenError):
                device.jacobi2d_band(banded[0], banded[1], k, r0, r1)
            return
        device.jacobi2d_band(banded[0], banded[1], k, r0, r1)
    np.testing.assert_array_equal(banded.cpu().numpy(), whole.cpu().numpy())
    # a single band touches only its own rows
    one = t(P)
    device.jacobi2d_band(one[0], one[1], k, 40 if M > 60 else 1, 60 if M > 60 else 17)
    got, ref = one.cpu().numpy(), whole.cpu().numpy()
    r0, r1 = (40, 60) if M > 60 else (1, 17)
    np.testing.assert_array_equal(got[1, r0:r1], ref[1, r0:r1])
    np.testing.assert_array_equal(got[1, :r0], P[1, :r0])
    np.testing.assert_array_equal(got[1, r1:], P[1, r1:])


@pytest.mark.parametrize("n", [4096, 16384])
def test_full_gemm(n):
    """M1 checked on every element (oracle over all rows, threads over rows);
    M2 (16384^3, infeasible on the host in full) on a row sample, as SURVEY
    §8c allows for that size only."""
    from paper_1902_10345_b200 import device
    g = torch.Generator(device=DEV).manual_seed(4)
    A = torch.rand(n, n, device=DEV, generator=g)
    B = torch.rand(n, n, device=DEV, generator=g)
    C = torch.empty(n, n, device=DEV)
    device.gemm(A, B, C, device.gemm_workspace(n, n, n, DEV))
    rows = list(range(n)) if n <= 4096 else [0, 1, n // 3, n // 2, n - 2, n - 1]
    a = A[rows].cpu().numpy()
    bh = B.cpu().numpy()
    ref = oracle.matmul(a, bh)
    got = C[rows].cpu().numpy()
    assert (np.abs(got - ref) / np.abs(ref)).max() < 1e-4


# ------------------------------------------------ pipelined host entries (C ABI)

def _vp(a):
    import ctypes
    return ctypes.c_void_p(a.ctypes.data)


def test_host_histogram_pipelined_chunks():
    """more than one 2^21-element chunk, ragged tail, existing counts kept"""
    from paper_1902_10345_b200 import _lib
    L = _lib.load()
    rng = np.random.default_rng(11)
    img = rng.random((2100, 1100))
    hist = rng.integers(0, 5, 256).astype(np.int64)
    ref, _ = oracle.histogram(img.astype(np.float32), hist.copy())
    got = hist.copy()
    _lib.check(L.sdfgb_host_histogram(_vp(img), _vp(got), 2100, 1100, 256, 256.0, 1.0, _lib.PREC_FP32))
    np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("M,N,K", [(2000, 96, 37), (1500, 130, 64), (130, 70, 5)])
def test_host_matmul_pipelined_panels(M, N, K):
    """row panels of A/C streamed through the copy streams; K % 4 != 0 pads"""
    from paper_1902_10345_b200 import _lib
    L = _lib.load()
    rng = np.random.default_rng(M + K)
    A = rng.random((M, K))
    B = rng.random((K, N))
    C = np.full((M, N), 3.0)
    _lib.check(L.sdfgb_host_matmul(_vp(A), _vp(B), _vp(C), M, N, K))
    ref = A.astype(np.float32).astype(np.float64) @ B.astype(np.float32).astype(np.float64)
    assert np.abs(C - ref).max() / np.abs(ref).max() < 1e-5
    C64 = np.zeros((M, N))
    _lib.check(L.sdfgb_host_matmul_f64(_vp(A), _vp(B), _vp(C64), M, N, K))
    seq = np.zeros((M, N))
    for k in range(K):
        seq = seq + A[:, k:k + 1] * B[k:k + 1, :]
    np.testing.assert_array_equal(C64, seq)


def test_gather_probe_runs_and_checks_arguments():
    """The bench's live L2-gather ceiling (sdfgb_probe_gather_f32): runs on a
    CSR-shaped stream and rejects unaligned / ragged inputs."""
    import ctypes
    from paper_1902_10345_b200 import _lib
    from paper_1902_10345_b200.errors import CodegenError
    L = _lib.load()
    x = torch.rand(1 << 16, device=DEV)
    col = torch.randint(0, 1 << 16, (1 << 20,), device=DEV, dtype=torch.int32)
    val = torch.rand(1 << 20, device=DEV)
    sink = torch.zeros(1, device=DEV)
    p = lambda t, off=0: ctypes.c_void_p(t.data_ptr() + off)  # noqa: E731
    _lib.check(L.sdfgb_probe_gather_f32(p(x), p(col), p(val), col.numel(), p(sink), None))
    torch.cuda.synchronize()
    with pytest.raises(CodegenError):
        _lib.check(L.sdfgb_probe_gather_f32(p(x), p(col), p(val), 6, p(sink), None))
    with pytest.raises(CodegenError):
        _lib.check(L.sdfgb_probe_gather_f32(p(x), p(col, 4), p(val), 8, p(sink), None))


@pytest.mark.parametrize("M,N,K", [(384, 256, 512), (300, 130, 96)])
def test_gemm_row_pieces_split_b_once(M, N, K):
    """sdfgb_gemm_f32_ex with SDFGB_GEMM_B_SPLIT: row pieces of one product
    (the multi-GPU A-piece pipeline) sharing one workspace split B once and
    give the whole product bit for bit (MN-major and transposed B paths)."""
    from paper_1902_10345_b200 import device
    g = torch.Generator(device=DEV).manual_seed(M + N)
    A = torch.rand(M, K, device=DEV, generator=g)
    B = torch.rand(K, N, device=DEV, generator=g)
    whole = torch.empty(M, N, device=DEV)
    device.gemm(A, B, whole, device.gemm_workspace(M, N, K, DEV))
    ws = device.gemm_workspace(M - 100, N, K, DEV)  # sized for the tallest piece
    pieces = torch.empty(M, N, device=DEV)
    device.gemm(A[:100].contiguous(), B, pieces[:100], ws)
    device.gemm(A[100:].contiguous(), B, pieces[100:], ws, b_split=True)
    torch.cuda.synchronize()
    assert torch.equal(pieces, whole)
