"""Randomised device-entry parity against the C oracle: sizes, alignments,
operators, thresholds and value ranges drawn from a seeded generator (many
small cases per run, each bit-exact)."""

import numpy as np
import pytest

import oracle

import os

DEV = "cuda"
OPS = ["<", "<=", ">", ">=", "==", "!="]
# SDFGB_FUZZ_SCALE=k runs k times the seeds (long campaigns on the box)
SCALE = max(1, int(os.environ.get("SDFGB_FUZZ_SCALE", "1")))


def t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(12 * SCALE))
def test_query_fuzz(seed, cuda_ok):
    import torch
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(1000 + seed)
    for _ in range(8):
        n = int(rng.choice([1, 3, 17, 255, 4096, 70001, 1 << 18]) + rng.integers(0, 5))
        off = int(rng.integers(0, 4))
        base = rng.random(n + off, dtype=np.float32) * 4 - 2
        if rng.random() < 0.3:
            base[rng.integers(0, n + off, 8)] = np.float32(0.25)  # ties for == / !=
        col = base[off:]
        op = OPS[int(rng.integers(0, 6))]
        thr = float(rng.choice([0.25, 0.0, -1.5, 1e-7, 0.1, np.float64(np.float32(0.3)) + 1e-12]))
        ordered = bool(rng.integers(0, 2))
        dcol = t(base)[off:]
        out = torch.zeros(n, dtype=torch.float32, device=DEV)
        cnt = torch.full((1,), 7, dtype=torch.int64, device=DEV)
        ws = device.query_workspace(n, 4, DEV)
        device.query(dcol, thr, out, cnt, ws, op, ordered=ordered)
        exp, ecnt = oracle.query(col, thr, np.zeros(n, np.float32), np.array([7], np.int64), op)
        k = int(ecnt[0] - 7)
        assert int(cnt.item()) == int(ecnt[0]), (n, op, thr)
        got = out[:k].cpu().numpy()
        if ordered:
            np.testing.assert_array_equal(got, exp[:k])
        else:
            np.testing.assert_array_equal(np.sort(got), np.sort(exp[:k]))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(4 * SCALE))
def test_query_ordered_multi_piece_fuzz(seed, cuda_ok):
    """FIFO order across several of the piece kernel's 16 MB pieces: random
    sizes (1-7 pieces, ragged tails), offsets, operators and thresholds"""
    import torch
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(5000 + seed)
    dtype = np.float32 if rng.random() < 0.7 else np.float64
    n = int(rng.integers(1, 7 * (16 << 20) // np.dtype(dtype).itemsize))
    off = int(rng.integers(0, 4)) * (16 // np.dtype(dtype).itemsize)  # 16 B-aligned views: the piece kernel
    base = (rng.random(n + off) * 4 - 2).astype(dtype)
    col = base[off:]
    op = OPS[int(rng.integers(0, 6))]
    thr = float(rng.choice([0.25, 0.0, -1.5, 1.9, -2.5]))
    dcol = t(base)[off:]
    out = torch.zeros(n, dtype=dcol.dtype, device=DEV)
    cnt = torch.full((1,), 5, dtype=torch.int64, device=DEV)
    device.query(dcol, thr, out, cnt, device.query_workspace(n, col.itemsize, DEV), op, ordered=True)
    exp, ecnt = oracle.query(col, thr, np.zeros(n, dtype), np.array([5], np.int64), op)
    assert int(cnt.item()) == int(ecnt[0]), (n, op, thr)
    np.testing.assert_array_equal(out.cpu().numpy(), exp)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(12 * SCALE))
def test_histogram_fuzz(seed, cuda_ok):
    import torch
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(2000 + seed)
    for _ in range(8):
        n = int(rng.choice([1, 5, 1000, 65537, 1 << 20]) + rng.integers(0, 9))
        off = int(rng.integers(0, 4))
        bins = int(rng.choice([1, 7, 256, 1000, 5000]))
        scale = float(rng.choice([256.0, 100.0, 1.0, 3.5, 1024.0]))
        div = float(rng.choice([1.0, 1.0, 3.0, 0.5]))
        base = (rng.random(n + off, dtype=np.float32) * 1.2 - 0.1).astype(np.float32)
        if rng.random() < 0.3:
            base[rng.integers(0, n + off, 4)] = np.float32(np.nan)
        img = base[off:]
        h0 = rng.integers(0, 3, bins).astype(np.int64)
        hist = t(h0)
        oob = torch.zeros(1, dtype=torch.int64, device=DEV)
        device.hist(t(base)[off:], hist, oob, scale, div)
        ref, roob = oracle.histogram(img, h0, scale, div)
        np.testing.assert_array_equal(hist.cpu().numpy(), ref, err_msg=f"{n} {bins} {scale} {div}")
        assert int(oob.item()) == roob


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(8 * SCALE))
def test_spmv_fuzz(seed, cuda_ok):
    """ragged rows (empty, short, > 64 nnz), unaligned row starts, duplicate columns"""
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(3000 + seed)
    for _ in range(6):
        H = int(rng.integers(1, 3000))
        W = int(rng.integers(1, 5000))
        lens = rng.choice([0, 1, 3, 16, 64, 65, 200], size=H, p=[.15, .15, .2, .2, .15, .1, .05])
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        nnz = int(rp[-1])
        col = rng.integers(0, W, max(nnz, 1)).astype(np.int32)[:nnz]
        val = rng.random(nnz, dtype=np.float32) - 0.5
        x = rng.random(W, dtype=np.float32)
        b0 = rng.random(H, dtype=np.float32)
        b = t(b0)
        device.spmv(t(rp), t(col), t(val), t(x), b)
        ref = b0.astype(np.float64).copy()
        for i in range(H):
            s, e = rp[i], rp[i + 1]
            ref[i] += float(np.dot(val[s:e].astype(np.float64), x[col[s:e]].astype(np.float64)))
        scale = np.abs(b0).astype(np.float64) + np.array(
            [np.abs(val[rp[i]:rp[i + 1]]).astype(np.float64) @ x[col[rp[i]:rp[i + 1]]] for i in range(H)])
        assert (np.abs(b.cpu().numpy() - ref) / (scale + 1e-30)).max() < 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6 * SCALE))
def test_jacobi_fuzz(seed, cuda_ok):
    """square sizes around the tile and vector widths, T around the temporal
    block lengths: bit-exact against the fp32 restatement"""
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(4000 + seed)
    for _ in range(3):
        N = int(rng.choice([3, 5, 8, 31, 100, 113, 128, 225, 300]))
        T = int(rng.choice([0, 1, 2, 3, 6, 7, 8, 15, 16]))
        A = rng.random((2, N, N), dtype=np.float32)
        ref = oracle.jacobi2d(A, T, fp32=True)
        At = t(A)
        device.jacobi2d(At, T)
        np.testing.assert_array_equal(At.cpu().numpy(), ref, err_msg=f"N={N} T={T}")


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6 * SCALE))
def test_matmul_host_entry_fuzz(seed, cuda_ok):
    """the reference-facing matmul entries on random shapes (K % 4 != 0 pads,
    one-row / one-column panels): 3xTF32 within 1e-5 of |A||B|, float64
    bit-exact in k order"""
    import ctypes
    from paper_1902_10345_b200 import _lib
    L = _lib.load()
    rng = np.random.default_rng(5000 + seed)
    for _ in range(3):
        M, N, K = (int(v) for v in rng.integers(1, 700, 3))
        A = rng.random((M, K)) - 0.5
        B = rng.random((K, N)) - 0.5
        C = np.zeros((M, N))
        p = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
        _lib.check(L.sdfgb_host_matmul(p(A), p(B), p(C), M, N, K))
        a32, b32 = A.astype(np.float32).astype(np.float64), B.astype(np.float32).astype(np.float64)
        err = np.abs(C - a32 @ b32) / (np.abs(a32) @ np.abs(b32) + 1e-30)
        assert err.max() < 1e-5, (M, N, K, err.max())
        if M * N * K <= 2_000_000:
            C64 = np.zeros((M, N))
            _lib.check(L.sdfgb_host_matmul_f64(p(A), p(B), p(C64), M, N, K))
            seq = np.zeros((M, N))
            for k in range(K):
                seq = seq + A[:, k:k + 1] * B[k:k + 1, :]
            np.testing.assert_array_equal(C64, seq)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(8 * SCALE))
def test_jacobi_strip_fuzz(seed, cuda_ok):
    """rectangular planes wide enough for the strip kernel (N >= 128), rows
    around its tile heights (16-row short tiles, 256-row tall tiles, border
    strips cut twice as fine), T around the 7/5/3 blocks; plus a random
    edge/interior band split of one launch: bit-exact against the fp32
    restatement / the whole-plane launch"""
    from paper_1902_10345_b200 import device
    rng = np.random.default_rng(9000 + seed)
    M = int(rng.integers(16, 1200))
    N = int(rng.integers(32, 420)) * 4
    T = int(rng.choice([4, 7, 8, 9, 13, 15, 22]))
    A = rng.random((2, M, N), dtype=np.float32)
    ref = A.copy()
    for tt in range(T):
        src, dst = ref[tt % 2], ref[(tt + 1) % 2]
        acc = src[1:-1, 1:-1] + src[0:-2, 1:-1]
        acc = acc + src[2:, 1:-1]
        acc = acc + src[1:-1, 0:-2]
        acc = acc + src[1:-1, 2:]
        dst[1:-1, 1:-1] = np.float32(0.2) * acc
    At = t(A)
    device.jacobi2d_rect(At, T)
    np.testing.assert_array_equal(At.cpu().numpy(), ref, err_msg=f"M={M} N={N} T={T}")
    if M >= 48:
        k = int(rng.choice([3, 5, 7]))
        e0 = int(rng.integers(9, M // 3))
        e1 = int(rng.integers(2 * M // 3, M - 9))
        whole, banded = t(A), t(A)
        device.jacobi2d_block(whole[0], whole[1], k)
        for r0, r1 in ((0, e0), (e1, M), (e0, e1)):
            device.jacobi2d_band(banded[0], banded[1], k, r0, r1)
        np.testing.assert_array_equal(banded.cpu().numpy(), whole.cpu().numpy(),
                                      err_msg=f"bands M={M} N={N} k={k} cuts={e0},{e1}")


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(3 * SCALE))
def test_jacobi_fused_p2p_slabs_fuzz(seed, cuda_ok):
    """the fused ghost exchange (multigpu.PeerJacobi) on 2-4 slabs of one
    device, blocks queued in turn on one stream: random grid shapes and step
    counts, bit-exact against the one-plane numpy restatement"""
    import torch
    from paper_1902_10345_b200 import multigpu as MG
    rng = np.random.default_rng(7000 + seed)
    nslabs = int(rng.integers(2, 5))
    Ng = int(rng.integers(50 * nslabs, 160 * nslabs))
    N = 4 * int(rng.integers(33, 150))
    T = int(rng.integers(1, 40))
    A = np.zeros((2, Ng, N), dtype=np.float32)
    A[:, 1:-1, 1:-1] = rng.random((Ng - 2, N - 2), dtype=np.float32)
    ref = A.copy()
    for s_ in range(T):
        src, dst = ref[s_ % 2], ref[(s_ + 1) % 2]
        acc = src[1:-1, 1:-1] + src[:-2, 1:-1]
        acc = acc + src[2:, 1:-1]
        acc = acc + src[1:-1, :-2]
        acc = acc + src[1:-1, 2:]
        dst[1:-1, 1:-1] = np.float32(0.2) * acc
    cuts = [round(i * Ng / nslabs) for i in range(nslabs + 1)]
    At = t(A)
    slabs = [MG.jacobi_slab(At[:, a:b], a, Ng) for a, b in zip(cuts, cuts[1:])]
    for up, lo in zip(slabs, slabs[1:]):
        up.A[:, up.top + up.rows:] = lo.A[:, lo.top:lo.top + up.bot]
        lo.A[:, :lo.top] = up.A[:, up.top + up.rows - lo.top:up.top + up.rows]
    peers = MG.PeerJacobi.chain(slabs)
    live = [MG.jacobi_p2p_blocks(s_, p, T) for s_, p in zip(slabs, peers)]
    while live:
        for g in list(live):
            try:
                next(g)
            except StopIteration:
                live.remove(g)
    torch.cuda.synchronize()
    got = np.concatenate([s_.A[:, s_.top:s_.top + s_.rows].cpu().numpy() for s_ in slabs], axis=1)
    np.testing.assert_array_equal(got[T % 2], ref[T % 2], err_msg=f"{Ng}x{N} T={T} slabs={nslabs}")
