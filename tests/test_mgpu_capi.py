"""Multi-GPU entries of the C ABI (csrc/mgpu.cu: one rank's share of a motif
plus its NCCL exchange).  This run has one GPU, so the GPU tests drive a
one-rank communicator: the collectives degenerate to copies, every other
line of the entry runs, and the result must equal the one-GPU entry bit for
bit.  The multi-rank index arithmetic is the same as multigpu.py's, which
the gloo world-size-2 tests (test_multigpu.py) cover."""

import ctypes

import numpy as np
import pytest

import oracle

from paper_1902_10345_b200 import _lib

DEV = "cuda"


def test_library_finds_nccl_at_run_time():
    """no link-time NCCL dependency; dlopen finds libnccl.so.2 here"""
    L = _lib.load()
    assert L.sdfgb_nccl_available() == 1
    assert L.sdfgb_hist_mgpu_workspace_bytes(256) == 257 * 8


@pytest.fixture(scope="module")
def comm(cuda_ok):
    import torch
    torch.cuda.init()
    L = _lib.load()
    uid = ctypes.create_string_buffer(128)
    _lib.check(L.sdfgb_nccl_unique_id(uid))
    c = ctypes.c_void_p()
    _lib.check(L.sdfgb_nccl_comm_init(ctypes.byref(c), 1, uid, 0))
    yield c
    _lib.check(L.sdfgb_nccl_comm_destroy(c))


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


def _s():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.mark.gpu
def test_hist_mgpu_one_rank(comm):
    import torch
    L = _lib.load()
    rng = np.random.default_rng(3)
    img = rng.random((1000, 1003), dtype=np.float32)
    img[0, :7] = [1.5, -0.1, np.nan, 0.999999, 0.0, 2.0, 0.5]
    h0 = rng.integers(0, 9, 256).astype(np.int64)
    ref, _ = oracle.histogram(img, h0.copy())
    hist, oob = t(h0), torch.zeros(1, dtype=torch.int64, device=DEV)
    ws = torch.empty(L.sdfgb_hist_mgpu_workspace_bytes(256), dtype=torch.uint8, device=DEV)
    dimg = t(img)  # (a temporary's pointer would dangle once ctypes holds only the address)
    _lib.check(L.sdfgb_hist_f32_mgpu(_p(dimg), img.size, 256.0, 1.0, _p(hist), 256, _p(oob), _p(ws),
                                     ws.numel(), comm, _s()))
    np.testing.assert_array_equal(hist.cpu().numpy(), ref)
    assert int(hist.sum()) - int(h0.sum()) + int(oob.item()) == img.size


@pytest.mark.gpu
def test_query_mgpu_one_rank(comm):
    import torch
    from paper_1902_10345_b200 import device
    L = _lib.load()
    col = np.random.default_rng(4).random(1 << 20, dtype=np.float32)
    out = torch.zeros(col.size, dtype=torch.float32, device=DEV)
    count = torch.full((1,), 5, dtype=torch.int64, device=DEV)
    offset = torch.full((1,), -1, dtype=torch.int64, device=DEV)
    counts = torch.zeros(1, dtype=torch.int64, device=DEV)
    ws = device.query_workspace(col.size, 4, DEV)
    dcol = t(col)
    _lib.check(L.sdfgb_query_f32_mgpu(_p(dcol), col.size, _lib.CMP["<"], 0.5, _p(out), _p(count), _p(offset),
                                      _p(counts), _p(ws), ws.numel(), comm, _s()))
    sel = col[col < 0.5]
    assert int(count.item()) == 5 + sel.size and int(offset.item()) == 0 and int(counts.item()) == sel.size
    np.testing.assert_array_equal(np.sort(out[:sel.size].cpu().numpy()), np.sort(sel))


@pytest.mark.gpu
def test_spmv_mgpu_one_rank(comm):
    import torch
    from paper_1902_10345_b200 import device
    L = _lib.load()
    rng = np.random.default_rng(5)
    H, W, nz = 3000, 2048, 24
    col = np.sort(rng.integers(0, W, (H, nz)), axis=1).astype(np.int32).reshape(-1)
    val = rng.random(H * nz, dtype=np.float32)
    x = rng.random(W, dtype=np.float32)
    rp = (np.arange(H + 1) * nz).astype(np.int32)
    b0 = rng.random(H, dtype=np.float32)
    drp, dcol, dval, dx = t(rp), t(col), t(val), t(x)
    ref = t(b0)
    device.spmv(drp, dcol, dval, dx, ref)
    b = t(b0)
    xf = torch.empty(W, dtype=torch.float32, device=DEV)
    _lib.check(L.sdfgb_spmv_csr_f32_mgpu(_p(drp), _p(dcol), _p(dval), _p(dx), W, _p(xf), _p(b), H,
                                         comm, _s()))
    np.testing.assert_array_equal(xf.cpu().numpy(), x)
    np.testing.assert_array_equal(b.cpu().numpy(), ref.cpu().numpy())


@pytest.mark.gpu
@pytest.mark.parametrize("T", [1, 2, 9, 16])
def test_jacobi_mgpu_one_rank(comm, T):
    """a one-rank slab has no ghost rows: the plane edge is the border"""
    L = _lib.load()
    rng = np.random.default_rng(T)
    A = rng.random((2, 300, 260), dtype=np.float32)
    ref = A.copy()
    for s in range(T):
        src, dst = ref[s % 2], ref[(s + 1) % 2]
        acc = src[1:-1, 1:-1] + src[:-2, 1:-1]
        acc = acc + src[2:, 1:-1]
        acc = acc + src[1:-1, :-2]
        acc = acc + src[1:-1, 2:]
        dst[1:-1, 1:-1] = np.float32(0.2) * acc
    At = t(A)
    _lib.check(L.sdfgb_jacobi2d_f32_mgpu(_p(At), 0, 300, 0, 260, T, 0.2, comm, _s()))
    got = At.cpu().numpy()
    np.testing.assert_array_equal(got[T % 2], ref[T % 2])
    np.testing.assert_array_equal(got[(T + 1) % 2], ref[(T + 1) % 2])


@pytest.mark.gpu
def test_jacobi_mgpu_rejects_bad_ghosts(comm):
    import torch
    L = _lib.load()
    A = torch.zeros((2, 40, 32), dtype=torch.float32, device=DEV)
    assert L.sdfgb_jacobi2d_f32_mgpu(_p(A), 3, 30, 7, 32, 4, 0.2, comm, _s()) == 1


@pytest.mark.gpu
def test_gemm_mgpu_one_rank(comm):
    import torch
    from paper_1902_10345_b200 import device
    L = _lib.load()
    rng = np.random.default_rng(6)
    M, N, K = 384, 256, 200
    A = rng.random((M, K), dtype=np.float32)
    B = rng.random((K, N), dtype=np.float32)
    ws = device.gemm_workspace(M, N, K, DEV)
    ref = torch.empty((M, N), dtype=torch.float32, device=DEV)
    dA, dB = t(A), t(B)
    device.gemm(dA, dB, ref, ws)
    Ap = torch.empty((M, K), dtype=torch.float32, device=DEV)
    Bp = torch.empty((K, N), dtype=torch.float32, device=DEV)
    C = torch.empty((M, N), dtype=torch.float32, device=DEV)
    _lib.check(L.sdfgb_gemm_f32_mgpu(_p(dA), M, _p(dB), K, K, N, _p(Ap), _p(Bp), _p(C), _p(ws), ws.numel(),
                                     comm, comm, _s()))
    np.testing.assert_array_equal(C.cpu().numpy(), ref.cpu().numpy())


def _p2p_worker(rank, world, port, shards, h0, out_q):
    import os
    import torch
    import torch.distributed as dist
    from paper_1902_10345_b200 import multigpu as MG
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        hist = torch.from_numpy(h0.copy()).cuda()
        oob = torch.zeros(1, dtype=torch.int64, device="cuda")
        peers = MG.PeerHist(dist, hist, oob)
        img = torch.from_numpy(shards[rank]).cuda()
        for _ in range(2):  # two calls: counts accumulate on every rank
            MG.histogram_p2p(dist, img, peers)
        MG.finish_histogram_p2p(dist)
        out_q.put((rank, hist.cpu().numpy(), int(oob.item())))
        dist.barrier()  # keep every exported buffer alive until all ranks have read
        dist.destroy_process_group()
    except Exception as exc:  # surfaced by the parent
        out_q.put((rank, repr(exc), -1))


@pytest.mark.gpu
def test_hist_p2p_two_processes_one_gpu(cuda_ok):
    """the fused compute + all-reduce histogram over CUDA IPC peer mappings:
    two processes (on the one GPU here) each add their shard's counts into
    both processes' hist from inside the kernel; no kernel waits on another"""
    import socket
    import torch.multiprocessing as mp
    rng = np.random.default_rng(8)
    shards = [rng.random((513, 700), dtype=np.float32) for _ in range(2)]
    shards[1][3, :4] = [1.5, -2.0, np.nan, 0.25]
    h0 = rng.integers(0, 4, 256).astype(np.int64)
    ref = h0.copy()
    oob_ref = 0
    for sh in shards:
        r, o = oracle.histogram(sh, np.zeros(256, np.int64))
        ref += 2 * r
        oob_ref += 2 * o
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_p2p_worker, args=(r, 2, port, shards, h0, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, hist, oob in sorted(res, key=lambda x: x[0]):
        assert not isinstance(hist, str), hist
        np.testing.assert_array_equal(hist, ref)
        assert oob == oob_ref


def _qgather_worker(rank, world, port, shards, out_q):
    import os
    import torch
    import torch.distributed as dist
    from paper_1902_10345_b200 import device
    from paper_1902_10345_b200 import multigpu as MG
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cap = sum(s.size for s in shards)
        out = torch.full((cap if rank == 0 else 1,), -1.0, dtype=torch.float32, device="cuda")
        reserve = torch.zeros(1, dtype=torch.int64, device="cuda")
        g = MG.QueryGather(dist, out, reserve, root=0)
        col = torch.from_numpy(shards[rank]).cuda()
        ws = device.query_workspace(col.numel(), 4, "cuda")
        count = torch.full((1,), 3, dtype=torch.int64, device="cuda")
        totals = []
        for _ in range(2):  # two rounds: the counter is re-zeroed between them
            MG.query_p2p(dist, col, 0.5, g, ws, "<")
            totals.append(MG.finish_query_p2p(dist, g, count))
        got = out[:totals[-1]].cpu().numpy() if rank == 0 else None
        out_q.put((rank, totals, int(count.item()), got))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:
        out_q.put((rank, repr(exc), -1, None))


@pytest.mark.gpu
def test_query_p2p_gather_two_processes_one_gpu(cuda_ok):
    """compaction + gather fused over CUDA IPC peer memory: both processes'
    survivors land in rank 0's output at slots reserved on rank 0's counter"""
    import socket
    import torch.multiprocessing as mp
    rng = np.random.default_rng(9)
    shards = [rng.random(300_000, dtype=np.float32), rng.random(123_457 * 4, dtype=np.float32)]
    sel = np.sort(np.concatenate([s[s < 0.5] for s in shards]))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_qgather_worker, args=(r, 2, port, shards, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    for rank, totals, count, got in res:
        assert not isinstance(totals, str), totals
        assert totals == [sel.size, sel.size]
        assert count == 3 + 2 * sel.size
    np.testing.assert_array_equal(np.sort(res[0][3]), sel)


def _numpy_jacobi(A, T):
    ref = A.copy()
    for s in range(T):
        src, dst = ref[s % 2], ref[(s + 1) % 2]
        acc = src[1:-1, 1:-1] + src[:-2, 1:-1]
        acc = acc + src[2:, 1:-1]
        acc = acc + src[1:-1, :-2]
        acc = acc + src[1:-1, 2:]
        dst[1:-1, 1:-1] = np.float32(0.2) * acc
    return ref


@pytest.mark.gpu
@pytest.mark.parametrize("T", [1, 2, 9, 23])
@pytest.mark.parametrize("nslabs", [2, 3])
def test_jacobi_fused_p2p_exchange_slabs_in_turn(T, nslabs):
    """multigpu.jacobi's fused ghost exchange (edge-band kernels storing the
    neighbours' ghost rows, sdfgb_jacobi2d_band_mirror_f32, ordered by
    sdfgb_flag_signal / _wait) on slabs of ONE device: every slab's blocks
    are queued in turn on one stream, so each flag wait is already satisfied
    when it runs (no kernel ever waits on another).  Bit-exact against the
    one-plane numpy restatement."""
    import torch
    from paper_1902_10345_b200 import multigpu as MG
    rng = np.random.default_rng(100 + T + nslabs)
    Ng, N = 64 * nslabs + 37, 260
    A = np.zeros((2, Ng, N), dtype=np.float32)
    A[:, 1:-1, 1:-1] = rng.random((Ng - 2, N - 2), dtype=np.float32)
    ref = _numpy_jacobi(A, T)
    cuts = [round(i * Ng / nslabs) for i in range(nslabs + 1)]
    At = t(A)
    slabs = [MG.jacobi_slab(At[:, a:b], a, Ng) for a, b in zip(cuts, cuts[1:])]
    # the initial ghost rows of both planes (what jacobi()'s first exchange does)
    for up, lo in zip(slabs, slabs[1:]):
        up.A[:, up.top + up.rows:] = lo.A[:, lo.top:lo.top + up.bot]
        lo.A[:, :lo.top] = up.A[:, up.top + up.rows - lo.top:up.top + up.rows]
    peers = MG.PeerJacobi.chain(slabs)
    gens = [MG.jacobi_p2p_blocks(s, p, T) for s, p in zip(slabs, peers)]
    live = list(gens)
    while live:
        for g in list(live):
            try:
                next(g)
            except StopIteration:
                live.remove(g)
    torch.cuda.synchronize()
    got = np.concatenate([s.A[:, s.top:s.top + s.rows].cpu().numpy() for s in slabs], axis=1)
    np.testing.assert_array_equal(got[T % 2], ref[T % 2])
    np.testing.assert_array_equal(got[(T + 1) % 2][1:-1, 1:-1], ref[(T + 1) % 2][1:-1, 1:-1])
    assert all(int(p.flags.max()) > 0 for p in peers) or T == 0
