"""Multi-rank decompositions (paper_1902_10345_b200/multigpu.py) on CPU with
the gloo backend: world sizes 2 and 4, per-shard compute by the C oracle.
Every sharded result must equal the single-domain oracle bit for bit (the
decompositions keep each element's operation order)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

from conftest import REPO
from paper_1902_10345_b200 import multigpu as MG


class OracleBackend:
    """Per-shard compute on CPU tensors through the C oracle (test only)."""

    def hist(self, img, hist, oob, scale=256.0, div=1.0):
        h, bad = oracle.histogram(img.numpy(), hist.numpy(), scale, div)
        hist.copy_(torch.from_numpy(h))
        oob += bad

    def query(self, col, thr, out, count, op="<"):
        o, c = oracle.query(col.numpy(), thr, out.numpy(), count.numpy(), op)
        out.copy_(torch.from_numpy(o))
        count.copy_(torch.from_numpy(c))

    def spmv(self, rowptr, col, val, x, b):
        r = oracle.spmv(rowptr.numpy(), col.numpy(), val.numpy(), x.numpy(), b.numpy(), fp32=True)
        b.copy_(torch.from_numpy(r))

    def jacobi_step(self, src, dst, N, rows, r0, r1, coef, terms):
        s = src.numpy()
        d = dst.numpy()
        c32 = np.float32(coef)
        for i in range(r0, r1):
            acc = s[i + terms[0][0], 1 + terms[0][1]:N - 1 + terms[0][1]].copy()
            for di, dj in terms[1:]:
                acc = acc + s[i + di, 1 + dj:N - 1 + dj]
            d[i, 1:N - 1] = c32 * acc

    def jacobi_block(self, src, dst, k, coef):
        """k steps from plane src to plane dst with the kernels' semantics:
        intermediate states alternate between the two planes' borders
        (plane edges), only dst is written (state t+k)."""
        P = [src.numpy().copy(), dst.numpy().copy()]
        c32 = np.float32(coef)
        for i in range(k):
            s_, d_ = P[i % 2], P[(i + 1) % 2]
            acc = s_[1:-1, 1:-1] + s_[0:-2, 1:-1]
            acc = acc + s_[2:, 1:-1]
            acc = acc + s_[1:-1, 0:-2]
            acc = acc + s_[1:-1, 2:]
            d_[1:-1, 1:-1] = c32 * acc
        dst.copy_(torch.from_numpy(P[k % 2]))

    def can_band(self, plane):
        return True

    def jacobi_band(self, src, dst, k, r0, r1, coef):
        """rows [r0, r1) (interior only) of the k-step block src -> dst"""
        tmp = dst.clone()
        self.jacobi_block(src, tmp, k, coef)
        r0, r1 = max(r0, 1), min(r1, dst.shape[0] - 1)
        dst[r0:r1] = tmp[r0:r1]

    def gemm(self, A, B, C, reuse_b=False, ws_rows=None):
        C.copy_(torch.from_numpy(oracle.matmul(A.numpy(), B.numpy()).astype(np.float32)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = ["histogram", "query", "spmv", "jacobi", "jacobi_overlap", "jacobi_p2p", "gemm", "gemm_uneven",
         "strong_shares"]


def _worker(rank, world, port, names, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    for name in names:
        try:
            res[name] = globals()["_case_" + name](rank, world)
        except Exception:  # surface worker failures to the test
            import traceback
            res[name] = "ERROR " + traceback.format_exc()
    q.put((rank, res))
    dist.destroy_process_group()


def run_ranks(names, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, names, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    return out  # rank -> {case: result}


_RESULTS = {}


def results(world):
    if world not in _RESULTS:
        _RESULTS[world] = run_ranks(CASES, world)
    return _RESULTS[world]


# ------------------------------------------------------------------ cases

def _case_histogram(rank, world):
    rng = np.random.default_rng(0)
    img = rng.random((64 * world, 48), dtype=np.float32)
    img[::37, ::5] = 1.5  # out of range
    rows = img.shape[0] // world
    hist = torch.full((256,), 3, dtype=torch.int64)
    oob = torch.zeros(1, dtype=torch.int64)
    MG.histogram(dist, torch.from_numpy(img[rank * rows:(rank + 1) * rows].copy()), hist, oob, OracleBackend())
    ref, bad = oracle.histogram(img, np.full(256, 3, np.int64))
    ok = bool(np.array_equal(hist.numpy(), ref) and oob.item() == bad)
    # deferred all_reduce over two calls
    hist2 = torch.full((256,), 3, dtype=torch.int64)
    oob2 = torch.zeros(1, dtype=torch.int64)
    pending = []
    for _ in range(2):
        MG.histogram(dist, torch.from_numpy(img[rank * rows:(rank + 1) * rows].copy()), hist2, oob2, OracleBackend(),
                     pending=pending)
    MG.finish_histogram(pending, hist2, oob2)
    ok = ok and np.array_equal(hist2.numpy() - 3, 2 * (ref - 3)) and oob2.item() == 2 * bad
    return ok


def _case_query(rank, world):
    rng = np.random.default_rng(1)
    col = rng.random(1000 * world + 0, dtype=np.float32)
    n = col.size // world
    shard = torch.from_numpy(col[rank * n:(rank + 1) * n].copy())
    out = torch.zeros(n, dtype=torch.float32)
    count = torch.full((1,), 5, dtype=torch.int64)
    k, off, full = MG.query(dist, shard, 0.5, out, count, OracleBackend(), "<", gather=True)
    ref = col[col < 0.5]
    ok = count.item() == 5 + ref.size and np.array_equal(out[:k].numpy(), ref[off:off + k])
    if rank == 0:
        ok = ok and np.array_equal(full.numpy(), ref)
    # device-tensor bookkeeping without the gather
    count2 = torch.full((1,), 5, dtype=torch.int64)
    k2, off2, none = MG.query(dist, shard, 0.5, out, count2, OracleBackend(), "<")
    ok = ok and none is None and int(k2) == k and int(off2) == off and count2.item() == count.item()
    # deferred count exchanges over three calls
    count3 = torch.full((1,), 5, dtype=torch.int64)
    pending = []
    for _ in range(3):
        MG.query(dist, shard, 0.5, out, count3, OracleBackend(), "<", pending=pending)
    MG.finish_query(pending, count3)
    ok = ok and count3.item() == 5 + 3 * ref.size and not pending
    return bool(ok)


def _case_spmv(rank, world):
    rng = np.random.default_rng(2)
    Hl, Wl, nz = 50, 40, 7
    H, W = Hl * world, Wl * world
    cols = np.sort(rng.integers(0, W, (H, nz)), axis=1).astype(np.int32)
    vals = rng.random((H, nz), dtype=np.float32)
    x = rng.random(W, dtype=np.float32)
    b0 = rng.random(H, dtype=np.float32)
    rp_local = torch.from_numpy((np.arange(Hl + 1) * nz).astype(np.int32))
    b = torch.from_numpy(b0[rank * Hl:(rank + 1) * Hl].copy())
    MG.spmv(dist, rp_local, torch.from_numpy(cols[rank * Hl:(rank + 1) * Hl].reshape(-1).copy()),
            torch.from_numpy(vals[rank * Hl:(rank + 1) * Hl].reshape(-1).copy()),
            torch.from_numpy(x[rank * Wl:(rank + 1) * Wl].copy()), b, OracleBackend())
    ref = oracle.spmv((np.arange(H + 1) * nz).astype(np.int32), cols.reshape(-1), vals.reshape(-1), x, b0, fp32=True)
    return bool(np.array_equal(b.numpy(), ref[rank * Hl:(rank + 1) * Hl]))


def _case_jacobi(rank, world):
    rng = np.random.default_rng(3)
    rows, N, T = 9, 12, 17  # two 7-step blocks, a 1-step block, the final step
    Ng = rows * world
    A = rng.random((2, Ng, N), dtype=np.float32)  # distinct planes, non-zero borders

    def restated(terms):
        # the whole domain is not square, so a non-square restatement with
        # the kernels' op order is the reference here
        ref = A.copy()
        for t in range(T):
            s, d = ref[t % 2], ref[(t + 1) % 2]
            acc = s[1 + terms[0][0]:Ng - 1 + terms[0][0], 1 + terms[0][1]:N - 1 + terms[0][1]].copy()
            for di, dj in terms[1:]:
                acc = acc + s[1 + di:Ng - 1 + di, 1 + dj:N - 1 + dj]
            d[1:-1, 1:-1] = np.float32(0.2) * acc
        return ref
    ok = True
    for terms in (((0, 0), (-1, 0), (1, 0), (0, -1), (0, 1)), ((0, 1), (0, 0), (1, 0), (-1, 0), (0, -1))):
        ref = restated(terms)
        slab = MG.jacobi_slab(torch.from_numpy(A[:, rank * rows:(rank + 1) * rows].copy()), rank * rows, Ng)
        MG.jacobi(dist, slab, T, OracleBackend(), terms=terms)
        got = slab.A[:, slab.top:slab.top + rows].numpy()
        ok = ok and bool(np.array_equal(got, ref[:, rank * rows:(rank + 1) * rows]))
    return ok


def _case_jacobi_overlap(rank, world):
    """The overlapped schedule (edge bands, exchange in flight, interior
    band) on uneven row shares of a grid: equals the restatement."""
    rng = np.random.default_rng(5)
    Ng, N, T = 61 * world + 3, 20, 23
    A = rng.random((2, Ng, N), dtype=np.float32)
    ref = A.copy()
    for t in range(T):
        s, d = ref[t % 2], ref[(t + 1) % 2]
        acc = s[1:-1, 1:-1] + s[0:-2, 1:-1]
        acc = acc + s[2:, 1:-1]
        acc = acc + s[1:-1, 0:-2]
        acc = acc + s[1:-1, 2:]
        d[1:-1, 1:-1] = np.float32(0.2) * acc
    lo, hi = MG.share(Ng, rank, world)
    slab = MG.jacobi_slab(torch.from_numpy(A[:, lo:hi].copy()), lo, Ng)
    calls = []
    be = OracleBackend()
    band = be.jacobi_band
    be.jacobi_band = lambda *a: (calls.append(a[3:5]), band(*a))
    MG.jacobi(dist, slab, T, be)
    got = slab.A[:, slab.top:slab.top + (hi - lo)].numpy()
    return bool(calls) and bool(np.array_equal(got, ref[:, lo:hi]))


class HostP2POps:
    """The fused exchange's four device operations on shared CPU tensors
    (test only): the band through the oracle backend, the mirror as a row
    copy into the neighbour's (shared-memory) plane, the flags as words of
    a shared tensor that the waiting rank polls."""

    def band(self, src, dst, k, r0, r1, coef, stream):
        OracleBackend().jacobi_band(src, dst, k, r0, r1, coef)

    def band_mirror(self, src, dst, k, r0, r1, mirror, m0, m1, coef, stream):
        self.band(src, dst, k, r0, r1, coef, stream)
        a, b = max(r0, m0, 1), min(r1, m1, dst.shape[0] - 1)
        if b > a:
            mirror[a - m0:b - m0] = dst[a:b]

    def signal(self, flag, value, stream):
        flag.fill_(value)

    def wait(self, flag, value, stream):
        import time
        t0 = time.time()
        while int(flag.item()) < value:
            if time.time() - t0 > 60:
                raise TimeoutError(f"flag stuck at {int(flag.item())} < {value}")
            time.sleep(1e-4)


def _case_jacobi_p2p(rank, world):
    """The fused ghost exchange (multigpu.PeerJacobi: mirrored edge bands and
    flag words, no collective) across processes, its planes and flags in
    shared memory mapped through pg like the CUDA IPC handles: equals the
    restatement, with every neighbour's waits really waiting."""
    rng = np.random.default_rng(8)
    Ng, N, T = 61 * world + 5, 20, 23
    A = rng.random((2, Ng, N), dtype=np.float32)
    ref = A.copy()
    for t in range(T):
        s_, d_ = ref[t % 2], ref[(t + 1) % 2]
        acc = s_[1:-1, 1:-1] + s_[0:-2, 1:-1]
        acc = acc + s_[2:, 1:-1]
        acc = acc + s_[1:-1, 0:-2]
        acc = acc + s_[1:-1, 2:]
        d_[1:-1, 1:-1] = np.float32(0.2) * acc
    # CPU storages cross processes by shared-memory file name here (the
    # handles travel through pg's pickles, as CUDA IPC handles do)
    torch.multiprocessing.set_sharing_strategy("file_system")
    lo, hi = MG.share(Ng, rank, world)
    slab = MG.jacobi_slab(torch.from_numpy(A[:, lo:hi].copy()), lo, Ng)
    peer = MG.PeerJacobi(dist, slab, ops=HostP2POps())
    MG.jacobi(dist, slab, T, OracleBackend(), p2p=peer)
    got = slab.A[:, slab.top:slab.top + (hi - lo)].numpy()
    # a second call continues the flag counts (peer.base)
    return bool(np.array_equal(got, ref[:, lo:hi])) and peer.base > 0


def _case_gemm_uneven(rank, world):
    """gemm_pieces on shapes that do not divide by the grid (uneven row and
    K pieces: broadcasts instead of all_gather), pipelined and not."""
    grid = MG.GemmGrid(dist)
    rng = np.random.default_rng(6)
    M, K, N = 4 * grid.P + 3, 11, 3 * grid.Q + 2
    A = rng.random((M, K), dtype=np.float32)
    B = rng.random((K, N), dtype=np.float32)
    ref = oracle.matmul(A, B).astype(np.float32)
    a, b = MG.gemm_pieces(torch.from_numpy(A), torch.from_numpy(B), grid)
    r0, r1 = MG.share(M, grid.i, grid.P)
    c0, c1 = MG.share(N, grid.j, grid.Q)
    ok = True
    for pipe in (True, False):
        C = torch.zeros((r1 - r0, c1 - c0), dtype=torch.float32)
        MG.gemm(dist, grid, a, b, C, OracleBackend(), pipeline=pipe)
        ok = ok and bool(np.array_equal(C.numpy(), ref[r0:r1, c0:c1]))
    return ok


def _case_strong_shares(rank, world):
    """share() tiles [0, total) exactly, in rank order, sizes within one."""
    ok = True
    for total in (0, 1, world - 1, 4096, 8190, 1 << 22, 16384 + 3):
        parts = [MG.share(total, r, world) for r in range(world)]
        ok = ok and parts[0][0] == 0 and parts[-1][1] == total
        ok = ok and all(parts[r][1] == parts[r + 1][0] for r in range(world - 1))
        ok = ok and max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1
    return ok


def _case_gemm(rank, world):
    grid = MG.GemmGrid(dist)
    rng = np.random.default_rng(4)
    n, K = 8, 12
    A = rng.random((grid.P * n, K), dtype=np.float32)
    B = rng.random((K, grid.Q * n), dtype=np.float32)
    Ai = A[grid.i * n:(grid.i + 1) * n]                 # A row panel i
    Bj = B[:, grid.j * n:(grid.j + 1) * n]              # B column panel j
    a_piece = Ai[grid.j * (n // grid.Q):(grid.j + 1) * (n // grid.Q)]
    b_piece = Bj[grid.i * (K // grid.P):(grid.i + 1) * (K // grid.P)]
    C = torch.zeros((n, n), dtype=torch.float32)
    MG.gemm(dist, grid, torch.from_numpy(a_piece.copy()), torch.from_numpy(b_piece.copy()), C, OracleBackend())
    ref = oracle.matmul(A, B).astype(np.float32)
    return bool(np.array_equal(C.numpy(), ref[grid.i * n:(grid.i + 1) * n, grid.j * n:(grid.j + 1) * n]))


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", CASES)
def test_sharded_equals_single_domain(case, world):
    per_rank = {r: v[case] for r, v in results(world).items()}
    for r, v in per_rank.items():
        assert v is True, f"rank {r}: {v}"


def test_grid_shapes():
    assert [MG.grid_shape(w) for w in (1, 2, 4, 8)] == [(1, 1), (1, 2), (2, 2), (2, 4)]


@pytest.mark.gpu
def test_bench_multi_rank_plumbing_on_one_gpu(tmp_path):
    """bench.py's N=2 path end to end (torchrun, per-rank shards, collectives,
    max-over-ranks timing, one JSON line from rank 0) with both ranks on the
    one GPU over gloo (SDFGB_BENCH_SHARE_GPU): a plumbing check, not a
    measurement -- no kernel waits on another rank's kernel."""
    import json
    import socket
    import subprocess
    import sys
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, SDFGB_BENCH_SHARE_GPU="1")
    detail = tmp_path / "detail.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(REPO, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e", "--detail", str(detail),
           "--motif", "histogram,query,spmv,jacobi2d,gemm4096"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=REPO)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    assert len(line) < 2800  # the whole line survives in the driver's tail
    d = json.loads(line)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    full = json.load(open(detail))["motifs"]
    for m in ("histogram", "query", "spmv", "jacobi2d", "gemm4096"):
        assert d["motifs"][m]["v"] > 0, m
        assert d["motifs"][m]["ok"] is True, (m, full[m]["check"])  # strong split, checked result
    assert full["histogram"]["config"]["exchange"].startswith("p2p")
    assert full["jacobi2d"]["config"]["rows"] in ([0, 4096], [4096, 8192])


@pytest.mark.gpu
def test_bench_nccl_two_gpus(tmp_path):
    """bench.py at N=2 exactly as the driver launches it (torchrun, NCCL, one
    rank per GPU, strong scaling): every motif's sharded result passes its
    check.  Needs two GPUs; skipped on a one-GPU box."""
    import json
    import socket
    import subprocess
    import sys
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (NCCL over NVLink)")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(REPO, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=REPO)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    for m, v in d["motifs"].items():
        assert v["ok"] in (True, None), (m, v)
