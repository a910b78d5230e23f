"""Multi-GPU decompositions of the motifs: one process per
GPU, ``torch.distributed`` (NCCL on GPUs) for the exchanges, libsdfgb200
kernels for the per-shard compute.

Each runner takes ``pg`` (the ``torch.distributed`` module) and a compute
``backend``; the default is the device kernels of :mod:`.device`.  The
decompositions keep every element's operation order, so a sharded result is
bit-identical to the one-device result for histogram, query and Jacobi (and
for SpMV, whose rows stay whole, and GEMM, whose K stays whole).  bench.py
splits the configured shapes across ranks with :func:`share` (strong
scaling) and can also give every rank the whole shape (weak scaling).

The exchange steps are the ones the north star names:
  histogram  per-GPU partial bins -> all_reduce(sum)
  query      per-shard compaction -> all_gather of counts -> global offsets
             (output stays sharded at its global offset; gather is optional)
  spmv       row blocks, x sharded -> all_gather(x) -> row kernel
  jacobi     row blocks with 7-row ghost zones -> one send/recv of ghost
             rows per temporal block (up to 7 steps), sent as soon as the
             edge bands are computed and overlapped with the interior band
  gemm       2-D process grid -> all_gather of the B column panel, then the
             A row panel's pieces broadcast one by one, each piece's C rows
             computed while the next piece is in flight
"""

from __future__ import annotations

import math
from dataclasses import dataclass


def share(total, rank, world):
    """[lo, hi) of ``total`` units owned by ``rank``: contiguous, sizes
    differing by at most one (the strong-scaling split of every motif)."""
    return total * rank // world, total * (rank + 1) // world


class DeviceBackend:
    """Per-shard compute on the local GPU through the C ABI."""

    def __init__(self):
        from . import device
        self.d = device
        self._ws = {}

    def hist(self, img, hist, oob, scale=256.0, div=1.0):
        self.d.hist(img, hist, oob, scale, div)

    def query(self, col, thr, out, count, op="<"):
        import torch
        key = ("q", col.numel(), col.element_size(), col.device)
        if key not in self._ws:
            self._ws[key] = self.d.query_workspace(col.numel(), col.element_size(), col.device)
        self.d.query(col, thr, out, count, self._ws[key], op)

    def spmv(self, rowptr, col, val, x, b):
        self.d.spmv(rowptr, col, val, x, b)

    def jacobi_step(self, src, dst, N, rows, r0, r1, coef, terms):
        self.d.jacobi2d_step(src, dst, N, rows, 0, r0, r1, coef, terms)

    def jacobi_block(self, src, dst, k, coef):
        self.d.jacobi2d_block(src, dst, k, coef)

    def can_band(self, plane):
        return plane.shape[-1] >= 128 and plane.shape[-1] % 4 == 0

    def jacobi_band(self, src, dst, k, r0, r1, coef):
        self.d.jacobi2d_band(src, dst, k, r0, r1, coef)

    def gemm(self, A, B, C, reuse_b=False, ws_rows=None):
        """C = A @ B.  Row pieces of one product pass ws_rows (the tallest
        piece, so they share one workspace) and reuse_b after the first, so
        B is split once."""
        M, K = A.shape
        N = B.shape[1]
        rows = max(M, ws_rows or 0)
        key = ("g", rows, N, K, A.device)
        if key not in self._ws:
            self._ws[key] = self.d.gemm_workspace(rows, N, K, A.device)
        self.d.gemm(A, B, C, self._ws[key], b_split=reuse_b)


def _rank_world(pg):
    return pg.get_rank(), pg.get_world_size()


# ----------------------------------------------------------------- histogram

def histogram(pg, img_shard, hist, oob, backend, scale=256.0, div=1.0, pending=None):
    """hist += counts of the union of all ranks' shards (every rank ends with
    the same hist); oob likewise.  With a ``pending`` list the all_reduce is
    left in flight, overlapping the next shard (finish_histogram folds it)."""
    import torch
    nb = hist.numel()
    part = torch.zeros(nb + 1, dtype=hist.dtype, device=hist.device)  # bins, then the out-of-range count
    backend.hist(img_shard, part[:nb], part[nb:], scale, div)
    if pending is not None:
        pending.append((part, pg.all_reduce(part, async_op=True)))
        return
    pg.all_reduce(part)  # one collective for bins + oob
    hist += part[:nb]
    oob += part[nb:].to(oob.dtype)


def finish_histogram(pending, hist, oob):
    nb = hist.numel()
    for part, work in pending:
        work.wait()
        hist += part[:nb]
        oob += part[nb:].to(oob.dtype)
    pending.clear()


def _peer_access(tensors):
    """IPC-rebuilt tensors live on the exporting rank's device: let this
    rank's kernels reach them (cudaDeviceEnablePeerAccess)."""
    import torch
    from . import _lib
    L = _lib.load()
    here = torch.cuda.current_device()
    for dev in sorted({t.device.index for t in tensors} - {here}):
        _lib.check(L.sdfgb_enable_peer_access(dev))


class PeerHist:
    """Every rank's ``hist`` / ``oob`` device tensors mapped into this process
    (CUDA IPC handles exchanged once through ``pg``), for
    :func:`histogram_p2p`.  The tensors must stay alive and keep their
    storage while the mapping is in use."""

    def __init__(self, pg, hist, oob):
        import ctypes
        import torch
        from torch.multiprocessing.reductions import reduce_tensor
        rank, world = _rank_world(pg)
        if world > 8:
            raise ValueError("hist_p2p maps at most 8 ranks")
        if hist.dtype != torch.int64 or oob.dtype != torch.int64 or not hist.is_cuda:
            raise TypeError("hist / oob must be int64 CUDA tensors")
        mine = (reduce_tensor(hist), reduce_tensor(oob))
        handles = [None] * world
        pg.all_gather_object(handles, mine)
        self.hists, self.oobs = [], []
        for r, ((hf, ha), (of, oa)) in enumerate(handles):
            if r == rank:
                self.hists.append(hist)
                self.oobs.append(oob)
            else:
                self.hists.append(hf(*ha))
                self.oobs.append(of(*oa))
        _peer_access(self.hists + self.oobs)
        self.world = world
        self.bins = hist.numel()
        self.hist_ptrs = (ctypes.c_void_p * world)(*[t.data_ptr() for t in self.hists])
        self.oob_ptrs = (ctypes.c_void_p * world)(*[t.data_ptr() for t in self.oobs])


def histogram_p2p(pg, img_shard, peers: PeerHist, scale=256.0, div=1.0, stream=None):
    """hist += counts of this rank's shard on EVERY rank, from inside the
    histogram kernel (sdfgb_hist_f32_p2p: system-scope atomics into the
    peers' bins over NVLink) -- the partial-bins all-reduce fused into the
    compute.  Every rank's hist is complete once all ranks' calls are:
    :func:`finish_histogram_p2p` synchronises and barriers."""
    import torch
    from . import _lib
    if img_shard.dtype != torch.float32:
        raise TypeError("histogram_p2p takes float32 images")
    L = _lib.load()
    st = stream if stream is not None else torch.cuda.current_stream()
    import ctypes
    _lib.check(L.sdfgb_hist_f32_p2p(img_shard.data_ptr(), img_shard.numel(), float(scale), float(div),
                                    ctypes.cast(peers.hist_ptrs, ctypes.c_void_p),
                                    ctypes.cast(peers.oob_ptrs, ctypes.c_void_p), peers.world, peers.bins,
                                    st.cuda_stream))


def finish_histogram_p2p(pg, stream=None):
    import torch
    (stream or torch.cuda.current_stream()).synchronize()  # this rank's remote adds are done
    pg.barrier()                                          # and every other rank's


# --------------------------------------------------------------------- query

def query(pg, col_shard, thr, out_shard, count, backend, op="<", gather=False, pending=None):
    """Per-shard compaction.  Returns (k_local, offset, full): this rank's
    survivors are out_shard[0:k_local] and belong at global
    out_vals[offset:offset+k].  ``count`` (replicated) is advanced by the
    global survivor count.  Without ``gather`` k_local and offset are device
    tensors (nothing waits for the host); with it they are ints and rank 0
    also receives the concatenated survivors.  With a ``pending`` list the
    count exchange is left in flight (finish_query completes it)."""
    import torch
    rank, world = _rank_world(pg)
    local = torch.zeros(1, dtype=torch.int64, device=col_shard.device)
    backend.query(col_shard, thr, out_shard, local, op)
    counts = torch.empty(world, dtype=torch.int64, device=col_shard.device)
    if pending is not None and not gather:
        # streaming use: the count exchange runs on the collective's own
        # stream and overlaps the next shard's compaction; finish_query()
        # folds the gathered counts into ``count``
        pending.append((counts, pg.all_gather_into_tensor(counts, local, async_op=True)))
        return local, None, None
    pg.all_gather_into_tensor(counts, local)
    if not gather:
        # device-side bookkeeping: no host round trip per call
        count += counts.sum()
        return counts[rank:rank + 1], counts[:rank].sum(), None
    cl = counts.tolist()
    offset = sum(cl[:rank])
    count += int(sum(cl))
    kmax = max(cl) if cl else 0
    pad = torch.zeros(max(kmax, 1), dtype=out_shard.dtype, device=out_shard.device)
    pad[:cl[rank]] = out_shard[:cl[rank]]
    allv = torch.empty(world * max(kmax, 1), dtype=out_shard.dtype, device=out_shard.device)
    pg.all_gather_into_tensor(allv, pad)
    full = torch.cat([allv[r * max(kmax, 1): r * max(kmax, 1) + cl[r]] for r in range(world)]) \
        if rank == 0 else None
    return cl[rank], offset, full


class QueryGather:
    """Rank ``root``'s gathered-output buffer and reservation counter mapped
    into every rank (CUDA IPC handles exchanged once through ``pg``), for
    :func:`query_p2p`.  ``out_root`` / ``reserve`` are only read on the root;
    the other ranks pass tensors of the right dtype (they are not used)."""

    def __init__(self, pg, out_root, reserve, root=0):
        import torch
        from torch.multiprocessing.reductions import reduce_tensor
        rank, world = _rank_world(pg)
        if out_root.dtype != torch.float32 or reserve.dtype != torch.int64 or not out_root.is_cuda:
            raise TypeError("out_root must be float32 and reserve int64 CUDA tensors")
        obj = [(reduce_tensor(out_root), reduce_tensor(reserve)) if rank == root else None]
        pg.broadcast_object_list(obj, src=root)
        if rank == root:
            self.out, self.reserve = out_root, reserve
        else:
            (of, oa), (rf, ra) = obj[0]
            self.out, self.reserve = of(*oa), rf(*ra)
        _peer_access([self.out, self.reserve])
        self.root = root


def query_p2p(pg, col_shard, thr, gather: QueryGather, ws, op="<", stream=None):
    """This rank's survivors of ``col OP thr`` go straight into the root's
    output (sdfgb_query_f32_p2p: slots reserved with system-scope atomics on
    the root's counter, survivors stored over NVLink): compaction and gather
    in one pass, no collective.  :func:`finish_query_p2p` completes it."""
    import torch
    from . import _lib
    if col_shard.dtype != torch.float32:
        raise TypeError("query_p2p takes float32 columns")
    L = _lib.load()
    st = stream if stream is not None else torch.cuda.current_stream()
    _lib.check(L.sdfgb_query_f32_p2p(col_shard.data_ptr(), col_shard.numel(), _lib.CMP[op], float(thr),
                                     gather.out.data_ptr(), gather.reserve.data_ptr(), ws.data_ptr(), ws.numel(),
                                     st.cuda_stream))


def finish_query_p2p(pg, gather: QueryGather, count, stream=None):
    """Wait for every rank's gather, advance ``count`` (replicated) by the
    number of survivors gathered, and re-zero the root's counter.  Returns
    that number (a host int)."""
    import torch
    (stream or torch.cuda.current_stream()).synchronize()
    pg.barrier()                        # every rank's survivors have landed
    total = int(gather.reserve.item())  # the root's counter, read over NVLink elsewhere
    count += total
    torch.cuda.synchronize()
    pg.barrier()                        # everyone has read it
    rank, _ = _rank_world(pg)
    if rank == gather.root:
        gather.reserve.zero_()
        torch.cuda.synchronize()
    pg.barrier()
    return total


def finish_query(pending, count):
    """Wait for the deferred count exchanges of query(..., pending=...) and
    advance ``count`` by every call's global survivor count."""
    for counts, work in pending:
        work.wait()
        count += counts.sum()
    pending.clear()


# ---------------------------------------------------------------------- spmv

def spmv(pg, rowptr_local, col, val, x_shard, b_local, backend):
    """Row-block SpMV: rowptr_local/col/val/b_local are this rank's rows (col
    holds GLOBAL column ids), x is sharded in equal contiguous blocks."""
    import torch
    rank, world = _rank_world(pg)
    x = torch.empty(x_shard.numel() * world, dtype=x_shard.dtype, device=x_shard.device)
    pg.all_gather_into_tensor(x, x_shard)
    backend.spmv(rowptr_local, col, val, x, b_local)
    return x


# -------------------------------------------------------------------- jacobi

GHOST = 7  # ghost rows per neighbour = the deepest temporal block


@dataclass
class JacobiSlab:
    """This rank's rows of the global [2, Ng, N] array plus ``top``/``bot``
    ghost rows towards its neighbours: planes [2, top + rows + bot, N].
    Local row l <-> global row g0 + l - top.  The first rank has no rows
    above it, so its plane's top edge IS the global border row 0 (and the
    last rank's bottom edge is row Ng-1): the kernels' plane-edge border
    is the reference's border exactly there."""
    A: object
    g0: int
    rows: int
    Ng: int
    top: int = 1
    bot: int = 1


def jacobi_slab(A_global_rows, g0, Ng, ghost=GHOST):
    """Build a slab from this rank's rows [2, rows, N] (a copy)."""
    import torch
    two, rows, N = A_global_rows.shape
    top = ghost if g0 > 0 else 0
    bot = ghost if g0 + rows < Ng else 0
    if (top or bot) and rows < ghost:
        raise ValueError(f"slab of {rows} rows is thinner than the {ghost} ghost rows")
    A = torch.zeros((2, top + rows + bot, N), dtype=A_global_rows.dtype, device=A_global_rows.device)
    A[:, top:top + rows] = A_global_rows
    return JacobiSlab(A, g0, rows, Ng, top, bot)


def jacobi(pg, slab: JacobiSlab, T, backend, coef=0.2, terms=((0, 0), (-1, 0), (1, 0), (0, -1), (0, 1)),
           overlap=True, p2p: "PeerJacobi" = None):
    """T steps of the guard loop (loops.py:31-61) over row blocks with
    ghost zones: the single-GPU temporal-blocking schedule (odd blocks of
    7/5/3 steps, then one final step so the other plane ends at state T-1)
    with one exchange of ghost rows per block of up to GHOST steps (GHOST
    rows of N fp32 per neighbour, instead of a halo per step).  Every owned
    row sits at least GHOST rows from a ghost edge, so after k <= GHOST
    steps it is exact; ghost rows are refreshed before they are read again.

    With ``overlap`` (and a backend that computes row bands) each block
    first computes the owned rows within EDGE of a neighbour -- the rows the
    neighbours' ghost zones need -- then posts the exchange of those rows
    and computes the interior band while it is in flight; the next block
    waits for it.  Non-canonical stencil orders take one step per block.

    With ``p2p`` (a :class:`PeerJacobi`, device backend) the exchange is
    fused into the edge-band kernels over NVLink instead
    (:func:`jacobi_p2p_blocks`)."""
    rank, world = _rank_world(pg)
    A = slab.A
    canon = tuple(map(tuple, terms)) == ((0, 0), (-1, 0), (1, 0), (0, -1), (0, 1))
    top, rows, bot = slab.top, slab.rows, slab.bot
    band = bool(overlap and canon and hasattr(backend, "jacobi_band") and backend.can_band(A[0])
                and (top or bot) and rows >= 3 * EDGE)
    # both planes' ghost rows once: the border columns of the ghost rows are
    # border values of their own plane, read by intermediate states of the
    # other parity and never exchanged again
    _ghost_exchange(pg, A[1], slab, rank, world)
    _ghost_exchange(pg, A[0], slab, rank, world)
    if p2p is not None and band:
        for _ in jacobi_p2p_blocks(slab, p2p, T, coef):
            pass
        if A.is_cuda:
            import torch
            torch.cuda.current_stream().synchronize()
        pg.barrier()  # no neighbour still writes into this rank's planes
        return
    t = 0
    pending = None
    while t < T:
        if not canon:
            k = 1
        elif T - t > 1:
            k = min(GHOST, T - 1 - t)
            k -= (k % 2 == 0)
        else:
            k = 1
        src, dst = A[t % 2], A[(t + 1) % 2]
        if pending is not None:
            _finish_exchange(pending)  # src's ghost rows have landed
            pending = None
        if band:
            lo, hi = top, top + rows  # owned rows
            e0 = lo + EDGE if top else lo
            e1 = hi - EDGE if bot else hi
            if top:
                backend.jacobi_band(src, dst, k, lo, e0, coef)
            if bot:
                backend.jacobi_band(src, dst, k, e1, hi, coef)
            pending = _ghost_exchange(pg, dst, slab, rank, world, wait=False)
            backend.jacobi_band(src, dst, k, e0, e1, coef)
        else:
            if canon:
                backend.jacobi_block(src, dst, k, coef)
            else:
                M = A.shape[1]
                backend.jacobi_step(src, dst, A.shape[-1], M, 1, M - 1, coef, terms)
            _ghost_exchange(pg, dst, slab, rank, world)
        t += k
    if pending is not None:
        _finish_exchange(pending)


EDGE = 16  # edge-band rows computed before the exchange (>= GHOST; the strip kernel's minimum band)


class PeerJacobi:
    """The neighbour slabs' planes and flag words mapped into this process
    (CUDA IPC handles exchanged once through ``pg``), for the fused ghost
    exchange of :func:`jacobi` (``p2p=``): the edge-band kernels store the
    rows a neighbour's ghost zone needs straight into that neighbour's
    planes over NVLink (sdfgb_jacobi2d_band_mirror_f32), and int32 flag words
    order the ranks (sdfgb_flag_signal / sdfgb_flag_wait) -- no collective.

    flags (this rank's, written by its neighbours): [0] blocks whose ghost
    rows the rank above has delivered, [1] the same from the rank below,
    [2] blocks the rank above has finished, [3] blocks the rank below has
    finished.  Counts only grow (``base`` carries them across calls)."""

    def __init__(self, pg=None, slab: "JacobiSlab" = None, _local=None, ops=None):
        import torch
        self.base = 0
        self.up = self.down = None
        self.ops = ops if ops is not None else DeviceP2POps()
        if _local is not None:  # one-process construction (tests): see chain()
            return
        import io
        import pickle
        from multiprocessing.reduction import ForkingPickler
        import torch.multiprocessing  # noqa: F401  (registers the tensor reductions)

        def export(t):
            # CUDA: an IPC handle; CPU (tests): a shared-memory segment
            if not t.is_cuda:
                t.share_memory_()
            buf = io.BytesIO()
            ForkingPickler(buf, pickle.HIGHEST_PROTOCOL).dump(t)
            return buf.getvalue()
        rank, world = _rank_world(pg)
        self.flags = torch.zeros(4, dtype=torch.int32, device=slab.A.device)
        mine = (export(slab.A), export(self.flags), slab.top, slab.rows, slab.bot)
        allh = [None] * world
        pg.all_gather_object(allh, mine)
        mapped = []
        for r in (rank - 1, rank + 1):
            if 0 <= r < world:
                a, f, top, rows, bot = allh[r]
                nb = {"A": pickle.loads(a), "flags": pickle.loads(f), "top": top, "rows": rows, "bot": bot}
                mapped += [nb["A"], nb["flags"]]
            else:
                nb = None
            if r == rank - 1:
                self.up = nb
            else:
                self.down = nb
        if slab.A.is_cuda:
            _peer_access(mapped)

    @classmethod
    def chain(cls, slabs):
        """Vertically adjacent slabs of ONE process (tests: their blocks are
        then driven in turn on one stream, see jacobi_p2p_blocks)."""
        import torch
        peers = [cls(_local=True) for _ in slabs]
        for p, s in zip(peers, slabs):
            p.flags = torch.zeros(4, dtype=torch.int32, device=s.A.device)
        for (a, up), (b, lo) in zip(zip(peers, slabs), zip(peers[1:], slabs[1:])):
            a.down = {"A": lo.A, "flags": b.flags, "top": lo.top, "rows": lo.rows, "bot": lo.bot}
            b.up = {"A": up.A, "flags": a.flags, "top": up.top, "rows": up.rows, "bot": up.bot}
        return peers


class DeviceP2POps:
    """The device side of the fused exchange (libsdfgb200); a test can swap
    in host implementations of the same four operations."""

    def band(self, src, dst, k, r0, r1, coef, stream):
        from . import device
        device.jacobi2d_band(src, dst, k, r0, r1, coef, stream)

    def band_mirror(self, src, dst, k, r0, r1, mirror, m0, m1, coef, stream):
        from . import device
        device.jacobi2d_band_mirror(src, dst, k, r0, r1, mirror.data_ptr(), m0, m1, coef, stream)

    def signal(self, flag, value, stream):
        from . import device
        device.flag_signal(flag.data_ptr(), value, stream)

    def wait(self, flag, value, stream):
        from . import device
        device.flag_wait(flag.data_ptr(), value, stream)


def jacobi_p2p_blocks(slab: "JacobiSlab", peer: PeerJacobi, T, coef=0.2, stream=None):
    """The canonical-stencil schedule of :func:`jacobi` with the fused ghost
    exchange, one temporal block per ``next()`` (a generator, so a test can
    interleave two slabs of one process on one stream).  Block b (k steps,
    src = A[t % 2] -> dst):

      1. wait until both neighbours delivered block b-1's ghost rows into
         src (flags[0], flags[1] >= b) and finished block b-1 -- the last
         reader of the ghost rows this block overwrites in their dst
         (flags[2], flags[3] >= b);
      2. the edge bands (EDGE rows at each neighbour), their first / last
         GHOST rows stored into the neighbour's dst ghost rows as well;
      3. signal the neighbours: ghost rows of block b delivered;
      4. the interior band;
      5. signal the neighbours: block b finished.
    Ghost rows of both planes must hold the initial state (one exchange
    before the first block, as jacobi() does)."""
    ops = peer.ops
    A = slab.A
    top, rows, bot = slab.top, slab.rows, slab.bot
    lo, hi = top, top + rows
    e0 = lo + EDGE if top else lo
    e1 = hi - EDGE if bot else hi
    up, down = peer.up, peer.down
    fl = peer.flags
    t, b = 0, 0
    while t < T:
        if T - t > 1:
            k = min(GHOST, T - 1 - t)
            k -= (k % 2 == 0)
        else:
            k = 1
        src, dst = A[t % 2], A[(t + 1) % 2]
        n = peer.base + b  # blocks before this one
        if b > 0:
            if up is not None:
                ops.wait(fl[0:1], n, stream)
                ops.wait(fl[2:3], n, stream)
            if down is not None:
                ops.wait(fl[1:2], n, stream)
                ops.wait(fl[3:4], n, stream)
        plane = (t + 1) % 2
        if up is not None:  # my rows [lo, lo + GHOST) -> the rank above's bottom ghost rows
            g = up["top"] + up["rows"]
            ops.band_mirror(src, dst, k, lo, e0, up["A"][plane][g:g + GHOST], lo, lo + GHOST, coef, stream)
        if down is not None:  # my rows [hi - GHOST, hi) -> the rank below's top ghost rows
            ops.band_mirror(src, dst, k, e1, hi, down["A"][plane][0:GHOST], hi - GHOST, hi, coef, stream)
        if up is not None:
            ops.signal(up["flags"][1:2], n + 1, stream)    # its [1]: delivered from below
        if down is not None:
            ops.signal(down["flags"][0:1], n + 1, stream)  # its [0]: delivered from above
        ops.band(src, dst, k, e0, e1, coef, stream)
        if up is not None:
            ops.signal(up["flags"][3:4], n + 1, stream)    # its [3]: below finished
        if down is not None:
            ops.signal(down["flags"][2:3], n + 1, stream)  # its [2]: above finished
        t += k
        b += 1
        yield b
    peer.base += b


def _ghost_exchange(pg, plane, slab: JacobiSlab, rank, world, wait=True):
    """Owned edge rows -> the neighbours' ghost rows (batched send/recv).
    With ``wait=False`` the exchange stays in flight and the returned
    handle goes to :func:`_finish_exchange` (NCCL: the sends/receives run on
    the collective stream, after the work already queued on this one)."""
    ops = []
    top, rows, bot = slab.top, slab.rows, slab.bot
    if rank > 0 and top:
        ops.append(pg.P2POp(pg.isend, plane[top:2 * top].contiguous(), rank - 1))
        ops.append(pg.P2POp(pg.irecv, plane[0:top], rank - 1))
    if rank < world - 1 and bot:
        ops.append(pg.P2POp(pg.isend, plane[top + rows - bot:top + rows].contiguous(), rank + 1))
        ops.append(pg.P2POp(pg.irecv, plane[top + rows:top + rows + bot], rank + 1))
    if not ops:
        return None
    back = []
    if plane.is_cuda and pg.get_backend() == "gloo":
        # gloo moves host memory only: stage the rows through the host
        import torch
        staged = []
        for op in ops:
            h = op.tensor.cpu() if op.op is pg.isend else torch.empty(op.tensor.shape, dtype=op.tensor.dtype)
            if op.op is pg.irecv:
                back.append((op.tensor, h))
            staged.append(pg.P2POp(op.op, h, op.peer))
        ops = staged
    handle = (pg.batch_isend_irecv(ops), back)
    if wait:
        _finish_exchange(handle)
        return None
    return handle


def _finish_exchange(handle):
    works, back = handle
    for r in works:
        r.wait()
    for dev, h in back:
        dev.copy_(h)


# ---------------------------------------------------------------------- gemm

def grid_shape(world):
    """P x Q process grid, P <= Q, as square as possible (2 -> 1x2, 4 -> 2x2, 8 -> 2x4)."""
    p = int(math.isqrt(world))
    while world % p:
        p -= 1
    return p, world // p


class GemmGrid:
    """Row / column sub-groups of the P x Q grid (rank = i * Q + j)."""

    def __init__(self, pg):
        rank, world = _rank_world(pg)
        self.P, self.Q = grid_shape(world)
        self.i, self.j = divmod(rank, self.Q)
        self.row_groups = [pg.new_group([i * self.Q + j for j in range(self.Q)]) for i in range(self.P)]
        self.col_groups = [pg.new_group([i * self.Q + j for i in range(self.P)]) for j in range(self.Q)]
        self.row_group = self.row_groups[self.i]
        self.col_group = self.col_groups[self.j]


def gemm_pieces(A, B, grid: GemmGrid):
    """This rank's inputs of the P x Q decomposition of C = A @ B, cut from
    the whole operands: A row panel i split by rows over the Q ranks of
    grid row i, B column panel j split by rows (of K) over the P ranks of
    grid column j.  Returns contiguous (A_piece, B_piece); this rank's C
    block is rows share(M, i, P) x columns share(N, j, Q)."""
    M, K = A.shape
    N = B.shape[1]
    a0, a1 = share(M, grid.i, grid.P)
    q0, q1 = share(a1 - a0, grid.j, grid.Q)
    b0, b1 = share(N, grid.j, grid.Q)
    k0, k1 = share(K, grid.i, grid.P)
    return A[a0 + q0:a0 + q1].contiguous(), B[k0:k1, b0:b1].contiguous()


def gemm(pg, grid: GemmGrid, A_piece, B_piece, C_block, backend, pipeline=True):
    """C block (i, j) = A row panel i x B column panel j (pieces as cut by
    :func:`gemm_pieces`).  The B panel is all-gathered inside grid column j
    (K whole).  With ``pipeline`` the A panel's pieces are then broadcast
    inside grid row i, all in flight at once, and the C rows of each piece
    are computed as soon as it has landed (this rank's own piece first), so
    the A exchange overlaps the MMA.  K is never split: every C element
    keeps the single-device summation."""
    import torch
    K = A_piece.shape[1]
    kp = [share(K, r, grid.P) for r in range(grid.P)]
    Bp = torch.empty((K, B_piece.shape[1]), dtype=B_piece.dtype, device=B_piece.device)
    _gather_rows(pg, [Bp[a:b] for a, b in kp], B_piece, grid.i, [i * grid.Q + grid.j for i in range(grid.P)],
                 grid.col_group)
    rows = [share(C_block.shape[0], q, grid.Q) for q in range(grid.Q)]
    if not pipeline or grid.Q == 1:
        Aq = torch.empty((C_block.shape[0], K), dtype=A_piece.dtype, device=A_piece.device)
        _gather_rows(pg, [Aq[a:b] for a, b in rows], A_piece, grid.j, [grid.i * grid.Q + q for q in range(grid.Q)],
                     grid.row_group)
        backend.gemm(Aq, Bp, C_block)
        return
    bufs = [A_piece.contiguous() if q == grid.j else
            torch.empty((b - a, K), dtype=A_piece.dtype, device=A_piece.device) for q, (a, b) in enumerate(rows)]
    works = [pg.broadcast(bufs[q], src=grid.i * grid.Q + q, group=grid.row_group, async_op=True)
             for q in range(grid.Q)]
    tallest = max(b - a for a, b in rows)
    first = True
    for q in [grid.j] + [q for q in range(grid.Q) if q != grid.j]:
        works[q].wait()
        a, b = rows[q]
        if b > a:  # B is split by the first piece's call, reused by the others
            backend.gemm(bufs[q], Bp, C_block[a:b], reuse_b=not first, ws_rows=tallest)
            first = False


def _gather_rows(pg, outs, mine, me, ranks, group):
    """outs[q] <- rank ranks[q]'s piece (row blocks of one tensor): one
    all_gather when the pieces are equal, else one broadcast per piece."""
    if all(o.shape == outs[0].shape for o in outs):
        pg.all_gather(outs, mine.contiguous(), group=group)
        return
    outs[me].copy_(mine)
    for q, o in enumerate(outs):
        pg.broadcast(o, src=ranks[q], group=group)
