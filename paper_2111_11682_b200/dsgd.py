"""Multi-GPU DSGD and sharded simLSH over torch.distributed.

One process per GPU.  With D ranks the matrix is cut into D row blocks and D column
blocks exactly as the reference's make_partition (parallel.py:99-107), and every stage
trains the same D disjoint (row block, column block) pairs as parallel_train(D)
(worker w: row block (w + s) % D, column block w; parallel.py:36-41).  Which side of
the model stays put and which one travels is a free choice -- the pairs per stage are
the same either way, so both are bit-identical to parallel_train(D) with the exact
stage kernel:

  side="cols" (north_star; the default whenever N(F+2K+1) < M(F+1), e.g. Netflix):
      rank d keeps row block d -- its ratings R[d, :], u_i, b_i -- resident, and at
      stage s trains column block (d - s) % D; after each stage the column block's
      v_j, w_j, c_j, b_hat_j move one step around the ring (to rank d+1).  At C3 with
      D = 8 that is 2,221 x (128 + 2*32 + 1) floats = 1.7 MB per stage per GPU.
  side="rows": rank d keeps column block d and trains row block (d + s) % D; u_i, b_i
      move (to rank d-1): 31 MB per stage per GPU at C3, D = 8.

Every rank initialises only the parameter blocks it owns (the PCG64 stream of
init_params jumped to the block's offset, csrc/init.cu).  With side="cols" a rank also
holds only its row block of the ratings: the explicit-neighbour lookups r(i, J[j, k]) of
a rating (i, j) read row i only, which is in the shard, so no rank ever materialises the
whole matrix or the whole model.  With side="rows" a rank trains column block d against
every row, and those lookups read whole rows, so the ratings are replicated.

simLSH is sharded by columns: row hashes are a pure function of (seed, g, m, i), so each
rank hashes its own column block with no exchange, ONE all-gather of the (q, N) group
keys gives every rank the buckets, each rank selects top-K for its own columns, and one
all-gather assembles J^K -- bit-identical to simlsh_topk.

The ring orchestration is device-agnostic (CPU tensors + gloo in the tests, CUDA
tensors + NCCL in production); a stage's computation is a callback.
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass

import numpy as np


@dataclass
class RingPlan:
    """Static DSGD plan for D ranks over an M x N matrix; ``side`` names the parameter
    blocks that travel ("rows": u/b, "cols": v/w/c/b_hat)."""

    D: int
    M: int
    N: int
    side: str = "rows"

    def __post_init__(self):
        if self.side not in ("rows", "cols"):
            raise ValueError(f"side must be 'rows' or 'cols', got {self.side!r}")
        self.row_bounds = np.array([(d * self.M) // self.D for d in range(self.D + 1)], np.int64)
        self.col_bounds = np.array([(d * self.N) // self.D for d in range(self.D + 1)], np.int64)

    def stage_block(self, rank: int, stage: int):
        """(row block, column block) rank trains at `stage` -- parallel_train's pair of
        worker (rank - stage) % D (side cols) or worker rank (side rows)."""
        if self.side == "rows":
            return (rank + stage) % self.D, rank
        return rank, (rank - stage) % self.D

    def row_block(self, rank: int, stage: int) -> int:
        return self.stage_block(rank, stage)[0]

    def moving_block(self, rank: int, stage: int) -> int:
        rb, cb = self.stage_block(rank, stage)
        return rb if self.side == "rows" else cb

    def send_peer(self, rank: int) -> int:
        return (rank - 1) % self.D if self.side == "rows" else (rank + 1) % self.D

    def recv_peer(self, rank: int) -> int:
        return (rank + 1) % self.D if self.side == "rows" else (rank - 1) % self.D

    def rows(self, rb: int) -> slice:
        return slice(int(self.row_bounds[rb]), int(self.row_bounds[rb + 1]))

    def cols(self, cb: int) -> slice:
        return slice(int(self.col_bounds[cb]), int(self.col_bounds[cb + 1]))

    def _sub(self, n: int, blk: int, part: int, parts: int) -> slice:
        """Part `part` of block blk cut into `parts`: block blk*parts + part of the
        D*parts-way partition, whose bounds contain the D-way ones
        ((k*n)//D == (k*parts*n)//(D*parts))."""
        k, m = blk * parts + part, self.D * parts
        return slice((k * n) // m, ((k + 1) * n) // m)

    def sub_rows(self, rb: int, part: int, parts: int) -> slice:
        return self._sub(self.M, rb, part, parts)

    def sub_cols(self, cb: int, part: int, parts: int) -> slice:
        return self._sub(self.N, cb, part, parts)

    def moving_span(self, blk: int, part: int = 0, parts: int = 1) -> slice:
        return self.sub_rows(blk, part, parts) if self.side == "rows" else self.sub_cols(blk, part, parts)


def choose_side(M: int, N: int, F: int, K: int) -> str:
    """Rotate the smaller parameter side: the column block (v, w, c, b_hat: F + 2K + 1
    values per column) unless the row block (u, b: F + 1 per row) is smaller."""
    return "cols" if N * (F + 2 * K + 1) < M * (F + 1) else "rows"


def _host_staging() -> bool:
    """Gloo has no CUDA send/recv: stage device tensors through host memory."""
    import torch.distributed as dist
    return dist.get_backend() == "gloo"


def _shift_part(plan: RingPlan, rank: int, stage: int, part: int, parts: int, tensors, group=None):
    """Start the ring shift of one sub-block of the moving side: send part `part` of the
    block trained at `stage` to send_peer, receive the same part of the next stage's block
    from recv_peer.  Returns a finisher.  With NCCL the requests run on NCCL's stream,
    which waits only for the work enqueued before this call (the sub-block's stage
    kernel), so the transfer overlaps the next sub-block's kernel; finishing makes the
    current stream wait for it."""
    import torch.distributed as dist
    send = plan.moving_span(plan.moving_block(rank, stage), part, parts)
    recv = plan.moving_span(plan.moving_block(rank, stage + 1), part, parts)
    dst, src = plan.send_peer(rank), plan.recv_peer(rank)
    stage_host = _host_staging()
    tensors = [t for t in tensors if t.numel()]
    ops, recv_bufs = [], []
    for t in tensors:
        out = t[send].contiguous()
        if stage_host and out.is_cuda:
            out = out.cpu()
        ops.append(dist.P2POp(dist.isend, out, dst, group))
    for t in tensors:
        buf = t[recv]
        if stage_host and buf.is_cuda:
            buf = buf.cpu()
        elif not buf.is_contiguous():
            buf = buf.contiguous()
        recv_bufs.append(buf)
        ops.append(dist.P2POp(dist.irecv, buf, src, group))
    reqs = dist.batch_isend_irecv(ops) if ops else []

    def finish():
        for req in reqs:
            req.wait()
        for t, buf in zip(tensors, recv_bufs):
            view = t[recv]
            if view.data_ptr() != buf.data_ptr():
                view.copy_(buf)
    return finish


def ring_shift(plan: RingPlan, rank: int, stage: int, tensors, group=None) -> None:
    """After stage `stage`: move the block just trained to send_peer and receive the next
    stage's block from recv_peer, in place, for every tensor given (first dim = M for
    side rows, N for side cols)."""
    if plan.D > 1:
        _shift_part(plan, rank, stage, 0, 1, tensors, group)()


def run_epoch(plan: RingPlan, rank: int, stage_fn, moving_tensors, group=None, parts: int = 1) -> None:
    """One DSGD epoch: D stages, each followed by the ring shift of the moving side.

    parts > 1 pipelines the shift: each stage runs as `parts` sub-blocks of the moving
    side (stage_fn(s, rb, cb, part)), and a sub-block is sent as soon as its kernel is
    enqueued while the next sub-block trains; a stage's sub-block waits only for its own
    part to arrive.  Each column still sees its entries of the block in row order and
    each row its columns in ascending order, so with the exact stage kernel the result is
    the same as parts = 1 (and parallel_train) bit for bit."""
    pending = {}
    for s in range(plan.D):
        rb, cb = plan.stage_block(rank, s)
        for h in range(parts):
            if h in pending:
                pending.pop(h)()
            stage_fn(s, rb, cb, h)
            if plan.D > 1:
                pending[h] = _shift_part(plan, rank, s, h, parts, moving_tensors, group)
    for h in sorted(pending):
        pending.pop(h)()


def allgather_blocks(t, bounds: np.ndarray, rank: int, D: int, group=None):
    """Every rank contributes rows [bounds[rank], bounds[rank+1]) of the full-size
    tensor t; on return t holds all blocks on every rank."""
    import torch
    import torch.distributed as dist
    if D == 1 or t.numel() == 0:
        return t
    sizes = np.diff(bounds)
    mx = int(sizes.max())
    tail = tuple(t.shape[1:])
    send = torch.zeros((mx,) + tail, dtype=t.dtype, device=t.device)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    send[:hi - lo] = t[lo:hi]
    if _host_staging() and send.is_cuda:
        send = send.cpu()
    outs = [torch.empty_like(send) for _ in range(D)]
    dist.all_gather(outs, send, group=group)
    for d in range(D):
        a, b = int(bounds[d]), int(bounds[d + 1])
        t[a:b] = outs[d][:b - a].to(t.device)
    return t


def _all_reduce_sum(t, group=None):
    import torch.distributed as dist
    if _host_staging() and t.is_cuda:
        h = t.cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, group=group)
    return t


# ------------------------------------------------------------------ shards ---

def shard_device_ratings(ratings, plan: RingPlan, rank: int, by: str):
    """This rank's shard of a host SparseRatings as a DeviceRatings over the global
    index space: by="rows" -> row block `rank` (a contiguous CSR slice), by="cols" ->
    column block `rank` (a contiguous CSC slice).  Baselines are left for the caller."""
    from . import _native as nat
    from .synth import device_ratings_from_sorted
    t = nat.torch()
    M, N = ratings.M, ratings.N
    if by == "rows":
        sl = plan.rows(rank)
        a, b = int(ratings.row_ptr[sl.start]), int(ratings.row_ptr[sl.stop])
        rows = np.repeat(np.arange(sl.start, sl.stop, dtype=np.int32), np.diff(ratings.row_ptr[sl.start:sl.stop + 1]))
        r = nat.to_dev(rows, np.int32)
        c = nat.to_dev(ratings.row_cols[a:b], np.int32)
        v = nat.to_dev(ratings.row_vals[a:b], np.float64)
        order = t.argsort(c.to(t.int64) * M + r.to(t.int64))
        r, c, v = r[order], c[order], v[order]
    else:
        sl = plan.cols(rank)
        a, b = int(ratings.col_ptr[sl.start]), int(ratings.col_ptr[sl.stop])
        c = nat.to_dev(np.repeat(np.arange(sl.start, sl.stop, dtype=np.int32),
                                 np.diff(ratings.col_ptr[sl.start:sl.stop + 1])), np.int32)
        r = nat.to_dev(ratings.col_rows[a:b], np.int32)
        v = nat.to_dev(ratings.col_vals[a:b], np.float64)
    return device_ratings_from_sorted(M, N, r, c, v, baselines=False)


def global_baselines(shard, group=None):
    """compute_baselines (data.py:289-309) of the whole matrix from the ranks' shards:
    per-row / per-column sums and counts, one all-reduce.  Exact (hence bit-identical to
    the reference) for integer-valued ratings; returns (mu, b, b_hat) device tensors."""
    from . import _native as nat
    t = nat.torch()
    M, N = shard.M, shard.N
    cs = nat.empty((max(N, 1),), "float64")
    rs = nat.empty((max(M, 1),), "float64")
    nat.call("culsh_segment_sums", N, nat.ptr(shard.col_ptr), nat.ptr(shard.col_vals), nat.ptr(cs), nat.stream_ptr())
    nat.call("culsh_segment_sums", M, nat.ptr(shard.row_ptr), nat.ptr(shard.row_vals), nat.ptr(rs), nat.stream_ptr())
    buf = t.cat([cs[:N], (shard.col_ptr[1:] - shard.col_ptr[:-1]).to(t.float64),
                 rs[:M], (shard.row_ptr[1:] - shard.row_ptr[:-1]).to(t.float64)])
    _all_reduce_sum(buf, group)
    cs, cc, rs, rc = buf[:N], buf[N:2 * N], buf[2 * N:2 * N + M], buf[2 * N + M:]
    mu = float(cs.sum().item()) / max(float(cc.sum().item()), 1.0)
    bb = t.where(rc > 0, rs / rc.clamp(min=1) - mu, t.zeros_like(rs))
    bh = t.where(cc > 0, cs / cc.clamp(min=1) - mu, t.zeros_like(cs))
    return mu, bb, bh


# ------------------------------------------------------------ sharded LSH ---

class _Offset:
    """A device pointer shifted by a byte offset (the accumulators of a column shard are
    indexed by global column; the kernel only touches the shard's own rows)."""

    def __init__(self, base: int):
        self._p = base

    def data_ptr(self) -> int:
        return self._p


def simlsh_topk_sharded(dev, config, K: int, rank: int, D: int, group=None):
    """Column-sharded simLSH top-K: local hashing of column block `rank` (``dev`` needs
    only those columns' ratings), one all-gather of group keys, local top-K for the
    rank's columns, one all-gather of J^K.  Returns the full (N*K,) int32 entries tensor
    on every rank (bit-identical to simlsh_topk)."""
    from . import _native as nat
    from .lsh import _accumulate, _topk_device, assign_row_hashes
    c = config
    N = dev.N
    cb = np.array([(d * N) // D for d in range(D + 1)], np.int64)
    lo, hi = int(cb[rank]), int(cb[rank + 1])
    W = c.q * c.p * c.G
    hashes = assign_row_hashes(dev.M, c)
    acc = nat.empty((max((hi - lo) * W, 1),), "float64")
    keys = nat.zeros((c.q * max(N, 1),), "uint64")
    if hi > lo:
        _accumulate(dev, hashes.table(), c, _Offset(acc.data_ptr() - lo * W * 8), None, keys, lo, hi - lo)
    keys2 = keys.view(c.q, N)
    gathered = allgather_blocks(keys2.t().contiguous(), cb, rank, D, group)   # (N, q)
    all_keys = gathered.t().contiguous().view(-1)
    ent, ncand = _topk_device(all_keys, c.q, N, c.p * c.G, lo, hi - lo, K, c.seed)
    full = nat.zeros((max(N * K, 1),), "int32")
    if hi > lo:
        full[lo * K:hi * K] = ent[:(hi - lo) * K]
    full2 = allgather_blocks(full[:N * K].view(N, K), cb, rank, D, group)
    return full2.reshape(-1), ncand


class PeerRing:
    """The ring shift as device-side peer-memory traffic (csrc/ring.cu): after stage s each
    rank's push kernel writes the block it trained straight into the next rank's receive
    slot (CUDA IPC mapping: NVLink P2P stores between GPUs) and raises a system-scope ready
    flag there; the next rank's pull kernel waits for the flag on the device, copies the block
    into its parameter arrays and acknowledges in the sender's memory.  Stage kernel -> push ->
    pull -> next stage are stream-ordered on every rank; no NCCL call and no host
    synchronisation between stages.  Same blocks and order as ring_shift, so the result is the
    same bytes (exact mode == parallel_train(D))."""

    def __init__(self, plan: RingPlan, rank: int, tensors, group=None):
        import ctypes
        import torch.distributed as dist
        from . import _native as nat
        self.plan, self.rank, self.tensors = plan, rank, [t for t in tensors if t.numel()]
        span = max(plan.moving_span(b).stop - plan.moving_span(b).start for b in range(plan.D))
        self.offs, off = [], 0
        for t in self.tensors:
            self.offs.append(off)
            row_bytes = (t[0].numel() if t.dim() > 1 else 1) * t.element_size()
            off += (span * row_bytes + 15) // 16 * 16
        self.slot = max(off, 16)
        hb = nat.load_library().culsh_ring_handle_bytes()
        handle = ctypes.create_string_buffer(hb)
        buf = ctypes.c_void_p()
        nat.call("culsh_ring_alloc", self.slot, ctypes.byref(buf), handle)
        self.buf = buf
        handles = [None] * plan.D
        dist.all_gather_object(handles, bytes(handle.raw), group=group)
        self.peers = {}
        for q in {plan.send_peer(rank), plan.recv_peer(rank)}:
            pb = ctypes.c_void_p()
            nat.call("culsh_ring_open", ctypes.create_string_buffer(handles[q], hb), ctypes.byref(pb))
            self.peers[q] = pb
        self.status = nat.zeros((1,), "int32")
        self.seq = 0

    def _pieces(self, span):
        import ctypes
        n = len(self.tensors)
        views = [t[span] for t in self.tensors]
        ptrs = (ctypes.c_void_p * n)(*[v.data_ptr() for v in views])
        nbytes = (ctypes.c_int64 * n)(*[v.numel() * v.element_size() for v in views])
        offs = (ctypes.c_int64 * n)(*self.offs)
        return n, ptrs, nbytes, offs

    def shift(self, stage: int) -> None:
        """Enqueue the shift after `stage` (push of its block, pull of the next one)."""
        from . import _native as nat
        p, r = self.plan, self.rank
        self.seq += 1
        send = p.moving_span(p.moving_block(r, stage))
        recv = p.moving_span(p.moving_block(r, stage + 1))
        n, ptrs, nb, offs = self._pieces(send)
        nat.call("culsh_ring_push", n, ptrs, nb, offs, self.buf, self.peers[p.send_peer(r)], self.slot, self.seq,
                 nat.ptr(self.status), nat.stream_ptr())
        n, ptrs, nb, offs = self._pieces(recv)
        nat.call("culsh_ring_pull", n, ptrs, nb, offs, self.buf, self.peers[p.recv_peer(r)], self.slot, self.seq,
                 nat.ptr(self.status), nat.stream_ptr())

    def close(self) -> None:
        from . import _native as nat
        nat.torch().cuda.synchronize()
        for pb in self.peers.values():
            nat.call("culsh_ring_close", pb)
        nat.call("culsh_ring_free", self.buf)
        self.peers = {}


# ------------------------------------------------------------- the trainer ---

class DistTrainer:
    """One rank's DSGD state: its ratings shard, the parameter blocks it owns (full-size
    arrays indexed globally; only owned / currently held blocks are valid) and the
    per-(stage, sub-block) launch plans.

    mode="exact": fp64, the deterministic stage kernel (csrc/sgd_exact.cu) -- the ranks
    together reproduce parallel_train(D) bit for bit.  mode="hogwild": fp32 Hogwild stage
    launches (csrc/sgd_hogwild.cu), the performance mode."""

    def __init__(self, shard, plan: RingPlan, rank: int, neighbors, config, baselines, mode: str = "exact",
                 parts: int = 1, group=None, exchange: str = "collective"):
        from . import _native as nat
        from .factorization import DeviceModel64, _check_model_dims, pcg64_uniform_device
        from .hogwild import DeviceModel32, HogwildTrainer
        t = nat.torch()
        if mode not in ("exact", "hogwild"):
            raise ValueError(f"unknown mode {mode!r}")
        if exchange not in ("collective", "peer", "auto"):
            raise ValueError(f"unknown exchange {exchange!r}")
        if exchange == "auto" and parts != 1:
            exchange = "collective"
        self.plan, self.rank, self.mode, self.group = plan, rank, mode, group
        self.parts = parts if plan.D > 1 else 1
        self.exchange = exchange if plan.D > 1 else "collective"
        if self.exchange == "peer" and self.parts != 1:
            raise ValueError("the peer-memory ring shifts whole blocks (parts=1)")
        self.config = config
        M, N, F = shard.M, shard.N, config.F
        K = neighbors.K if neighbors is not None else 0
        _check_model_dims(F, K)
        self.M, self.N, self.F, self.K = M, N, F, K
        mu, bb, bh = baselines
        shard.mu, shard.base_b, shard.base_bhat = float(mu), bb, bh
        shard.struct = shard._make_struct()
        self.dev = shard
        dt = "float64" if mode == "exact" else "float32"
        tdt = getattr(t, dt)
        # own blocks at start: row block `rank`, column block `rank` (both sides)
        r0, r1 = plan.rows(rank).start, plan.rows(rank).stop
        c0, c1 = plan.cols(rank).start, plan.cols(rank).stop
        scale = config.effective_init_scale
        U = t.zeros(max(M * F, 1), dtype=tdt, device=nat.device())
        V = t.zeros(max(N * F, 1), dtype=tdt, device=nat.device())
        U[r0 * F:r1 * F] = pcg64_uniform_device(config.seed, r0 * F, (r1 - r0) * F, scale, dt)[:(r1 - r0) * F]
        V[c0 * F:c1 * F] = pcg64_uniform_device(config.seed, M * F + c0 * F, (c1 - c0) * F, scale, dt)[:(c1 - c0) * F]
        b = bb[:M].to(tdt).clone() if M else t.zeros(1, dtype=tdt, device=nat.device())
        bhat = bh[:N].to(tdt).clone() if N else t.zeros(1, dtype=tdt, device=nat.device())
        arrays = {"b": b, "b_hat": bhat, "U": U, "V": V,
                  "W": t.zeros(max(N * K, 1), dtype=tdt, device=nat.device()),
                  "C": t.zeros(max(N * K, 1), dtype=tdt, device=nat.device())}
        nbr = neighbors.device_entries() if K else None
        self.neighbors = neighbors
        self.mu = float(mu)
        if mode == "exact":
            self.model = DeviceModel64(arrays=arrays, mu=mu, M=M, N=N, F=F, K=K, nbr=nbr)
            self._build_exact()
        else:
            from .factorization import ModelParams
            m32 = DeviceModel32.from_arrays(arrays, mu, M, N, F, K, nbr)
            p = ModelParams._from_device(mu, m32, M, N, neighbors)
            self.hw = HogwildTrainer(None, neighbors, config, dev=shard, params=p, split=False)
            self.model = self.hw.model
            self._build_hogwild()
        self.ring = None
        if self.exchange in ("peer", "auto"):
            self.ring = self._peer_ring(strict=self.exchange == "peer")
            self.exchange = "peer" if self.ring is not None else "collective"

    def _peer_ring(self, strict: bool):
        """The peer-memory ring, or None when a rank cannot map its neighbours' buffers
        (strict: raise instead).  All ranks agree (one all-reduce of the failures)."""
        import torch.distributed as dist
        from . import _native as nat
        ring, err = None, None
        try:
            ring = PeerRing(self.plan, self.rank, self.moving_tensors(), self.group)
        except Exception as ex:   # e.g. no P2P between the GPUs: fall back to the collective path
            err = ex
        bad = nat.torch().tensor([0.0 if err is None else 1.0], dtype=nat.torch().float64)
        if dist.get_backend(self.group) == "nccl":
            bad = bad.cuda()
        dist.all_reduce(bad, group=self.group)
        if float(bad.item()):
            if ring is not None:
                ring.close()
            if strict:
                raise nat.NativeError(f"peer-memory ring unavailable: {err!r}")
            return None
        return ring

    # -- per-(stage, part) block ranges --------------------------------------
    def _block(self, s: int, h: int):
        """(row slice, column slice) of stage s, sub-block h."""
        rb, cb = self.plan.stage_block(self.rank, s)
        if self.plan.side == "rows":
            return self.plan.sub_rows(rb, h, self.parts), self.plan.cols(cb)
        return self.plan.rows(rb), self.plan.sub_cols(cb, h, self.parts)

    def _build_exact(self):
        from . import _native as nat
        from .factorization import _Scratch, _exact_lookups
        d = self.dev
        self.sc = _Scratch(self.M, self.N)
        self.plans = {}
        for s in range(self.plan.D):
            for h in range(self.parts):
                rs, cs = self._block(s, h)
                seg = nat.zeros((2 * max(self.N, 1),), "int64")
                chain = nat.zeros((max(self.N, 1),), "int32")
                nat.call("culsh_pass_plan", nat.ptr(d.col_ptr), nat.ptr(d.col_rows), self.N, 0, cs.start, cs.stop,
                         rs.start, rs.stop, None, None, 1, 0, nat.ptr(seg), nat.ptr(chain), nat.stream_ptr())
                self.plans[(s, h)] = (seg, chain, cs)
        self.pre = _exact_lookups(d, self.model, 0, self.N, 0.25)

    def _build_hogwild(self):
        from . import _native as nat
        t = nat.torch()
        d = self.dev
        self.works = {}
        cp = nat.to_host(d.col_ptr).astype(np.int64)
        for s in range(self.plan.D):
            for h in range(self.parts):
                rs, cs = self._block(s, h)
                if self.plan.side == "cols":     # the shard holds exactly the stage's rows
                    lo, hi = cp[:-1].copy(), cp[1:].copy()
                else:
                    bnd = nat.to_dev(np.array([rs.start, rs.stop], np.int64))
                    bp = nat.empty((max(self.N * 2, 1),), "int64")
                    nat.call("culsh_block_pointers", nat.ptr(d.col_ptr), nat.ptr(d.col_rows), self.N, nat.ptr(bnd),
                             2, nat.ptr(bp), nat.stream_ptr())
                    bph = nat.to_host(bp)[:self.N * 2].reshape(self.N, 2)
                    lo, hi = bph[:, 0], bph[:, 1]
                seg = np.zeros((self.N, 2), np.int64)
                seg[cs, 0], seg[cs, 1] = lo[cs], hi[cs]
                counts = hi[cs] - lo[cs]
                own = (np.argsort(-counts, kind="stable") + cs.start).astype(np.int32)
                self.works[(s, h)] = self.hw.block_work(nat.to_dev(seg.reshape(-1)), nat.to_dev(own, np.int32))

    def moving_tensors(self):
        m, M, N, F, K = self.model, self.M, self.N, self.F, self.K
        if self.plan.side == "rows":
            return [m.U[:M * F].view(M, F), m.b[:M]]
        return [m.V[:N * F].view(N, F), m.W[:N * K].view(N, K), m.C[:N * K].view(N, K), m.bhat[:N]]

    def epoch(self, ep: int) -> None:
        from . import _native as nat
        from .factorization import TrainingDivergedError, _colpass, _rates_struct
        if self.mode == "exact":
            rates = _rates_struct(self.config.rates_at(ep), self.config.regs)

            def fn(s, rb, cb, h):
                seg, chain, cs = self.plans[(s, h)]
                self.sc.seg, self.sc.chain = seg, chain
                _colpass(self.dev, self.model, self.sc, rates, cs.start, cs.stop, 1, pre=self.pre)
        else:
            def fn(s, rb, cb, h):
                self.hw.launch_work(ep, self.works[(s, h)])
        if self.ring is not None:
            for s_ in range(self.plan.D):
                rb, cb = self.plan.stage_block(self.rank, s_)
                fn(s_, rb, cb, 0)
                self.ring.shift(s_)
            if int(self.ring.status.item()):
                raise nat.NativeError("peer-memory ring shift timed out waiting for a neighbour")
        else:
            run_epoch(self.plan, self.rank, fn, self.moving_tensors(), self.group, self.parts)
        status = self.sc.status_value() if self.mode == "exact" else int(self.hw.status.item())
        bad = nat.torch().tensor([float(status & 1)], dtype=nat.torch().float64, device=nat.device())
        if self.plan.D > 1:
            _all_reduce_sum(bad, self.group)
        if float(bad.item()):
            raise TrainingDivergedError(epoch=ep)

    def gather(self) -> None:
        """Assemble the whole model on every rank (after whole epochs rank d holds row
        block d and column block d again)."""
        m, M, N, F, K = self.model, self.M, self.N, self.F, self.K
        D, r = self.plan.D, self.rank
        allgather_blocks(m.U[:M * F].view(M, F), self.plan.row_bounds, r, D, self.group)
        allgather_blocks(m.b[:M], self.plan.row_bounds, r, D, self.group)
        for x, w in ((m.V, F), (m.W, K), (m.C, K)):
            allgather_blocks(x[:N * w].view(N, w), self.plan.col_bounds, r, D, self.group)
        allgather_blocks(m.bhat[:N], self.plan.col_bounds, r, D, self.group)

    def params(self):
        from .factorization import ModelParams
        return ModelParams._from_device(self.mu, self.model, self.M, self.N, self.neighbors)


def parallel_train_distributed(ratings, neighbors, config, epoch_callback=None, mode: str = "exact",
                               side: str = "auto", parts: int = 1, group=None, exchange: str = "collective"):
    """parallel_train (parallel.py:166-227) across the ranks of a torch.distributed group,
    one GPU per rank, D = world size.  Called on every rank with the same arguments
    (SPMD); each rank uploads only its shard of ``ratings``.  mode="exact" returns the
    same bytes as parallel_train(ratings, neighbors, config, D); mode="hogwild" is the
    fp32 performance mode.  ``epoch_callback(t, params)`` runs on every rank with the
    whole (gathered, device-backed) model; edits it makes are kept.  Returns the whole
    model (device-backed ModelParams) on every rank.  exchange="collective": torch.distributed
    send/recv ring shift (NCCL; sub-block pipelining with parts > 1); exchange="peer": the
    block is pushed by this package's own kernels into the neighbour's memory (PeerRing,
    CUDA IPC / NVLink P2P, device-side flags, parts = 1)."""
    import torch.distributed as dist
    from . import _native as nat
    from dataclasses import replace
    config.validate()
    D = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    K = neighbors.K if neighbors is not None else 0
    if K != config.K:
        config = replace(config, K=K)
    if D < 1 or D > min(ratings.M, ratings.N):
        raise ValueError(f"D={D} out of range for a {ratings.M}x{ratings.N} matrix")
    if side == "auto":
        side = choose_side(ratings.M, ratings.N, config.F, K)
    plan = RingPlan(D, ratings.M, ratings.N, side)
    if side == "cols":
        shard = shard_device_ratings(ratings, plan, rank, "rows")
    else:   # whole rows are read by the lookups: the ratings are replicated
        from .data import DeviceRatings
        shard = DeviceRatings(ratings, with_baselines=False)
    st = ratings.baselines()     # the reference's host statistics (any values)
    base = (st.mu, nat.to_dev(st.b, np.float64), nat.to_dev(st.b_hat, np.float64))
    tr = DistTrainer(shard, plan, rank, neighbors, config, base, mode=mode, parts=parts, group=group,
                     exchange=exchange)
    try:
        for ep in range(config.epochs):
            tr.epoch(ep)
            if epoch_callback is not None:
                tr.gather()
                p = tr.params()
                epoch_callback(ep, p)
                p._device(0)      # edits made by the callback (identical on every rank)
    finally:
        if tr.ring is not None:
            tr.ring.close()
    tr.gather()
    return tr.params()


# --------------------------------------------------------------- the bench ---

def _max_over_ranks(x: float) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def bench_main(args, metric, workload, rates):
    """Multi-GPU DSGD benchmark (launched by torchrun, one rank per GPU).  Every rank
    generates only its own shards of the synthetic matrix (its column block for the
    simLSH build, its row block for SGD), builds its part of J^K (sharded simLSH),
    initialises its own parameter blocks, and runs Hogwild DSGD epochs with the column
    side rotating (1.7 MB per stage per GPU at C3, D = 8)."""
    import json
    import torch
    import torch.distributed as dist
    from . import _native as nat
    from . import synth, lsh
    from .factorization import TrainConfig
    from .similarity import NeighborTable

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # CULSH_DIST_BACKEND=gloo + CULSH_SHARE_GPU=1 lets a 1-GPU box run the N-rank
    # orchestration end to end (ranks time-share cuda:0, exchanges staged via host)
    backend = os.environ.get("CULSH_DIST_BACKEND", "nccl")
    if os.environ.get("CULSH_SHARE_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    D = world
    M, N, nnz_t, F, K, e = synth.SHAPES[args.config]
    side = os.environ.get("CULSH_DSGD_SIDE", choose_side(M, N, F, K))
    plan = RingPlan(D, M, N, side)
    # ---- simLSH on the column shard
    cs = plan.cols(rank)
    r_, c_, v_, _ = synth.hashed_shard(M, N, nnz_t, seed=0, cols=(cs.start, cs.stop))
    col_shard = synth.device_ratings_from_sorted(M, N, r_, c_, v_, baselines=False)
    del r_, c_, v_
    lcfg = lsh.LshConfig(G=8, p=3, q=100, psi_exponent=e, seed=0)
    simlsh_topk_sharded(col_shard, lcfg, K, rank, D)          # warm
    dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    ent, _ = simlsh_topk_sharded(col_shard, lcfg, K, rank, D)
    ev1.record()
    torch.cuda.synchronize()
    lsh_s = _max_over_ranks(ev0.elapsed_time(ev1) / 1e3)
    nbr = NeighborTable(N, K, nat.to_host(ent)[:N * K].reshape(N, K).astype(np.int32))
    # ---- SGD shard (row block for side cols; the column shard itself for side rows)
    if side == "cols":
        del col_shard
        rs = plan.rows(rank)
        r_, c_, v_, _ = synth.hashed_shard(M, N, nnz_t, seed=0, rows=(rs.start, rs.stop))
        shard = synth.device_ratings_from_sorted(M, N, r_, c_, v_, baselines=False)
        del r_, c_, v_
        base = global_baselines(shard)
    else:   # side rows: the lookups read whole rows -> every rank holds the whole matrix
        del col_shard
        shard = synth.random_sparse_device(M, N, nnz_t, seed=0).dev
        base = (shard.mu, shard.base_b, shard.base_bhat)
    local_nnz = torch.tensor([float(shard.nnz)], dtype=torch.float64, device="cuda")
    _all_reduce_sum(local_nnz)
    nnz = int(local_nnz.item()) if side == "cols" else shard.nnz
    cfg = TrainConfig(F=F, K=K, epochs=args.warmup + args.steps, seed=0, **rates)
    parts = int(os.environ.get("CULSH_DSGD_PARTS", "2")) if D > 1 else 1
    # own push/pull kernels over peer memory unless a rank cannot map its neighbours
    exchange = os.environ.get("CULSH_DSGD_EXCHANGE", "auto")
    if exchange in ("peer", "auto"):
        parts = 1
    tr = DistTrainer(shard, plan, rank, nbr, cfg, base, mode="hogwild", parts=parts, exchange=exchange)
    hw = tr.hw

    for w in range(args.warmup):
        tr.epoch(w)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    from bench import Clocks   # noqa: E402  (repo root is on sys.path under bench.py)
    clk = Clocks(f"/tmp/culsh_clocks_rank{rank}.csv")
    with clk:
        t0.record()
        for s in range(args.steps):
            tr.epoch(args.warmup + s)
        t1.record()
        torch.cuda.synchronize()
    dist.barrier()
    total = _max_over_ranks(t0.elapsed_time(t1) / 1e3)
    ups = nnz * args.steps / total
    b_upd = hw.bytes_per_update()

    # e2e: every step each rank copies ITS shard's rating stream (packed records, masks,
    # residuals) from pinned host memory, runs the epoch, reads the loss back
    if hw.packed is not None:
        pk = hw.packed
        dev_views = {"words": pk["words"][:shard.nnz], "cmask": pk["cmask"], "resid": hw.resid}
    else:
        dev_views = {"rows": shard.col_rows, "vals": hw.vals32, "mask": hw.mask, "resid": hw.resid}
    host = {k: v.cpu().pin_memory() for k, v in dev_views.items()}
    e_steps = max(1, min(args.steps, 3))
    torch.cuda.synchronize()
    dist.barrier()
    w0 = time.perf_counter()
    for s in range(e_steps):
        for k, v in dev_views.items():
            v.copy_(host[k], non_blocking=True)
        hw.loss.zero_()
        tr.epoch(args.warmup + args.steps + s)
        float(hw.loss.item())
    torch.cuda.synchronize()
    e_dt = _max_over_ranks(time.perf_counter() - w0)
    h2d = torch.tensor([float(sum(int(v.numel() * v.element_size()) for v in host.values()))],
                       dtype=torch.float64, device="cuda")
    _all_reduce_sum(h2d)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pk_path = os.path.join(root, "MEASURED_PEAKS.json")
    peak = float(json.load(open(pk_path))["hbm_gbs"]) if os.path.exists(pk_path) else 6650.0
    ach = b_upd * nnz / D / (total / args.steps) / 1e9
    moving = ((N // D) * (F + 2 * K + 1) * 4) if side == "cols" else ((M // D) * (F + 1) * 4)
    if rank == 0:
        line = {"metric": metric, "value": ups, "unit": "updates/s", "n_gpus": D, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp32",
                "data": "synthetic (random_sparse distribution, each rank generates its own shards in HBM)",
                "config": workload,
                "impl_config": {"nnz_generated": nnz, "parallelism": f"dsgd{D}",
                           "ring_parts": parts, "rotating_side": side,
                           "moving_bytes_per_stage_per_gpu": moving,
                           "exchange": (f"peer-memory push/pull kernels (csrc/ring.cu): the {side} block written "
                                        "into the neighbour's memory over IPC/NVLink, device-side flags"
                                        if tr.exchange == "peer" else
                                        f"NCCL send/recv ring shift of the {side} parameter sub-blocks, each "
                                        "overlapping the next sub-block's kernel" if backend == "nccl" else
                                        f"{backend} ring shift of the {side} parameter sub-blocks (host-staged)"),
                           "l2": "inputs larger than L2, no flush"},
                "lsh_build_s": lsh_s,
                "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                             "frac": ach / peak, "traffic": None,
                             "note": "per GPU: B_upd x nnz/D per epoch / epoch time (incl. ring shifts)"},
                "gpu_launches": args.steps * D * parts,
                "e2e": {"value": nnz * e_steps / e_dt, "unit": "updates/s",
                        "h2d_bytes_per_step": int(h2d.item()), "d2h_bytes_per_step": 8 * D,
                        "api": "per-rank pinned shard stream -> DSGD epoch -> loss"},
                "clocks": clk.summary(local)}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0
