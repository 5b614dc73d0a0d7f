"""Multi-GPU DSGD and sharded simLSH over torch.distributed.

One process per GPU.  With D ranks the matrix is cut into D row blocks and D
column blocks exactly as the reference's make_partition (parallel.py:99-107):

  * rank d owns column block d for the whole run: its ratings R[:, d], and the
    column parameters v_j, w_j, c_j, b_hat_j of those columns;
  * at stage s rank d trains row block (d + s) % D (parallel.py:36-41), so no
    two ranks ever touch the same row or column parameter;
  * after every stage the row-block parameters (u_i, b_i) rotate one step
    around the ring: rank d sends its block to rank d-1 and receives block
    (d + s + 1) % D from rank d+1 (one NCCL send/recv pair over NVLink; the
    paper's "U-block transfer directly in the GPUs").

With the exact stage kernel this reproduces parallel_train(D) bit for bit;
with the Hogwild stage kernel it is the multi-GPU performance mode.

simLSH is sharded by columns: row hashes are a pure function of (seed, g, m,
i), so each rank hashes its own columns with no exchange, then ONE all-gather
of the (q, N) group keys gives every rank the buckets, each rank selects top-K
for its own columns, and one all-gather assembles J^K.

The orchestration below is device-agnostic (CPU tensors + gloo in the tests,
CUDA tensors + NCCL in production); the stage computation is a callback.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass

import numpy as np


@dataclass
class RingPlan:
    """Static DSGD plan for D ranks over an M x N matrix."""

    D: int
    M: int
    N: int

    def __post_init__(self):
        self.row_bounds = np.array([(d * self.M) // self.D for d in range(self.D + 1)], np.int64)
        self.col_bounds = np.array([(d * self.N) // self.D for d in range(self.D + 1)], np.int64)

    def row_block(self, rank: int, stage: int) -> int:
        return (rank + stage) % self.D

    def send_peer(self, rank: int) -> int:
        return (rank - 1) % self.D

    def recv_peer(self, rank: int) -> int:
        return (rank + 1) % self.D

    def rows(self, rb: int) -> slice:
        return slice(int(self.row_bounds[rb]), int(self.row_bounds[rb + 1]))

    def cols(self, cb: int) -> slice:
        return slice(int(self.col_bounds[cb]), int(self.col_bounds[cb + 1]))

    def sub_rows(self, rb: int, part: int, parts: int) -> slice:
        """Part `part` of row block rb cut into `parts`: block rb*parts + part of the
        D*parts-way partition (whose bounds contain the D-way bounds: (k*M)//D ==
        (k*parts*M)//(D*parts))."""
        k, n = rb * parts + part, self.D * parts
        return slice((k * self.M) // n, ((k + 1) * self.M) // n)


def _host_staging() -> bool:
    """Gloo has no CUDA send/recv: stage device tensors through host memory."""
    import torch.distributed as dist
    return dist.get_backend() == "gloo"


def ring_shift(plan: RingPlan, rank: int, stage: int, tensors, group=None) -> None:
    """After stage `stage`: send the row block just trained to rank-1 and receive the
    next stage's row block from rank+1, in place, for every (M, ...) tensor given."""
    import torch.distributed as dist
    if plan.D == 1:
        return
    send_rb = plan.row_block(rank, stage)
    recv_rb = plan.row_block(rank, stage + 1)
    dst, src = plan.send_peer(rank), plan.recv_peer(rank)
    stage_host = _host_staging()
    ops = []
    for t in tensors:
        out = t[plan.rows(send_rb)].contiguous()
        if stage_host and out.is_cuda:
            out = out.cpu()
        ops.append(dist.P2POp(dist.isend, out, dst, group))
    recv_bufs = []
    for t in tensors:
        buf = t[plan.rows(recv_rb)]
        if stage_host and buf.is_cuda:
            buf = buf.cpu()
        elif not buf.is_contiguous():
            buf = buf.contiguous()
        recv_bufs.append(buf)
        ops.append(dist.P2POp(dist.irecv, buf, src, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    for t, buf in zip(tensors, recv_bufs):
        view = t[plan.rows(recv_rb)]
        if view.data_ptr() != buf.data_ptr():
            view.copy_(buf)


def _shift_part(plan: RingPlan, rank: int, stage: int, part: int, parts: int, tensors, group=None):
    """Start the ring shift of one row sub-block: send part `part` of the block trained at
    `stage` to rank-1, receive the same part of the next stage's block from rank+1.
    Returns a finisher.  With NCCL the requests run on NCCL's stream, which waits only for
    the work enqueued before this call (the sub-block's stage kernel), so the transfer
    overlaps the next sub-block's kernel; finishing makes the current stream wait for it."""
    import torch.distributed as dist
    send_rows = plan.sub_rows(plan.row_block(rank, stage), part, parts)
    recv_rows = plan.sub_rows(plan.row_block(rank, stage + 1), part, parts)
    dst, src = plan.send_peer(rank), plan.recv_peer(rank)
    stage_host = _host_staging()
    ops, recv_bufs = [], []
    for t in tensors:
        out = t[send_rows].contiguous()
        if stage_host and out.is_cuda:
            out = out.cpu()
        ops.append(dist.P2POp(dist.isend, out, dst, group))
    for t in tensors:
        buf = t[recv_rows]
        if stage_host and buf.is_cuda:
            buf = buf.cpu()
        elif not buf.is_contiguous():
            buf = buf.contiguous()
        recv_bufs.append(buf)
        ops.append(dist.P2POp(dist.irecv, buf, src, group))
    reqs = dist.batch_isend_irecv(ops)

    def finish():
        for req in reqs:
            req.wait()
        for t, buf in zip(tensors, recv_bufs):
            view = t[recv_rows]
            if view.data_ptr() != buf.data_ptr():
                view.copy_(buf)
    return finish


def run_epoch(plan: RingPlan, rank: int, stage_fn, row_tensors, group=None, parts: int = 1) -> None:
    """One DSGD epoch: D stages, each followed by the ring shift.

    parts > 1 pipelines the shift: each stage runs as `parts` row sub-blocks
    (stage_fn(s, rb, part)), and a sub-block is sent as soon as its kernel is enqueued,
    while the next sub-block trains; a stage's sub-block waits only for its own part to
    arrive.  Each column still sees its entries of the block in row order and each row
    its columns in ascending order, so with the exact stage kernel the result is the
    same as parts = 1 (and parallel_train) bit for bit."""
    if parts == 1:
        for s in range(plan.D):
            stage_fn(s, plan.row_block(rank, s))
            ring_shift(plan, rank, s, row_tensors, group)
        return
    pending = {}
    for s in range(plan.D):
        rb = plan.row_block(rank, s)
        for h in range(parts):
            if h in pending:
                pending.pop(h)()
            stage_fn(s, rb, h)
            if plan.D > 1:
                pending[h] = _shift_part(plan, rank, s, h, parts, row_tensors, group)
    for h in sorted(pending):
        pending.pop(h)()


def allgather_blocks(t, bounds: np.ndarray, rank: int, D: int, group=None):
    """Every rank contributes rows [bounds[rank], bounds[rank+1]) of the full-size
    tensor t; on return t holds all blocks on every rank."""
    import torch
    import torch.distributed as dist
    if D == 1:
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


# ------------------------------------------------------------ sharded LSH ---

def simlsh_topk_sharded(dev, config, K: int, rank: int, D: int, group=None):
    """Column-sharded simLSH top-K: local hashing, one all-gather of group keys,
    local top-K for the rank's columns, one all-gather of J^K.  Returns the full
    (N*K,) int32 entries tensor on every rank (bit-identical to simlsh_topk)."""
    import torch
    import torch.distributed as dist
    from . import _native as nat
    from .lsh import _accumulate, _ns, _topk_device, assign_row_hashes
    c = config
    N = dev.N
    cb = np.array([(d * N) // D for d in range(D + 1)], np.int64)
    lo, hi = int(cb[rank]), int(cb[rank + 1])
    W = c.q * c.p * c.G
    hashes = assign_row_hashes(dev.M, c)
    acc = nat.empty((max((hi - lo) * W, 1),), "float64")
    keys = nat.zeros((c.q * max(N, 1),), "uint64")
    if hi > lo:
        # acc rows are indexed by global column: offset the base pointer
        base = acc.data_ptr() - lo * W * 8

        class _Shift:
            def data_ptr(self):
                return base
        _accumulate(dev, hashes.table(), c, _Shift(), None, keys, lo, hi - lo)
    keys2 = keys.view(c.q, N)
    gathered = allgather_blocks(keys2.t().contiguous(), cb, rank, D, group)   # (N, q)
    all_keys = gathered.t().contiguous().view(-1)
    ent, ncand = _topk_device(all_keys, c.q, N, c.p * c.G, lo, hi - lo, K, c.seed)
    full = nat.zeros((max(N * K, 1),), "int32")
    if hi > lo:
        full[lo * K:hi * K] = ent[:(hi - lo) * K]
    full2 = allgather_blocks(full[:N * K].view(N, K), cb, rank, D, group)
    return full2.reshape(-1), ncand


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
    """Multi-GPU DSGD benchmark (launched by torchrun, one rank per GPU)."""
    import json
    import torch
    import torch.distributed as dist
    from . import _native as nat
    from . import synth, lsh
    from .data import BaselineStats
    from .factorization import TrainConfig, init_params
    from .hogwild import HogwildTrainer
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
    dm = synth.random_sparse_device(M, N, nnz_t, seed=0)   # same seed: identical matrix on every rank
    nnz = dm.nnz
    lcfg = lsh.LshConfig(G=8, p=3, q=100, psi_exponent=e, seed=0)
    simlsh_topk_sharded(dm.dev, lcfg, K, rank, D)          # warm
    dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    ent, _ = simlsh_topk_sharded(dm.dev, lcfg, K, rank, D)
    ev1.record()
    torch.cuda.synchronize()
    lsh_s = _max_over_ranks(ev0.elapsed_time(ev1) / 1e3)
    nbr = NeighborTable(N, K, nat.to_host(ent)[:N * K].reshape(N, K).astype(np.int32))

    cfg = TrainConfig(F=F, K=K, epochs=args.warmup + args.steps, seed=0, **rates)
    tr = HogwildTrainer(None, nbr, cfg, dev=dm.dev)
    plan = RingPlan(D, M, N)
    d = dm.dev
    # per-(stage, row sub-block) work lists of the own column block: entry ranges from the
    # block pointers of the D*parts-way row partition, split when the block has fewer
    # columns than the GPU has resident warps (HogwildTrainer.block_work); the ring shift
    # of each sub-block overlaps the next sub-block's kernel (run_epoch parts)
    parts = int(os.environ.get("CULSH_DSGD_PARTS", "2")) if D > 1 else 1
    nb = D * parts + 1
    fine = np.array([(k * M) // (D * parts) for k in range(nb)], np.int64)
    bp = nat.empty((N * nb,), "int64")
    nat.call("culsh_block_pointers", nat.ptr(d.col_ptr), nat.ptr(d.col_rows), N, nat.ptr(nat.to_dev(fine)), nb,
             nat.ptr(bp), nat.stream_ptr())
    bp_h = nat.to_host(bp).reshape(N, nb)
    cs = plan.cols(rank)
    counts = (d.col_ptr[1:] - d.col_ptr[:-1])[cs]
    own = (torch.argsort(counts, descending=True, stable=True) + cs.start).to(torch.int32)
    U = tr.model.U.view(M, F)
    b = tr.model.b
    works = {}
    for s in range(D):
        rb = plan.row_block(rank, s)
        for h in range(parts):
            k = rb * parts + h
            seg = np.zeros((N, 2), np.int64)
            seg[cs, 0], seg[cs, 1] = bp_h[cs, k], bp_h[cs, k + 1]
            works[(s, h)] = tr.block_work(nat.to_dev(seg.reshape(-1)), own)

    def stage(ep):
        def fn(s, rb, h=0):
            tr.launch_work(ep, works[(s, h)])
        return fn

    def epoch(ep):
        run_epoch(plan, rank, stage(ep), [U, b], parts=parts)

    for w in range(args.warmup):
        epoch(w)
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
            epoch(args.warmup + s)
        t1.record()
        torch.cuda.synchronize()
    dist.barrier()
    total = _max_over_ranks(t0.elapsed_time(t1) / 1e3)
    ups = nnz * args.steps / total
    b_upd = tr.bytes_per_update()

    # e2e: every step each rank copies ITS column block's rating stream (rows,
    # values, masks) from pinned host memory, runs the epoch, reads the loss back
    lo_e, hi_e = int(d.col_ptr[cs.start].item()), int(d.col_ptr[cs.stop].item())
    r_lo, r_hi = int(tr.resid_ptr[cs.start].item()), int(tr.resid_ptr[cs.stop].item())
    if tr.packed is not None:   # the arrays the stage kernels read: packed records, masks, residuals
        pk = tr.packed
        m_lo, m_hi = int(pk["mptr"][cs.start].item()) * tr.MW, int(pk["mptr"][cs.stop].item()) * tr.MW
        dev_views = {"words": pk["words"][lo_e:hi_e], "cmask": pk["cmask"][m_lo:m_hi],
                     "resid": tr.resid[r_lo:r_hi]}
    else:
        dev_views = {"rows": d.col_rows[lo_e:hi_e], "vals": tr.vals32[lo_e:hi_e],
                     "mask": tr.mask[lo_e * tr.MW:hi_e * tr.MW], "resid": tr.resid[r_lo:r_hi]}
    host = {k: v.cpu().pin_memory() for k, v in dev_views.items()}
    e_steps = max(1, min(args.steps, 3))
    torch.cuda.synchronize()
    dist.barrier()
    w0 = time.perf_counter()
    for s in range(e_steps):
        for k, v in dev_views.items():
            v.copy_(host[k], non_blocking=True)
        tr.loss.zero_()
        epoch(args.warmup + args.steps + s)
        float(tr.loss.item())
    torch.cuda.synchronize()
    e_dt = _max_over_ranks(time.perf_counter() - w0)
    h2d = sum(int(v.numel() * v.element_size()) for v in host.values())
    peak = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]) if os.path.exists(os.path.join(
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6650.0
    ach = b_upd * nnz / D / (total / args.steps) / 1e9
    if rank == 0:
        line = {"metric": metric, "value": ups, "unit": "updates/s", "n_gpus": D, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp32",
                "data": "synthetic (random_sparse distribution generated in HBM)",
                "config": {"workload": workload[args.config], "parallelism": f"dsgd{D}", "ring_parts": parts,
                           "exchange": ("NCCL send/recv ring shift of u/b row sub-blocks, each overlapping the next "
                                        "sub-block's kernel" if backend == "nccl" else
                                        f"{backend} ring shift of u/b row sub-blocks (host-staged)"),
                           "l2": "inputs larger than L2, no flush"},
                "lsh_build_s": lsh_s,
                "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                             "frac": ach / peak, "traffic": None,
                             "note": "per GPU: B_upd x nnz/D per epoch / epoch time (incl. ring shifts)"},
                "gpu_launches": args.steps * D,
                "e2e": {"value": nnz * e_steps / e_dt, "unit": "updates/s",
                        "h2d_bytes_per_step": h2d * D, "d2h_bytes_per_step": 8 * D,
                        "api": "per-rank pinned column-block stream -> DSGD epoch -> loss"},
                "clocks": clk.summary(local)}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0
