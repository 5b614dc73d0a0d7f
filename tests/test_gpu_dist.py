"""GPU: the multi-GPU DSGD product path (dsgd.py) with 2 and 3 ranks time-sharing one
GPU over gloo (the only multi-rank setup a 1-GPU box offers; the orchestration is the
same one NCCL drives on 8 GPUs).  Exact mode must equal the single-process
parallel_train(D) bit for bit for both rotation sides, and the column-sharded simLSH must
equal simlsh_topk."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(P, seed=0, M=300, N=90, dens=0.2, integer=True):
    rng = np.random.default_rng(seed)
    rows, cols = np.nonzero(rng.random((M, N)) < dens)
    vals = (rng.integers(1, 6, len(rows)).astype(np.float64) if integer
            else np.round(rng.random(len(rows)) * 5, 3))
    return P.SparseRatings(M, N, rows, cols, vals)


def _worker(rank, world, port, job, out_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2111_11682_b200 as P
        from paper_2111_11682_b200 import _native as nat
        from paper_2111_11682_b200.dsgd import parallel_train_distributed, simlsh_topk_sharded, RingPlan, \
            shard_device_ratings
        kind = job["kind"]
        r = _case(P, **job.get("data", {}))
        if kind == "lsh":
            lc = P.LshConfig(**job["lsh"])
            plan = RingPlan(world, r.M, r.N)
            shard = shard_device_ratings(r, plan, rank, "cols")
            ent, _ = simlsh_topk_sharded(shard, lc, job["K"], rank, world)
            out = {"entries": nat.to_host(ent)[:r.N * job["K"]].tobytes()}
        else:
            tbl, _ = P.simlsh_topk(r, P.LshConfig(G=4, p=2, q=8, seed=3), job["K"])
            cfg = P.TrainConfig(F=job["F"], K=job["K"], epochs=job["epochs"], seed=1)
            seen = []
            p = parallel_train_distributed(r, tbl, cfg, mode=kind, side=job["side"], parts=job["parts"],
                                           epoch_callback=lambda t, q: seen.append(P.rmse(q, r.triplets(), r)),
                                           exchange=job.get("exchange", "collective"))
            out = {n: getattr(p, n).tobytes() for n in ("b", "b_hat", "U", "V", "W", "C")}
            out["curve"] = seen
        if rank == 0:
            out_q.put(out)
    finally:
        dist.barrier()
        dist.destroy_process_group()


def _run(world, job):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, job, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2111_11682_b200 as p
    return p


@pytest.mark.parametrize("world,side,parts,integer", [(2, "cols", 1, True), (2, "rows", 1, True),
                                                      (3, "cols", 2, True), (3, "rows", 2, False),
                                                      (2, "cols", 3, False)])
def test_distributed_exact_equals_parallel_train(P, world, side, parts, integer):
    job = {"kind": "exact", "side": side, "parts": parts, "F": 12, "K": 5, "epochs": 3,
           "data": {"seed": world + parts, "integer": integer}}
    res = _run(world, job)
    r = _case(P, seed=world + parts, integer=integer)
    tbl, _ = P.simlsh_topk(r, P.LshConfig(G=4, p=2, q=8, seed=3), 5)
    seen = []
    ref = P.parallel_train(r, tbl, P.TrainConfig(F=12, K=5, epochs=3, seed=1), world,
                           epoch_callback=lambda t, q: seen.append(P.rmse(q, r.triplets(), r)))
    for n in ("b", "b_hat", "U", "V", "W", "C"):
        assert res[n] == getattr(ref, n).tobytes(), (side, parts, n)
    assert res["curve"] == seen


@pytest.mark.parametrize("world,side,integer", [(2, "cols", True), (3, "cols", False), (3, "rows", True)])
def test_peer_ring_exact_equals_parallel_train(P, world, side, integer):
    """exchange="peer": the ring shift done by csrc/ring.cu's push / pull kernels over CUDA
    IPC-mapped neighbour memory with device-side flags (ranks share one GPU here; NVLink P2P
    between GPUs) -- the same bytes as parallel_train(D)."""
    job = {"kind": "exact", "side": side, "parts": 1, "F": 12, "K": 5, "epochs": 3, "exchange": "peer",
           "data": {"seed": world + 7, "integer": integer}}
    res = _run(world, job)
    r = _case(P, seed=world + 7, integer=integer)
    tbl, _ = P.simlsh_topk(r, P.LshConfig(G=4, p=2, q=8, seed=3), 5)
    seen = []
    ref = P.parallel_train(r, tbl, P.TrainConfig(F=12, K=5, epochs=3, seed=1), world,
                           epoch_callback=lambda t, q: seen.append(P.rmse(q, r.triplets(), r)))
    for n in ("b", "b_hat", "U", "V", "W", "C"):
        assert res[n] == getattr(ref, n).tobytes(), (side, n)
    assert res["curve"] == seen


def test_distributed_hogwild_trains(P):
    res = _run(2, {"kind": "hogwild", "side": "cols", "parts": 2, "F": 32, "K": 5, "epochs": 4,
                   "data": {"seed": 9, "M": 2000, "N": 300, "dens": 0.1}})
    curve = res["curve"]
    assert np.isfinite(curve).all() and curve[-1] < curve[0]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_simlsh_equals_simlsh_topk(P, world):
    lsh = {"G": 8, "p": 3, "q": 12, "psi_exponent": 2, "seed": 5}
    res = _run(world, {"kind": "lsh", "lsh": lsh, "K": 7, "data": {"seed": 4, "M": 500, "N": 130}})
    r = _case(P, seed=4, M=500, N=130)
    tbl, _ = P.simlsh_topk(r, P.LshConfig(**lsh), 7)
    assert res["entries"] == tbl.entries.tobytes()
