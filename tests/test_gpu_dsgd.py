"""Multi-rank DSGD on the GPU: D processes share cuda:0 (this build has one GPU),
exchange the (u, b) row blocks with dsgd.ring_shift over gloo (host-staged), and
run the exact stage kernel on their own column block.  The result must equal the
reference's parallel_train(D) bit for bit (golden fixtures).  On a multi-GPU box
the same code runs one rank per GPU over NCCL (bench.py / dsgd.bench_main)."""

import os
import socket

import numpy as np
import pytest

from conftest import ROOT, load_golden

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import ctypes
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2111_11682_b200 as P
    from paper_2111_11682_b200 import _native as nat
    from paper_2111_11682_b200.dsgd import RingPlan, allgather_blocks, run_epoch
    from paper_2111_11682_b200.factorization import (DeviceModel64, _Scratch, _colpass,
                                                     _rates_struct, init_params)
    z = load_golden("sgd_small.npz")
    pre = f"s{case}_"
    F, K, epochs, seed = (int(x) for x in z[pre + "cfg"])
    r = P.SparseRatings(int(z[pre + "M"]), int(z[pre + "N"]), z[pre + "rows"], z[pre + "cols"],
                        z[pre + "vals"])
    nbr = P.NeighborTable(r.N, K, z[pre + "nbr"]) if K else None
    cfg = P.TrainConfig(F=F, K=K, epochs=epochs, seed=seed)
    params = init_params(r.M, r.N, F, K, nbr, r.baselines(), cfg)
    dev = r.device()
    dm = DeviceModel64(params)
    sc = _Scratch(r.M, r.N)
    plan = RingPlan(world, r.M, r.N)
    part = P.make_partition(r, world)
    segs = []
    for s in range(world):
        seg = nat.zeros((2 * r.N,), "int64")
        chain = nat.zeros((r.N,), "int32")
        nat.call("culsh_pass_plan", nat.ptr(dev.col_ptr), nat.ptr(dev.col_rows), r.N, 1, 0, r.N, 0,
                 r.M, nat.ptr(part._dev_block_ptr), nat.ptr(part._dev_col_bounds), world, s,
                 nat.ptr(seg), nat.ptr(chain), nat.stream_ptr())
        segs.append((seg, chain))
    cs = plan.cols(rank)
    U, b = dm.U.view(r.M, F), dm.b
    for t in range(epochs):
        rates = _rates_struct(cfg.rates_at(t), cfg.regs)

        def stage(s, rb):
            sc.seg, sc.chain = segs[s]
            _colpass(dev, dm, sc, rates, cs.start, cs.stop, 1)
            assert sc.status_value() == 0
        run_epoch(plan, rank, stage, [U, b])
    torch.cuda.synchronize()
    allgather_blocks(U, plan.row_bounds, rank, world)
    allgather_blocks(b, plan.row_bounds, rank, world)
    for name, F_ in (("V", F), ("W", K), ("C", K)):
        t = getattr(dm, name)
        if F_:
            allgather_blocks(t.view(r.N, F_), plan.col_bounds, rank, world)
    allgather_blocks(dm.bhat, plan.col_bounds, rank, world)
    dm.download(params)
    if rank == 0:
        q.put({n: getattr(params, n).tobytes() for n in ("b", "b_hat", "U", "V", "W", "C")})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(2, 0), (3, 1)])
def test_multirank_exact_dsgd_equals_reference(world, case):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    z = load_golden("sgd_small.npz")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for n in ("b", "b_hat", "U", "V", "W", "C"):
        assert res[n] == z[f"s{case}_D{world}_{n}"].tobytes(), (world, case, n)
