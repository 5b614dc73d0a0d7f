"""Multi-rank DSGD orchestration (dsgd.py) on CPU: world_size 2 and 3 over gloo.
The per-stage compute is the oracle's _stage_pass restatement, so the test
isolates the ring schedule, the U/b ring shift and the final block gather:
the result must equal the reference's parallel_train(D) bit for bit (golden)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, load_golden

REGS = (0.02, 0.02, 0.02, 0.02, 0.002, 0.002)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, out_q, parts=1, side="rows"):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    from paper_2111_11682_b200.dsgd import RingPlan, allgather_blocks, run_epoch
    z = load_golden("sgd_small.npz")
    pre = f"s{case}_"
    F, K, epochs, seed = (int(x) for x in z[pre + "cfg"])
    d, mu = orc.build_csr(int(z[pre + "M"]), int(z[pre + "N"]), z[pre + "rows"], z[pre + "cols"],
                          z[pre + "vals"])
    m = orc.init_model(d.M, d.N, F, K, z[pre + "nbr"], mu, d.base_b, d.base_bhat, seed)
    plan = RingPlan(world, d.M, d.N, side)
    _, col_bounds, bp = orc.partition(d, world)
    assert np.array_equal(col_bounds, plan.col_bounds)
    bp_fine = orc.partition(d, world * parts)[2]   # row sub-blocks of the pipelined shift
    U, b = torch.from_numpy(m.U), torch.from_numpy(m.b)
    moving = [U, b] if side == "rows" else [torch.from_numpy(x) for x in (m.V, m.W, m.C, m.bhat)]
    for t in range(epochs):
        rates = orc.make_rates(tuple(a / (1.0 + 0.3 * t ** 1.5)
                                     for a in (0.035, 0.035, 0.035, 0.035, 0.002, 0.002)), REGS)

        def stage(s, rb, cb, h):
            if side == "rows":
                cs = plan.cols(cb)
                assert orc.stage_pass(d, m, rates, cs.start, cs.stop, rb * parts + h, bp_fine) == 0
            else:
                cs = plan.sub_cols(cb, h, parts)
                assert orc.stage_pass(d, m, rates, cs.start, cs.stop, rb, bp) == 0
        run_epoch(plan, rank, stage, moving, parts=parts)
    # after D stages per epoch every rank holds row block `rank` again
    allgather_blocks(U, plan.row_bounds, rank, world)
    allgather_blocks(b, plan.row_bounds, rank, world)
    for arr in (m.V, m.W, m.C, m.bhat):
        allgather_blocks(torch.from_numpy(arr), plan.col_bounds, rank, world)
    if rank == 0:
        out_q.put({n: getattr(m, n).tobytes() for n in ("b", "bhat", "U", "V", "W", "C")})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("side", ["rows", "cols"])
@pytest.mark.parametrize("world,case,parts", [(2, 0, 1), (3, 0, 1), (2, 1, 1), (3, 3, 1), (2, 0, 2), (3, 3, 3)])
def test_dsgd_ring_equals_reference_parallel_train(world, case, parts, side):
    """Both rotation sides (u/b row blocks or v/w/c/b_hat column blocks travel) give the
    same bytes as the reference's parallel_train(D); parts > 1: the pipelined ring
    (sub-blocks shifted while the next one trains) too."""
    z = load_golden("sgd_small.npz")
    if world not in (2, 3):
        pytest.skip()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q, parts, side)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pre = f"s{case}_D{world}_"
    names = {"b": "b", "bhat": "b_hat", "U": "U", "V": "V", "W": "W", "C": "C"}
    for k, n in names.items():
        assert res[k] == z[pre + n].tobytes(), (world, case, n)


@pytest.mark.parametrize("side", ["rows", "cols"])
def test_ring_plan_covers_every_block(side):
    from paper_2111_11682_b200.dsgd import RingPlan
    for D in (1, 2, 3, 8):
        p = RingPlan(D, 1000, 700, side)
        seen = set()
        for s in range(D):
            blocks = [p.stage_block(r, s) for r in range(D)]
            # the stage's pairs are parallel_train's: worker w takes ((w + s) % D, w)
            assert sorted(blocks) == sorted(((w + s) % D, w) for w in range(D))
            seen |= set(blocks)
            for r in range(D):   # the block rank r trains next is the one its recv peer trained now
                assert p.moving_block(r, s + 1) == p.moving_block(p.recv_peer(r), s)
                assert p.send_peer(p.recv_peer(r)) == r
        assert len(seen) == D * D
        for parts in (1, 2, 3):   # sub-blocks tile each block
            for blk in range(D):
                for sub, whole in ((p.sub_rows, p.rows), (p.sub_cols, p.cols)):
                    sl = [sub(blk, h, parts) for h in range(parts)]
                    assert sl[0].start == whole(blk).start and sl[-1].stop == whole(blk).stop
                    assert all(sl[h].stop == sl[h + 1].start for h in range(parts - 1))


def test_choose_side():
    from paper_2111_11682_b200.dsgd import choose_side
    assert choose_side(480_189, 17_770, 128, 32) == "cols"      # Netflix: move v/w/c (1.7 MB / stage)
    assert choose_side(1_000, 600_000, 32, 64) == "rows"
