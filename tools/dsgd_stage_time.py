"""Per-GPU compute of the multi-GPU DSGD Hogwild epoch, measured on one GPU: for D = 2, 4, 8
the stage kernel of rank 0 (its column block x one row block) is timed with CUDA events,
both as a per-column block launch (wide stream) and as the block_work list dsgd.bench_main
launches (packed stream, columns split when the block has fewer columns than warps), and the D stages of rank 0 give its compute per
epoch.  The ring shift moves M/D rows of u (F fp32) + b per stage; its NVLink time is not
measurable on one GPU and is reported as bytes.

  python tools/dsgd_stage_time.py [c3]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_11682_b200 import _native as nat, lsh, synth  # noqa: E402
from paper_2111_11682_b200.data import BaselineStats  # noqa: E402
from paper_2111_11682_b200.dsgd import RingPlan  # noqa: E402
from paper_2111_11682_b200.factorization import TrainConfig, init_params  # noqa: E402
from paper_2111_11682_b200.hogwild import HogwildTrainer  # noqa: E402
from paper_2111_11682_b200.similarity import NeighborTable  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    M, N, nnz, F, K, e = synth.SHAPES[name]
    dm = synth.random_sparse_device(M, N, nnz, seed=0)
    d = dm.dev
    ent, _, _ = lsh.simlsh_topk_device(d, lsh.LshConfig(psi_exponent=e), K)
    nbr = NeighborTable(N, K, nat.to_host(ent)[:N * K].reshape(N, K))
    cfg = TrainConfig(F=F, K=K, epochs=20, seed=0)
    stats = BaselineStats(d.mu, nat.to_host(d.base_b), nat.to_host(d.base_bhat))
    tr = HogwildTrainer(None, nbr, cfg, dev=d, params=init_params(M, N, F, K, nbr, stats, cfg))
    for _ in range(2):
        tr.launch_epoch(0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for t in range(5):
        tr.launch_epoch(t)
    b.record()
    torch.cuda.synchronize()
    out = {"config": name, "single_gpu_epoch_ms": a.elapsed_time(b) / 5}
    for D in (2, 4, 8):
        plan = RingPlan(D, M, N)
        rb_t = nat.to_dev(plan.row_bounds)
        bp = nat.empty((N * (D + 1),), "int64")
        nat.call("culsh_block_pointers", nat.ptr(d.col_ptr), nat.ptr(d.col_rows), N, nat.ptr(rb_t), D + 1,
                 nat.ptr(bp), nat.stream_ptr())
        cbt = nat.to_dev(plan.col_bounds)
        cs = plan.cols(0)
        counts = (d.col_ptr[1:] - d.col_ptr[:-1])[cs]
        own = (torch.argsort(counts, descending=True, stable=True) + cs.start).to(torch.int32)
        stage_ms, work_ms, split = [], [], 0
        for s in range(D):
            seg = nat.zeros((2 * N,), "int64")
            chain = nat.zeros((N,), "int32")
            nat.call("culsh_pass_plan", nat.ptr(d.col_ptr), nat.ptr(d.col_rows), N, 1, 0, N, 0, M,
                     nat.ptr(bp), nat.ptr(cbt), D, s, nat.ptr(seg), nat.ptr(chain), nat.stream_ptr())
            tr.launch_epoch(0, seg=seg, col_order=own, n_cols=own.numel())   # warm
            torch.cuda.synchronize()
            a.record()
            for t in range(5):
                tr.launch_epoch(t, seg=seg, col_order=own, n_cols=own.numel())
            b.record()
            torch.cuda.synchronize()
            stage_ms.append(a.elapsed_time(b) / 5)
            w = tr.block_work(seg, own)
            tr.launch_work(0, w)
            torch.cuda.synchronize()
            a.record()
            for t in range(5):
                tr.launch_work(t, w)
            b.record()
            torch.cuda.synchronize()
            work_ms.append(a.elapsed_time(b) / 5)
            split = w["split_cols"]
        shift_bytes = int((plan.row_bounds[1] - plan.row_bounds[0]) * (F + 1) * 4)
        out[f"D{D}"] = {"stage_ms": [round(x, 4) for x in stage_ms], "compute_ms_per_epoch": sum(stage_ms),
                        "work_stage_ms": [round(x, 4) for x in work_ms], "work_compute_ms_per_epoch": sum(work_ms),
                        "work_split_cols": split,
                        "columns_per_rank": own.numel(), "ratings_per_stage": int(nnz / D / D),
                        "shift_bytes_per_stage": shift_bytes,
                        "ideal_ms_per_epoch": out["single_gpu_epoch_ms"] / D}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
