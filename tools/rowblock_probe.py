"""Probe: the C3 Hogwild epoch run as B row-block sub-epochs (each column's entries with rows in
block b, blocks in ascending order -- every column still meets its entries in row order) so
that each sub-epoch's u rows (246 MB / B) stay L2-resident, against the one-launch epoch.
Uses the DSGD block path (HogwildTrainer.block_work / launch_work); times 5 epochs per B with
CUDA events and reports ms/epoch and the training loss after them.

  python tools/rowblock_probe.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_11682_b200 import lsh, synth  # noqa: E402
from paper_2111_11682_b200.factorization import TrainConfig  # noqa: E402
from paper_2111_11682_b200.hogwild import HogwildTrainer  # noqa: E402
from paper_2111_11682_b200.similarity import NeighborTable  # noqa: E402
from paper_2111_11682_b200 import _native as nat  # noqa: E402

RATES = dict(alpha_b=0.02, alpha_b_hat=0.02, alpha_u=0.02, alpha_v=0.02, alpha_w=0.001, alpha_c=0.001,
             lambda_b=0.01, lambda_b_hat=0.01, lambda_u=0.01, lambda_v=0.01, lambda_w=0.05, lambda_c=0.05,
             beta=0.3)


def main():
    torch.cuda.set_device(0)
    M, N, nnz_t, F, K, e = synth.SHAPES["c3"]
    dm = synth.random_sparse_device(M, N, nnz_t, seed=0)
    d = dm.dev
    ent, _, _ = lsh.simlsh_topk_device(d, lsh.LshConfig(psi_exponent=e), K)
    nbr = NeighborTable(N, K, nat.to_host(ent)[:N * K].reshape(N, K).astype(np.int32))
    cols = torch.repeat_interleave(torch.arange(N, device="cuda", dtype=torch.int64), d.col_ptr[1:] - d.col_ptr[:-1])
    key = cols * M + d.col_rows.to(torch.int64)
    out = {}
    for B in (1, 2, 4, 8):
        cfg = TrainConfig(F=F, K=K, epochs=8, seed=0, **RATES)
        tr = HogwildTrainer(None, nbr, cfg, dev=d)
        works = []
        if B > 1:
            jj = torch.arange(N, device="cuda", dtype=torch.int64)
            bounds = [(b * M) // B for b in range(B + 1)]
            pos = [torch.searchsorted(key, jj * M + r) for r in bounds]
            allc = torch.arange(N, device="cuda", dtype=torch.int32)
            for b in range(B):
                seg = torch.stack([pos[b], pos[b + 1]], 1).reshape(-1).contiguous()
                works.append(tr.block_work(seg, allc))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for t in range(cfg.epochs):
            if t == 3:
                tr.loss.zero_()
                ev[0].record()
            if B == 1:
                tr.launch_epoch(t)
            else:
                for w in works:
                    tr.launch_work(t, w)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / (cfg.epochs - 3)
        out[f"B{B}"] = {"ms_per_epoch": ms, "train_rmse_last5": (float(tr.loss.item()) / (d.nnz * 5)) ** 0.5,
                        "status": int(tr.status.item())}
        print(json.dumps({f"B{B}": out[f"B{B}"]}), flush=True)
        del tr, works
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
