"""C3-shape skewed data (lognormal row activity / column popularity, SURVEY's perf-stress
generator): Hogwild epoch time with work segments started from per-plan stream cursors (the
default) vs the in-kernel cursor scan, same trainer.

  python tools/skew_epoch_probe.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_11682_b200 as P  # noqa: E402
from paper_2111_11682_b200 import lsh, synth, _native as nat  # noqa: E402
from paper_2111_11682_b200.factorization import TrainConfig  # noqa: E402
from paper_2111_11682_b200.hogwild import HogwildTrainer  # noqa: E402
from paper_2111_11682_b200.similarity import NeighborTable  # noqa: E402

RATES = dict(alpha_b=0.02, alpha_b_hat=0.02, alpha_u=0.02, alpha_v=0.02, alpha_w=0.001, alpha_c=0.001,
             lambda_b=0.01, lambda_b_hat=0.01, lambda_u=0.01, lambda_v=0.01, lambda_w=0.05, lambda_c=0.05,
             beta=0.3)


def main():
    torch.cuda.set_device(0)
    M, N, nnz_t, F, K, e = synth.SHAPES["c3"]
    r, c, v = synth.structured_triplets_device(M, N, nnz_t, seed=0)
    dsr = P.DeviceSparseRatings(M, N, r, c, v)
    d = dsr.device()
    ent, _, _ = lsh.simlsh_topk_device(d, lsh.LshConfig(psi_exponent=e), K)
    nbr = NeighborTable(N, K, nat.to_host(ent)[:N * K].reshape(N, K).astype(np.int32))
    cfg = TrainConfig(F=F, K=K, epochs=8, seed=0, **RATES)
    tr = HogwildTrainer(None, nbr, cfg, dev=d)
    out = {"nnz": d.nnz, "max_col": int((d.col_ptr[1:] - d.col_ptr[:-1]).max().item()),
           "segments": tr.work["n"] if tr.work else 0, "split_cols": tr.work["split_cols"] if tr.work else 0}
    cfg.epochs = 20
    for rep, mode in enumerate(("cursors", "scan", "cursors", "scan")):   # alternating: same model age
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for t in range(5 * rep, 5 * rep + 5):
            if t == 5 * rep + 1:
                ev[0].record()
            if mode == "cursors":
                tr.launch_epoch(t)
            else:   # the work list without cursors: the kernel scans from each column start
                tr._launch_packed(tr.work["n"], tr._stream_buffers(resident=True), tr.work["col"], tr._rates(t),
                                  tr.loss, tr.work["seg"])
        ev[1].record()
        torch.cuda.synchronize()
        out.setdefault(f"{mode}_ms_per_epoch", []).append(ev[0].elapsed_time(ev[1]) / 4)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
