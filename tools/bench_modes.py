"""Per-epoch throughput of the exact (bit-identical) training modes through the public
API on device-built uniform synthetic data: train_full (serial column-major order),
parallel_train (DSGD, D blocks) and train_basic (CUSGD++ row-major, exact and racy).
Per-epoch time = (T(1 + n epochs) - T(1 epoch)) / n (n = 2 for the exact modes, 10 for the
fast ones), which cancels the per-call setup.

  python tools/bench_modes.py [c2|c3]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_11682_b200 as P  # noqa: E402
from paper_2111_11682_b200 import _native as nat, lsh, synth  # noqa: E402
from paper_2111_11682_b200.data import DeviceSparseRatings  # noqa: E402

RATES = dict(alpha_b=0.02, alpha_b_hat=0.02, alpha_u=0.02, alpha_v=0.02, alpha_w=0.001, alpha_c=0.001,
             lambda_b=0.01, lambda_b_hat=0.01, lambda_u=0.01, lambda_v=0.01, lambda_w=0.05, lambda_c=0.05)


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t0


def per_epoch(make, extra=2):
    t1 = timed(lambda: make(1))
    tn = timed(lambda: make(1 + extra))
    return (tn - t1) / extra


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    M, N, nnz, F, K, e = synth.SHAPES[name]
    if "--structured" in sys.argv:   # skewed, low-rank-plus-noise stars (SURVEY §8(d) perf-stress)
        rows, cols, vals = synth.structured_triplets_device(M, N, nnz, seed=0)
        r = DeviceSparseRatings(M, N, rows, cols, vals)
        del rows, cols, vals
    else:
        dm = synth.random_sparse_device(M, N, nnz, seed=0)
        d = dm.dev
        col = torch.repeat_interleave(torch.arange(N, device="cuda"), d.col_ptr[1:] - d.col_ptr[:-1]).to(torch.int32)
        r = DeviceSparseRatings(M, N, d.col_rows, col, d.col_vals)
        del col, dm
    d = r.device()
    ent, _, _ = lsh.simlsh_topk_device(d, P.LshConfig(psi_exponent=e), K)
    nbr = P.NeighborTable(N, K, nat.to_host(ent)[:N * K].reshape(N, K))
    cfg = lambda ep: P.TrainConfig(F=F, K=K, epochs=ep, seed=0, **RATES)
    out = {"config": name, "data": "structured" if "--structured" in sys.argv else "uniform", "M": M, "N": N,
           "nnz": int(d.nnz), "F": F, "K": K}
    if "--exact-only" in sys.argv:
        s = per_epoch(lambda ep: P.train_full(r, nbr, cfg(ep)))
        out["train_full_exact_s_per_epoch"] = s
        s = per_epoch(lambda ep: P.parallel_train(r, nbr, cfg(ep), 4))
        out["parallel_train_D4_exact_s_per_epoch"] = s
        print(json.dumps(out), flush=True)
        return
    s = per_epoch(lambda ep: P.train_full(r, nbr, cfg(ep)))
    out["train_full_exact_s_per_epoch"] = s
    out["train_full_exact_updates_per_s"] = d.nnz / s
    s = per_epoch(lambda ep: P.parallel_train(r, nbr, cfg(ep), 4))
    out["parallel_train_D4_exact_s_per_epoch"] = s
    s = per_epoch(lambda ep: P.train_basic(r, P.TrainConfig(F=F, K=0, epochs=ep, seed=0)))
    out["train_basic_exact_s_per_epoch"] = s
    out["train_basic_exact_updates_per_s"] = d.nnz / s
    s = per_epoch(lambda ep: P.train_basic(r, P.TrainConfig(F=F, K=0, epochs=ep, seed=0), racy_workers=8), 10)
    out["train_basic_racy_s_per_epoch"] = s
    out["train_basic_racy_updates_per_s"] = d.nnz / s
    s = per_epoch(lambda ep: P.train_full(r, nbr, cfg(ep), mode="hogwild"), 10)
    out["train_full_hogwild_api_s_per_epoch"] = s
    out["reference_note"] = ("SURVEY.md §6/§8: reference serial train_full 0.31M upd/s (C2), 0.24M (C3), "
                             "1 core; parallel_train D=8 at C2 9.57 s/epoch")
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
