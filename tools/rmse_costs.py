"""Per-call cost of rmse() on the resident model at C3 (train set = ratings.triplets(),
and held-out sets of 1 % / 10 %), for an exact (fp64) and a Hogwild (fp32) fit.

  python tools/rmse_costs.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_11682_b200 as P  # noqa: E402
from paper_2111_11682_b200 import _native as nat, synth  # noqa: E402


def timed(fn, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        out.append(time.perf_counter() - t0)
    return out


def main():
    torch.cuda.set_device(0)
    M, N, nnz, F, K, e = synth.SHAPES["c3"]
    r = synth.random_sparse_ratings(M, N, nnz, seed=0)
    tbl, _ = P.simlsh_topk(r, P.LshConfig(psi_exponent=e), K)
    rng = np.random.default_rng(1)
    er, ec, ev = (nat.to_host(x) for x in r.device_entries())
    res = {}
    tests = {}
    for frac in (100, 10):
        sel = np.sort(rng.choice(r.nnz, r.nnz // frac, replace=False))
        tests[f"test_{100 // frac}pct"] = P.Triplets(er[sel].copy(), ec[sel].copy(), ev[sel].copy())
    for mode in ("exact", "hogwild"):
        p = P.train_full(r, tbl, P.TrainConfig(F=F, K=K, epochs=1, seed=0), mode=mode)
        res[f"{mode}_train"] = timed(lambda: P.rmse(p, r.triplets(), r))
        for k, te in tests.items():
            res[f"{mode}_{k}"] = timed(lambda: P.rmse(p, te, r))
        res[f"{mode}_device_model"] = timed(lambda: p._device(64))
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
