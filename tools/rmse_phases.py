"""Kernel-level cost of the per-epoch callback's two rmse calls at C3 (cli.py:204-210):
train RMSE over the training set and test RMSE over a 1 % split_holdout-style test set,
on an exact-mode (fp64) model and a Hogwild (fp32) model.  Kernel times from the CUPTI
activity records (torch.profiler), wall times with a sync on both sides.

  python tools/rmse_phases.py
"""
import json
import os
import sys
import time
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2111_11682_b200 as P  # noqa: E402
from paper_2111_11682_b200 import _native as nat, synth  # noqa: E402

RATES = dict(alpha_b=0.02, alpha_b_hat=0.02, alpha_u=0.02, alpha_v=0.02, alpha_w=0.001, alpha_c=0.001,
             lambda_b=0.01, lambda_b_hat=0.01, lambda_u=0.01, lambda_v=0.01, lambda_w=0.05, lambda_c=0.05,
             beta=0.3)


def wall(fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def kernels(fn):
    fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    agg = defaultdict(float)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            agg[ev.name[:60]] += ev.device_time_total / 1e6
    return {k: round(v, 5) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]}


def main():
    torch.cuda.set_device(0)
    M, N, nnz, F, K, e = synth.SHAPES["c3"]
    r = synth.random_sparse_ratings(M, N, nnz, seed=0)
    tbl, _ = P.simlsh_topk(r, P.LshConfig(psi_exponent=e), K)
    rng = np.random.default_rng(1)
    er, ec, ev = (nat.to_host(x) for x in r.device_entries())
    sel = np.sort(rng.choice(r.nnz, r.nnz // 100, replace=False))
    arrs = [er[sel].copy(), ec[sel].copy(), ev[sel].copy()]
    for a in arrs:
        a.flags.writeable = False      # split_holdout's test sets are immutable (cached device copy)
    test = P.Triplets(*arrs)
    test_w = P.Triplets(*(a.copy() for a in arrs))   # writeable (a CLI --test file): uploaded per call
    train_t = r.triplets()
    out = {"config": "C3", "test_n": len(test)}
    for mode in ("exact", "hogwild"):
        p = P.train_full(r, tbl, P.TrainConfig(F=F, K=K, epochs=1, seed=0, **RATES), mode=mode)
        out[mode] = {
            "train_wall_s": wall(lambda: P.rmse(p, train_t, r)),
            "test_wall_s": wall(lambda: P.rmse(p, test, r)),
            "test_writeable_wall_s": wall(lambda: P.rmse(p, test_w, r)),
            "train_kernels_s": kernels(lambda: P.rmse(p, train_t, r)),
            "test_kernels_s": kernels(lambda: P.rmse(p, test, r)),
        }
    # the same two calls from inside a fit's per-epoch callback (cli.py:204-210), timed per call
    for mode in ("exact", "hogwild"):
        seen = []

        def cb(t, q):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            P.rmse(q, train_t, r)
            t1 = time.perf_counter()
            P.rmse(q, test_w, r)
            t2 = time.perf_counter()
            seen.append((t1 - t0, t2 - t1))

        P.train_full(r, tbl, P.TrainConfig(F=F, K=K, epochs=4, seed=0, **RATES), mode=mode, epoch_callback=cb)
        out[mode]["in_callback_s"] = seen
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
