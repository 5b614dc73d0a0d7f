"""Where the time of one C3 train_full(mode="hogwild", 20 epochs) goes, through the public
API, with the parameters read back to host numpy (the per-fit work the epoch-only bench
line excludes): trainer prep (device init + explicit-neighbour stream + packing), the 20
epochs, and the host materialisation of U, V, W, C, b, b_hat (fp64 numpy), each timed with
a device sync on both sides.  Also times the materialisation strategies it chooses between.

  python tools/fit_breakdown.py
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
from paper_2111_11682_b200.hogwild import HogwildTrainer  # noqa: E402

RATES = dict(alpha_b=0.02, alpha_b_hat=0.02, alpha_u=0.02, alpha_v=0.02, alpha_w=0.001, alpha_c=0.001,
             lambda_b=0.01, lambda_b_hat=0.01, lambda_u=0.01, lambda_v=0.01, lambda_w=0.05, lambda_c=0.05,
             beta=0.3)


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def main():
    torch.cuda.set_device(0)
    M, N, nnz, F, K, e = synth.SHAPES["c3"]
    r = synth.random_sparse_ratings(M, N, nnz, seed=0)
    tbl, _ = P.simlsh_topk(r, P.LshConfig(psi_exponent=e), K)
    cfg = P.TrainConfig(F=F, K=K, epochs=20, seed=0, **RATES)
    P.train_full(r, tbl, P.TrainConfig(F=F, K=K, epochs=1, seed=0, **RATES), mode="hogwild")   # warm
    out = {"config": "C3", "nnz": r.nnz}
    tr, out["prep_s"] = timed(lambda: HogwildTrainer(r, tbl, cfg))
    _, out["epochs_s"] = timed(lambda: [tr.epoch(t) for t in range(cfg.epochs)])
    p = P.ModelParams._from_device(tr.model.mu, tr.model, r.M, r.N, tbl)
    _, out["materialise_s"] = timed(lambda: [getattr(p, n) for n in ("b", "b_hat", "U", "V", "W", "C")])
    # the whole public call, as a user makes it
    def fit():
        q = P.train_full(r, tbl, cfg, mode="hogwild")
        return [getattr(q, n) for n in ("b", "b_hat", "U", "V", "W", "C")]
    _, out["fit_s"] = timed(fit)
    _, out["fit_s_2"] = timed(fit)
    # materialisation strategies for U (61.5M fp32 values -> fp64 host array)
    U = tr.model.U[:M * F]
    _, out["U_cpu_then_astype_s"] = timed(lambda: U.cpu().numpy().astype(np.float64))
    _, out["U_dev_f64_then_cpu_s"] = timed(lambda: U.double().cpu().numpy())
    host = torch.empty((M * F,), dtype=torch.float64, pin_memory=True)
    _, out["U_dev_f64_to_pinned_s"] = timed(lambda: host.copy_(U.double(), non_blocking=True))
    _, out["pinned_alloc_492MB_s"] = timed(lambda: torch.empty((M * F,), dtype=torch.float64, pin_memory=True))
    dst = np.empty(M * F, np.float64)
    _, out["pinned_to_numpy_memcpy_s"] = timed(lambda: np.copyto(dst, host.numpy()))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
