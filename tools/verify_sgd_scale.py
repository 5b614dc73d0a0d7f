"""Full-scale exact-SGD parity evidence: one parallel_train(D) epoch at C3 (100M ratings,
F=128, K=32) on the GPU against the oracle's parallel_epoch (pinned to the reference's
parallel_train), all parameters compared byte for byte.

  python tools/verify_sgd_scale.py [c3] [D]
"""
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_11682_b200 as P  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2111_11682_b200 import _native as nat, lsh, synth  # noqa: E402
from paper_2111_11682_b200.data import DeviceSparseRatings  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    D = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    M, N, nnz, F, K, e = synth.SHAPES[name]
    dm = synth.random_sparse_device(M, N, nnz, seed=0)
    d = dm.dev
    col = torch.repeat_interleave(torch.arange(N, device="cuda"), d.col_ptr[1:] - d.col_ptr[:-1]).to(torch.int32)
    r = DeviceSparseRatings(M, N, d.col_rows, col, d.col_vals)
    ent, _, _ = lsh.simlsh_topk_device(r.device(), P.LshConfig(psi_exponent=e), K)
    nbr = P.NeighborTable(N, K, nat.to_host(ent)[:N * K].reshape(N, K))
    cfg = P.TrainConfig(F=F, K=K, epochs=1, seed=0, alpha_b=0.02, alpha_b_hat=0.02, alpha_u=0.02,
                        alpha_v=0.02, alpha_w=0.001, alpha_c=0.001, lambda_b=0.01, lambda_b_hat=0.01,
                        lambda_u=0.01, lambda_v=0.01, lambda_w=0.05, lambda_c=0.05)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = P.parallel_train(r, nbr, cfg, D)
    gpu_s = time.perf_counter() - t0
    cp, cr, cv = nat.to_host(d.col_ptr), nat.to_host(d.col_rows), nat.to_host(d.col_vals)
    cols = np.repeat(np.arange(N, dtype=np.int32), np.diff(cp))
    csr, mu = orc.build_csr(M, N, cr, cols, cv)
    t0 = time.perf_counter()
    m = orc.parallel_train(csr, mu, nbr.entries, F, K, 1, 0, cfg.rates_at, cfg.regs, D)
    cpu_s = time.perf_counter() - t0
    eq = {k: getattr(p, k).tobytes() == getattr(m, k2).tobytes()
          for k, k2 in (("b", "b"), ("b_hat", "bhat"), ("U", "U"), ("V", "V"), ("W", "W"), ("C", "C"))}
    print(json.dumps({"case": f"{name} parallel_train D={D}, 1 epoch", "nnz": int(d.nnz), "F": F, "K": K,
                      "gpu_api_s_incl_setup": gpu_s, "oracle_s": cpu_s, "oracle_threads": orc.n_threads(),
                      "U_sha": sha(p.U), "equal": eq, "all_equal": all(eq.values())}), flush=True)


if __name__ == "__main__":
    main()
