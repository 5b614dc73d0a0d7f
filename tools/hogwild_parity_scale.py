"""Hogwild (fp32, the performance mode) vs exact (bit-identical to the reference)
test RMSE at C2 / C3 scale on a synthetic 90/10 split built in HBM (GPU).

  python tools/hogwild_parity_scale.py c2 10
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2111_11682_b200 as P
from paper_2111_11682_b200 import _native as nat, lsh, synth
from paper_2111_11682_b200.data import DeviceSparseRatings
from paper_2111_11682_b200.hogwild import HogwildTrainer

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 10
M, N, nnz, F, K, e = synth.SHAPES[cfg_name]
rows, cols, vals = synth.structured_triplets_device(M, N, nnz, seed=0)
n_test = rows.numel() // 10          # entries are in random order: last 10% = test
tr_rows, tr_cols, tr_vals = rows[n_test:], cols[n_test:], vals[n_test:]
te = P.Triplets(nat.to_host(rows[:n_test]), nat.to_host(cols[:n_test]), nat.to_host(vals[:n_test]))


tr = DeviceSparseRatings(M, N, tr_rows, tr_cols, tr_vals)
ent, _, _ = lsh.simlsh_topk_device(tr.device(), lsh.LshConfig(psi_exponent=e), K)
nbr = P.NeighborTable(N, K, nat.to_host(ent)[:N * K].reshape(N, K))
rates = dict(alpha_b=0.02, alpha_b_hat=0.02, alpha_u=0.02, alpha_v=0.02, alpha_w=0.001,
             alpha_c=0.001, lambda_b=0.01, lambda_b_hat=0.01, lambda_u=0.01, lambda_v=0.01,
             lambda_w=0.05, lambda_c=0.05, beta=0.3)
cfg = P.TrainConfig(F=F, K=K, epochs=epochs, seed=0, **rates)
t0 = time.perf_counter()
ex = P.train_full(tr, nbr, cfg)
torch.cuda.synchronize()
t_ex = time.perf_counter() - t0
r_ex = P.rmse(ex, te, tr)
print(f"{cfg_name}: train nnz {tr.nnz}, test {len(te)}; exact {epochs} epochs {t_ex:.1f}s "
      f"({t_ex / epochs * 1e3:.0f} ms/epoch) test RMSE {r_ex:.5f}", flush=True)
for rot, at in ((1, 1), (1, 0), (0, 1)):
    h = HogwildTrainer(tr, nbr, cfg, rotate=bool(rot), atomic_rows=bool(at))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for t in range(epochs):
        h.epoch(t)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / epochs
    r = P.rmse(h.to_params(), te, tr)
    print(f"  hogwild rotate={rot} atomic={at}: test RMSE {r:.5f}  diff {r - r_ex:+.5f}  "
          f"{dt * 1e3:.1f} ms/epoch", flush=True)
