"""Hogwild vs exact test RMSE on the C1 golden split (GPU).  Usage: python tools/hogwild_rmse.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_11682_b200 as P
from paper_2111_11682_b200.hogwild import HogwildTrainer

z = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "c1.npz"))
tr = P.SparseRatings(int(z["train_M"]), int(z["train_N"]), z["train_rows"].astype(np.int32),
                     z["train_cols"].astype(np.int32), z["train_vals"].astype(np.float64))
te = P.Triplets(z["test_rows"].astype(np.int32), z["test_cols"].astype(np.int32),
                z["test_vals"].astype(np.float64))
for K, ent in ((16, z["lsh_entries16"]), (32, z["lsh_entries32"])):
    nbr = P.NeighborTable(tr.N, K, ent)
    for epochs in (5, 20, 50):
        cfg = P.TrainConfig(F=32, K=K, epochs=epochs, seed=0)
        ex = P.rmse(P.train_full(tr, nbr, cfg), te, tr)
        out = [f"K={K} epochs={epochs} exact={ex:.5f}"]
        for rot, MW in ((1, 0), (1, 58), (0, 58)):
            h = HogwildTrainer(tr, nbr, cfg, rotate=bool(rot), max_warps=MW)
            for t in range(epochs):
                h.epoch(t)
            r = P.rmse(h.to_params(), te, tr)
            out.append(f"rot{rot}mw{MW}={r:.5f} (d={r - ex:+.5f})")
        print("  ".join(out), flush=True)
