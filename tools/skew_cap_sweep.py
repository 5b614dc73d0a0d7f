"""Work-segment length cap on the skewed C3-shape data: ms/epoch and held-out RMSE of the
Hogwild fit for several caps (default = 2 x nnz / resident warps), against the exact
(serial-order) fit after the same epochs.

  python tools/skew_cap_sweep.py [epochs] [c2|c3]
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
from paper_2111_11682_b200.hogwild import HogwildTrainer  # noqa: E402

epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 6
shape = sys.argv[2] if len(sys.argv) > 2 else "c3"
M, N, nnz, F, K, e = synth.SHAPES[shape]
rows, cols, vals = synth.structured_triplets_device(M, N, nnz, seed=0)
nt = rows.numel() // 10
tr = DeviceSparseRatings(M, N, rows[nt:], cols[nt:], vals[nt:])
te = P.Triplets(nat.to_host(rows[:nt]).astype(np.int32), nat.to_host(cols[:nt]).astype(np.int32),
                nat.to_host(vals[:nt]).astype(np.float64))
d = tr.device()
ent, _, _ = lsh.simlsh_topk_device(d, P.LshConfig(psi_exponent=e), K)
nbr = P.NeighborTable(N, K, nat.to_host(ent)[:N * K].reshape(N, K))
cfg = P.TrainConfig(F=F, K=K, epochs=epochs, seed=0, alpha_b=0.02, alpha_b_hat=0.02, alpha_u=0.02,
                    alpha_v=0.02, alpha_w=0.001, alpha_c=0.001, lambda_b=0.01, lambda_b_hat=0.01,
                    lambda_u=0.01, lambda_v=0.01, lambda_w=0.05, lambda_c=0.05)
warps = 32 * torch.cuda.get_device_properties(0).multi_processor_count
mean = -(-d.nnz // warps)
out = {"shape": shape, "nnz": int(d.nnz), "max_col": int((d.col_ptr[1:] - d.col_ptr[:-1]).max()), "epochs": epochs}
t0 = time.perf_counter()
pe = P.train_full(tr, nbr, cfg)
out["exact_s"] = time.perf_counter() - t0
out["exact_rmse"] = float(P.rmse(pe, te, tr))
for mult in [float(x) for x in os.environ.get("CAPS", "2,1,0.5,0.25").split(",")]:
    cap = max(1024, int(mult * mean))
    h = HogwildTrainer(tr, nbr, cfg, split_cap=cap)
    h.launch_epoch(0)   # warm-up epoch is part of the fit (epochs counted below)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for t in range(1, epochs):
        h.launch_epoch(t)
    ev1.record()
    torch.cuda.synchronize()
    out[f"cap_{mult}x"] = {"cap": cap, "segments": None if h.work is None else h.work["n"],
                          "ms_per_epoch": ev0.elapsed_time(ev1) / max(1, epochs - 1),
                          "status": int(h.status.item()), "rmse": float(P.rmse(h.to_params(), te, tr))}
    del h
print(json.dumps(out), flush=True)
