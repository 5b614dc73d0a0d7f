"""Hogwild on the C3-shape structured (skewed) data: packed vs wide stream, per-epoch
loss and divergence status (debug aid for TestHogwildAtScale)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2111_11682_b200 as P  # noqa: E402
from paper_2111_11682_b200 import _native as nat, lsh, synth  # noqa: E402
from paper_2111_11682_b200.data import DeviceSparseRatings  # noqa: E402
from paper_2111_11682_b200.hogwild import HogwildTrainer  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "c3"
M, N, nnz, F, K, e = synth.SHAPES[shape]
rows, cols, vals = synth.structured_triplets_device(M, N, nnz, seed=0)
nt = rows.numel() // 10
tr = DeviceSparseRatings(M, N, rows[nt:], cols[nt:], vals[nt:])
d = tr.device()
cnt = (d.col_ptr[1:] - d.col_ptr[:-1])
rc = (d.row_ptr[1:] - d.row_ptr[:-1])
print("nnz", d.nnz, "max col", int(cnt.max()), "max row", int(rc.max()), flush=True)
ent, _, _ = lsh.simlsh_topk_device(d, P.LshConfig(psi_exponent=e), K)
nbr = P.NeighborTable(N, K, nat.to_host(ent)[:N * K].reshape(N, K))
cfg = P.TrainConfig(F=F, K=K, epochs=3, seed=0, alpha_b=0.02, alpha_b_hat=0.02,
                    alpha_u=0.02, alpha_v=0.02, alpha_w=0.001, alpha_c=0.001,
                    lambda_b=0.01, lambda_b_hat=0.01, lambda_u=0.01, lambda_v=0.01,
                    lambda_w=0.05, lambda_c=0.05)
import time
if "--stress" in sys.argv:
    # divergence frequency of the first (largest-step) epoch, fresh model each trial
    for rotate in (False, True):
        fails = 0
        for trial in range(int(sys.argv[sys.argv.index("--stress") + 1])):
            h = HogwildTrainer(tr, nbr, cfg, rotate=rotate)
            h.launch_epoch(0)
            torch.cuda.synchronize()
            fails += int(h.status.item()) != 0
            del h
        print("rotate", rotate, "diverged", fails, flush=True)
    sys.exit(0)
for packed in (True,):
    for atomic, rotate, split in ((True, False, False), (True, False, True)):
        h = HogwildTrainer(tr, nbr, cfg, packed=packed, atomic_rows=atomic, rotate=rotate, split=split)
        print("work list:", None if h.work is None else {k: v for k, v in h.work.items() if k in ("n", "cap", "split_cols")})
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = []
        for t in range(3):
            h.loss.zero_()
            h.launch_epoch(t)
            torch.cuda.synchronize()
            out.append((float(h.loss.item()) / d.nnz, int(h.status.item())))
        ms = (time.perf_counter() - t0) / 3 * 1e3
        p = h.to_params()
        print("packed", h.packed is not None, "atomic", atomic, "rotate", rotate, "split", split, "ms/epoch %.2f" % ms, out,
              "finite U", bool(np.isfinite(p.U).all()), "max|U|", float(np.nanmax(np.abs(p.U))),
              "max|V|", float(np.nanmax(np.abs(p.V))), "max|C|", float(np.nanmax(np.abs(p.C))), flush=True)
