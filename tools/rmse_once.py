"""One train RMSE and one test RMSE call on a C3 exact-mode model (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_11682_b200 as P  # noqa: E402
from paper_2111_11682_b200 import _native as nat, synth  # noqa: E402
from rmse_phases import RATES  # noqa: E402

M, N, nnz, F, K, e = synth.SHAPES["c3"]
r = synth.random_sparse_ratings(M, N, nnz, seed=0)
tbl, _ = P.simlsh_topk(r, P.LshConfig(psi_exponent=e), K)
p = P.train_full(r, tbl, P.TrainConfig(F=F, K=K, epochs=1, seed=0, **RATES), mode=sys.argv[1] if len(sys.argv) > 1 else "exact")
rng = np.random.default_rng(1)
er, ec, ev = (nat.to_host(x) for x in r.device_entries())
sel = np.sort(rng.choice(r.nnz, r.nnz // 100, replace=False))
test = P.Triplets(er[sel].copy(), ec[sel].copy(), ev[sel].copy())
print(P.rmse(p, r.triplets(), r), P.rmse(p, test, r))
torch.cuda.synchronize()
