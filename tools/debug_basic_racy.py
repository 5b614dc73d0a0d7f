"""train_basic racy mode (CUSGD++ lock-free on V) at C2/C3 scale: divergence and loss
per epoch with the rotated visiting order on / off (debug aid)."""
import sys
from dataclasses import replace

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_11682_b200 as P  # noqa: E402
from paper_2111_11682_b200 import synth  # noqa: E402
from paper_2111_11682_b200 import factorization as fz  # noqa: E402
from paper_2111_11682_b200.data import DeviceSparseRatings  # noqa: E402
from paper_2111_11682_b200.hogwild import HogwildTrainer  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
M, N, nnz, F, K, e = synth.SHAPES[name]
dm = synth.random_sparse_device(M, N, nnz, seed=0)
d = dm.dev
col = torch.repeat_interleave(torch.arange(N, device="cuda"), d.col_ptr[1:] - d.col_ptr[:-1]).to(torch.int32)
r = DeviceSparseRatings(M, N, d.col_rows, col, d.col_vals)
config = P.TrainConfig(F=F, K=0, epochs=3, seed=0)
rng = np.random.default_rng(0)
U = rng.uniform(0.0, config.effective_init_scale, size=(M, F))
V = rng.uniform(0.0, config.effective_init_scale, size=(N, F))
tdev = fz._transposed_device(r)
tcfg = replace(config, K=0, alpha_b=1e-300, alpha_b_hat=1e-300, alpha_u=config.alpha_v, alpha_v=config.alpha_u,
               lambda_u=config.lambda_v, lambda_v=config.lambda_u)
for rotate in (False, True):
    tp = P.ModelParams(mu=0.0, b=np.zeros(N), b_hat=np.zeros(M), U=V.copy(), V=U.copy(), W=np.zeros((M, 0)),
                       C=np.zeros((M, 0)), neighbors=None)
    tr = HogwildTrainer(None, None, tcfg, dev=tdev, params=tp, rotate=rotate)
    out = []
    for t in range(4):
        tr.loss.zero_()
        tr.launch_epoch(t)
        torch.cuda.synchronize()
        out.append((round(float(tr.loss.item()) / tdev.nnz, 5), int(tr.status.item())))
    print("rotate", rotate, out, flush=True)

if "--full" in sys.argv:
    # the neighbourhood model (train_full mode="hogwild") with the default TrainConfig rates
    from paper_2111_11682_b200 import lsh, _native as nat
    ent, _, _ = lsh.simlsh_topk_device(r.device(), P.LshConfig(psi_exponent=e), 32)
    nbr = P.NeighborTable(N, 32, nat.to_host(ent)[:N * 32].reshape(N, 32))
    for rotate in (False, True):
        tr = HogwildTrainer(r, nbr, P.TrainConfig(F=F, K=32, epochs=4, seed=0), rotate=rotate)
        out = []
        for t in range(4):
            tr.loss.zero_()
            tr.launch_epoch(t)
            torch.cuda.synchronize()
            out.append((round(float(tr.loss.item()) / r.device().nnz, 5), int(tr.status.item())))
        print("full model, default rates, rotate", rotate, out, flush=True)
