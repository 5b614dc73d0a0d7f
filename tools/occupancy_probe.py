"""Is the C3 Hogwild epoch latency-bound?  Time it with the resident warps capped
(HogwildTrainer.max_warps -> grid of max_warps/8 CTAs: 4 / 3 / 2 / 1 CTAs per SM).

  python tools/occupancy_probe.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_11682_b200 import lsh, synth, _native as nat  # noqa: E402
from paper_2111_11682_b200.factorization import TrainConfig  # noqa: E402
from paper_2111_11682_b200.hogwild import HogwildTrainer  # noqa: E402
from paper_2111_11682_b200.similarity import NeighborTable  # noqa: E402

RATES = dict(alpha_b=0.02, alpha_b_hat=0.02, alpha_u=0.02, alpha_v=0.02, alpha_w=0.001, alpha_c=0.001,
             lambda_b=0.01, lambda_b_hat=0.01, lambda_u=0.01, lambda_v=0.01, lambda_w=0.05, lambda_c=0.05,
             beta=0.3)


def main():
    torch.cuda.set_device(0)
    M, N, nnz_t, F, K, e = synth.SHAPES["c3"]
    d = synth.random_sparse_device(M, N, nnz_t, seed=0).dev
    ent, _, _ = lsh.simlsh_topk_device(d, lsh.LshConfig(psi_exponent=e), K)
    nbr = NeighborTable(N, K, nat.to_host(ent)[:N * K].reshape(N, K).astype(np.int32))
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    out = {}
    for per_sm in (4, 3, 2, 1):
        cfg = TrainConfig(F=F, K=K, epochs=8, seed=0, **RATES)
        tr = HogwildTrainer(None, nbr, cfg, dev=d, max_warps=per_sm * 8 * sms)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for t in range(cfg.epochs):
            if t == 3:
                ev[0].record()
            tr.launch_epoch(t)
        ev[1].record()
        torch.cuda.synchronize()
        out[f"{per_sm}_ctas_per_sm"] = ev[0].elapsed_time(ev[1]) / 5
        print(json.dumps(out), flush=True)
        del tr


if __name__ == "__main__":
    main()
