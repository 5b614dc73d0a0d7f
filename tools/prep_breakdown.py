"""Per-stage device time of one Hogwild fit's preparation at C3 (HogwildTrainer.__init__)
plus the simLSH build, with CUDA events around each stage."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_11682_b200 import _native as nat, lsh, synth  # noqa: E402
from paper_2111_11682_b200 import hogwild as hw  # noqa: E402
from paper_2111_11682_b200.data import BaselineStats  # noqa: E402
from paper_2111_11682_b200.factorization import TrainConfig, init_params  # noqa: E402
from paper_2111_11682_b200.similarity import NeighborTable  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c3"
M, N, nnz, F, K, e = synth.SHAPES[cfgname]
dm = synth.random_sparse_device(M, N, nnz, seed=0)
ent, _, _ = lsh.simlsh_topk_device(dm.dev, lsh.LshConfig(psi_exponent=e), K)
nbr = NeighborTable(N, K, nat.to_host(ent)[:N * K].reshape(N, K))
cfg = TrainConfig(F=F, K=K, epochs=1, seed=0)
stats = BaselineStats(dm.dev.mu, nat.to_host(dm.dev.base_b), nat.to_host(dm.dev.base_bhat))
t0 = time.perf_counter()
params = init_params(M, N, F, K, nbr, stats, cfg)
t_init = time.perf_counter() - t0

marks = {}
orig_call = nat.call


def timed_call(name, *a):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = orig_call(name, *a)
    torch.cuda.synchronize()
    marks[name] = marks.get(name, 0.0) + time.perf_counter() - t
    return r


hw.HogwildTrainer(None, nbr, cfg, dev=dm.dev, params=params)   # warm
torch.cuda.synchronize()
nat.call = timed_call
hw.nat.call = timed_call
t0 = time.perf_counter()
tr = hw.HogwildTrainer(None, nbr, cfg, dev=dm.dev, params=params)
torch.cuda.synchronize()
total = time.perf_counter() - t0
print(json.dumps({"config": cfgname, "init_params_host_s": t_init, "trainer_init_s": total,
                  "native_calls_s": marks}), flush=True)
