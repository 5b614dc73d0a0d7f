"""Reference-written 20-epoch learning curve at C1 (the Hogwild RMSE contract's anchor).

Run in the build container only (the reference is not on the GPU box):

    cp -r /root/reference/pkg /tmp/refpkg
    NUMBA_CACHE_DIR=/tmp/numba PYTHONPATH=/tmp/refpkg/src python tests/golden/make_golden_ref20.py

The unmodified reference's train_full (F=32, K=16, 20 epochs, TrainConfig defaults) on
the C1 split of c1.npz, with its own simLSH J^K, recording the reference's test and
train RMSE after every epoch (the CLI's callback, cli.py:204-210).  tests compare the
CUDA Hogwild mode's curve against it (north_star: within 0.005 after the same epochs).
"""

from __future__ import annotations

import os
import sys

import numpy as np

import lshmf
from lshmf.data import split_holdout
from lshmf.datasets import synthetic_movielens_100k
from lshmf.factorization import TrainConfig, rmse, train_full
from lshmf.lsh import LshConfig, simlsh_topk

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    print("lshmf", lshmf.__version__, "numpy", np.__version__)
    data = synthetic_movielens_100k(seed=0)
    train, test = split_holdout(data, 0.1, seed=0)
    table, _ = simlsh_topk(train, LshConfig(G=8, p=3, q=100, psi_exponent=2, seed=0), K=16)
    out = {"entries16": table.entries}
    for F, epochs in ((32, 20),):
        cfg = TrainConfig(F=F, K=16, epochs=epochs, seed=0)
        seen = []
        train_full(train, table, cfg,
                   epoch_callback=lambda t, q: seen.append((rmse(q, test, train), rmse(q, train.triplets(), train))))
        out[f"F{F}_rmse_test"] = np.array([a for a, _ in seen])
        out[f"F{F}_rmse_train"] = np.array([b for _, b in seen])
    np.savez_compressed(os.path.join(OUT, "c1_ref20.npz"), **out)
    print({k: v[-1] for k, v in out.items() if k.startswith("F")})


if __name__ == "__main__":
    sys.exit(main())
