"""Generate tests/golden/similarity.npz FROM THE REFERENCE ITSELF (build container only):

    cp -r /root/reference/pkg /tmp/refpkg
    NUMBA_CACHE_DIR=/tmp/numba PYTHONPATH=/tmp/refpkg/src python tests/golden/make_golden_similarity.py

Pins the exact-similarity path (similarity.py: pearson, shrunk_similarity,
gsm_topk, random_topk) and the LSHMF-R text format (data.py:238-257) on stored
inputs: small integer and non-integer matrices (every pair's pearson / shrunk
value, GSM top-K for several K and lambda), GSM on the C1 training matrix, and
random_topk draws.
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

from lshmf.data import Triplets, build_indices, split_holdout
from lshmf.datasets import planted_clusters, random_sparse, synthetic_movielens_100k
from lshmf.similarity import (SimilarityConfig, gsm_topk, pearson, random_topk,
                              shrunk_similarity)

OUT = os.path.dirname(os.path.abspath(__file__))


def trip(r, pre):
    return {f"{pre}M": r.M, f"{pre}N": r.N, f"{pre}rows": r.entry_rows.astype(np.int32),
            f"{pre}cols": r.entry_cols.astype(np.int32), f"{pre}vals": r.entry_values.astype(np.float64)}


def main():
    out = {}
    rng = np.random.default_rng(11)
    cases = []
    # integer stars, non-integer values, planted clusters (many ties / strong similarities)
    cases.append(("int", random_sparse(60, 40, 0.3, seed=3)))
    r = random_sparse(50, 35, 0.35, seed=4)
    vals = r.entry_values * 0.37 + rng.normal(0, 0.2, r.nnz)
    cases.append(("real", build_indices(Triplets(r.entry_rows, r.entry_cols, vals), M=r.M, N=r.N)))
    cases.append(("planted", planted_clusters(seed=5, M=80, N=48, n_clusters=6, fans_per_cluster=8)[0]))
    cases.append(("sparse", random_sparse(40, 30, 0.05, seed=6)))   # many zero-support pairs
    out["cases"] = np.array([c[0] for c in cases])
    for name, r in cases:
        out.update(trip(r, name + "_"))
        N = r.N
        P = np.zeros((N, N))
        S = np.zeros((N, N))
        for a in range(N):
            for b in range(N):
                if a != b:
                    P[a, b] = pearson(r, a, b)
                    S[a, b] = shrunk_similarity(r, a, b, 25.0)
        out[name + "_pearson"] = P
        out[name + "_shrunk25"] = S
        for K in (1, 5, min(16, N - 1)):
            for lam in (100.0, 25.0, 0.0):
                out[f"{name}_gsm_K{K}_l{int(lam)}"] = gsm_topk(r, SimilarityConfig(K=K, lambda_rho=lam)).entries
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "m.txt")
            r.save(p)
            out[name + "_lshmfr"] = np.frombuffer(open(p, "rb").read(), dtype=np.uint8)
    data = synthetic_movielens_100k(seed=0)
    train, _ = split_holdout(data, 0.1, seed=0)
    out.update({"c1_" + k: v for k, v in trip(train, "").items()})
    out["c1_gsm_K16"] = gsm_topk(train, SimilarityConfig(K=16)).entries
    out["c1_gsm_K32_l50"] = gsm_topk(train, SimilarityConfig(K=32, lambda_rho=50.0)).entries
    # checkpoint / hash-state binary formats (factorization.py:154-185, lsh.py:209-228)
    from lshmf.factorization import ModelParams
    from lshmf.lsh import LshConfig, compute_hash_state
    from lshmf.similarity import NeighborTable
    g = np.random.default_rng(3)
    nb = NeighborTable(N=6, K=2, entries=np.array([[1, 2], [0, 2], [0, 1], [4, 5], [3, 5], [3, 4]], np.int32))
    mp = ModelParams(mu=3.25, b=g.random(7), b_hat=g.random(6), U=g.random((7, 4)), V=g.random((6, 4)),
                     W=g.random((6, 2)), C=g.random((6, 2)), neighbors=nb)
    for k in ("b", "b_hat", "U", "V", "W", "C"):
        out["mp_" + k] = getattr(mp, k)
    out["mp_entries"] = nb.entries
    r0 = cases[0][1]
    hs = compute_hash_state(r0, LshConfig(G=8, p=3, q=7, psi_exponent=2, seed=4))
    with tempfile.TemporaryDirectory() as d:
        mp.save(os.path.join(d, "m.bin"))
        out["mp_bytes"] = np.frombuffer(open(os.path.join(d, "m.bin"), "rb").read(), dtype=np.uint8)
        hs.save(os.path.join(d, "h.bin"))
        out["hs_bytes"] = np.frombuffer(open(os.path.join(d, "h.bin"), "rb").read(), dtype=np.uint8)
    out["rand_2_1_0"] = random_topk(2, 1, seed=0).entries
    out["rand_50_5_9"] = random_topk(50, 5, seed=9).entries
    out["rand_1682_16_0"] = random_topk(1682, 16, seed=0).entries
    np.savez_compressed(os.path.join(OUT, "similarity.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    sys.exit(main())
