"""Generate the golden fixtures under tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container only (the reference is not on the GPU box):

    cp -r /root/reference/pkg /tmp/refpkg
    NUMBA_CACHE_DIR=/tmp/numba PYTHONPATH=/tmp/refpkg/src python tests/golden/make_golden.py

Every array here is an output of the unmodified reference package (lshmf) on
inputs that are stored alongside it, so the fixtures pin both the CPU oracle
(oracle/) and the CUDA path to the reference's exact behaviour.  Large outputs
are stored as sha256 digests of their little-endian bytes plus small samples.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

import lshmf
from lshmf.data import SparseRatings, Triplets, build_indices, split_holdout
from lshmf.datasets import random_sparse, synthetic_movielens_100k, planted_clusters
from lshmf.factorization import TrainConfig, rmse, train_full, predict
from lshmf.lsh import (LshConfig, _state_group_keys, assign_row_hashes,
                       compute_hash_state, simlsh_topk)
from lshmf.online import (absorb_increment, holdback_variables,
                          update_hashes_incremental, topk_for_new, extend_ratings)
from lshmf.parallel import parallel_train
from lshmf.similarity import random_topk

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def triplets_of(r: SparseRatings, prefix: str) -> dict:
    return {f"{prefix}M": r.M, f"{prefix}N": r.N,
            f"{prefix}rows": r.entry_rows.astype(np.int32),
            f"{prefix}cols": r.entry_cols.astype(np.int32),
            f"{prefix}vals": r.entry_values.astype(np.float64)}


def params_of(p, prefix: str, full: bool) -> dict:
    d = {f"{prefix}mu": p.mu}
    for n in ("b", "b_hat", "U", "V", "W", "C"):
        a = getattr(p, n)
        d[f"{prefix}{n}_sha"] = sha(a)
        if full:
            d[f"{prefix}{n}"] = a
    return d


def lsh_small():
    """simlsh_topk on small matrices: integer and non-integer values, several configs."""
    cases = []
    rng = np.random.default_rng(42)
    M, N = 12, 9
    mask = rng.random((M, N)) < 0.5
    rows, cols = np.nonzero(mask)
    vals = rng.integers(1, 6, size=len(rows)).astype(float)
    cases.append((build_indices(Triplets(rows.astype(np.int32), cols.astype(np.int32), vals), M=M, N=N),
                  [(6, 2, 4, 2, 9, 3), (5, 2, 3, 2, 8, 3), (4, 2, 3, 1, 5, 3), (8, 1, 1, 1, 0, 3)]))
    cases.append((random_sparse(30, 22, 0.25, seed=3),
                  [(8, 3, 10, 2, 0, 5), (16, 4, 7, 4, 11, 4), (3, 5, 9, 1, 2, 6)]))
    cases.append((random_sparse(40, 60, 0.2, seed=4, integer_values=False),
                  [(8, 3, 20, 2, 0, 8), (64, 1, 5, 4, 1, 4), (13, 2, 6, 1, 7, 5)]))
    pc, _ = planted_clusters(seed=0, M=120, N=150, n_clusters=6, fans_per_cluster=10)
    cases.append((pc, [(8, 3, 100, 2, 0, 16), (4, 2, 50, 1, 3, 8)]))
    out = {"n_cases": len(cases)}
    k = 0
    for ci, (r, cfgs) in enumerate(cases):
        out.update(triplets_of(r, f"c{ci}_"))
        for (G, p, q, e, seed, K) in cfgs:
            cfg = LshConfig(G=G, p=p, q=q, psi_exponent=e, seed=seed)
            table, state = simlsh_topk(r, cfg, K=K)
            keys = _state_group_keys(state)
            pre = f"k{k}_"
            out[pre + "case"] = ci
            out[pre + "cfg"] = np.array([G, p, q, e, seed, K], np.int64)
            out[pre + "acc"] = state.acc
            out[pre + "sig"] = state.sig
            out[pre + "keys"] = keys
            out[pre + "entries"] = table.entries
            k += 1
    out["n_runs"] = k
    np.savez_compressed(os.path.join(OUT, "lsh_small.npz"), **out)


def c1_data():
    data = synthetic_movielens_100k(seed=0)
    train, test = split_holdout(data, 0.1, seed=0)
    return train, test


def lsh_c1(train):
    cfg = LshConfig(G=8, p=3, q=100, psi_exponent=2, seed=0)
    table, state = simlsh_topk(train, cfg, K=16)
    keys = _state_group_keys(state)
    table32, _ = simlsh_topk(train, cfg, K=32)
    return {"acc_sha": sha(state.acc), "sig_sha": sha(state.sig), "keys": keys,
            "entries16": table.entries, "entries32": table32.entries,
            "acc_sample": state.acc[::97, 3, 1, :].copy()}, table


def sgd_small():
    out = {}
    for s, (integer, F, K, epochs) in enumerate([(True, 4, 4, 6), (False, 3, 2, 4), (True, 8, 0, 3),
                                                  (True, 5, 7, 3)]):
        r = random_sparse(60, 40, 0.25, seed=s, integer_values=integer)
        nbr = random_topk(r.N, K, seed=s) if K else None
        cfg = TrainConfig(F=F, K=K, epochs=epochs, seed=s)
        out.update(triplets_of(r, f"s{s}_"))
        out[f"s{s}_cfg"] = np.array([F, K, epochs, s], np.int64)
        out[f"s{s}_nbr"] = nbr.entries if nbr is not None else np.zeros((r.N, 0), np.int32)
        p = train_full(r, nbr, cfg)
        out.update(params_of(p, f"s{s}_full_", True))
        for D in (2, 3):
            pd = parallel_train(r, nbr, cfg, D=D)
            out.update(params_of(pd, f"s{s}_D{D}_", True))
        t = r.triplets()
        out[f"s{s}_rmse"] = rmse(p, t, r)
        out[f"s{s}_rmse_clamp"] = rmse(p, t, r, unscale=2.0, clamp=(1.5, 4.5))
    out["n_cases"] = 4
    np.savez_compressed(os.path.join(OUT, "sgd_small.npz"), **out)


def sgd_c1(train, test, table16):
    cfg = TrainConfig(F=32, K=16, epochs=3, seed=0)
    seen = []
    p = train_full(train, table16, cfg,
                   epoch_callback=lambda t, q: seen.append((rmse(q, test, train), rmse(q, train.triplets(), train))))
    out = params_of(p, "full_", False)
    out["rmse_test"] = np.array([a for a, _ in seen])
    out["rmse_train"] = np.array([b for _, b in seen])
    out["U_sample"] = p.U[::37].copy()
    out["V_sample"] = p.V[::41].copy()
    out["W_sample"] = p.W[::29].copy()
    out["C_sample"] = p.C[::29].copy()
    cfg2 = TrainConfig(F=32, K=16, epochs=2, seed=0)
    pd = parallel_train(train, table16, cfg2, D=4)
    out.update(params_of(pd, "D4_", False))
    out["D4_rmse_test"] = rmse(pd, test, train)
    return out


def online_small():
    out = {}
    n = 0
    for seed in range(4):
        full = random_sparse(30, 22, 0.25, seed=seed, integer_values=(seed % 2 == 0))
        orig, batch, _, _ = holdback_variables(full, 3, 4, seed=seed)
        lsh = LshConfig(G=6, p=2, q=4, psi_exponent=1 + (seed % 2), seed=seed)
        cfg = TrainConfig(F=3, K=4, epochs=6, seed=seed)
        tbl, state = simlsh_topk(orig, lsh, K=4)
        params = train_full(orig, tbl, cfg)
        pre = f"o{seed}_"
        out.update(triplets_of(orig, pre))
        out[pre + "b_rows"] = batch.rows
        out[pre + "b_cols"] = batch.cols
        out[pre + "b_vals"] = batch.values
        out[pre + "b_shape"] = np.array([batch.base_M, batch.base_N, batch.new_row_count,
                                         batch.new_col_count], np.int64)
        out[pre + "lsh"] = np.array([lsh.G, lsh.p, lsh.q, lsh.psi_exponent, lsh.seed], np.int64)
        out[pre + "cfg"] = np.array([cfg.F, cfg.K, cfg.epochs, cfg.seed], np.int64)
        out[pre + "state_acc"] = state.acc
        out[pre + "table"] = tbl.entries
        out.update(params_of(params, pre + "p0_", True))
        pe, se, re_, ne = absorb_increment(params, state, orig, batch, cfg)
        out[pre + "ext_acc"] = se.acc
        out[pre + "ext_entries"] = ne.entries
        out.update(params_of(pe, pre + "ext_", True))
        n += 1
    out["n_cases"] = n
    np.savez_compressed(os.path.join(OUT, "online_small.npz"), **out)


def online_c1(train):
    lc = LshConfig(G=8, p=3, q=100, psi_exponent=2, seed=0)
    cfg = TrainConfig(F=32, K=32, epochs=4, seed=0)
    n_r, n_c = max(1, train.M // 100), max(1, train.N // 100)
    orig, batch, row_map, col_map = holdback_variables(train, n_r, n_c, seed=7)
    table0, state0 = simlsh_topk(orig, lc, K=32)
    p0 = train_full(orig, table0, cfg)
    pe, se, re_, ne = absorb_increment(p0, state0, orig, batch, cfg)
    out = {"row_map": row_map, "col_map": col_map,
           "b_rows": batch.rows, "b_cols": batch.cols, "b_vals": batch.values,
           "b_shape": np.array([batch.base_M, batch.base_N, batch.new_row_count,
                                batch.new_col_count], np.int64),
           "orig_entries": table0.entries, "ext_entries": ne.entries,
           "ext_acc_sha": sha(se.acc), "state0_acc_sha": sha(state0.acc)}
    out.update(params_of(p0, "p0_", False))
    out.update(params_of(pe, "ext_", False))
    return out


def basic():
    """train_basic (factorization.py:476-527): serial row-major, +/- biases, sorted rows."""
    from lshmf.factorization import train_basic
    out = {}
    cases = [(0, True, 4, 5, False, False), (1, False, 3, 4, True, False), (2, True, 8, 3, False, True),
             (3, False, 2, 6, True, True)]
    for s, (seed, integer, F, epochs, wb, srt) in enumerate(cases):
        r = random_sparse(50, 35, 0.3, seed=seed, integer_values=integer)
        cfg = TrainConfig(F=F, K=0, epochs=epochs, seed=seed, alpha_u=0.04, alpha_v=0.04,
                          lambda_u=0.035, lambda_v=0.035)
        p = train_basic(r, cfg, with_biases=wb, sort_rows_by_count=srt)
        out.update(triplets_of(r, f"b{s}_"))
        out[f"b{s}_cfg"] = np.array([F, epochs, seed, int(wb), int(srt)], np.int64)
        out.update(params_of(p, f"b{s}_", True))
    out["n_cases"] = len(cases)
    np.savez_compressed(os.path.join(OUT, "basic.npz"), **out)


def main():
    np.set_printoptions(precision=17)
    print("lshmf", lshmf.__version__, "numpy", np.__version__)
    if "--only-basic" in sys.argv:
        basic()
        return
    lsh_small()
    print("lsh_small done")
    sgd_small()
    print("sgd_small done")
    online_small()
    print("online_small done")
    basic()
    print("basic done")
    train, test = c1_data()
    c1 = {"train_M": train.M, "train_N": train.N,
          "train_rows": train.entry_rows.astype(np.int16), "train_cols": train.entry_cols.astype(np.int16),
          "train_vals": train.entry_values.astype(np.int8),
          "test_rows": test.rows.astype(np.int16), "test_cols": test.cols.astype(np.int16),
          "test_vals": test.values.astype(np.int8)}
    assert np.array_equal(c1["train_vals"].astype(np.float64), train.entry_values)
    lsh, table16 = lsh_c1(train)
    c1.update({"lsh_" + k: v for k, v in lsh.items()})
    print("lsh_c1 done")
    c1.update({"sgd_" + k: v for k, v in sgd_c1(train, test, table16).items()})
    print("sgd_c1 done")
    c1.update({"online_" + k: v for k, v in online_c1(train).items()})
    print("online_c1 done")
    np.savez_compressed(os.path.join(OUT, "c1.npz"), **c1)


if __name__ == "__main__":
    sys.exit(main())
