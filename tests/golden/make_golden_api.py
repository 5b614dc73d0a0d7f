"""Generate tests/golden/api.npz FROM THE REFERENCE ITSELF (build container only):

    cp -r /root/reference/pkg /tmp/refpkg
    NUMBA_CACHE_DIR=/tmp/numba PYTHONPATH=/tmp/refpkg/src python tests/golden/make_golden_api.py

Pins the public functions the composite fixtures reach only indirectly, each called
standalone on stored inputs: compute_baselines, split_neighbors, predict (with and
without clamp), sgd_update, objective_value, parallel_train(instrument=True), and the
online stages update_hashes_incremental, topk_for_new, extend_ratings, extend_params,
train_incremental (online.py:84-314).
"""

from __future__ import annotations

import os
import sys

import numpy as np

from lshmf.data import compute_baselines
from lshmf.datasets import random_sparse
from lshmf.factorization import (TrainConfig, objective_value, predict, sgd_update,
                                 split_neighbors, train_full)
from lshmf.lsh import LshConfig, assign_row_hashes, simlsh_topk
from lshmf.online import (extend_params, extend_ratings, holdback_variables, topk_for_new,
                          train_incremental, update_hashes_incremental)
from lshmf.parallel import parallel_train

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    out = {}
    full = random_sparse(48, 30, 0.3, seed=21)
    orig, batch, _, _ = holdback_variables(full, 4, 3, seed=5)
    for k, v in (("rows", orig.entry_rows), ("cols", orig.entry_cols), ("vals", orig.entry_values)):
        out["orig_" + k] = v
    out["orig_shape"] = np.array([orig.M, orig.N], np.int64)
    out["b_rows"], out["b_cols"], out["b_vals"] = batch.rows, batch.cols, batch.values
    out["b_shape"] = np.array([batch.base_M, batch.base_N, batch.new_row_count, batch.new_col_count],
                              np.int64)
    lc = LshConfig(G=6, p=2, q=5, psi_exponent=2, seed=3)
    cfg = TrainConfig(F=4, K=5, epochs=3, seed=2)
    tbl, state = simlsh_topk(orig, lc, K=5)
    out["table"] = tbl.entries
    st = compute_baselines(orig)
    out["base_mu"], out["base_b"], out["base_bhat"] = np.float64(st.mu), st.b, st.b_hat
    p = train_full(orig, tbl, cfg)
    for k in ("b", "b_hat", "U", "V", "W", "C"):
        out["p_" + k] = getattr(p, k)
    out["p_mu"] = np.float64(p.mu)
    pairs = np.array([[i, j] for i in range(0, orig.M, 5) for j in range(0, orig.N, 4)], np.int64)
    out["pairs"] = pairs
    out["pred"] = np.array([predict(int(i), int(j), p, orig) for i, j in pairs])
    out["pred_clamped"] = np.array([predict(int(i), int(j), p, orig, clamp=(2.0, 4.0)) for i, j in pairs])
    expl, impl = [], []
    for i, j in pairs:
        s = split_neighbors(int(i), int(j), tbl, orig)
        m = np.zeros(5, np.int8)
        m[s.explicit] = 1
        expl.append(m)
    out["split_explicit"] = np.array(expl)
    regs = cfg.regs if hasattr(cfg, "regs") else (cfg.lambda_b, cfg.lambda_b_hat, cfg.lambda_u,
                                                   cfg.lambda_v, cfg.lambda_w, cfg.lambda_c)
    out["objective"] = np.float64(objective_value(p, orig, tuple(regs)))
    # one sgd_update at the first rated pair
    i0, j0 = int(orig.entry_rows[7]), int(orig.entry_cols[7])
    q = p.copy()
    rates = (0.03, 0.031, 0.032, 0.033, 0.004, 0.005)
    out["sgd_err"] = np.float64(sgd_update(i0, j0, q, rates, tuple(regs), orig))
    out["sgd_ij"] = np.array([i0, j0], np.int64)
    out["sgd_rates"] = np.array(rates)
    for k in ("b", "b_hat", "U", "V", "W", "C"):
        out["sgd_" + k] = getattr(q, k)
    # instrumented DSGD
    pp, rep = parallel_train(orig, tbl, cfg, 3, instrument=True)
    out["instr"] = np.array([rep.stages_checked, rep.disjoint_violations, rep.epochs_checked,
                             rep.coverage_violations], np.int64)
    out["par_U"] = pp.U
    # online stages, standalone
    hashes = assign_row_hashes(batch.M_hat, lc)
    se = update_hashes_incremental(state, batch, hashes)
    out["inc_acc"] = se.acc
    ne = topk_for_new(se, tbl, 5, lc.seed)
    out["new_entries"] = ne.entries
    re_ = extend_ratings(orig, batch)
    out["ext_rows"], out["ext_cols"], out["ext_vals"] = re_.entry_rows, re_.entry_cols, re_.entry_values
    pe = extend_params(p, batch, ne, cfg)
    for k in ("b", "b_hat", "U", "V", "W", "C"):
        out["extp_" + k] = getattr(pe, k).copy()   # train_incremental trains pe in place
    pt = train_incremental(pe, batch, ne, re_, cfg)
    out["inc_in_place"] = np.int64(pt is pe)
    for k in ("b", "b_hat", "U", "V", "W", "C"):
        out["inc_" + k] = getattr(pt, k)
    # holdout split (data.py:312-346) and value transform (data.py:150-163)
    from lshmf.data import split_holdout, transform_ratings, Triplets
    big = random_sparse(400, 300, 0.08, seed=9)
    for k, v in (("rows", big.entry_rows), ("cols", big.entry_cols), ("vals", big.entry_values)):
        out["split_in_" + k] = v
    for frac, sd in ((0.1, 0), (0.3, 4), (0.0, 1)):
        tr_, te_ = split_holdout(big, frac, sd)
        out[f"split_{int(frac * 10)}_{sd}_test_rows"] = te_.rows
        out[f"split_{int(frac * 10)}_{sd}_test_cols"] = te_.cols
        out[f"split_{int(frac * 10)}_{sd}_train_rows"] = tr_.entry_rows
    tt = transform_ratings(Triplets(np.array([0, 1, 2]), np.array([0, 1, 1]), np.array([0.0, 50.0, 100.0])),
                           zero_floor=0.5, scale=20.0)
    out["transform_vals"] = tt.values
    np.savez_compressed(os.path.join(OUT, "api.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    sys.exit(main())
