"""Per-stage cost of the public absorb_increment at C4 (online.py:317-332 stages, each timed
with a device sync on both sides), batches 2..6 of the bench's C4 split.

  python tools/absorb_breakdown.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_11682_b200 as P  # noqa: E402
from paper_2111_11682_b200 import _native as nat, online, synth  # noqa: E402

RATES = dict(alpha_b=0.02, alpha_b_hat=0.02, alpha_u=0.02, alpha_v=0.02, alpha_w=0.001, alpha_c=0.001,
             lambda_b=0.01, lambda_b_hat=0.01, lambda_u=0.01, lambda_v=0.01, lambda_w=0.05, lambda_c=0.05,
             beta=0.3)


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def main():
    t = torch
    M, N, nnz_t, F, K, e = synth.SHAPES["c3"]
    d = synth.random_sparse_device(M, N, nnz_t, seed=0).dev
    col = t.repeat_interleave(t.arange(N, device="cuda"), d.col_ptr[1:] - d.col_ptr[:-1]).to(t.int32)
    row = d.col_rows
    M0, N0 = int(M * 0.9), int(N * 0.9)
    dM, dN = (M - M0) // 10, (N - N0) // 10
    br = t.where(row >= M0, (row - M0) // dM, t.full_like(row, -1)).clamp(max=9)
    bc = t.where(col >= N0, (col - N0) // dN, t.full_like(col, -1)).clamp(max=9)
    bidx = t.maximum(br, bc)
    init = bidx < 0
    base = P.DeviceSparseRatings(M0, N0, row[init], col[init], d.col_vals[init])
    ratings = P.SparseRatings._from_device(base.device(), (row[init].contiguous(), col[init].contiguous(),
                                                           d.col_vals[init].contiguous()))
    ratings.device().exact_baselines = True
    lc = P.LshConfig(psi_exponent=e)
    tbl, state = P.simlsh_topk(ratings, lc, K)
    cfg = P.TrainConfig(F=F, K=K, epochs=1, seed=0, **RATES)
    params = P.train_full(ratings, tbl, P.TrainConfig(F=F, K=K, epochs=3, seed=0, **RATES), mode="hogwild")
    Mb, Nb = M0, N0
    rows_out = []
    for b in range(6):
        sel = bidx == b
        nr_ = dM
        nc_ = dN
        batch = P.IncrementBatch(Mb, Nb, nr_, nc_, nat.to_host(row[sel]), nat.to_host(col[sel]),
                                 nat.to_host(d.col_vals[sel]))
        st = {}
        hashes, st["row_hashes"] = timed(lambda: P.assign_row_hashes(batch.M_hat, state.config))
        state_ext, st["update_hashes"] = timed(lambda: online.update_hashes_incremental(state, batch, hashes))
        nbr_ext, st["topk_for_new"] = timed(lambda: online.topk_for_new(state_ext, params.neighbors, params.K,
                                                                        state.config.seed))
        ratings_ext, st["extend_ratings"] = timed(lambda: online.extend_ratings(ratings, batch))
        pe, st["extend_params"] = timed(lambda: online.extend_params(params, batch, nbr_ext, cfg))
        pt, st["train_incremental"] = timed(lambda: online.train_incremental(pe, batch, nbr_ext, ratings_ext, cfg))
        st["total"] = sum(st.values())
        if b >= 1:
            rows_out.append(st)
        params, state, ratings = pt, state_ext, ratings_ext
        Mb, Nb = Mb + nr_, Nb + nc_
    med = {k: float(np.median([r[k] for r in rows_out])) for k in rows_out[0]}
    print(json.dumps({"config": "C4 public absorb_increment stages (median of batches 2-6, s)", **med}))


if __name__ == "__main__":
    main()
