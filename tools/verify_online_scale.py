"""Full-scale online parity evidence (C4 setting): the device OnlineSession absorbing the
first 1 % increment of the Netflix-shape matrix against the oracle's absorb_increment
(pinned to the reference's), hash state, neighbour table and every parameter byte.

  python tools/verify_online_scale.py
"""
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as orc  # noqa: E402
from paper_2111_11682_b200 import _native as nat, lsh, synth  # noqa: E402
from paper_2111_11682_b200.data import DeviceSparseRatings  # noqa: E402
from paper_2111_11682_b200.factorization import TrainConfig  # noqa: E402
from paper_2111_11682_b200.hogwild import HogwildTrainer  # noqa: E402
from paper_2111_11682_b200.online import IncrementBatch  # noqa: E402
from paper_2111_11682_b200.online_device import OnlineSession  # noqa: E402
from paper_2111_11682_b200.similarity import NeighborTable  # noqa: E402

RATES = dict(alpha_b=0.02, alpha_b_hat=0.02, alpha_u=0.02, alpha_v=0.02, alpha_w=0.001, alpha_c=0.001,
             lambda_b=0.01, lambda_b_hat=0.01, lambda_u=0.01, lambda_v=0.01, lambda_w=0.05, lambda_c=0.05,
             beta=0.3)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main():
    M, N, nnz_t, F, K, e = synth.SHAPES["c3"]
    dm = synth.random_sparse_device(M, N, nnz_t, seed=0)
    d = dm.dev
    col = torch.repeat_interleave(torch.arange(N, device="cuda"), d.col_ptr[1:] - d.col_ptr[:-1]).to(torch.int32)
    row = d.col_rows
    M0, N0 = int(M * 0.9), int(N * 0.9)
    dM, dN = (M - M0) // 10, (N - N0) // 10
    br = torch.where(row >= M0, (row - M0) // dM, torch.full_like(row, -1)).clamp(max=9)
    bc = torch.where(col >= N0, (col - N0) // dN, torch.full_like(col, -1)).clamp(max=9)
    bidx = torch.maximum(br, bc)
    init = bidx < 0
    orig_trip = (nat.to_host(row[init]), nat.to_host(col[init]), nat.to_host(d.col_vals[init]))
    base = DeviceSparseRatings(M0, N0, row[init], col[init], d.col_vals[init])
    lc = lsh.LshConfig(psi_exponent=e)
    ent, state, _ = lsh.simlsh_topk_device(base.device(), lc, K)
    nbr = NeighborTable(N0, K, nat.to_host(ent)[:N0 * K].reshape(N0, K))
    cfg = TrainConfig(F=F, K=K, epochs=1, seed=0, **RATES)
    tr = HogwildTrainer(base, nbr, cfg)
    for t in range(2):
        tr.epoch(t)
    params = tr.to_params()
    acc0 = np.array(state.acc, copy=True)
    m0 = orc.Model(params.mu, params.b.copy(), params.b_hat.copy(), params.U.copy(), params.V.copy(),
                   params.W.copy(), params.C.copy(), nbr.entries.copy())
    sess = OnlineSession(base.device(), state, ent, K, params, cfg)
    sel = bidx == 0
    batch = IncrementBatch(M0, N0, dM, dN, nat.to_host(row[sel]), nat.to_host(col[sel]), nat.to_host(d.col_vals[sel]))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tm = sess.absorb(batch)
    gpu_s = time.perf_counter() - t0
    pe = sess.to_params()
    t0 = time.perf_counter()
    me, acc_ext, entries_ext, _ = orc.absorb_increment(
        m0, acc0, (lc.G, lc.p, lc.q, lc.psi_exponent, lc.seed), None, orig_trip,
        (M0, N0, dM, dN, batch.rows, batch.cols, batch.values), F, K, cfg.epochs, cfg.seed, cfg.rates_at,
        cfg.regs)
    cpu_s = time.perf_counter() - t0
    eq = {"acc": sess.state.acc.tobytes() == acc_ext.tobytes(),
          "entries": pe.neighbors.entries.tobytes() == entries_ext.tobytes()}
    for k, k2 in (("b", "b"), ("b_hat", "bhat"), ("U", "U"), ("V", "V"), ("W", "W"), ("C", "C")):
        eq[k] = getattr(pe, k).tobytes() == getattr(me, k2).tobytes()
    print(json.dumps({"case": "C4 batch 0 (1 % new rows + 1 % new columns of the C3 shape)",
                      "batch_ratings": int(len(batch.rows)), "gpu_absorb_s": gpu_s, "gpu_stages": tm,
                      "oracle_absorb_s": cpu_s, "oracle_threads": orc.n_threads(), "U_sha": sha(pe.U),
                      "equal": eq, "all_equal": all(eq.values())}), flush=True)


if __name__ == "__main__":
    main()
