"""GPU parity at the configs' full scale (BASELINE.json configs C3, C4, C5), against the
CPU oracle (itself pinned to reference-written fixtures, tests/test_oracle.py), plus the
Hogwild mode against the reference's own 20-epoch C1 learning curve.

  C3  the whole simLSH state (341 MB of fp64 accumulators, signatures) and J^K of the
      100.48M-rating Netflix-shape matrix; one exact parallel_train(D=16) epoch, every
      parameter byte
  C4  the first 1 % increment absorbed into the 90 % fit, through the public
      absorb_increment AND the resident OnlineSession: hash state, J^K, every parameter
  C5  Yahoo shape (K=64, psi exponent 4): accumulators, signatures and group keys of a
      2,000-column range, and J^K of those columns from the full key matrix; Hogwild vs
      exact held-out RMSE on a 1/16 row sample

Each test runs the oracle on the box's host cores (seconds to about a minute each)."""

import os

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

RATES = dict(alpha_b=0.02, alpha_b_hat=0.02, alpha_u=0.02, alpha_v=0.02, alpha_w=0.001, alpha_c=0.001,
             lambda_b=0.01, lambda_b_hat=0.01, lambda_u=0.01, lambda_v=0.01, lambda_w=0.05, lambda_c=0.05,
             beta=0.3)
TOL_RMSE = 0.005


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2111_11682_b200 as p
    return p


@pytest.fixture(scope="module")
def orc():
    from oracle import oracle
    return oracle


@pytest.fixture(scope="module")
def c3(P):
    """The C3 matrix as a device-built SparseRatings + its host CSC for the oracle."""
    from paper_2111_11682_b200 import _native as nat, synth
    M, N, nnz, F, K, e = synth.SHAPES["c3"]
    r = synth.random_sparse_ratings(M, N, nnz, seed=0)
    d = r.device()
    host = tuple(nat.to_host(x) for x in (d.col_ptr, d.col_rows, d.col_vals))
    return r, host


def test_c1_hogwild_tracks_reference_20_epoch_curve(P):
    """Exact mode reproduces the reference's 20-epoch curve bit for bit; the Hogwild
    mode's test RMSE stays within 0.005 of it after the same epochs (north_star)."""
    z = load_golden("c1.npz")
    ref = load_golden("c1_ref20.npz")
    tr = P.SparseRatings(int(z["train_M"]), int(z["train_N"]), z["train_rows"].astype(np.int32),
                         z["train_cols"].astype(np.int32), z["train_vals"].astype(np.float64))
    te = P.Triplets(z["test_rows"].astype(np.int32), z["test_cols"].astype(np.int32),
                    z["test_vals"].astype(np.float64))
    nbr = P.NeighborTable(tr.N, 16, ref["entries16"])
    cfg = P.TrainConfig(F=32, K=16, epochs=20, seed=0)
    ex, hw = [], []
    P.train_full(tr, nbr, cfg, epoch_callback=lambda t, p: ex.append((P.rmse(p, te, tr), P.rmse(p, tr.triplets(), tr))))
    P.train_full(tr, nbr, cfg, mode="hogwild", epoch_callback=lambda t, p: hw.append(P.rmse(p, te, tr)))
    np.testing.assert_array_equal([a for a, _ in ex], ref["F32_rmse_test"])
    np.testing.assert_array_equal([b for _, b in ex], ref["F32_rmse_train"])
    gap = np.abs(np.array(hw) - ref["F32_rmse_test"])
    assert gap[-1] <= TOL_RMSE, (hw[-1], ref["F32_rmse_test"][-1])
    assert gap[5:].max() <= TOL_RMSE, gap


def test_c3_simlsh_state_and_topk_bit_exact(P, orc, c3):
    r, (cp, cr, cv) = c3
    from paper_2111_11682_b200 import synth
    M, N, _, _, K, e = synth.SHAPES["c3"]
    tbl, state = P.simlsh_topk(r, P.LshConfig(psi_exponent=e, seed=0), K)
    ref = orc.simlsh_topk(cp, cr, cv, M, 8, 3, 100, e, 0, K)
    assert state.acc.tobytes() == ref.acc.tobytes()
    assert state.sig.tobytes() == ref.sig.tobytes()
    assert tbl.entries.tobytes() == ref.entries.tobytes()


def test_c3_exact_dsgd_epoch_bit_exact(P, orc, c3):
    r, (cp, cr, cv) = c3
    from paper_2111_11682_b200 import _native as nat, lsh, synth
    M, N, _, F, K, e = synth.SHAPES["c3"]
    ent, _, _ = lsh.simlsh_topk_device(r.device(), P.LshConfig(psi_exponent=e), K)
    nbr = P.NeighborTable(N, K, nat.to_host(ent)[:N * K].reshape(N, K))
    cfg = P.TrainConfig(F=F, K=K, epochs=1, seed=0, **RATES)
    p = P.parallel_train(r, nbr, cfg, 16)
    csr, mu = orc.build_csr(M, N, cr, np.repeat(np.arange(N, dtype=np.int32), np.diff(cp)), cv)
    m = orc.parallel_train(csr, mu, nbr.entries, F, K, 1, 0, cfg.rates_at, cfg.regs, 16)
    for a, b in ((p.b, m.b), (p.b_hat, m.bhat), (p.U, m.U), (p.V, m.V), (p.W, m.W), (p.C, m.C)):
        assert a.tobytes() == b.tobytes()


def test_c4_first_increment_public_api_and_session(P, orc):
    """The first C4 increment (1 % new rows + 1 % new columns into the 90 % fit) through
    absorb_increment and through OnlineSession, both against the oracle's absorb."""
    import torch
    from paper_2111_11682_b200 import _native as nat, synth
    from paper_2111_11682_b200.online_device import OnlineSession
    M, N, nnz_t, F, K, e = synth.SHAPES["c3"]
    d = synth.random_sparse_device(M, N, nnz_t, seed=0).dev
    col = torch.repeat_interleave(torch.arange(N, device="cuda"), d.col_ptr[1:] - d.col_ptr[:-1]).to(torch.int32)
    row = d.col_rows
    M0, N0 = int(M * 0.9), int(N * 0.9)
    dM, dN = (M - M0) // 10, (N - N0) // 10
    first = ((row >= M0) & (row < M0 + dM) & (col < N0 + dN)) | ((col >= N0) & (col < N0 + dN) & (row < M0 + dM))
    init = (row < M0) & (col < N0)
    trip = tuple(x[init].contiguous() for x in (row, col, d.col_vals))
    base = P.DeviceSparseRatings(M0, N0, *trip)
    ratings = P.SparseRatings._from_device(base.device(), trip)
    ratings.device().exact_baselines = True
    lc = P.LshConfig(psi_exponent=e)
    tbl, state = P.simlsh_topk(ratings, lc, K)
    cfg = P.TrainConfig(F=F, K=K, epochs=1, seed=0, **RATES)
    params = P.train_full(ratings, tbl, P.TrainConfig(F=F, K=K, epochs=2, seed=0, **RATES), mode="hogwild")
    m0 = orc.Model(params.mu, params.b.copy(), params.b_hat.copy(), params.U.copy(), params.V.copy(),
                   params.W.copy(), params.C.copy(), tbl.entries.copy())
    acc0 = np.array(state.acc, copy=True)
    batch = P.IncrementBatch(M0, N0, dM, dN, nat.to_host(row[first]), nat.to_host(col[first]),
                             nat.to_host(d.col_vals[first]))
    sess = OnlineSession(ratings.device(), state, tbl.device_entries(), K, params, cfg)
    sess.absorb(batch)
    ps = sess.to_params()
    pe, se, re_, ne = P.absorb_increment(params, state, ratings, batch, cfg)
    me, acc_ext, ent_ext, _ = orc.absorb_increment(
        m0, acc0, (lc.G, lc.p, lc.q, lc.psi_exponent, lc.seed), None, tuple(nat.to_host(x) for x in trip),
        (M0, N0, dM, dN, batch.rows, batch.cols, batch.values), F, K, cfg.epochs, cfg.seed, cfg.rates_at, cfg.regs)
    assert se.acc.tobytes() == acc_ext.tobytes()
    assert sess.state.acc.tobytes() == acc_ext.tobytes()
    assert ne.entries.tobytes() == ent_ext.tobytes() == ps.neighbors.entries.tobytes()
    for n, n2 in (("b", "b"), ("b_hat", "bhat"), ("U", "U"), ("V", "V"), ("W", "W"), ("C", "C")):
        ref = getattr(me, n2).tobytes()
        assert getattr(pe, n).tobytes() == ref, ("absorb_increment", n)
        assert getattr(ps, n).tobytes() == ref, ("OnlineSession", n)
    assert re_.nnz == ratings.nnz + len(batch.rows)


@pytest.fixture(scope="module")
def c5_cols(P):
    """Columns [c0, c0 + 2000) of the C5 matrix (full columns), plus the full key matrix."""
    from paper_2111_11682_b200 import synth
    M, N, nnz, F, K, e = synth.SHAPES["c5"]
    c0, n = 312_000, 2000
    rows, cols, vals, cp = synth.hashed_shard(M, N, nnz, seed=0, cols=(c0, c0 + n))
    dev = synth.device_ratings_from_sorted(M, N, rows, cols, vals, baselines=False)
    return dev, (c0, n)


def test_c5_column_range_hash_state_bit_exact(P, orc, c5_cols):
    """C5 (K=64, psi exponent 4): accumulators / signatures / group keys of 2,000 whole
    columns against orc.accumulate_all on those columns."""
    from paper_2111_11682_b200 import _native as nat, synth
    from paper_2111_11682_b200.dsgd import _Offset
    from paper_2111_11682_b200.lsh import _accumulate, assign_row_hashes
    dev, (c0, n) = c5_cols
    M, N, _, _, K, e = synth.SHAPES["c5"]
    c = P.LshConfig(psi_exponent=e, seed=0)
    W = c.q * c.p * c.G
    acc = nat.empty((n * W,), "float64")
    sig = nat.empty((n * W,), "uint8")
    keys = nat.zeros((c.q * N,), "uint64")
    _accumulate(dev, assign_row_hashes(M, c).table(), c, _Offset(acc.data_ptr() - c0 * W * 8),
                _Offset(sig.data_ptr() - c0 * W), keys, c0, n)
    cp = nat.to_host(dev.col_ptr)
    lo, hi = int(cp[c0]), int(cp[c0 + n])
    sub_ptr = (cp[c0:c0 + n + 1] - lo).astype(np.int64)
    bits = orc.assign_bits(0, c.q, c.p, M, c.G)
    ref = orc.accumulate_all(sub_ptr, nat.to_host(dev.col_rows)[lo:hi].copy(), nat.to_host(dev.col_vals)[lo:hi].copy(),
                             bits, e)
    del bits
    assert nat.to_host(acc).tobytes() == ref.tobytes()
    ref_sig = orc.threshold(ref)
    assert nat.to_host(sig).tobytes() == ref_sig.tobytes()
    gk = nat.to_host(keys).reshape(c.q, N)[:, c0:c0 + n]
    assert gk.tobytes() == np.ascontiguousarray(orc.group_keys(ref_sig)).tobytes()


def test_c5_topk_of_column_range_bit_exact(P, orc):
    """J^K of 2,000 C5 columns from the full (q, N) key matrix of the whole C5 build,
    against the oracle's _topk_from_group_keys for the same target range."""
    from paper_2111_11682_b200 import _native as nat, lsh, synth
    M, N, nnz, F, K, e = synth.SHAPES["c5"]
    d = synth.random_sparse_device(M, N, nnz, seed=0).dev
    c = P.LshConfig(psi_exponent=e, seed=0)
    ent, state, _ = lsh.simlsh_topk_device(d, c, K)
    keys = nat.to_host(state.device_keys()).view(np.uint64).reshape(c.q, N)
    c0, n = 312_000, 2000
    ref, _ = orc.topk_from_group_keys(np.ascontiguousarray(keys), K, c.seed, c0, n)
    got = nat.to_host(ent)[:N * K].reshape(N, K)[c0:c0 + n]
    assert got.tobytes() == np.ascontiguousarray(ref).tobytes()


def test_c5_row_sample_hogwild_vs_exact_rmse(P):
    """A 1/16 row sample of C5 (~16M ratings, 625K columns, K=64): held-out RMSE of the
    Hogwild mode within 0.005 of the exact (reference-order) fit after the same epochs."""
    import torch
    from paper_2111_11682_b200 import _native as nat, synth
    M, N, nnz, F, K, e = synth.SHAPES["c5"]
    Ms = M // 16
    rows, cols, vals, _ = synth.hashed_shard(M, N, nnz, seed=0, rows=(0, Ms))
    test = (rows * 7919 + cols * 104729) % 10 == 0            # deterministic 10 % holdout
    keep = ~test
    tr_dev = synth.device_ratings_from_sorted(Ms, N, rows[keep], cols[keep], vals[keep])
    r = P.SparseRatings._from_device(tr_dev, (rows[keep], cols[keep], vals[keep]))
    te = P.Triplets(nat.to_host(rows[test]), nat.to_host(cols[test]), nat.to_host(vals[test]))
    tbl, _ = P.simlsh_topk(r, P.LshConfig(psi_exponent=e), K)
    cfg = P.TrainConfig(F=F, K=K, epochs=3, seed=0, **RATES)
    ex = P.rmse(P.train_full(r, tbl, cfg), te, r)
    hw = P.rmse(P.train_full(r, tbl, cfg, mode="hogwild"), te, r)
    print(f"C5 row sample: {r.nnz} ratings, held-out RMSE exact {ex:.5f} hogwild {hw:.5f}")
    assert np.isfinite(ex) and abs(hw - ex) <= TOL_RMSE, (hw, ex)
