"""K above two mask words (65 <= K <= 128) and F above 256 (up to 512): the exact
(reference-order) kernels, the online
path and rmse / predict take four explicit-neighbour mask words per rating and stay
bit-identical to the oracle (itself pinned to the reference); the fp32 Hogwild mode keeps
K <= 64 and says so.  The reference accepts any K (factorization.py:75-82)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2111_11682_b200 as p
    return p


def _case(P, seed, M=220, N=150, dens=0.25):
    rng = np.random.default_rng(seed)
    mask = rng.random((M, N)) < dens
    rows, cols = np.nonzero(mask)
    vals = rng.integers(1, 6, len(rows)).astype(float)
    return P.SparseRatings(M, N, rows, cols, vals), rows, cols, vals


@pytest.mark.parametrize("F,K", [(40, 100), (128, 128), (8, 65), (300, 32), (512, 70)])
def test_exact_train_full_wide_k_vs_oracle(P, orc, F, K):
    r, rows, cols, vals = _case(P, seed=K)
    tbl, _ = P.simlsh_topk(r, P.LshConfig(G=8, p=3, q=20, psi_exponent=2, seed=1), K)
    tc = P.TrainConfig(F=F, K=K, epochs=2, seed=3)
    p = P.train_full(r, tbl, tc)
    d, mu = orc.build_csr(r.M, r.N, rows, cols, vals)
    m = orc.train_full(d, mu, tbl.entries, F, K, 2, 3, tc.rates_at, tc.regs)
    for a, b in ((p.U, m.U), (p.V, m.V), (p.W, m.W), (p.C, m.C), (p.b, m.b), (p.b_hat, m.bhat)):
        assert a.tobytes() == b.tobytes()
    # rmse (training set, a held-out style subset) and predict on the same fit
    te = r.triplets()
    mo = orc.rmse(d, m, te.rows, te.cols, te.values)
    assert P.rmse(p, te, r) == mo
    sub = P.Triplets(te.rows[::3].copy(), te.cols[::3].copy(), te.values[::3].copy())
    assert P.rmse(p, sub, r, clamp=(1.0, 5.0)) == orc.rmse(d, m, sub.rows, sub.cols, sub.values, clamp=(1.0, 5.0))


@pytest.mark.parametrize("F,K", [(32, 96), (384, 16)])
def test_parallel_train_wide_k_vs_oracle(P, orc, F, K):
    r, rows, cols, vals = _case(P, seed=5)
    tbl, _ = P.simlsh_topk(r, P.LshConfig(G=8, p=3, q=20, psi_exponent=2, seed=1), K)
    tc = P.TrainConfig(F=F, K=K, epochs=2, seed=0)
    p = P.parallel_train(r, tbl, tc, 3)
    p = p[0] if isinstance(p, tuple) else p
    d, mu = orc.build_csr(r.M, r.N, rows, cols, vals)
    m = orc.parallel_train(d, mu, tbl.entries, F, K, 2, 0, tc.rates_at, tc.regs, 3)
    for a, b in ((p.U, m.U), (p.V, m.V), (p.W, m.W), (p.C, m.C), (p.b, m.b), (p.b_hat, m.bhat)):
        assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("F,K", [(16, 80), (272, 24)])
def test_absorb_increment_wide_k_vs_oracle(P, orc, F, K):
    full, *_ = _case(P, seed=9, M=240, N=160, dens=0.2)
    lc = P.LshConfig(G=4, p=2, q=10, psi_exponent=2, seed=2)
    cfg = P.TrainConfig(F=F, K=K, epochs=2, seed=3)
    orig, batch3, _, _ = P.holdback_variables(full, 12, 6, seed=0)
    tbl, state = P.simlsh_topk(orig, lc, K)
    params = P.train_full(orig, tbl, cfg)
    acc0 = state.acc.copy()
    d0, mu0 = orc.build_csr(orig.M, orig.N, orig.entry_rows, orig.entry_cols, orig.entry_values)
    m = orc.train_full(d0, mu0, tbl.entries, F, K, 2, 3, cfg.rates_at, cfg.regs)
    batch = P.IncrementBatch(orig.M, orig.N, 12, 6, batch3.rows, batch3.cols, batch3.values)
    params, state, _, tbl = P.absorb_increment(params, state, orig, batch, cfg)
    m, acc, ent, _ = orc.absorb_increment(
        m, acc0, (lc.G, lc.p, lc.q, lc.psi_exponent, lc.seed), None,
        (orig.entry_rows, orig.entry_cols, orig.entry_values),
        (batch.base_M, batch.base_N, batch.new_row_count, batch.new_col_count, batch.rows, batch.cols,
         batch.values), F, K, 2, 3, cfg.rates_at, cfg.regs)
    assert state.acc.tobytes() == acc.tobytes()
    assert tbl.entries.tobytes() == ent.tobytes()
    for a, b in ((params.U, m.U), (params.V, m.V), (params.W, m.W), (params.C, m.C),
                 (params.b, m.b), (params.b_hat, m.bhat)):
        assert a.tobytes() == b.tobytes()


def test_hogwild_rejects_wide_k(P):
    r, *_ = _case(P, seed=1, M=120, N=90)
    tbl = P.random_topk(r.N, 70, seed=1)
    with pytest.raises(ValueError, match="K <= 64"):
        P.train_full(r, tbl, P.TrainConfig(F=32, K=70, epochs=1, seed=0), mode="hogwild")
