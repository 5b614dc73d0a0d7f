"""GPU: the drop-in API on device-resident objects -- live device-backed ModelParams in
epoch callbacks, rmse/predict on the resident model, and the online step
(extend_ratings / extend_params / train_incremental / absorb_increment) built in HBM --
all bit-identical to the oracle / the reference-written fixtures."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


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


def _case(P, seed=0, M=120, N=60, dens=0.15, integer=True):
    rng = np.random.default_rng(seed)
    rows, cols = np.nonzero(rng.random((M, N)) < dens)
    vals = (rng.integers(1, 6, len(rows)).astype(np.float64) if integer
            else np.round(rng.random(len(rows)) * 5, 3))
    return P.SparseRatings(M, N, rows, cols, vals), rows, cols, vals


def test_callback_gets_live_device_params(P, orc):
    """The callback's rmse runs on the resident model; the fit equals the oracle's."""
    r, rows, cols, vals = _case(P)
    tbl, _ = P.simlsh_topk(r, P.LshConfig(G=4, p=2, q=8, seed=3), 6)
    cfg = P.TrainConfig(F=8, K=6, epochs=4, seed=1)
    seen, ids = [], []

    def cb(t, p):
        ids.append(id(p))
        seen.append(P.rmse(p, r.triplets(), r))
        assert all(s == "D" for s in p._state.values())     # nothing copied to the host

    p = P.train_full(r, tbl, cfg, epoch_callback=cb)
    assert len(set(ids)) == 1 and ids[0] == id(p)            # the live object, as in the reference
    d, mu = orc.build_csr(r.M, r.N, rows, cols, vals)
    ref_rmse = []
    m = orc.train_full(d, mu, tbl.entries, 8, 6, 4, 1, cfg.rates_at, cfg.regs,
                       callback=lambda t, mm: ref_rmse.append(
                           orc.rmse(d, mm, r.entry_rows, r.entry_cols, r.entry_values)))
    assert p.U.tobytes() == m.U.tobytes() and p.W.tobytes() == m.W.tobytes()
    assert np.array_equal(np.array(seen), np.array(ref_rmse))


def test_callback_edits_reach_the_device(P, orc):
    """Edits the callback makes to the host arrays are trained on (reference: live arrays)."""
    r, rows, cols, vals = _case(P, seed=2)
    tbl, _ = P.simlsh_topk(r, P.LshConfig(G=4, p=2, q=8, seed=3), 5)
    cfg = P.TrainConfig(F=8, K=5, epochs=3, seed=4)

    def edit(U, W):
        U[3] *= 2.0
        W[:, 0] = 0.25

    def cb(t, p):
        if t == 0:
            edit(p.U, p.W)

    p = P.train_full(r, tbl, cfg, epoch_callback=cb)
    d, mu = orc.build_csr(r.M, r.N, rows, cols, vals)
    m = orc.train_full(d, mu, tbl.entries, 8, 5, 3, 4, cfg.rates_at, cfg.regs,
                       callback=lambda t, mm: edit(mm.U, mm.W) if t == 0 else None)
    for a, b in ((p.U, m.U), (p.V, m.V), (p.W, m.W), (p.C, m.C), (p.b, m.b), (p.b_hat, m.bhat)):
        assert a.tobytes() == b.tobytes()


def test_hogwild_callback_edit_applied(P):
    r, *_ = _case(P, seed=5, M=300, N=80)
    tbl, _ = P.simlsh_topk(r, P.LshConfig(G=4, p=2, q=8, seed=3), 4)
    cfg = P.TrainConfig(F=16, K=4, epochs=2, seed=0)
    seen = []

    def cb(t, p):
        seen.append(P.rmse(p, r.triplets(), r))
        if t == 0:
            p.U[:] = 0.0            # an edit the next epoch must start from
            p.V[:] = 0.0
    p = P.train_full(r, tbl, cfg, epoch_callback=cb, mode="hogwild")
    # with u = v = 0 every u/v gradient is 0: they stay exactly 0 through epoch 1
    assert not p.U.any() and not p.V.any()
    assert np.isfinite(seen).all()


def test_rmse_predict_reuse_resident_model(P, orc):
    r, rows, cols, vals = _case(P, seed=6)
    tbl, _ = P.simlsh_topk(r, P.LshConfig(G=4, p=2, q=8, seed=3), 6)
    cfg = P.TrainConfig(F=8, K=6, epochs=2, seed=1)
    p = P.train_full(r, tbl, cfg)
    dev = p._dev
    x = P.rmse(p, r.triplets(), r)
    y = P.predict(3, int(r.entry_cols[r.entry_rows == 3][0]), p, r)
    assert p._dev is dev and all(s == "D" for s in p._state.values())
    d, mu = orc.build_csr(r.M, r.N, rows, cols, vals)
    m = orc.train_full(d, mu, tbl.entries, 8, 6, 2, 1, cfg.rates_at, cfg.regs)
    assert x == orc.rmse(d, m, r.entry_rows, r.entry_cols, r.entry_values)
    # a host edit after the fit is seen by the next evaluation
    p.U[:] = 0.0
    m.U[:] = 0.0
    assert P.rmse(p, r.triplets(), r) == orc.rmse(d, m, r.entry_rows, r.entry_cols, r.entry_values)
    assert np.isfinite(y)


@pytest.mark.parametrize("integer", [True, False])
def test_extend_ratings_on_device_equals_rebuild(P, integer):
    """Device append == the reference's full rebuild: entries, CSR, CSC and baselines."""
    full, *_ = _case(P, seed=8, M=90, N=50, dens=0.3, integer=integer)
    orig, batch, _, _ = P.holdback_variables(full, 7, 5, seed=1)
    ext = P.extend_ratings(orig, batch)
    ref = P.SparseRatings(batch.M_hat, batch.N_hat, np.concatenate([orig.entry_rows, batch.rows]),
                          np.concatenate([orig.entry_cols, batch.cols]),
                          np.concatenate([orig.entry_values, batch.values]))
    for name in ("entry_rows", "entry_cols", "entry_values", "row_ptr", "row_cols", "row_vals",
                 "col_ptr", "col_rows", "col_vals"):
        assert getattr(ext, name).tobytes() == getattr(ref, name).tobytes(), name
    a, b = ext.baselines(), ref.baselines()
    assert a.mu == b.mu and a.b.tobytes() == b.b.tobytes() and a.b_hat.tobytes() == b.b_hat.tobytes()
    d = ext.device()
    from paper_2111_11682_b200 import _native as nat
    assert nat.to_host(d.base_b)[:ext.M].tobytes() == b.b.tobytes()
    assert nat.to_host(d.csc2csr)[:ext.nnz].tobytes() == nat.to_host(ref.device().csc2csr)[:ext.nnz].tobytes()


def test_absorb_increment_chain_matches_oracle(P, orc):
    """Three increments through the public API, each bit-identical to the oracle."""
    full, *_ = _case(P, seed=11, M=160, N=70, dens=0.2)
    lc = P.LshConfig(G=4, p=2, q=10, psi_exponent=2, seed=2)
    cfg = P.TrainConfig(F=8, K=5, epochs=2, seed=3)
    orig, b3, _, _ = P.holdback_variables(full, 12, 6, seed=0)
    tbl, state = P.simlsh_topk(orig, lc, 5)
    params = P.train_full(orig, tbl, cfg)
    ratings = orig
    # split the held-back variables into three successive batches
    M0, N0 = orig.M, orig.N
    m_, c_ = [M0, M0 + 4, M0 + 8, M0 + 12], [N0, N0 + 2, N0 + 4, N0 + 6]
    d0, mu0 = orc.build_csr(orig.M, orig.N, orig.entry_rows, orig.entry_cols, orig.entry_values)
    m = orc.train_full(d0, mu0, tbl.entries, 8, 5, 2, 3, cfg.rates_at, cfg.regs)
    acc = state.acc.copy()
    trip = (orig.entry_rows, orig.entry_cols, orig.entry_values)
    for k in range(3):
        sel = ((b3.rows < m_[k + 1]) & (b3.cols < c_[k + 1])) & ~((b3.rows < m_[k]) & (b3.cols < c_[k]))
        batch = P.IncrementBatch(m_[k], c_[k], m_[k + 1] - m_[k], c_[k + 1] - c_[k],
                                 b3.rows[sel], b3.cols[sel], b3.values[sel])
        params, state, ratings, tbl = P.absorb_increment(params, state, ratings, batch, cfg)
        m, acc, ent, _ = orc.absorb_increment(
            m, acc, (lc.G, lc.p, lc.q, lc.psi_exponent, lc.seed), None, trip,
            (batch.base_M, batch.base_N, batch.new_row_count, batch.new_col_count, batch.rows,
             batch.cols, batch.values), 8, 5, 2, 3, cfg.rates_at, cfg.regs)
        trip = tuple(np.concatenate([a, b]) for a, b in zip(trip, (batch.rows, batch.cols, batch.values)))
        assert state.acc.tobytes() == acc.tobytes(), k
        assert tbl.entries.tobytes() == ent.tobytes(), k
        for a, b in ((params.U, m.U), (params.V, m.V), (params.W, m.W), (params.C, m.C),
                     (params.b, m.b), (params.b_hat, m.bhat)):
            assert a.tobytes() == b.tobytes(), k


@pytest.mark.parametrize("seed", [0, 7, (3, 0x0B1)])
def test_pcg64_device_draws_equal_numpy(P, seed):
    """init_params' U then V (and extend_params' stream) drawn in HBM == numpy's PCG64."""
    from paper_2111_11682_b200 import _native as nat
    from paper_2111_11682_b200.factorization import pcg64_uniform_device
    n, skip, scale = 200_003, 12_345, 1.0 / np.sqrt(128)
    ref = np.random.default_rng(seed).uniform(0.0, scale, skip + n)[skip:]
    assert nat.to_host(pcg64_uniform_device(seed, skip, n, scale))[:n].tobytes() == ref.tobytes()
    assert (nat.to_host(pcg64_uniform_device(seed, skip, n, scale, "float32"))[:n].tobytes()
            == ref.astype(np.float32).tobytes())


def test_init_params_equals_reference_draws(P):
    r, *_ = _case(P, seed=3, M=700, N=300)
    tbl, _ = P.simlsh_topk(r, P.LshConfig(G=4, p=2, q=8, seed=3), 6)
    cfg = P.TrainConfig(F=24, K=6, epochs=0, seed=9)
    p = P.init_params(r.M, r.N, 24, 6, tbl, r.baselines(), cfg)
    rng = np.random.default_rng(9)
    sc = 1.0 / np.sqrt(24)
    assert p.U.tobytes() == rng.uniform(0.0, sc, (r.M, 24)).tobytes()
    assert p.V.tobytes() == rng.uniform(0.0, sc, (r.N, 24)).tobytes()
    st = r.baselines()
    assert p.b.tobytes() == st.b.tobytes() and p.b_hat.tobytes() == st.b_hat.tobytes()
    assert not p.W.any() and p.W.shape == (r.N, 6)
    # the Hogwild trainer's fp32 model holds the same draws rounded to float
    from paper_2111_11682_b200.hogwild import HogwildTrainer
    tr = HogwildTrainer(r, tbl, P.TrainConfig(F=32, K=6, epochs=1, seed=9))
    rng = np.random.default_rng(9)
    sc = 1.0 / np.sqrt(32)
    U = rng.uniform(0.0, sc, (r.M, 32))
    assert tr.model.download("U").astype(np.float32).tobytes() == U.astype(np.float32).tobytes()


@pytest.mark.parametrize("K", [0, 7, 40])
def test_train_set_rmse_path_equals_generic(P, orc, K):
    """rmse(params, ratings.triplets(), ratings) -- the cached-lookup training-set path --
    equals the generic path on a copy of the same triplets and the oracle (sequential sum)."""
    r, rows, cols, vals = _case(P, seed=12, M=400, N=90, dens=0.3)
    if K:
        tbl, _ = P.simlsh_topk(r, P.LshConfig(G=4, p=2, q=6, seed=1), K)
    else:
        tbl = None
    p = P.train_full(r, tbl, P.TrainConfig(F=40, K=K, epochs=2, seed=2))
    a = P.rmse(p, r.triplets(), r, clamp=(1.0, 5.0))
    t = r.triplets()
    b = P.rmse(p, P.Triplets(t.rows.copy(), t.cols.copy(), t.values.copy()), r, clamp=(1.0, 5.0))
    d, mu = orc.build_csr(r.M, r.N, rows, cols, vals)
    m = orc.Model(p.mu, p.b, p.b_hat, p.U, p.V, p.W, p.C,
                  tbl.entries if K else np.zeros((r.N, 0), np.int32))
    ref = orc.rmse(d, m, r.entry_rows, r.entry_cols, r.entry_values, clamp=(1.0, 5.0))
    assert a == b == ref


@pytest.mark.parametrize("K,F,mode,order", [(0, 8, "exact", "csr"), (7, 40, "exact", "random"),
                                          (40, 33, "exact", "csc"), (64, 64, "exact", "random"),
                                          (16, 64, "hogwild", "random"), (33, 32, "hogwild", "csr")])
def test_train_set_rmse_row_kernel_equals_lookup_kernel(P, orc, monkeypatch, K, F, mode, order):
    """The row-order kernel (one warp per row, row bitmap) returns the same float as the
    CSC-order lookup-cache kernel (training set) / the ungrouped kernel (a test set) and the
    oracle: empty rows and columns, rows longer than 32, K spanning two 32-wide halves, entry
    orders CSR / CSC / random, duplicate and unrated test pairs, fp64 and fp32 (Hogwild)
    models, clamp + unscale."""
    from paper_2111_11682_b200 import factorization as fz
    rng = np.random.default_rng(5)
    M, N = 300, 120
    dense = rng.random((M, N)) < 0.25
    dense[7] = False                      # empty row
    dense[:, 11] = False                  # empty column
    dense[3, :100] = True                 # long row (4 chunks of 32)
    rows, cols = np.nonzero(dense)
    if order == "csc":
        o = np.lexsort((rows, cols))
    elif order == "random":
        o = rng.permutation(len(rows))
    else:
        o = np.arange(len(rows))
    rows, cols = rows[o], cols[o]
    vals = rng.integers(1, 6, len(rows)).astype(np.float64)
    r = P.SparseRatings(M, N, rows, cols, vals)
    tbl = P.simlsh_topk(r, P.LshConfig(G=4, p=2, q=6, seed=1), K)[0] if K else None
    p = P.train_full(r, tbl, P.TrainConfig(F=F, K=K, epochs=2, seed=2), mode=mode)
    kw = dict(clamp=(1.0, 5.0), unscale=2.0)
    # a held-out-style test set: random rows / cols (rated or not, duplicates, unsorted)
    nt = 6000
    te = P.Triplets(rng.integers(0, M, nt).astype(np.int32), rng.integers(0, N, nt).astype(np.int32),
                    rng.integers(1, 6, nt).astype(np.float64))
    a = P.rmse(p, r.triplets(), r, **kw)
    at = P.rmse(p, te, r, **kw)
    monkeypatch.setattr(fz, "_ROWS_RMSE_MAX_N", 0)
    b = P.rmse(p, r.triplets(), r, **kw)
    bt = P.rmse(p, te, r, **kw)
    assert a == b and at == bt
    if mode == "exact":
        d, _ = orc.build_csr(r.M, r.N, rows, cols, vals)
        m = orc.Model(p.mu, p.b, p.b_hat, p.U, p.V, p.W, p.C, tbl.entries if K else np.zeros((N, 0), np.int32))
        assert a == orc.rmse(d, m, r.entry_rows, r.entry_cols, r.entry_values, **kw)
        assert at == orc.rmse(d, m, te.rows, te.cols, te.values, **kw)


@pytest.mark.parametrize("n", [10, 5000])
def test_rmse_rejects_out_of_range_test_pairs(P, n):
    """Both test-set routes (ungrouped below 4,096 targets, row-grouped above) raise
    IndexError for a pair outside the ratings' index space instead of reading out of bounds."""
    r, rows, cols, vals = _case(P, seed=4, M=200, N=50, dens=0.2)
    p = P.train_full(r, None, P.TrainConfig(F=8, K=0, epochs=1, seed=0))
    rng = np.random.default_rng(0)
    tr = rng.integers(0, r.M, n).astype(np.int32)
    tc = rng.integers(0, r.N, n).astype(np.int32)
    tv = np.ones(n)
    assert np.isfinite(P.rmse(p, P.Triplets(tr, tc, tv), r))
    bad_r, bad_c = tr.copy(), tc.copy()
    bad_r[n // 2] = r.M
    bad_c[n // 3] = -1
    with pytest.raises(IndexError):
        P.rmse(p, P.Triplets(bad_r, tc, tv), r)
    with pytest.raises(IndexError):
        P.rmse(p, P.Triplets(tr, bad_c, tv), r)


def test_train_set_rmse_large_tree_sum(P):
    """Above 2^22 ratings both paths use the same fixed tree over entry order."""
    rng = np.random.default_rng(3)
    M, N = 60_000, 700
    rows, cols = np.nonzero(rng.random((M, N)) < 0.11)
    perm = rng.permutation(len(rows))          # entry order != CSC order
    r = P.SparseRatings(M, N, rows[perm], cols[perm], rng.integers(1, 6, len(rows)).astype(float))
    assert r.nnz > (1 << 22)
    tbl, _ = P.simlsh_topk(r, P.LshConfig(G=4, p=2, q=6, seed=1), 16)
    p = P.train_full(r, tbl, P.TrainConfig(F=32, K=16, epochs=1, seed=2), mode="hogwild")
    t = r.triplets()
    a = P.rmse(p, t, r)
    b = P.rmse(p, P.Triplets(t.rows.copy(), t.cols.copy(), t.values.copy()), r)
    assert a == b and np.isfinite(a)
    from paper_2111_11682_b200 import factorization as fz
    old = fz._ROWS_RMSE_MAX_N
    fz._ROWS_RMSE_MAX_N = 0                    # the CSC lookup-cache kernel
    try:
        assert P.rmse(p, t, r) == a
    finally:
        fz._ROWS_RMSE_MAX_N = old


@pytest.mark.parametrize("n", [1, 7, 8, 9, 127, 128, 129, 1000, 65536, 65537, 300001, 3_000_017])
def test_pairwise_sum_device_equals_numpy(P, n):
    """numpy's np.add.reduce (pairwise) restated on the device, bit for bit, across the leaf,
    split and chunk-combine boundaries (values spread over 12 orders of magnitude)."""
    from paper_2111_11682_b200 import _native as nat
    from paper_2111_11682_b200.data import pairwise_sum_device
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) * 10.0 ** rng.integers(-6, 6, n)
    assert pairwise_sum_device(nat.to_dev(x)) == float(np.add.reduce(x))
    assert pairwise_sum_device(nat.to_dev(x)) / n == float(x.mean())


def test_device_sparse_ratings_real_values_exact_baselines(P):
    """DeviceSparseRatings from device triplets in arbitrary entry order, real values:
    mu, b and b_hat equal compute_baselines of the same triplets byte for byte (numpy
    pairwise mean, np.add.at in entry order), and the index views equal the host build."""
    import torch
    from paper_2111_11682_b200 import _native as nat
    rng = np.random.default_rng(5)
    M, N, nnz = 3000, 700, 120000
    key = rng.choice(M * N, nnz, replace=False)          # random entry order, no duplicates
    rows, cols = (key // N).astype(np.int32), (key % N).astype(np.int32)
    vals = rng.random(nnz) * 4.7 + 0.3
    host = P.SparseRatings(M, N, rows, cols, vals)
    ref = host.baselines()
    dsr = P.DeviceSparseRatings(M, N, torch.from_numpy(rows.copy()).cuda(), torch.from_numpy(cols.copy()).cuda(),
                                torch.from_numpy(vals.copy()).cuda())
    got = dsr.baselines()
    assert got.mu == ref.mu
    assert got.b.tobytes() == ref.b.tobytes() and got.b_hat.tobytes() == ref.b_hat.tobytes()
    d = dsr.device()
    for name, want in (("col_ptr", host.col_ptr), ("col_rows", host.col_rows), ("col_vals", host.col_vals),
                       ("row_ptr", host.row_ptr), ("row_cols", host.row_cols), ("row_vals", host.row_vals)):
        n = len(want)
        assert nat.to_host(getattr(d, name))[:n].tobytes() == np.ascontiguousarray(want).tobytes(), name


@pytest.mark.parametrize("F", [32, 50])
def test_rmse_on_fp32_model_equals_widened(P, F):
    """rmse() on a Hogwild fit reads its fp32 arrays directly (culsh_rmse[_train]_m32; F = 50
    runs on zero-padded 64-wide rows) and returns the same float as on a widened fp64 copy
    of the same parameters, for a held-out set and for the training set."""
    r, rows, cols, vals = _case(P, seed=21, M=400, N=90, dens=0.2)
    tbl, _ = P.simlsh_topk(r, P.LshConfig(G=4, p=2, q=8, seed=3), 6)
    ph = P.train_full(r, tbl, P.TrainConfig(F=F, K=6, epochs=3, seed=0), mode="hogwild")
    host = ph.copy()                                   # fp64 host arrays -> DeviceModel64 path
    rng = np.random.default_rng(2)
    sel = rng.choice(len(rows), 300, replace=False)
    te = P.Triplets(rows[sel].astype(np.int32), cols[sel].astype(np.int32), vals[sel])
    assert P.rmse(ph, te, r) == P.rmse(host, te, r)
    assert P.rmse(ph, r.triplets(), r) == P.rmse(host, r.triplets(), r)
    assert P.rmse(ph, te, r, clamp=(1.0, 5.0), unscale=2.0) == P.rmse(host, te, r, clamp=(1.0, 5.0), unscale=2.0)


@pytest.mark.parametrize("dtype", [np.float64, np.int32])
def test_staged_copies_round_trip(P, dtype):
    """Large host <-> device copies go through the reused pinned chunks (to_dev /
    copy_to_device / to_host): a multi-chunk array (> 2 x 64 MB, ragged tail) survives both
    directions byte for byte, twice in a row (chunk reuse), and a small one takes the plain path."""
    from paper_2111_11682_b200 import _native as nat
    rng = np.random.default_rng(0)
    n = (200 << 20) // np.dtype(dtype).itemsize + 12345
    for _ in range(2):
        a = (rng.standard_normal(n) if dtype == np.float64 else rng.integers(-2**31, 2**31 - 1, n)).astype(dtype)
        d = nat.to_dev(a)
        b = nat.to_host(d)
        assert b.dtype == a.dtype and b.tobytes() == a.tobytes()
    small = np.arange(1000, dtype=dtype)
    assert nat.to_host(nat.to_dev(small)).tobytes() == small.tobytes()


@pytest.mark.parametrize("integer", [True, False])
def test_sparse_ratings_device_build_equals_host_build(P, integer, monkeypatch):
    """SparseRatings from host triplets >= 1M entries builds CSR / CSC / baselines on the
    device: every host view (materialised on first read) and the baselines equal the host
    lexsort build byte for byte, including duplicate (row, col) entries (ties in entry order)."""
    import paper_2111_11682_b200.data as D
    rng = np.random.default_rng(11)
    M, N, n = 5000, 900, 1_300_000
    rows = rng.integers(0, M, n).astype(np.int32)       # duplicates included on purpose
    cols = rng.integers(0, N, n).astype(np.int32)
    vals = (rng.integers(1, 6, n).astype(np.float64) if integer else rng.random(n) * 5)
    dev = P.SparseRatings(M, N, rows.copy(), cols.copy(), vals.copy())
    assert dev._dev is not None and "row_ptr" not in dev.__dict__
    monkeypatch.setattr(D, "_DEVICE_BUILD_MIN", 1 << 62)
    host = P.SparseRatings(M, N, rows.copy(), cols.copy(), vals.copy())
    assert host._dev is None
    for name in ("entry_rows", "entry_cols", "entry_values", "row_ptr", "row_cols", "row_vals",
                 "col_ptr", "col_rows", "col_vals"):
        assert getattr(dev, name).tobytes() == getattr(host, name).tobytes(), name
        assert not getattr(dev, name).flags.writeable
    a, b = dev.baselines(), host.baselines()
    assert a.mu == b.mu and a.b.tobytes() == b.b.tobytes() and a.b_hat.tobytes() == b.b_hat.tobytes()


def test_build_indices_duplicate_check_on_device(P):
    """build_indices on >= 1M triplets checks duplicates on the device and reports the same
    first duplicate as the reference's lexsort (data.py:269-286)."""
    rng = np.random.default_rng(4)
    M, N = 4000, 3000
    key = rng.choice(M * N, 1_200_000, replace=False)
    rows, cols = (key // N).astype(np.int32), (key % N).astype(np.int32)
    vals = rng.integers(1, 6, len(key)).astype(np.float64)
    r = P.build_indices(P.Triplets(rows, cols, vals), M=M, N=N)
    assert r.nnz == len(key)
    rows2, cols2 = rows.copy(), cols.copy()
    rows2[1_000_000], cols2[1_000_000] = rows2[17], cols2[17]        # entry 17 duplicated later
    rows2[500_000], cols2[500_000] = rows2[900_000], cols2[900_000]  # and another pair
    order = np.lexsort((cols2, rows2))
    same = (np.diff(rows2[order]) == 0) & (np.diff(cols2[order]) == 0)
    k = order[int(np.flatnonzero(same)[0])]
    import re
    with pytest.raises(ValueError, match=re.escape(f"duplicate entry at (row={rows2[k]}, col={cols2[k]})")):
        P.build_indices(P.Triplets(rows2, cols2, vals), M=M, N=N)


def _seq_sum_device(x):
    from paper_2111_11682_b200 import _native as nat
    xd = nat.to_dev(np.ascontiguousarray(x, np.float64))
    out = nat.empty((1,), "float64")
    nat.call("culsh_sequential_sum", nat.ptr(xd), len(x), nat.ptr(out), nat.stream_ptr())
    return float(out.item())


def _seq_cases():
    rng = np.random.default_rng(42)
    e = rng.standard_normal(3_000_000)
    yield "squares_3M", e * e
    # ties to even: on a grid where S ~ 1, terms of 0.5 / 1.5 / 2.5 ulp
    u = 2.0 ** -52
    t = rng.choice(np.array([0.5, 1.5, 2.5, 1.0, 0.0]) * u, 400_000)
    t[0] = 1.0
    yield "ties", t
    # many binade changes: geometric growth, then tiny terms
    yield "binades", np.concatenate([2.0 ** (np.arange(200_000) / 4000.0), rng.random(100_000) * 1e-12])
    # leading zeros, subnormals, a huge term mid-way
    z = np.zeros(150_000)
    sub = rng.random(120_000) * 1e-310
    mid = rng.random(90_000)
    mid[45_000] = 1e300
    yield "zeros_subnormal_huge", np.concatenate([z, sub, mid])
    for n in (1, 7, 8192, 32768, 32769, 40_000, 100_003):
        yield f"n{n}", rng.random(n) * 3.0


@pytest.mark.parametrize("name,x", list(_seq_cases()), ids=lambda v: v if isinstance(v, str) else "")
def test_exact_sequential_sum(P, name, x):
    """culsh_sequential_sum (every rmse's sum) == numpy's sequential accumulate, bit for bit,
    through ties-to-even, binade changes, zeros, subnormals and a huge term."""
    ref = np.add.accumulate(x)[-1]
    assert _seq_sum_device(x) == ref, name


def test_exact_sequential_sum_nonfinite(P):
    x = np.random.default_rng(1).random(200_000)
    x[150_000] = np.inf
    assert _seq_sum_device(x) == np.inf
    x[170_000] = np.nan
    assert np.isnan(_seq_sum_device(x))


def test_exact_sequential_sum_100m(P):
    """At the C3 training-set size (rmse over 100M squared errors, cli.py's train RMSE)."""
    e = np.random.default_rng(3).standard_normal(100_000_000) * 0.9
    x = e * e
    del e
    assert _seq_sum_device(x) == np.add.accumulate(x)[-1]
