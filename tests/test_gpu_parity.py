"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
fixtures and the CPU oracle, bit-exact for hashes / keys / top-K / exact-mode
SGD / online, and RMSE within 0.005 for the Hogwild mode."""

import numpy as np
import pytest

from conftest import load_golden, sha

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2111_11682_b200 as p
    return p


def ratings_of(P, z, pre):
    return P.SparseRatings(int(z[pre + "M"]), int(z[pre + "N"]), z[pre + "rows"], z[pre + "cols"],
                           z[pre + "vals"])


@pytest.fixture(scope="module")
def c1(P):
    z = load_golden("c1.npz")
    tr = P.SparseRatings(int(z["train_M"]), int(z["train_N"]), z["train_rows"].astype(np.int32),
                         z["train_cols"].astype(np.int32), z["train_vals"].astype(np.float64))
    te = P.Triplets(z["test_rows"].astype(np.int32), z["test_cols"].astype(np.int32),
                    z["test_vals"].astype(np.float64))
    return z, tr, te


REF_TOL_RMSE = 0.005


# ------------------------------------------------------------------ hashes ---

class TestHashKat:
    def test_worked_example_fig3(self, P):
        # test_lsh.py:63-66
        r = P.SparseRatings(3, 1, np.array([0, 1, 2]), np.array([0, 0, 0]), np.array([3., 4., 5.]))
        H = np.array([[0, 0, 1], [0, 1, 0], [1, 0, 0]], dtype=np.uint8)
        acc, sig = P.simlsh_signature(0, r, H, psi_exponent=1)
        np.testing.assert_array_equal(acc, [-2.0, -4.0, -6.0])
        np.testing.assert_array_equal(sig, [0, 0, 0])

    def test_empty_column_all_ones(self, P):
        r = P.SparseRatings(3, 1, np.zeros(0), np.zeros(0), np.zeros(0))
        acc, sig = P.simlsh_signature(0, r, np.eye(3, dtype=np.uint8), 1)
        np.testing.assert_array_equal(acc, [0, 0, 0])
        np.testing.assert_array_equal(sig, [1, 1, 1])

    def test_single_rating_matches_row_hash(self, P):
        H = np.array([[0, 0, 1], [0, 1, 0], [1, 0, 0]], dtype=np.uint8)
        r = P.SparseRatings(3, 1, np.array([1]), np.array([0]), np.array([2.5]))
        _, sig = P.simlsh_signature(0, r, H, 1)
        np.testing.assert_array_equal(sig, H[1])

    def test_psi_exponents(self, P):
        r = P.SparseRatings(1, 1, np.array([0]), np.array([0]), np.array([3.0]))
        H = np.ones((1, 2), dtype=np.uint8)
        for e, want in [(1, 3.0), (2, 9.0), (4, 81.0)]:
            acc, _ = P.simlsh_signature(0, r, H, e)
            assert acc[0] == want

    def test_row_hashes_match_oracle(self, P, orc):
        for (M, G, p, q, seed) in [(50, 8, 2, 3, 11), (37, 13, 2, 5, 3), (20, 64, 1, 2, 9),
                                   (0, 4, 2, 2, 0)]:
            h = P.assign_row_hashes(M, P.LshConfig(G=G, p=p, q=q, seed=seed))
            assert h.bits.shape == (M, q, p, G)
            np.testing.assert_array_equal(h.bits, orc.assign_bits(seed, q, p, M, G))
        h = P.assign_row_hashes(50, P.LshConfig(G=8, p=2, q=3, seed=11))
        np.testing.assert_array_equal(h.extended(80).bits[:50], h.bits)

    def test_ones_fraction(self, P):
        h = P.assign_row_hashes(10_000, P.LshConfig(G=8, p=2, q=2, seed=0))
        frac = h.bits.reshape(10_000, -1).mean(axis=0)
        assert frac.min() >= 0.48 and frac.max() <= 0.52


class TestHashGolden:
    def test_lsh_small_bit_exact(self, P):
        z = load_golden("lsh_small.npz")
        for k in range(int(z["n_runs"])):
            pre = f"k{k}_"
            G, p, q, e, seed, K = (int(x) for x in z[pre + "cfg"])
            r = ratings_of(P, z, f"c{int(z[pre + 'case'])}_")
            table, state = P.simlsh_topk(r, P.LshConfig(G=G, p=p, q=q, psi_exponent=e, seed=seed), K)
            assert state.acc.tobytes() == z[pre + "acc"].tobytes(), k
            assert state.sig.tobytes() == z[pre + "sig"].tobytes(), k
            keys = P._native.to_host(state.device_keys()).view(np.uint64).reshape(q, r.N)
            assert keys.tobytes() == z[pre + "keys"].tobytes(), k
            assert table.entries.tobytes() == z[pre + "entries"].tobytes(), k
            table.validate()

    def test_c1_bit_exact(self, P, c1):
        z, tr, _ = c1
        cfg = P.LshConfig(G=8, p=3, q=100, psi_exponent=2, seed=0)
        table, state = P.simlsh_topk(tr, cfg, 16)
        assert sha(state.acc) == str(z["lsh_acc_sha"])
        assert sha(state.sig) == str(z["lsh_sig_sha"])
        assert table.entries.tobytes() == z["lsh_entries16"].tobytes()
        t32, _ = P.simlsh_topk(tr, cfg, 32)
        assert t32.entries.tobytes() == z["lsh_entries32"].tobytes()

    def test_fp64_path_equals_int_path(self, P, orc):
        """Integer ratings take the exact-integer kernel; the ordered fp64 kernel
        (used for non-integer data) must give the identical bytes."""
        from paper_2111_11682_b200 import lsh as L, _native as nat
        rng = np.random.default_rng(5)
        M, N = 200, 150
        mask = rng.random((M, N)) < 0.1
        rows, cols = np.nonzero(mask)
        vals = rng.integers(1, 6, size=len(rows)).astype(float)
        r = P.SparseRatings(M, N, rows, cols, vals)
        c = P.LshConfig(G=8, p=3, q=20, psi_exponent=2, seed=4)
        st = P.compute_hash_state(r, c)
        dev = r.device()
        h = P.assign_row_hashes(M, c)
        W = c.q * c.p * c.G
        acc = nat.zeros((N * W,), "float64")
        nat.call("culsh_hash_accumulate", nat.ptr(dev.col_ptr), nat.ptr(dev.col_rows),
                 nat.ptr(dev.col_vals), 0, N, None, nat.ptr(h.table()), c.q, c.p, c.G, 2, 0, 0,
                 nat.ptr(acc), None, None, N, nat.stream_ptr())
        assert nat.to_host(acc).tobytes() == st.acc.tobytes()
        ref = orc.accumulate_all(r.col_ptr, r.col_rows, r.col_vals, orc.assign_bits(4, 20, 3, M, 8), 2)
        assert ref.tobytes() == st.acc.tobytes()

    def test_injected_hashes(self, P, orc):
        """compute_hash_state with user-supplied RowHashes (lsh.py:231-239)."""
        rng = np.random.default_rng(1)
        bits = (rng.random((30, 2, 2, 5)) < 0.5).astype(np.uint8)
        rows = rng.integers(0, 30, 60)
        cols = rng.integers(0, 12, 60)
        key = np.unique(rows * 100 + cols)
        r = P.SparseRatings(30, 12, key // 100, key % 100, rng.uniform(0.5, 5, len(key)))
        st = P.compute_hash_state(r, P.LshConfig(G=5, p=2, q=2, psi_exponent=4),
                                  P.RowHashes(bits=bits, seed=0))
        ref = orc.accumulate_all(r.col_ptr, r.col_rows, r.col_vals, bits, 4)
        assert st.acc.tobytes() == ref.tobytes()


# --------------------------------------------------------------------- SGD ---

REGS = (0.02, 0.02, 0.02, 0.02, 0.002, 0.002)


class TestSgdExact:
    def test_sgd_small_bit_exact(self, P):
        z = load_golden("sgd_small.npz")
        for s in range(int(z["n_cases"])):
            pre = f"s{s}_"
            F, K, epochs, seed = (int(x) for x in z[pre + "cfg"])
            r = ratings_of(P, z, pre)
            nbr = P.NeighborTable(r.N, K, z[pre + "nbr"]) if K else None
            cfg = P.TrainConfig(F=F, K=K, epochs=epochs, seed=seed)
            p = P.train_full(r, nbr, cfg)
            for n in ("b", "b_hat", "U", "V", "W", "C"):
                assert getattr(p, n).tobytes() == z[f"{pre}full_{n}"].tobytes(), (s, n)
            assert P.rmse(p, r.triplets(), r) == float(z[pre + "rmse"])
            assert P.rmse(p, r.triplets(), r, unscale=2.0, clamp=(1.5, 4.5)) == float(z[pre + "rmse_clamp"])
            for D in (2, 3):
                pd = P.parallel_train(r, nbr, cfg, D=D)
                for n in ("b", "b_hat", "U", "V", "W", "C"):
                    assert getattr(pd, n).tobytes() == z[f"{pre}D{D}_{n}"].tobytes(), (s, D, n)
            p1 = P.parallel_train(r, nbr, cfg, D=1)
            assert p1.U.tobytes() == p.U.tobytes()

    def test_c1_train_full_bit_exact(self, P, c1):
        z, tr, te = c1
        nbr = P.NeighborTable(tr.N, 16, z["lsh_entries16"])
        seen = []
        p = P.train_full(tr, nbr, P.TrainConfig(F=32, K=16, epochs=3, seed=0),
                         epoch_callback=lambda t, q: seen.append(P.rmse(q, te, tr)))
        np.testing.assert_array_equal(seen, z["sgd_rmse_test"])
        for n in ("b", "b_hat", "U", "V", "W", "C"):
            assert sha(getattr(p, n)) == str(z[f"sgd_full_{n}_sha"]), n

    def test_c1_dsgd_d4_bit_exact(self, P, c1):
        z, tr, te = c1
        nbr = P.NeighborTable(tr.N, 16, z["lsh_entries16"])
        times = []
        pd, rep = P.parallel_train(tr, nbr, P.TrainConfig(F=32, K=16, epochs=2, seed=0), D=4,
                                   instrument=True, stage_times=times)
        assert rep.ok and rep.stages_checked == 8
        assert len(times) == 8
        for n in ("b", "U", "V", "W", "C"):
            assert sha(getattr(pd, n)) == str(z[f"sgd_D4_{n}_sha"]), n
        assert P.rmse(pd, te, tr) == float(z["sgd_D4_rmse_test"])

    def test_predict_hand_value(self, P):
        # test_factorization.py:148-158 -> 3.8
        r = P.SparseRatings(3, 3, np.array([0, 0, 1, 1, 1, 2, 2]), np.array([0, 2, 0, 1, 2, 1, 2]),
                            np.array([4, 2, 2, 3, 4, 3, 3.0]))
        nbr = P.NeighborTable(3, 2, np.array([[1, 2], [0, 2], [0, 1]], dtype=np.int32))
        p = P.ModelParams(mu=3.0, b=np.zeros(3), b_hat=np.zeros(3),
                          U=np.array([[0.5], [0.0], [0.0]]), V=np.array([[0.0], [0.0], [1.0]]),
                          W=np.array([[0.0, 0.0], [0.0, 0.0], [0.1, 0.0]]),
                          C=np.array([[0.0, 0.0], [0.0, 0.0], [0.0, 0.2]]), neighbors=nbr)
        assert P.predict(0, 2, p, r) == pytest.approx(3.8, abs=1e-12)
        with pytest.raises(IndexError):
            P.predict(5, 0, p, r)

    def test_scalar_sgd_step(self, P):
        # test_factorization.py:197-207
        r = P.SparseRatings(1, 1, np.array([0]), np.array([0]), np.array([4.0]))
        p = P.ModelParams(mu=0.0, b=np.zeros(1), b_hat=np.zeros(1), U=np.array([[1.0]]),
                          V=np.array([[2.0]]), W=np.zeros((1, 0)), C=np.zeros((1, 0)))
        e = P.sgd_update(0, 0, p, rates=(0.0, 0.0, 0.1, 0.1, 0.0, 0.0), regs=(0.0,) * 6, ratings=r)
        assert e == pytest.approx(2.0)
        assert p.U[0, 0] == pytest.approx(1.4)
        assert p.V[0, 0] == pytest.approx(2.2)

    def test_gradient_directions_fd(self, P):
        # test_factorization.py:214-235 (A1 oracle): analytic step == central FD
        rng = np.random.default_rng(3)
        for F, K in [(1, 0), (2, 2), (8, 4)]:
            M, N = 7, 9
            mask = rng.random((M, N)) < 0.5
            rows, cols = np.nonzero(mask)
            r = P.SparseRatings(M, N, rows, cols, rng.integers(1, 6, len(rows)).astype(float))
            nbr = None
            if K:
                ent = np.stack([rng.choice(np.delete(np.arange(N), j), K, replace=False)
                                for j in range(N)]).astype(np.int32)
                nbr = P.NeighborTable(N, K, ent)
            p = P.ModelParams(mu=3.0, b=rng.normal(0, .2, M), b_hat=rng.normal(0, .2, N),
                              U=rng.uniform(0, .3, (M, F)), V=rng.uniform(0, .3, (N, F)),
                              W=rng.normal(0, .1, (N, K)), C=rng.normal(0, .1, (N, K)), neighbors=nbr)
            k = rng.integers(0, r.nnz)
            i, j = int(r.entry_rows[k]), int(r.entry_cols[k])
            q = p.copy()
            P.sgd_update(i, j, q, rates=(1.0,) * 6, regs=(0.0,) * 6, ratings=r)
            rv = r.rating(i, j)

            def fd(mut, h=1e-5):
                def sq(dl):
                    t = p.copy()
                    mut(t, dl)
                    return (rv - P.predict(i, j, t, r)) ** 2
                return -0.5 * (sq(h) - sq(-h)) / (2 * h)

            assert q.b[i] - p.b[i] == pytest.approx(fd(lambda t, d: t.b.__setitem__(i, t.b[i] + d)),
                                                    rel=1e-4, abs=1e-9)
            for f in range(F):
                assert q.U[i, f] - p.U[i, f] == pytest.approx(
                    fd(lambda t, d, f=f: t.U.__setitem__((i, f), t.U[i, f] + d)), rel=1e-4, abs=1e-9)
            for kk in range(K):
                assert q.W[j, kk] - p.W[j, kk] == pytest.approx(
                    fd(lambda t, d, kk=kk: t.W.__setitem__((j, kk), t.W[j, kk] + d)), rel=1e-4, abs=1e-9)
                assert q.C[j, kk] - p.C[j, kk] == pytest.approx(
                    fd(lambda t, d, kk=kk: t.C.__setitem__((j, kk), t.C[j, kk] + d)), rel=1e-4, abs=1e-9)

    def test_divergence_raises(self, P):
        rng = np.random.default_rng(42)
        mask = rng.random((12, 9)) < 0.5
        rows, cols = np.nonzero(mask)
        r = P.SparseRatings(12, 9, rows, cols, rng.integers(1, 6, len(rows)).astype(float))
        ent = np.stack([np.delete(np.arange(9), j)[:2] for j in range(9)]).astype(np.int32)
        cfg = P.TrainConfig(F=3, K=2, alpha_b=1e12, alpha_b_hat=1e12, alpha_u=1e12, alpha_v=1e12,
                            alpha_w=1e12, alpha_c=1e12, epochs=3, seed=1)
        with pytest.raises(P.TrainingDivergedError):
            P.train_full(r, P.NeighborTable(9, 2, ent), cfg)
        with pytest.raises(P.TrainingDivergedError):
            P.parallel_train(r, P.NeighborTable(9, 2, ent), cfg, D=2)


# ------------------------------------------------------------------ online ---

class TestOnline:
    def test_online_small_bit_exact(self, P):
        z = load_golden("online_small.npz")
        for s in range(int(z["n_cases"])):
            pre = f"o{s}_"
            G, p_, q, e, lseed = (int(x) for x in z[pre + "lsh"])
            F, K, epochs, seed = (int(x) for x in z[pre + "cfg"])
            orig = ratings_of(P, z, pre)
            lc = P.LshConfig(G=G, p=p_, q=q, psi_exponent=e, seed=lseed)
            cfg = P.TrainConfig(F=F, K=K, epochs=epochs, seed=seed)
            tbl, state = P.simlsh_topk(orig, lc, K)
            assert tbl.entries.tobytes() == z[pre + "table"].tobytes()
            params = P.train_full(orig, tbl, cfg)
            assert params.U.tobytes() == z[pre + "p0_U"].tobytes()
            before = params.copy()
            bM, bN, nr_, nc_ = (int(x) for x in z[pre + "b_shape"])
            batch = P.IncrementBatch(bM, bN, nr_, nc_, z[pre + "b_rows"], z[pre + "b_cols"],
                                     z[pre + "b_vals"])
            pe, se, re_, ne = P.absorb_increment(params, state, orig, batch, cfg)
            assert se.acc.tobytes() == z[pre + "ext_acc"].tobytes(), s
            assert ne.entries.tobytes() == z[pre + "ext_entries"].tobytes(), s
            for n in ("b", "b_hat", "U", "V", "W", "C"):
                assert getattr(pe, n).tobytes() == z[f"{pre}ext_{n}"].tobytes(), (s, n)
            assert pe.U[:orig.M].tobytes() == before.U.tobytes()
            assert pe.V[:orig.N].tobytes() == before.V.tobytes()

    def test_incremental_equals_recompute(self, P):
        # A7a (test_acceptance.py:201-220) on 40 random increments
        rng = np.random.default_rng(7)
        for trial in range(40):
            M = int(rng.integers(6, 16))
            N = int(rng.integers(5, 12))
            mask = rng.random((M, N)) < 0.35
            rows, cols = np.nonzero(mask)
            full = P.SparseRatings(M, N, rows, cols, rng.integers(1, 6, len(rows)).astype(float))
            orig, batch, _, _ = P.holdback_variables(full, int(rng.integers(1, 3)),
                                                     int(rng.integers(1, 3)), seed=trial)
            cfg = P.LshConfig(G=int(rng.integers(2, 9)), p=int(rng.integers(1, 3)),
                              q=int(rng.integers(1, 4)), psi_exponent=int(rng.choice([1, 2, 4])),
                              seed=trial)
            state = P.compute_hash_state(orig, cfg)
            inc = P.update_hashes_incremental(state, batch, P.assign_row_hashes(batch.M_hat, cfg))
            ref = P.compute_hash_state(P.extend_ratings(orig, batch), cfg)
            assert inc.acc.tobytes() == ref.acc.tobytes(), trial
            assert inc.sig.tobytes() == ref.sig.tobytes(), trial

    def test_online_c1(self, P, c1):
        z, tr, _ = c1
        row_map, col_map = z["online_row_map"], z["online_col_map"]
        bM, bN, nr_, nc_ = (int(x) for x in z["online_b_shape"])
        rr, cc = row_map[tr.entry_rows], col_map[tr.entry_cols]
        keep = (rr < bM) & (cc < bN)
        orig = P.SparseRatings(bM, bN, rr[keep], cc[keep], tr.entry_values[keep])
        lc = P.LshConfig(G=8, p=3, q=100, psi_exponent=2, seed=0)
        cfg = P.TrainConfig(F=32, K=32, epochs=4, seed=0)
        t0, s0 = P.simlsh_topk(orig, lc, 32)
        assert sha(s0.acc) == str(z["online_state0_acc_sha"])
        assert t0.entries.tobytes() == z["online_orig_entries"].tobytes()
        p0 = P.train_full(orig, t0, cfg)
        assert sha(p0.U) == str(z["online_p0_U_sha"])
        batch = P.IncrementBatch(bM, bN, nr_, nc_, z["online_b_rows"], z["online_b_cols"],
                                 z["online_b_vals"])
        pe, se, _, ne = P.absorb_increment(p0, s0, orig, batch, cfg)
        assert sha(se.acc) == str(z["online_ext_acc_sha"])
        assert ne.entries.tobytes() == z["online_ext_entries"].tobytes()
        for n in ("b", "b_hat", "U", "V", "W", "C"):
            assert sha(getattr(pe, n)) == str(z[f"online_ext_{n}_sha"]), n


# ----------------------------------------------------------------- Hogwild ---

class TestHogwild:
    def test_c1_rmse_within_tolerance(self, P, c1):
        """Hogwild fp32 test RMSE within 0.005 of the exact (== reference) run after
        the same epochs (BASELINE.json north_star)."""
        z, tr, te = c1
        nbr = P.NeighborTable(tr.N, 16, z["lsh_entries16"])
        cfg = P.TrainConfig(F=32, K=16, epochs=20, seed=0)
        exact = P.rmse(P.train_full(tr, nbr, cfg), te, tr)
        hog = P.rmse(P.train_full(tr, nbr, cfg, mode="hogwild"), te, tr)
        assert abs(hog - exact) <= REF_TOL_RMSE, (hog, exact)

    def test_f128_k32_runs(self, P):
        from paper_2111_11682_b200.hogwild import HogwildTrainer
        rng = np.random.default_rng(0)
        M, N = 3000, 800
        mask = rng.random((M, N)) < 0.02
        rows, cols = np.nonzero(mask)
        r = P.SparseRatings(M, N, rows, cols, rng.integers(1, 6, len(rows)).astype(float))
        tbl, _ = P.simlsh_topk(r, P.LshConfig(), 32)
        cfg = P.TrainConfig(F=128, K=32, epochs=3, seed=0, alpha_b=0.02, alpha_b_hat=0.02,
                            alpha_u=0.02, alpha_v=0.02, alpha_w=0.001, alpha_c=0.001,
                            lambda_b=0.01, lambda_b_hat=0.01, lambda_u=0.01, lambda_v=0.01,
                            lambda_w=0.05, lambda_c=0.05)
        tr = HogwildTrainer(r, tbl, cfg)
        first = None
        for t in range(cfg.epochs):
            tr.loss.zero_()
            tr.epoch(t)
            l = float(tr.loss.item())
            first = first or l
        assert l < first
        pe = P.train_full(r, tbl, P.TrainConfig(**{**cfg.__dict__, "epochs": 3}))
        rm_exact = P.rmse(pe, r.triplets(), r)
        rm_hog = P.rmse(tr.to_params(), r.triplets(), r)
        assert abs(rm_exact - rm_hog) <= REF_TOL_RMSE, (rm_exact, rm_hog)


class TestPackedStream:
    """The packed per-epoch stream (culsh_pack_stream) carries exactly the wide
    stream's information, and the packed kernel makes exactly the wide kernel's
    updates (columns run one launch at a time, so both are deterministic)."""

    def _problem(self, P, K, nvals=5, M=700, N=90, dens=0.08):
        rng = np.random.default_rng(3)
        mask = rng.random((M, N)) < dens
        rows, cols = np.nonzero(mask)
        vals = rng.integers(1, nvals + 1, len(rows)).astype(float) * 0.5
        r = P.SparseRatings(M, N, rows, cols, vals)
        tbl, _ = P.simlsh_topk(r, P.LshConfig(q=20), K)
        cfg = P.TrainConfig(F=64, K=K, epochs=2, seed=0)
        return r, tbl, cfg

    @pytest.mark.parametrize("K", [16, 40])
    def test_decode_equals_wide(self, P, K):
        from paper_2111_11682_b200 import _native as nat
        from paper_2111_11682_b200.hogwild import HogwildTrainer
        r, tbl, cfg = self._problem(P, K)
        tr = HogwildTrainer(r, tbl, cfg)
        pk = tr.packed
        assert pk is not None
        w = nat.to_host(pk["words"]).view(np.uint32)[:r.nnz]
        lut = nat.to_host(pk["lut"])
        rows = nat.to_host(tr.dev.col_rows)[:r.nnz]
        vals = nat.to_host(tr.vals32)[:r.nnz]
        MW = tr.MW
        mask = nat.to_host(tr.mask).view(np.uint32)[:r.nnz * MW].reshape(r.nnz, MW)
        assert np.array_equal(w & 0x07FFFFFF, rows)
        assert np.array_equal(lut[(w >> 27) & 15], vals)
        hm = (w >> 31).astype(bool)
        assert np.array_equal(hm, mask.any(axis=1))
        assert hm.any() and not hm.all()
        cm = nat.to_host(pk["cmask"]).view(np.uint32)[:hm.sum() * MW].reshape(-1, MW)
        assert np.array_equal(cm, mask[hm])
        mptr = nat.to_host(pk["mptr"])
        assert np.array_equal(mptr, np.concatenate([[0], np.cumsum(np.add.reduceat(hm, r.col_ptr[:-1])
                                                                   * (np.diff(r.col_ptr) > 0))]))
        # the 2-byte records: rows = first_row + running deltas per column, same codes / flags
        assert pk["w16"] is not None
        w16 = nat.to_host(pk["w16"]).view(np.uint16)[:r.nnz].astype(np.int64)
        first = nat.to_host(pk["first_row"])[:r.N]
        col_of = np.repeat(np.arange(r.N), np.diff(r.col_ptr))
        delta = w16 & 0xFFF
        run = np.cumsum(delta) - np.repeat(np.cumsum(delta)[r.col_ptr[:-1]] - delta[r.col_ptr[:-1]],
                                           np.diff(r.col_ptr))
        assert np.array_equal(first[col_of] + run, rows)
        assert np.array_equal(lut[(w16 >> 12) & 7], vals)
        assert np.array_equal((w16 >> 15).astype(bool), hm)

    def _serial(self, P, r, tbl, cfg, streamed=False, **kw):
        """Columns one launch at a time (deterministic).  streamed: through the stream
        format the host path ships (2-byte records when they fit) instead of the
        device-resident one."""
        import torch
        from paper_2111_11682_b200.factorization import _rates_struct
        from paper_2111_11682_b200.hogwild import HogwildTrainer
        tr = HogwildTrainer(r, tbl, cfg, **kw)
        for t in range(2):
            for j in range(r.N):
                col = torch.tensor([j], dtype=torch.int32, device="cuda")
                if streamed:
                    tr._launch_packed(1, tr._stream_buffers(), col, _rates_struct(cfg.rates_at(t), cfg.regs),
                                      tr.loss)
                else:
                    tr.launch_epoch(t, col_order=col, n_cols=1)
        torch.cuda.synchronize()
        return tr, tr.to_params()

    @pytest.mark.parametrize("p16", [True, False])
    @pytest.mark.parametrize("rotate", [False, True])
    @pytest.mark.parametrize("K", [16, 40])
    def test_packed_kernel_equals_wide(self, P, K, rotate, p16):
        """4-byte and (unrotated) 2-byte records make the wide kernel's updates."""
        r, tbl, cfg = self._problem(P, K)
        ta, a = self._serial(P, r, tbl, cfg, streamed=True, packed=True, rotate=rotate, p16=p16)
        tb, b = self._serial(P, r, tbl, cfg, packed=False, rotate=rotate)
        assert ta.packed is not None and tb.packed is None
        assert (ta.packed["w16"] is not None) == (p16 and not rotate)
        for name in ("b", "b_hat", "U", "V", "W", "C"):
            assert getattr(a, name).tobytes() == getattr(b, name).tobytes(), name

    def test_work_segments_packed_equals_wide(self, P):
        """Columns split into work segments (skew handling): one segment at a time, the
        packed and wide kernels make identical updates, including the atomic merge of
        the column parameters of partial segments."""
        import ctypes
        import torch
        from paper_2111_11682_b200 import _native as nat
        from paper_2111_11682_b200.factorization import _rates_struct
        from paper_2111_11682_b200.hogwild import HogwildTrainer
        r, tbl, cfg = self._problem(P, 16, M=900, N=40, dens=0.3)
        out = []
        # packed / wide stream x cursor scan in the kernel / precomputed segment cursors
        for packed, cursors in ((True, False), (True, True), (False, False), (False, True)):
            tr = HogwildTrainer(r, tbl, cfg, packed=packed, split_cap=50, p16=False)
            wk = tr.work
            assert wk is not None and wk["split_cols"] > 0
            seg4 = tr._seg_cursors(wk) if cursors else None
            for ep in range(2):
                rates = _rates_struct(cfg.rates_at(ep), cfg.regs)
                for s_ in range(wk["n"]):
                    col = wk["col"][s_:s_ + 1]
                    seg = seg4[4 * s_:4 * s_ + 4] if cursors else wk["seg"][2 * s_:2 * s_ + 2]
                    if packed:
                        tr._launch_packed(1, tr._stream_buffers(resident=True), col, rates, tr.loss, seg,
                                          cursors=cursors)
                    else:
                        d = tr.dev
                        nat.call("culsh_sgd_hogwild_epoch", 1, nat.ptr(d.col_ptr), nat.ptr(seg),
                                 nat.ptr(d.col_rows), nat.ptr(tr.vals32), nat.ptr(tr.mask),
                                 nat.ptr(tr.resid_ptr), nat.ptr(tr.resid), nat.ptr(col),
                                 ctypes.byref(tr.model.struct), ctypes.byref(rates),
                                 2 | 8 | (16 if cursors else 0), 0,
                                 nat.ptr(tr.ticket), nat.ptr(tr.loss), nat.ptr(tr.status), nat.stream_ptr())
            torch.cuda.synchronize()
            out.append(tr.to_params())
        for b in out[1:]:
            for name in ("b", "b_hat", "U", "V", "W", "C"):
                assert getattr(out[0], name).tobytes() == getattr(b, name).tobytes(), name

    def test_work_segments_train(self, P):
        """Concurrent epochs with split columns still train (same data, same epochs).  A
        split column's parameters move by the average of its segments' changes, so on
        this tiny all-split problem (2 segments of ~300 ratings per column; production
        segments are >= 1024 and only long columns split) training is slightly slower:
        within 0.015 RMSE of unsplit.  The accuracy bar on skewed data at scale is
        TestHogwildAtScale (C3 structured data, long columns split)."""
        from paper_2111_11682_b200.hogwild import HogwildTrainer
        r, tbl, cfg = self._problem(P, 16, M=3000, N=60, dens=0.2)
        res = []
        for cap in (None, 320):
            tr = HogwildTrainer(r, tbl, cfg, split_cap=cap)
            assert (tr.work is not None) == (cap is not None)
            for ep in range(6):
                tr.epoch(ep)
            res.append(P.rmse(tr.to_params(), r.triplets(), r))
        assert res[1] <= res[0] + 0.015, res

    @pytest.mark.parametrize("K", [16, 40])
    def test_explicit_stream_matches_host(self, P, K):
        """Explicit-neighbour masks and residuals (shared-memory intersection for columns
        up to 6,144 ratings, per-rating search above) equal a host restatement of
        factorization.py:287-298's test and residual, bit for bit."""
        from paper_2111_11682_b200 import _native as nat
        from paper_2111_11682_b200.hogwild import HogwildTrainer
        rng = np.random.default_rng(5)
        M, N = 9000, 50
        mask = rng.random((M, N)) < 0.05
        mask[:7000, 3] = True                      # one column above the shared-memory cap
        rows, cols = np.nonzero(mask)
        r = P.SparseRatings(M, N, rows, cols, rng.integers(1, 6, len(rows)).astype(float))
        tbl, _ = P.simlsh_topk(r, P.LshConfig(q=20), K)
        tr = HogwildTrainer(r, tbl, P.TrainConfig(F=64, K=K, epochs=1, seed=0))
        d = tr.dev
        mu, bb, bh = d.mu, nat.to_host(d.base_b), nat.to_host(d.base_bhat)
        MW = tr.MW
        got_m = nat.to_host(tr.mask).view(np.uint32)[:r.nnz * MW].reshape(r.nnz, MW)
        got_r = nat.to_host(tr.resid)[:tr.n_explicit]
        exp_m = np.zeros((r.nnz, MW), np.uint32)
        exp_r = []
        dense = {(int(i), int(j)): v for i, j, v in zip(r.entry_rows, r.entry_cols, r.entry_values)}
        for j in range(N):
            for e in range(r.col_ptr[j], r.col_ptr[j + 1]):
                i = int(r.col_rows[e])
                for k in range(K):
                    J = int(tbl.entries[j, k])
                    v = dense.get((i, J))
                    if v is not None:
                        exp_m[e, k >> 5] |= np.uint32(1 << (k & 31))
                        exp_r.append(np.float32(v - (mu + bb[i] + bh[J])))
        assert np.array_equal(got_m, exp_m)
        assert np.array_equal(got_r, np.array(exp_r, np.float32))
        assert tr.n_explicit == len(exp_r)

    def test_host_stream_epochs(self, P):
        """train_from_host (per-epoch H2D of the packed stream) == device-resident epochs
        in expectation: same loss trajectory within Hogwild noise, finite model."""
        from paper_2111_11682_b200.hogwild import HogwildTrainer
        r, tbl, cfg = self._problem(P, 16, M=3000, N=400, dens=0.03)
        tr = HogwildTrainer(r, tbl, cfg)
        host = tr.pinned_stream()
        assert set(host) == {"w16", "first_row", "cmask", "resid"}
        losses, h2d, d2h = tr.train_from_host(host, 0, 3)
        assert h2d == sum(v.numel() * v.element_size() for v in host.values())
        assert np.all(np.isfinite(losses)) and losses[-1] < losses[0]


class TestHogwildAtScale:
    """The performance mode against the exact mode (== reference) at C2 / C3 shape on
    structured (skewed, low-rank + noise) data, 90/10 split: |test RMSE diff| <= 0.005."""

    @pytest.mark.parametrize("shape,epochs", [("c2", 8), ("c3", 3)])
    def test_rmse_parity(self, P, shape, epochs):
        from paper_2111_11682_b200 import _native as nat, lsh, synth
        from paper_2111_11682_b200.data import DeviceSparseRatings
        M, N, nnz, F, K, e = synth.SHAPES[shape]
        rows, cols, vals = synth.structured_triplets_device(M, N, nnz, seed=0)
        nt = rows.numel() // 10
        te = P.Triplets(nat.to_host(rows[:nt]), nat.to_host(cols[:nt]), nat.to_host(vals[:nt]))
        tr = DeviceSparseRatings(M, N, rows[nt:], cols[nt:], vals[nt:])
        del rows, cols, vals
        ent, _, _ = lsh.simlsh_topk_device(tr.device(), P.LshConfig(psi_exponent=e), K)
        nbr = P.NeighborTable(N, K, nat.to_host(ent)[:N * K].reshape(N, K))
        cfg = P.TrainConfig(F=F, K=K, epochs=epochs, seed=0, alpha_b=0.02, alpha_b_hat=0.02,
                            alpha_u=0.02, alpha_v=0.02, alpha_w=0.001, alpha_c=0.001,
                            lambda_b=0.01, lambda_b_hat=0.01, lambda_u=0.01, lambda_v=0.01,
                            lambda_w=0.05, lambda_c=0.05)
        r_ex = P.rmse(P.train_full(tr, nbr, cfg), te, tr)
        r_hw = P.rmse(P.train_full(tr, nbr, cfg, mode="hogwild"), te, tr)
        assert abs(r_hw - r_ex) <= REF_TOL_RMSE, (shape, r_hw, r_ex)


class TestBitCountPath:
    """The Harley-Seal bit-count kernel (integer ratings, <= 16 distinct values) must
    equal the ordered-fp64 kernel byte for byte, including the counter-overflow fold."""

    def _fp64(self, P, r, c):
        from paper_2111_11682_b200 import _native as nat
        dev = r.device()
        h = P.assign_row_hashes(r.M, c)
        acc = nat.zeros((r.N * c.q * c.p * c.G,), "float64")
        nat.call("culsh_hash_accumulate", nat.ptr(dev.col_ptr), nat.ptr(dev.col_rows),
                 nat.ptr(dev.col_vals), 0, r.N, None, nat.ptr(h.table()), c.q, c.p, c.G,
                 c.psi_exponent, 0, 0, nat.ptr(acc), None, None, r.N, nat.stream_ptr())
        return nat.to_host(acc)

    @pytest.mark.parametrize("G,p,q,e,nvals", [(8, 3, 100, 2, 5), (5, 2, 4, 4, 16), (16, 2, 6, 1, 9),
                                                (4, 4, 10, 2, 17)])
    def test_matches_fp64(self, P, G, p, q, e, nvals):
        from paper_2111_11682_b200 import lsh as L
        rng = np.random.default_rng(G * 100 + nvals)
        M, N = 700, 90
        mask = rng.random((M, N)) < 0.2
        rows, cols = np.nonzero(mask)
        vals = rng.integers(1, nvals + 1, len(rows)).astype(float) - (nvals // 3)
        r = P.SparseRatings(M, N, rows, cols, vals)
        c = P.LshConfig(G=G, p=p, q=q, psi_exponent=e, seed=3)
        st = P.compute_hash_state(r, c)
        uses_count = (nvals <= 16) and ((q * p * ((G + 7) // 8)) % 4 == 0)
        assert (L._value_classes(r.device()) is not None) == (nvals <= 16)
        assert st.acc.tobytes() == self._fp64(P, r, c).tobytes(), uses_count

    def test_counter_fold_long_column(self, P):
        M = 300_000                   # one class > 16*(2^14-1) ratings in column 0
        rows = np.concatenate([np.arange(M), np.arange(0, M, 7)])
        cols = np.concatenate([np.zeros(M, np.int64), np.ones(len(rows) - M, np.int64)])
        vals = np.concatenate([np.full(M, 3.0), np.full(len(rows) - M, 5.0)])
        vals[::1000] = 1.0
        r = P.SparseRatings(M, 2, rows, cols, vals)
        c = P.LshConfig(G=8, p=2, q=2, psi_exponent=2, seed=0)
        assert P.compute_hash_state(r, c).acc.tobytes() == self._fp64(P, r, c).tobytes()


class TestStageApis:
    """coarse_candidates / fine_topk (lsh.py:290-305, 377-398) as in test_lsh.py:111-257."""

    def test_equal_signatures_bucket_together(self, P):
        sig = np.zeros((3, 4), dtype=np.uint8)
        sig[2, 1] = 1
        out = P.coarse_candidates([sig])
        assert list(out[0]) == [1] and list(out[1]) == [0] and list(out[2]) == []

    def test_any_differing_bit_separates(self, P):
        s1 = np.zeros((2, 4), dtype=np.uint8)
        s2 = np.zeros((2, 4), dtype=np.uint8)
        s2[1, 3] = 1
        out = P.coarse_candidates([s1, s2])
        assert list(out[0]) == [] and list(out[1]) == []

    def test_fine_topk_rules(self, P):
        groups = [[np.array([5, 2]), *[np.array([], int)] * 9],
                  [np.array([5, 2, 7]), *[np.array([], int)] * 9],
                  [np.array([5]), *[np.array([], int)] * 9]]
        assert list(P.fine_topk(groups, K=2, N=10, seed=0).entries[0]) == [5, 2]
        assert P.fine_topk([[np.array([7, 3]), *[np.array([], int)] * 9]], K=1, N=10, seed=0).entries[0, 0] == 3
        t = P.fine_topk([[np.array([4]), *[np.array([], int)] * 4]], K=3, N=5, seed=1)
        assert t.entries[0, 0] == 4 and len(set(t.entries[0])) == 3 and 0 not in t.entries[0]
        P.fine_topk([[np.array([], int)] * 6], K=3, N=6, seed=2).validate()
        with pytest.raises(ValueError):
            P.fine_topk([[np.array([], int)] * 3], K=3, N=3, seed=0)

    def test_pipeline_equals_composition(self, P):
        # test_lsh.py:233-257: one call == per-map signatures -> per-group buckets -> top-K
        rng = np.random.default_rng(42)
        mask = rng.random((12, 9)) < 0.5
        rows, cols = np.nonzero(mask)
        r = P.SparseRatings(12, 9, rows, cols, rng.integers(1, 6, len(rows)).astype(float))
        cfg = P.LshConfig(G=5, p=2, q=3, psi_exponent=2, seed=8)
        table, state = P.simlsh_topk(r, cfg, K=3)
        hashes = P.assign_row_hashes(r.M, cfg)
        groups = []
        for g in range(cfg.q):
            sigs = []
            for m in range(cfg.p):
                H = hashes.map_bits(g, m)
                sigs.append(np.stack([P.simlsh_signature(j, r, H, cfg.psi_exponent)[1]
                                      for j in range(r.N)]))
            groups.append(P.coarse_candidates(sigs))
        composed = P.fine_topk(groups, K=3, N=r.N, seed=cfg.seed)
        np.testing.assert_array_equal(composed.entries, table.entries)


class TestTrainBasic:
    """train_basic (CUSGD++ basic MF, factorization.py:476-527): the serial mode must
    equal the reference bit for bit; the racy (Hogwild) mode must train comparably."""

    def test_serial_bit_exact(self, P):
        z = load_golden("basic.npz")
        for s in range(int(z["n_cases"])):
            pre = f"b{s}_"
            F, epochs, seed, wb, srt = (int(x) for x in z[pre + "cfg"])
            r = ratings_of(P, z, pre)
            cfg = P.TrainConfig(F=F, K=0, epochs=epochs, seed=seed, alpha_u=0.04, alpha_v=0.04,
                                lambda_u=0.035, lambda_v=0.035)
            p = P.train_basic(r, cfg, with_biases=bool(wb), sort_rows_by_count=bool(srt))
            for n in ("b", "b_hat", "U", "V"):
                assert getattr(p, n).tobytes() == z[f"{pre}{n}"].tobytes(), (s, n)

    def test_racy_mode_trains(self, P, c1):
        z, tr, te = c1
        cfg = P.TrainConfig(F=32, K=0, alpha_u=0.04, alpha_v=0.04, lambda_u=0.035, lambda_v=0.035,
                            epochs=20, seed=0)
        exact = P.rmse(P.train_basic(tr, cfg, with_biases=True), te, tr)
        racy = P.rmse(P.train_basic(tr, cfg, with_biases=True, racy_workers=4), te, tr)
        assert abs(racy - exact) <= REF_TOL_RMSE, (racy, exact)


class TestOnlineSession:
    """Device-resident online session (append instead of rebuild) == the reference's
    absorb_increment, bit for bit, on integer-valued data (golden fixtures)."""

    @pytest.mark.parametrize("s", [0, 2])
    def test_matches_reference(self, P, s):
        from paper_2111_11682_b200.online_device import OnlineSession
        from paper_2111_11682_b200 import lsh as L
        z = load_golden("online_small.npz")
        pre = f"o{s}_"
        G, p_, q, e, lseed = (int(x) for x in z[pre + "lsh"])
        F, K, epochs, seed = (int(x) for x in z[pre + "cfg"])
        orig = ratings_of(P, z, pre)
        lc = P.LshConfig(G=G, p=p_, q=q, psi_exponent=e, seed=lseed)
        cfg = P.TrainConfig(F=F, K=K, epochs=epochs, seed=seed)
        ent, state, _ = L.simlsh_topk_device(orig.device(), lc, K)
        tbl = P.NeighborTable(orig.N, K, P._native.to_host(ent)[:orig.N * K].reshape(orig.N, K))
        params = P.train_full(orig, tbl, cfg)
        sess = OnlineSession(orig.device(), state, ent, K, params, cfg)
        bM, bN, nr_, nc_ = (int(x) for x in z[pre + "b_shape"])
        batch = P.IncrementBatch(bM, bN, nr_, nc_, z[pre + "b_rows"], z[pre + "b_cols"], z[pre + "b_vals"])
        tm = sess.absorb(batch)
        assert tm["total"] > 0
        assert sess.state.acc.tobytes() == z[pre + "ext_acc"].tobytes()
        pe = sess.to_params()
        assert pe.neighbors.entries.tobytes() == z[pre + "ext_entries"].tobytes()
        for n in ("b", "b_hat", "U", "V", "W", "C"):
            assert getattr(pe, n).tobytes() == z[f"{pre}ext_{n}"].tobytes(), n
        # the appended index views, csc2csr map and baselines == a from-scratch build
        nat = P._native
        full = P.extend_ratings(orig, batch).device()
        d = sess.dev
        for a in ("col_ptr", "col_rows", "col_vals", "row_ptr", "row_cols", "row_vals", "csc2csr",
                  "base_b", "base_bhat"):
            assert nat.to_host(getattr(d, a)).tobytes() == nat.to_host(getattr(full, a)).tobytes(), a
        assert d.mu == full.mu


# -------------------------------------------------------- GSM similarity ---

def _sim_ratings(P, z, pre):
    return P.SparseRatings(int(z[pre + "M"]), int(z[pre + "N"]), z[pre + "rows"], z[pre + "cols"],
                           z[pre + "vals"])


class TestGsm:
    """GPU exact similarity (similarity.py) against the reference's own outputs
    (tests/golden/similarity.npz): bit-exact similarities, identical top-K tables
    by both the count (int8 tensor-core GEMM) and the merge route."""

    def test_pearson_shrunk_bitwise(self, P):
        z = load_golden("similarity.npz")
        for name in ("int", "real"):
            r = _sim_ratings(P, z, name + "_")
            Pm, Sm = z[name + "_pearson"], z[name + "_shrunk25"]
            for a in range(0, r.N, 3):
                for b in range(r.N):
                    if a != b:
                        assert P.pearson(r, a, b) == Pm[a, b], (name, a, b)
                        assert P.shrunk_similarity(r, a, b, 25.0) == Sm[a, b], (name, a, b)
        with pytest.raises(ValueError):
            P.pearson(r, 1, 1)

    def test_gsm_small_cases_both_routes(self, P):
        z = load_golden("similarity.npz")
        n_count = 0
        for name in z["cases"]:
            r = _sim_ratings(P, z, str(name) + "_")
            integral = bool(np.all(r.col_vals == np.round(r.col_vals)))
            for key in z.files:
                if not key.startswith(f"{name}_gsm_K"):
                    continue
                K = int(key.split("_K")[1].split("_")[0])
                cfg = P.SimilarityConfig(K=K, lambda_rho=float(key.split("_l")[1]))
                assert np.array_equal(P.gsm_topk(r, cfg, method="merge").entries, z[key]), key
                if integral:
                    assert np.array_equal(P.gsm_topk(r, cfg, method="count").entries, z[key]), key
                    n_count += 1
        assert n_count >= 20
        with pytest.raises(ValueError):
            P.gsm_topk(_sim_ratings(P, z, "real_"), P.SimilarityConfig(K=3), method="count")

    def test_gsm_c1(self, P):
        z = load_golden("similarity.npz")
        r = _sim_ratings(P, z, "c1_")
        for meth in ("count", "merge"):
            assert np.array_equal(P.gsm_topk(r, P.SimilarityConfig(K=16), method=meth).entries,
                                  z["c1_gsm_K16"]), meth
            assert np.array_equal(P.gsm_topk(r, P.SimilarityConfig(K=32, lambda_rho=50.0), method=meth).entries,
                                  z["c1_gsm_K32_l50"]), meth

    @pytest.mark.parametrize("ld,w,passes", [(128, 64, 1), (384, 1024, 1), (1664, 192, 2), (256, 4096, 3)])
    def test_gsm_stats_tc_products(self, P, ld, w, passes):
        """culsh_gsm_stats_tc (tcgen05 kind::i8, TMEM accumulators) == the four int32
        products computed independently (torch integer matmul in int64), with row-pass
        accumulation; 1664 = 13 blocks -> 169 tiles, more than one tile per CTA."""
        import torch
        from paper_2111_11682_b200 import _native as nat
        gen = torch.Generator().manual_seed(ld + w)
        g = torch.zeros((6, ld, ld), dtype=torch.int32, device="cuda")
        want = torch.zeros((6, ld, ld), dtype=torch.int64)
        for ps in range(passes):
            pan = torch.randint(-11, 12, (3, ld, w), generator=gen, dtype=torch.int8)
            pan[0] = (pan[0] > 0).to(torch.int8)           # indicator
            pan[2] = (pan[1].to(torch.int16) ** 2).to(torch.int8)   # squares <= 121
            x, r, q = (pan[i].to(torch.int64) for i in range(3))
            want[0] += x @ x.T
            want[1] += r @ x.T
            want[2] += r @ r.T
            want[3] += q @ x.T
            want[4] += x @ r.T          # transposed copies for the select kernel
            want[5] += x @ q.T
            dpan = pan.cuda()
            tiles = torch.empty_like(dpan)
            nat.call("culsh_gsm_tile_panels", nat.ptr(dpan), ld, w, nat.ptr(tiles), nat.stream_ptr())
            nat.call("culsh_gsm_stats_tc", nat.ptr(tiles), ld, w, int(ps > 0), nat.ptr(g[0]), nat.ptr(g[1]),
                     nat.ptr(g[2]), nat.ptr(g[3]), nat.ptr(g[4]), nat.ptr(g[5]), nat.stream_ptr())
        torch.cuda.synchronize()
        got = g.cpu().to(torch.int64)
        for i, name in enumerate(("xx", "rx", "rr", "qx", "xr", "xq")):
            assert torch.equal(got[i], want[i]), name

    @pytest.mark.parametrize("K", [50, 100])
    def test_gsm_large_k_vs_oracle(self, P, orc, K):
        """K > 32 (two / four top-K entries per lane in the warp select): count route ==
        merge route == oracle."""
        rng = np.random.default_rng(K)
        M, N = 3000, 160
        mask = rng.random((M, N)) < 0.05
        rows, cols = np.nonzero(mask)
        r = P.SparseRatings(M, N, rows, cols, rng.integers(1, 6, len(rows)).astype(np.float64))
        cfg = P.SimilarityConfig(K=K, lambda_rho=10.0)
        a = P.gsm_topk(r, cfg, method="count").entries
        assert np.array_equal(a, P.gsm_topk(r, cfg, method="merge").entries)
        assert np.array_equal(a, orc.gsm_topk(r.col_ptr, r.col_rows, r.col_vals, N, K, 10.0))

    def test_gsm_mid_scale_vs_oracle(self, P, orc):
        """20,000 x 3,000, ~600k integer ratings: count route == merge route == oracle."""
        rng = np.random.default_rng(7)
        M, N, nnz = 20000, 3000, 600000
        key = np.unique(rng.integers(0, M * N, nnz))
        rows, cols = (key % M).astype(np.int32), (key // M).astype(np.int32)
        vals = rng.integers(1, 6, len(key)).astype(np.float64)
        r = P.SparseRatings(M, N, rows, cols, vals)
        cfg = P.SimilarityConfig(K=32)
        a = P.gsm_topk(r, cfg, method="count").entries
        b = P.gsm_topk(r, cfg, method="merge").entries
        assert np.array_equal(a, b)
        ref = orc.gsm_topk(r.col_ptr, r.col_rows, r.col_vals, N, 32, 100.0)
        assert np.array_equal(a, ref)


def test_hash_state_file_bytes_match_reference(P, tmp_path):
    """compute_hash_state on the GPU + HashState.save == the reference's file bytes
    (lsh.py:209-216), and load re-thresholds to the same state."""
    z = load_golden("similarity.npz")
    r = _sim_ratings(P, z, "int_")
    hs = P.compute_hash_state(r, P.LshConfig(G=8, p=3, q=7, psi_exponent=2, seed=4))
    hs.save(tmp_path / "h.bin")
    assert (tmp_path / "h.bin").read_bytes() == z["hs_bytes"].tobytes()
    back = P.HashState.load(tmp_path / "h.bin")
    assert back.sig.tobytes() == hs.sig.tobytes()


class TestEdgeCases:
    def test_gsm_empty_columns_negative_values_full_k(self, P, orc):
        """Empty columns, negative integer ratings, K = N-1: both GSM routes == oracle."""
        rng = np.random.default_rng(9)
        M, N = 120, 24
        mask = rng.random((M, N)) < 0.3
        mask[:, [3, 17]] = False                      # two empty columns
        rows, cols = np.nonzero(mask)
        vals = rng.integers(-11, 12, len(rows)).astype(float)
        r = P.SparseRatings(M, N, rows, cols, vals)
        for K in (1, N - 1):
            ref = orc.gsm_topk(r.col_ptr, r.col_rows, r.col_vals, N, K, 100.0)
            for meth in ("count", "merge"):
                got = P.gsm_topk(r, P.SimilarityConfig(K=K), method=meth).entries
                assert np.array_equal(got, ref), (K, meth)

    def test_hogwild_empty_columns_and_rows(self, P):
        """Empty columns / rows in every Hogwild stream form: parameters of untouched
        columns keep their initial values except regularisation-free ones, and the
        packed kernel equals the wide kernel."""
        import torch
        from paper_2111_11682_b200.hogwild import HogwildTrainer
        rng = np.random.default_rng(4)
        M, N = 400, 60
        mask = rng.random((M, N)) < 0.1
        mask[:, [0, 31, 59]] = False
        mask[[5, 77], :] = False
        rows, cols = np.nonzero(mask)
        r = P.SparseRatings(M, N, rows, cols, rng.integers(1, 6, len(rows)).astype(float))
        tbl, _ = P.simlsh_topk(r, P.LshConfig(q=20), 8)
        cfg = P.TrainConfig(F=64, K=8, epochs=2, seed=0)
        out = []
        for packed in (True, False):
            tr = HogwildTrainer(r, tbl, cfg, packed=packed)
            for t in range(2):
                for j in range(N):
                    tr.launch_epoch(t, col_order=torch.tensor([j], dtype=torch.int32, device="cuda"), n_cols=1)
            torch.cuda.synchronize()
            assert int(tr.status.item()) == 0
            out.append(tr.to_params())
        init = P.init_params(M, N, 64, 8, tbl, r.baselines(), cfg)
        for p in out:
            assert np.allclose(p.V[[0, 31, 59]], init.V[[0, 31, 59]].astype(np.float32))
            assert np.allclose(p.U[[5, 77]], init.U[[5, 77]].astype(np.float32))
        for name in ("b", "b_hat", "U", "V", "W", "C"):
            assert getattr(out[0], name).tobytes() == getattr(out[1], name).tobytes(), name


@pytest.fixture(scope="module")
def api_case(P):
    z = load_golden("api.npz")
    M, N = (int(x) for x in z["orig_shape"])
    orig = P.SparseRatings(M, N, z["orig_rows"], z["orig_cols"], z["orig_vals"])
    tbl = P.NeighborTable(N, 5, z["table"])
    p = P.ModelParams(float(z["p_mu"]), z["p_b"].copy(), z["p_b_hat"].copy(), z["p_U"].copy(),
                      z["p_V"].copy(), z["p_W"].copy(), z["p_C"].copy(), tbl)
    s = z["b_shape"]
    batch = P.IncrementBatch(int(s[0]), int(s[1]), int(s[2]), int(s[3]), z["b_rows"], z["b_cols"],
                             z["b_vals"])
    lc = P.LshConfig(G=6, p=2, q=5, psi_exponent=2, seed=3)
    cfg = P.TrainConfig(F=4, K=5, epochs=3, seed=2)
    return z, orig, tbl, p, batch, lc, cfg


class TestApiGolden:
    """Public functions called standalone vs the reference's outputs on stored inputs
    (tests/golden/api.npz, tests/golden/make_golden_api.py), bit for bit."""

    def test_baselines_predict_split_objective(self, P, api_case):
        z, orig, tbl, p, batch, lc, cfg = api_case
        st = P.compute_baselines(orig)
        assert st.mu == float(z["base_mu"]) and st.b.tobytes() == z["base_b"].tobytes()
        assert st.b_hat.tobytes() == z["base_bhat"].tobytes()
        pairs = z["pairs"]
        pred = np.array([P.predict(int(i), int(j), p, orig) for i, j in pairs])
        assert pred.tobytes() == z["pred"].tobytes()
        pc = np.array([P.predict(int(i), int(j), p, orig, clamp=(2.0, 4.0)) for i, j in pairs])
        assert pc.tobytes() == z["pred_clamped"].tobytes()
        for (i, j), m in zip(pairs, z["split_explicit"]):
            s = P.split_neighbors(int(i), int(j), tbl, orig)
            assert np.array_equal(np.flatnonzero(m), s.explicit)
            assert np.array_equal(np.flatnonzero(m == 0), s.implicit)
        assert P.objective_value(p, orig, cfg.regs) == float(z["objective"])

    def test_sgd_update(self, P, api_case):
        z, orig, tbl, p, batch, lc, cfg = api_case
        q = p.copy()
        i0, j0 = (int(x) for x in z["sgd_ij"])
        err = P.sgd_update(i0, j0, q, tuple(z["sgd_rates"]), cfg.regs, orig)
        assert err == float(z["sgd_err"])
        for k in ("b", "b_hat", "U", "V", "W", "C"):
            assert getattr(q, k).tobytes() == z["sgd_" + k].tobytes(), k

    def test_parallel_train_instrumented(self, P, api_case):
        z, orig, tbl, p, batch, lc, cfg = api_case
        pp, rep = P.parallel_train(orig, tbl, cfg, 3, instrument=True)
        assert [rep.stages_checked, rep.disjoint_violations, rep.epochs_checked,
                rep.coverage_violations] == list(z["instr"])
        assert rep.ok
        assert pp.U.tobytes() == z["par_U"].tobytes()

    def test_online_stages_standalone(self, P, api_case):
        z, orig, tbl, p, batch, lc, cfg = api_case
        state = P.compute_hash_state(orig, lc)
        hashes = P.assign_row_hashes(batch.M_hat, lc)
        se = P.update_hashes_incremental(state, batch, hashes)
        assert se.acc.tobytes() == z["inc_acc"].tobytes()
        ne = P.topk_for_new(se, tbl, 5, lc.seed)
        assert np.array_equal(ne.entries, z["new_entries"])
        re_ = P.extend_ratings(orig, batch)
        assert np.array_equal(re_.entry_rows, z["ext_rows"]) and np.array_equal(re_.entry_cols, z["ext_cols"])
        assert re_.entry_values.tobytes() == z["ext_vals"].tobytes()
        pe = P.extend_params(p, batch, ne, cfg)
        for k in ("b", "b_hat", "U", "V", "W", "C"):
            assert getattr(pe, k).tobytes() == z["extp_" + k].tobytes(), k
        pt = P.train_incremental(pe, batch, ne, re_, cfg)
        assert (pt is pe) == bool(z["inc_in_place"])          # trains its argument in place
        for k in ("b", "b_hat", "U", "V", "W", "C"):
            assert getattr(pt, k).tobytes() == z["inc_" + k].tobytes(), k


@pytest.mark.parametrize("F,K", [(8, 8), (32, 48), (256, 64), (50, 16), (96, 32), (200, 8)])
def test_hogwild_shapes_c1(P, c1, F, K):
    """Every Hogwild kernel instantiation family (F < 32 masked lanes, K > 32 two mask
    words, F = 256) and the zero-padded widths (F = 50 / 96 / 200 run as 64 / 128 / 256)
    train to the exact mode's test RMSE within the 0.005 bar."""
    z, tr, te = c1
    nbr = P.NeighborTable(tr.N, 32, z["lsh_entries32"])
    if K != 32:
        tbl, _ = P.simlsh_topk(tr, P.LshConfig(), K)
        nbr = tbl
    cfg = P.TrainConfig(F=F, K=K, epochs=12, seed=0)
    exact = P.rmse(P.train_full(tr, nbr, cfg), te, tr)
    ph = P.train_full(tr, nbr, cfg, mode="hogwild")
    hog = P.rmse(ph, te, tr)
    assert abs(hog - exact) <= REF_TOL_RMSE, (F, K, hog, exact)
    assert ph.U.shape == (tr.M, F) and ph.V.shape == (tr.N, F)
    if F in (50, 96, 200):    # padded storage: the extra features stay exactly zero
        m = ph._dev
        U = m.U[:tr.M * m.Fp].view(tr.M, m.Fp)[:, F:]
        assert m.Fp > F and bool((U == 0).all())
        ph.U[0, :] = 0.5                           # a host edit reaches the padded device copy
        j = int(tr.row_cols[0])
        assert P.predict(0, j, ph, tr) == P.predict(0, j, ph.copy(), tr)


@pytest.mark.parametrize("work", [False, True])
def test_hogwild_dsgd_stages_c1(P, c1, work):
    """The multi-GPU DSGD performance path (dsgd.bench_main): each stage runs the Hogwild
    kernel on (row block, column block) entry ranges from culsh_pass_plan.  Here one process
    runs every rank's block of a stage in one launch; the D stages cover every rating once
    per epoch and the fit lands within the RMSE bar of the exact mode."""
    import torch
    from paper_2111_11682_b200 import _native as nat
    from paper_2111_11682_b200.dsgd import RingPlan
    from paper_2111_11682_b200.hogwild import HogwildTrainer
    z, tr, te = c1
    nbr = P.NeighborTable(tr.N, 32, z["lsh_entries32"])
    cfg = P.TrainConfig(F=32, K=32, epochs=12, seed=0)
    exact = P.rmse(P.train_full(tr, nbr, cfg), te, tr)
    D = 3
    ht = HogwildTrainer(tr, nbr, cfg)
    d = ht.dev
    M, N = d.M, d.N
    plan = RingPlan(D, M, N)
    rb_t = nat.to_dev(plan.row_bounds)
    bp = nat.empty((N * (D + 1),), "int64")
    nat.call("culsh_block_pointers", nat.ptr(d.col_ptr), nat.ptr(d.col_rows), N, nat.ptr(rb_t), D + 1,
             nat.ptr(bp), nat.stream_ptr())
    cbt = nat.to_dev(plan.col_bounds)
    segs = []
    for s in range(D):
        seg = nat.zeros((2 * N,), "int64")
        chain = nat.zeros((N,), "int32")
        nat.call("culsh_pass_plan", nat.ptr(d.col_ptr), nat.ptr(d.col_rows), N, 1, 0, N, 0, M,
                 nat.ptr(bp), nat.ptr(cbt), D, s, nat.ptr(seg), nat.ptr(chain), nat.stream_ptr())
        segs.append(seg)
    sh = nat.to_host
    covered = sum(sh(sg)[1::2].astype(np.int64) - sh(sg)[0::2] for sg in segs)
    assert np.array_equal(covered, np.diff(sh(d.col_ptr)))          # every rating once per epoch
    cols = torch.arange(N, dtype=torch.int32, device="cuda")
    if work:   # block_work lists (packed stream; C1 has fewer columns than warps: split)
        works = [ht.block_work(sg, cols) for sg in segs]
        assert all(w["split_cols"] > 0 for w in works)
    for ep in range(cfg.epochs):
        for s in range(D):
            if work:
                ht.launch_work(ep, works[s])
            else:
                ht.launch_epoch(ep, seg=segs[s], col_order=cols, n_cols=N)
    assert int(ht.status.item()) == 0
    hog = P.rmse(ht.to_params(), te, tr)
    assert abs(hog - exact) <= REF_TOL_RMSE, (hog, exact)


def test_hogwild_divergence_raises(P):
    """A diverging Hogwild fit (non-finite partials take the fp32 shuffle reduction, not the
    fixed-point redux) raises TrainingDivergedError like the exact modes."""
    rng = np.random.default_rng(42)
    mask = rng.random((40, 30)) < 0.5
    rows, cols = np.nonzero(mask)
    r = P.SparseRatings(40, 30, rows, cols, rng.integers(1, 6, len(rows)).astype(float))
    ent = np.stack([np.delete(np.arange(30), j)[:4] for j in range(30)]).astype(np.int32)
    cfg = P.TrainConfig(F=128, K=4, alpha_b=1e12, alpha_b_hat=1e12, alpha_u=1e12, alpha_v=1e12,
                        alpha_w=1e12, alpha_c=1e12, epochs=3, seed=1)
    with pytest.raises(P.TrainingDivergedError):
        P.train_full(r, P.NeighborTable(30, 4, ent), cfg, mode="hogwild")


def test_hogwild_large_magnitude_ratings(P, c1):
    """Ratings on a 0-100 scale (the Yahoo-style values of C5): per-lane partial sums can
    leave the fixed-point reduction's +-32 window, where the kernel falls back to the fp32
    shuffle tree; Hogwild still lands within the tolerance (scaled by 20) of the exact fit."""
    z, tr, te = c1
    s = 20.0
    tr2 = P.SparseRatings(tr.M, tr.N, z["train_rows"].astype(np.int32), z["train_cols"].astype(np.int32),
                          z["train_vals"].astype(np.float64) * s)
    te2 = P.Triplets(te.rows, te.cols, te.values * s)
    nbr = P.NeighborTable(tr.N, 32, z["lsh_entries32"])
    cfg = P.TrainConfig(F=128, K=32, epochs=8, seed=0, alpha_b=0.002, alpha_b_hat=0.002, alpha_u=0.002,
                        alpha_v=0.002, alpha_w=0.0001, alpha_c=0.0001)
    exact = P.rmse(P.train_full(tr2, nbr, cfg), te2, tr2)
    hog = P.rmse(P.train_full(tr2, nbr, cfg, mode="hogwild"), te2, tr2)
    assert np.isfinite(hog) and abs(hog - exact) <= REF_TOL_RMSE * s, (hog, exact)


@pytest.mark.parametrize("F,K", [(128, 40), (256, 64), (1, 1)])
def test_exact_mode_large_shapes_vs_oracle(P, orc, F, K):
    """Exact mode at shapes the reference fixtures do not reach (F up to 256, K > 32 with
    two mask words, F = K = 1): bit-identical to the oracle (itself pinned to the
    reference)."""
    rng = np.random.default_rng(F + K)
    M, N = 90, 70
    mask = rng.random((M, N)) < 0.2
    rows, cols = np.nonzero(mask)
    vals = rng.integers(1, 6, len(rows)).astype(float)
    r = P.SparseRatings(M, N, rows, cols, vals)
    tbl = P.random_topk(N, K, seed=1)
    tc = P.TrainConfig(F=F, K=K, epochs=2, seed=3)
    p = P.train_full(r, tbl, tc)
    d, mu = orc.build_csr(M, N, rows, cols, vals)
    m = orc.train_full(d, mu, tbl.entries, F, K, 2, 3, tc.rates_at, tc.regs)
    assert p.U.tobytes() == m.U.tobytes() and p.V.tobytes() == m.V.tobytes()
    assert p.W.tobytes() == m.W.tobytes() and p.C.tobytes() == m.C.tobytes()
    assert p.b.tobytes() == m.b.tobytes() and p.b_hat.tobytes() == m.bhat.tobytes()


@pytest.fixture(scope="module")
def c2_uniform(P):
    from paper_2111_11682_b200 import _native as nat, synth
    M, N, nnz, F, K, e = synth.SHAPES["c2"]
    dm = synth.random_sparse_device(M, N, nnz, seed=0)
    d = dm.dev
    return dm, (nat.to_host(d.col_ptr), nat.to_host(d.col_rows), nat.to_host(d.col_vals)), (M, N, F, K, e)


class TestAtScaleVsOracle:
    """Full C2-shape parity (20M ratings), where no reference fixture exists: the GPU
    against the oracle (pinned to the reference) on the same device-generated matrix."""

    def test_simlsh_topk_c2_bit_exact(self, P, orc, c2_uniform):
        from paper_2111_11682_b200 import _native as nat, lsh
        dm, (cp, cr, cv), (M, N, F, K, e) = c2_uniform
        ent, state, _ = lsh.simlsh_topk_device(dm.dev, P.LshConfig(psi_exponent=e, seed=0), K)
        ref = orc.simlsh_topk(cp, cr, cv, M, 8, 3, 100, e, 0, K)
        assert state.acc.tobytes() == ref.acc.tobytes()
        assert state.sig.tobytes() == ref.sig.tobytes()
        assert np.array_equal(nat.to_host(ent)[:N * K].reshape(N, K), ref.entries)

    def test_dsgd_epoch_c2_bit_exact(self, P, orc, c2_uniform):
        """parallel_train(D=16), one exact epoch at C2 scale == the oracle's parallel_epoch."""
        import torch
        from paper_2111_11682_b200 import _native as nat, lsh
        from paper_2111_11682_b200.data import DeviceSparseRatings
        dm, (cp, cr, cv), (M, N, F, K, e) = c2_uniform
        d = dm.dev
        col = torch.repeat_interleave(torch.arange(N, device="cuda"), d.col_ptr[1:] - d.col_ptr[:-1]).to(torch.int32)
        r = DeviceSparseRatings(M, N, d.col_rows, col, d.col_vals)
        ent, _, _ = lsh.simlsh_topk_device(r.device(), P.LshConfig(psi_exponent=e), K)
        nbr = P.NeighborTable(N, K, nat.to_host(ent)[:N * K].reshape(N, K))
        cfg = P.TrainConfig(F=F, K=K, epochs=1, seed=0)
        p = P.parallel_train(r, nbr, cfg, 16)
        rows = np.repeat(np.arange(N, dtype=np.int32), np.diff(cp))
        csr, mu = orc.build_csr(M, N, cr, rows, cv)
        m = orc.parallel_train(csr, mu, nbr.entries, F, K, 1, 0, cfg.rates_at, cfg.regs, 16)
        assert p.U.tobytes() == m.U.tobytes() and p.V.tobytes() == m.V.tobytes()
        assert p.W.tobytes() == m.W.tobytes() and p.C.tobytes() == m.C.tobytes()


def test_api_edge_behaviour_matches_reference(P):
    """Small-edge behaviour of the public API, as the reference behaves (recorded from
    lshmf on the same 3x2 matrix): tiny top-K tables, K > N-1, K = 0, zero epochs, empty
    test set, out-of-range predict, config validation, D out of range."""
    r = P.build_indices(P.Triplets(np.array([0, 1, 2]), np.array([0, 1, 0]), np.array([3., 4., 5.])), M=3, N=2)
    tbl, _ = P.simlsh_topk(r, P.LshConfig(q=4), 1)
    assert tbl.entries.tolist() == [[1], [0]]
    with pytest.raises(ValueError):
        P.simlsh_topk(r, P.LshConfig(q=4), 2)
    assert P.train_full(r, None, P.TrainConfig(F=3, K=0, epochs=2)).U.shape == (3, 3)
    assert P.train_full(r, None, P.TrainConfig(F=3, K=0, epochs=0)).U.shape == (3, 3)
    p = P.train_full(r, None, P.TrainConfig(F=3, K=0, epochs=1))
    with pytest.raises(ValueError):
        P.rmse(p, P.Triplets(np.array([], int), np.array([], int), np.array([])), r)
    with pytest.raises(IndexError):
        P.predict(5, 0, p, r)
    assert P.gsm_topk(r, P.SimilarityConfig(K=1)).entries.tolist() == [[1], [0]]
    with pytest.raises(ValueError):
        P.LshConfig(G=65).validate()
    for D in (0, 5):
        with pytest.raises(ValueError):
            P.parallel_train(r, None, P.TrainConfig(F=3, K=0, epochs=1), D)
