"""Pin the CPU oracle (oracle/) to the reference: golden fixtures produced by the
unmodified reference package (tests/golden/make_golden.py) and the reference's own
known-answer tests (cited per test).  CPU only."""

import numpy as np
import pytest

from conftest import load_golden, sha


def _csr(orc, z, pre):
    d, mu = orc.build_csr(int(z[pre + "M"]), int(z[pre + "N"]), z[pre + "rows"], z[pre + "cols"],
                          z[pre + "vals"])
    return d, mu


def _rates(alpha=(0.035, 0.035, 0.035, 0.035, 0.002, 0.002), beta=0.3):
    return lambda t: tuple(a / (1.0 + beta * t ** 1.5) for a in alpha)


REGS = (0.02, 0.02, 0.02, 0.02, 0.002, 0.002)


class TestHashKat:
    def test_splitmix_known(self, orc):
        # lsh.py:465-469 restated in Python integers is the definition
        def sm(x):
            m = 0xFFFFFFFFFFFFFFFF
            z = (x + 0x9E3779B97F4A7C15) & m
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
            return (z ^ (z >> 31)) & m
        for x in (0, 1, 2, 12345, 2**63, 2**64 - 1):
            assert orc.splitmix64(x) == sm(x)

    def test_worked_example_fig3(self, orc):
        # test_lsh.py:63-66 / test_acceptance.py:111-118: acc (-2,-4,-6), sig 000
        bits = np.array([[0, 0, 1], [0, 1, 0], [1, 0, 0]], np.uint8).reshape(3, 1, 1, 3)
        acc = orc.accumulate_all(np.array([0, 3]), np.array([0, 1, 2]), np.array([3., 4., 5.]),
                                 bits, 1)
        np.testing.assert_array_equal(acc.ravel(), [-2.0, -4.0, -6.0])
        np.testing.assert_array_equal(orc.threshold(acc).ravel(), [0, 0, 0])

    def test_empty_column_all_ones(self, orc):
        # test_lsh.py:68-72
        bits = np.zeros((3, 1, 1, 3), np.uint8)
        acc = orc.accumulate_all(np.array([0, 0]), np.zeros(0, np.int32), np.zeros(0), bits, 1)
        np.testing.assert_array_equal(orc.threshold(acc).ravel(), [1, 1, 1])

    def test_psi_exponents(self, orc):
        # test_lsh.py:79-84
        bits = np.ones((1, 1, 1, 2), np.uint8)
        for e, want in [(1, 3.0), (2, 9.0), (4, 81.0)]:
            acc = orc.accumulate_all(np.array([0, 1]), np.array([0]), np.array([3.0]), bits, e)
            assert acc.ravel()[0] == want

    def test_incremental_hand_case(self, orc):
        # test_online.py:64-76: (-2,-4,-6) + 10 with row hash 111 -> (8,6,4)
        acc = np.array([-2.0, -4.0, -6.0]).reshape(1, 1, 1, 3)
        bits = np.zeros((4, 1, 1, 3), np.uint8)
        bits[3] = 1
        orc.accumulate_into(acc, np.array([0, 1]), np.array([3]), np.array([10.0]), bits, 1)
        np.testing.assert_array_equal(acc.ravel(), [8.0, 6.0, 4.0])

    def test_row_hash_prefix_and_balance(self, orc):
        # test_lsh.py:32-59
        a = orc.assign_bits(11, 3, 2, 50, 8)
        b = orc.assign_bits(11, 3, 2, 80, 8)
        np.testing.assert_array_equal(a, b[:50])
        h = orc.assign_bits(0, 2, 2, 10_000, 8)
        frac = h.reshape(10_000, -1).mean(axis=0)
        assert frac.min() >= 0.48 and frac.max() <= 0.52

    def test_topk_frequency_and_ties(self, orc):
        # test_lsh.py:153-169 through keys: columns 5 and 2 share buckets with 0
        q, N = 3, 10
        keys = np.arange(q * N, dtype=np.uint64).reshape(q, N) + 1000
        keys[0, [0, 5, 2]] = 1
        keys[1, [0, 5, 2, 7]] = 2
        keys[2, [0, 5]] = 3
        ent, total = orc.topk_from_group_keys(keys, 2, 0)
        assert list(ent[0]) == [5, 2]
        keys = np.arange(N, dtype=np.uint64).reshape(1, N) + 1000
        keys[0, [0, 7, 3]] = 1
        ent, _ = orc.topk_from_group_keys(keys, 1, 0)
        assert ent[0, 0] == 3

    def test_supplement_valid(self, orc):
        keys = np.arange(6, dtype=np.uint64).reshape(1, 6)
        ent, total = orc.topk_from_group_keys(keys, 3, 2)
        assert total == 0
        for j in range(6):
            assert len(set(ent[j])) == 3 and j not in ent[j]
            assert ent[j].min() >= 0 and ent[j].max() < 6


class TestHashGolden:
    def test_lsh_small(self, orc):
        z = load_golden("lsh_small.npz")
        for k in range(int(z["n_runs"])):
            pre = f"k{k}_"
            ci = int(z[pre + "case"])
            G, p, q, e, seed, K = (int(x) for x in z[pre + "cfg"])
            d, _ = _csr(orc, z, f"c{ci}_")
            r = orc.simlsh_topk(d.col_ptr, d.col_rows, d.col_vals, d.M, G, p, q, e, seed, K)
            assert r.acc.tobytes() == z[pre + "acc"].tobytes(), k
            assert r.sig.tobytes() == z[pre + "sig"].tobytes(), k
            assert r.keys.tobytes() == z[pre + "keys"].tobytes(), k
            assert r.entries.tobytes() == z[pre + "entries"].tobytes(), k

    def test_c1_lsh(self, orc):
        z = load_golden("c1.npz")
        d, _ = orc.build_csr(int(z["train_M"]), int(z["train_N"]), z["train_rows"], z["train_cols"],
                             z["train_vals"])
        r = orc.simlsh_topk(d.col_ptr, d.col_rows, d.col_vals, d.M, 8, 3, 100, 2, 0, 16)
        assert sha(r.acc) == str(z["lsh_acc_sha"])
        assert sha(r.sig) == str(z["lsh_sig_sha"])
        assert r.keys.tobytes() == z["lsh_keys"].tobytes()
        assert r.entries.tobytes() == z["lsh_entries16"].tobytes()
        ent32, _ = orc.topk_from_group_keys(r.keys, 32, 0)
        assert ent32.tobytes() == z["lsh_entries32"].tobytes()


class TestSgdGolden:
    def test_sgd_small_serial_and_dsgd(self, orc):
        z = load_golden("sgd_small.npz")
        for s in range(int(z["n_cases"])):
            pre = f"s{s}_"
            F, K, epochs, seed = (int(x) for x in z[pre + "cfg"])
            d, mu = _csr(orc, z, pre)
            nbr = z[pre + "nbr"]
            m = orc.train_full(d, mu, nbr, F, K, epochs, seed, _rates(), REGS)
            for n, a in (("b", m.b), ("b_hat", m.bhat), ("U", m.U), ("V", m.V), ("W", m.W),
                         ("C", m.C)):
                assert a.tobytes() == z[f"{pre}full_{n}"].tobytes(), (s, n)
            rm = orc.rmse(d, m, z[pre + "rows"], z[pre + "cols"], z[pre + "vals"])
            assert rm == float(z[pre + "rmse"])
            rm2 = orc.rmse(d, m, z[pre + "rows"], z[pre + "cols"], z[pre + "vals"],
                           clamp=(1.5, 4.5), unscale=2.0)
            assert rm2 == float(z[pre + "rmse_clamp"])
            for D in (2, 3):
                md = orc.parallel_train(d, mu, nbr, F, K, epochs, seed, _rates(), REGS, D)
                for n, a in (("b", md.b), ("U", md.U), ("V", md.V), ("W", md.W), ("C", md.C)):
                    assert a.tobytes() == z[f"{pre}D{D}_{n}"].tobytes(), (s, D, n)

    def test_sgd_c1(self, orc):
        z = load_golden("c1.npz")
        d, mu = orc.build_csr(int(z["train_M"]), int(z["train_N"]), z["train_rows"], z["train_cols"],
                              z["train_vals"])
        nbr = z["lsh_entries16"]
        tr, tc, tv = (z["test_rows"].astype(np.int32), z["test_cols"].astype(np.int32),
                      z["test_vals"].astype(np.float64))
        seen = []
        m = orc.train_full(d, mu, nbr, 32, 16, 3, 0, _rates(), REGS,
                           callback=lambda t, mm: seen.append(orc.rmse(d, mm, tr, tc, tv)))
        np.testing.assert_array_equal(seen, z["sgd_rmse_test"])
        for n, a in (("b", m.b), ("b_hat", m.bhat), ("U", m.U), ("V", m.V), ("W", m.W), ("C", m.C)):
            assert sha(a) == str(z[f"sgd_full_{n}_sha"]), n
        md = orc.parallel_train(d, mu, nbr, 32, 16, 2, 0, _rates(), REGS, 4)
        for n, a in (("b", md.b), ("U", md.U), ("V", md.V), ("W", md.W), ("C", md.C)):
            assert sha(a) == str(z[f"sgd_D4_{n}_sha"]), n
        assert orc.rmse(d, md, tr, tc, tv) == float(z["sgd_D4_rmse_test"])


    def test_c1_20_epoch_curve(self, orc):
        """The oracle reproduces the reference's whole 20-epoch learning curve (test and
        train RMSE after every epoch, c1_ref20.npz written by the reference)."""
        z = load_golden("c1.npz")
        ref = load_golden("c1_ref20.npz")
        assert ref["entries16"].tobytes() == z["lsh_entries16"].tobytes()
        d, mu = orc.build_csr(int(z["train_M"]), int(z["train_N"]), z["train_rows"], z["train_cols"],
                              z["train_vals"])
        tr, tc, tv = (z["test_rows"].astype(np.int32), z["test_cols"].astype(np.int32),
                      z["test_vals"].astype(np.float64))
        rr, rc, rv = (z["train_rows"].astype(np.int32), z["train_cols"].astype(np.int32),
                      z["train_vals"].astype(np.float64))
        seen = []
        orc.train_full(d, mu, ref["entries16"], 32, 16, 20, 0, _rates(), REGS,
                       callback=lambda t, mm: seen.append((orc.rmse(d, mm, tr, tc, tv),
                                                           orc.rmse(d, mm, rr, rc, rv))))
        np.testing.assert_array_equal([a for a, _ in seen], ref["F32_rmse_test"])
        np.testing.assert_array_equal([b for _, b in seen], ref["F32_rmse_train"])


class TestOnlineGolden:
    def test_online_small(self, orc):
        z = load_golden("online_small.npz")
        for s in range(int(z["n_cases"])):
            pre = f"o{s}_"
            G, p, q, e, lseed = (int(x) for x in z[pre + "lsh"])
            F, K, epochs, seed = (int(x) for x in z[pre + "cfg"])
            d, mu = _csr(orc, z, pre)
            r = orc.simlsh_topk(d.col_ptr, d.col_rows, d.col_vals, d.M, G, p, q, e, lseed, K)
            assert r.acc.tobytes() == z[pre + "state_acc"].tobytes()
            assert r.entries.tobytes() == z[pre + "table"].tobytes()
            m = orc.train_full(d, mu, r.entries, F, K, epochs, seed, _rates(), REGS)
            assert m.U.tobytes() == z[pre + "p0_U"].tobytes()
            bM, bN, nr_, nc_ = (int(x) for x in z[pre + "b_shape"])
            batch = (bM, bN, nr_, nc_, z[pre + "b_rows"], z[pre + "b_cols"], z[pre + "b_vals"])
            me, acc_e, ent_e, _ = orc.absorb_increment(
                m, r.acc, (G, p, q, e, lseed), d, (z[pre + "rows"], z[pre + "cols"], z[pre + "vals"]),
                batch, F, K, epochs, seed, _rates(), REGS)
            assert acc_e.tobytes() == z[pre + "ext_acc"].tobytes(), s
            assert ent_e.tobytes() == z[pre + "ext_entries"].tobytes(), s
            for n, a in (("b", me.b), ("b_hat", me.bhat), ("U", me.U), ("V", me.V), ("W", me.W),
                         ("C", me.C)):
                assert a.tobytes() == z[f"{pre}ext_{n}"].tobytes(), (s, n)

    def test_online_c1(self, orc):
        z = load_golden("c1.npz")
        from numpy import asarray
        M, N = int(z["train_M"]), int(z["train_N"])
        rows = z["train_rows"].astype(np.int32)
        cols = z["train_cols"].astype(np.int32)
        vals = z["train_vals"].astype(np.float64)
        bM, bN, nr_, nc_ = (int(x) for x in z["online_b_shape"])
        row_map, col_map = z["online_row_map"], z["online_col_map"]
        # holdback_variables (online.py:335-368): original = entries touching no held variable
        rr, cc = row_map[rows], col_map[cols]
        keep = (rr < bM) & (cc < bN)
        d, mu = orc.build_csr(bM, bN, rr[keep], cc[keep], vals[keep])
        r = orc.simlsh_topk(d.col_ptr, d.col_rows, d.col_vals, d.M, 8, 3, 100, 2, 0, 32)
        assert sha(r.acc) == str(z["online_state0_acc_sha"])
        assert r.entries.tobytes() == z["online_orig_entries"].tobytes()
        m = orc.train_full(d, mu, r.entries, 32, 32, 4, 0, _rates(), REGS)
        assert sha(m.U) == str(z["online_p0_U_sha"])
        batch = (bM, bN, nr_, nc_, z["online_b_rows"], z["online_b_cols"], z["online_b_vals"])
        me, acc_e, ent_e, _ = orc.absorb_increment(
            m, r.acc, (8, 3, 100, 2, 0), d, (asarray(rr[keep]), asarray(cc[keep]), vals[keep]),
            batch, 32, 32, 4, 0, _rates(), REGS)
        assert sha(acc_e) == str(z["online_ext_acc_sha"])
        assert ent_e.tobytes() == z["online_ext_entries"].tobytes()
        for n, a in (("b", me.b), ("b_hat", me.bhat), ("U", me.U), ("V", me.V), ("W", me.W),
                     ("C", me.C)):
            assert sha(a) == str(z[f"online_ext_{n}_sha"]), n


class TestBasicGolden:
    def test_train_basic(self, orc):
        z = load_golden("basic.npz")
        for s in range(int(z["n_cases"])):
            pre = f"b{s}_"
            F, epochs, seed, wb, srt = (int(x) for x in z[pre + "cfg"])
            d, mu = _csr(orc, z, pre)
            m = orc.train_basic(d, mu, F, epochs, seed, _rates((0.035, 0.035, 0.04, 0.04, 0.002, 0.002)),
                                (0.02, 0.02, 0.035, 0.035, 0.002, 0.002), bool(wb), bool(srt))
            for n, a in (("b", m.b), ("b_hat", m.bhat), ("U", m.U), ("V", m.V)):
                assert a.tobytes() == z[f"{pre}{n}"].tobytes(), (s, n)


# ------------------------------------------------------- similarity (GSM) ---

def _col_view(z, pre):
    M, N = int(z[pre + "M"]), int(z[pre + "N"])
    rows, cols, vals = z[pre + "rows"], z[pre + "cols"], z[pre + "vals"]
    order = np.lexsort((rows, cols))
    col_ptr = np.zeros(N + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=N), out=col_ptr[1:])
    return M, N, col_ptr, rows[order].astype(np.int32), vals[order].astype(np.float64)


class TestOracleSimilarity:
    """oracle GSM restatement == reference similarity.py outputs (tests/golden/similarity.npz)."""

    def test_pearson_and_shrunk_bitwise(self, orc):
        z = load_golden("similarity.npz")
        for name in z["cases"]:
            M, N, cp, cr, cv = _col_view(z, str(name) + "_")
            P = np.zeros((N, N))
            S = np.zeros((N, N))
            for a in range(N):
                for b in range(N):
                    if a == b:
                        continue
                    st = orc.pair_stats(cr[cp[a]:cp[a + 1]], cv[cp[a]:cp[a + 1]],
                                        cr[cp[b]:cp[b + 1]], cv[cp[b]:cp[b + 1]])
                    P[a, b] = orc.pearson_from_stats(st)
                    S[a, b] = 0.0 if st[0] == 0 else st[0] / (st[0] + 25.0) * P[a, b]
            assert P.tobytes() == z[f"{name}_pearson"].tobytes(), name
            assert S.tobytes() == z[f"{name}_shrunk25"].tobytes(), name

    def test_gsm_small_cases(self, orc):
        z = load_golden("similarity.npz")
        n = 0
        for name in z["cases"]:
            M, N, cp, cr, cv = _col_view(z, str(name) + "_")
            for key in z.files:
                if key.startswith(f"{name}_gsm_K"):
                    K = int(key.split("_K")[1].split("_")[0])
                    lam = float(key.split("_l")[1])
                    assert np.array_equal(orc.gsm_topk(cp, cr, cv, N, K, lam), z[key]), key
                    n += 1
        assert n >= 30

    def test_gsm_c1(self, orc):
        z = load_golden("similarity.npz")
        M, N, cp, cr, cv = _col_view(z, "c1_")
        assert np.array_equal(orc.gsm_topk(cp, cr, cv, N, 16, 100.0), z["c1_gsm_K16"])
        assert np.array_equal(orc.gsm_topk(cp, cr, cv, N, 32, 50.0), z["c1_gsm_K32_l50"])
