"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
the product path refuses to run without a GPU (no CPU fallback), and the
host-side logic (configs, schedules, file formats) mirrors the reference."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden


def header_functions():
    src = open(os.path.join(ROOT, "include", "culsh.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(culsh_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_2111_11682_b200 import _native as nat
    lib = nat.load_library()
    names = header_functions()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(nat.exported_symbols())
    assert lib.culsh_version().decode().startswith("culsh")


def test_error_reporting_without_launch():
    """Argument validation happens before any CUDA call (CULSH_EINVAL path)."""
    import ctypes
    from paper_2111_11682_b200 import _native as nat
    lib = nat.load_library()
    st = lib.culsh_row_hash_table(ctypes.c_uint64(0), 1, 9, 8, 0, 10, None, None)  # p*G = 72
    assert st == nat.CULSH_EINVAL
    assert "LSH config" in lib.culsh_last_error().decode()
    st = lib.culsh_topk(None, 0, 5, 24, 0, 5, 3, ctypes.c_uint64(0), None, None, None)
    assert st == nat.CULSH_EINVAL


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    import paper_2111_11682_b200 as P
    from paper_2111_11682_b200._native import NativeUnavailable
    r = P.SparseRatings(3, 2, np.array([0, 1, 2]), np.array([0, 1, 1]), np.array([1., 2., 3.]))
    with pytest.raises(NativeUnavailable):
        P.compute_hash_state(r, P.LshConfig(G=4, p=1, q=2))
    with pytest.raises(NativeUnavailable):
        P.train_full(r, None, P.TrainConfig(F=2, K=0, epochs=1))


def test_configs_mirror_reference():
    import paper_2111_11682_b200 as P
    P.LshConfig().validate()
    for bad in (dict(G=0), dict(G=32, p=3), dict(psi_exponent=3), dict(seed=-1)):
        with pytest.raises(ValueError):
            P.LshConfig(**bad).validate()
    # test_factorization.py:56-66 / A10
    assert P.learning_rate(0.04, 0.3, 0) == 0.04
    assert P.learning_rate(0.04, 0.3, 1) == pytest.approx(0.030769230769230771, rel=1e-12)
    assert P.learning_rate(0.04, 0.3, 4) == pytest.approx(0.04 / 3.4, rel=1e-12)
    vals = [P.learning_rate(0.04, 0.3, t) for t in range(1001)]
    assert all(a > b for a, b in zip(vals, vals[1:]))
    with pytest.raises(ValueError):
        P.TrainConfig(alpha_u=0).validate()
    assert P.TrainConfig(F=16).effective_init_scale == 0.25


def test_rotation_schedule():
    import paper_2111_11682_b200 as P
    s = P.RotationSchedule(3)
    assert [s.row_block(d, 1) for d in range(3)] == [1, 2, 0]
    P.RotationSchedule(4).validate()
    assert P.RotationSchedule(1).stage_assignments(0) == [(0, 0, 0)]


def test_sparse_ratings_and_baselines(orc):
    import paper_2111_11682_b200 as P
    rng = np.random.default_rng(42)
    mask = rng.random((12, 9)) < 0.5
    rows, cols = np.nonzero(mask)
    vals = rng.integers(1, 6, size=len(rows)).astype(float)
    r = P.build_indices(P.Triplets(rows.astype(np.int32), cols.astype(np.int32), vals), M=12, N=9)
    d, mu = orc.build_csr(12, 9, rows, cols, vals)
    np.testing.assert_array_equal(r.col_rows, d.col_rows)
    np.testing.assert_array_equal(r.row_cols, d.row_cols)
    st = r.baselines()
    assert st.mu == mu
    assert st.b.tobytes() == d.base_b.tobytes()
    with pytest.raises(ValueError):
        P.build_indices(P.Triplets(np.array([0, 0]), np.array([1, 1]), np.array([1., 2.])))


def test_checkpoint_and_hashstate_formats(tmp_path):
    import paper_2111_11682_b200 as P
    rng = np.random.default_rng(0)
    nbr = P.NeighborTable(4, 2, np.array([[1, 2], [0, 2], [0, 1], [0, 1]], np.int32))
    p = P.ModelParams(3.5, rng.random(5), rng.random(4), rng.random((5, 3)), rng.random((4, 3)),
                      rng.random((4, 2)), rng.random((4, 2)), nbr)
    p.save(tmp_path / "m.bin")
    q = P.ModelParams.load(tmp_path / "m.bin")
    assert q.mu == p.mu and q.U.tobytes() == p.U.tobytes()
    np.testing.assert_array_equal(q.neighbors.entries, nbr.entries)
    acc = rng.normal(size=(4, 3, 2, 5))
    h = P.HashState(acc=acc, sig=(acc >= 0).astype(np.uint8), config=P.LshConfig(G=5, p=2, q=3))
    h.save(tmp_path / "h.bin")
    back = P.HashState.load(tmp_path / "h.bin")
    assert back.acc.tobytes() == acc.tobytes() and back.config == h.config
    nbr.write_csv(tmp_path / "n.csv")
    np.testing.assert_array_equal(P.NeighborTable.read_csv(tmp_path / "n.csv").entries, nbr.entries)
    nbr.validate()
    with pytest.raises(ValueError):
        P.NeighborTable(2, 1, np.array([[0], [0]], np.int32)).validate()


def test_increment_batch_validation():
    import paper_2111_11682_b200 as P
    t = P.Triplets(np.array([0], np.int32), np.array([1], np.int32), np.array([3.0]))
    with pytest.raises(ValueError, match="no new variable"):
        P.make_increment(2, 2, t, new_row_count=1, new_col_count=0)
    b = P.make_increment(2, 2, P.Triplets(np.array([2, 0]), np.array([0, 3]), np.array([1., 2.])))
    assert (b.new_row_count, b.new_col_count, b.M_hat, b.N_hat) == (1, 2, 3, 4)


def test_random_topk_matches_reference():
    """random_topk is defined by numpy's PCG64 stream (similarity.py:203-213)."""
    import paper_2111_11682_b200 as P
    z = load_golden("similarity.npz")
    assert np.array_equal(P.random_topk(2, 1, seed=0).entries, z["rand_2_1_0"])
    assert np.array_equal(P.random_topk(50, 5, seed=9).entries, z["rand_50_5_9"])
    assert np.array_equal(P.random_topk(1682, 16, seed=0).entries, z["rand_1682_16_0"])
    P.random_topk(1000, 32, seed=4).validate()
    with pytest.raises(ValueError):
        P.random_topk(4, 4, seed=0)


def test_lshmfr_format_byte_identical(tmp_path):
    """SparseRatings.save writes the reference's LSHMF-R v1 bytes (data.py:238-243)
    and load reads them back (data.py:245-257)."""
    import paper_2111_11682_b200 as P
    z = load_golden("similarity.npz")
    for name in z["cases"]:
        pre = str(name) + "_"
        r = P.SparseRatings(int(z[pre + "M"]), int(z[pre + "N"]), z[pre + "rows"], z[pre + "cols"],
                            z[pre + "vals"])
        path = tmp_path / f"{name}.txt"
        r.save(path)
        assert path.read_bytes() == z[pre + "lshmfr"].tobytes(), name
        back = P.SparseRatings.load(path)
        assert (back.M, back.N) == (r.M, r.N)
        assert back.entry_values.tobytes() == r.entry_values.tobytes()
        assert np.array_equal(back.entry_rows, r.entry_rows)
    bad = tmp_path / "bad.txt"
    bad.write_text("NOPE v1 1 1 0\n")
    with pytest.raises(ValueError):
        P.SparseRatings.load(bad)


def test_checkpoint_bytes_match_reference(tmp_path):
    """ModelParams.save writes the reference's LSHMF-M bytes (factorization.py:154-161)."""
    import paper_2111_11682_b200 as P
    z = load_golden("similarity.npz")
    nb = P.NeighborTable(6, 2, z["mp_entries"])
    p = P.ModelParams(3.25, z["mp_b"], z["mp_b_hat"], z["mp_U"], z["mp_V"], z["mp_W"], z["mp_C"], nb)
    p.save(tmp_path / "m.bin")
    assert (tmp_path / "m.bin").read_bytes() == z["mp_bytes"].tobytes()
    q = P.ModelParams.load(tmp_path / "m.bin")
    assert q.V.tobytes() == p.V.tobytes()


def test_split_holdout_and_transform_match_reference():
    """split_holdout (native sequential core, numpy PCG64 permutation) and
    transform_ratings reproduce the reference's outputs exactly (api.npz)."""
    import paper_2111_11682_b200 as P
    z = load_golden("api.npz")
    r = P.SparseRatings(400, 300, z["split_in_rows"], z["split_in_cols"], z["split_in_vals"])
    for frac, sd in ((0.1, 0), (0.3, 4), (0.0, 1)):
        tr, te = P.split_holdout(r, frac, sd)
        key = f"split_{int(frac * 10)}_{sd}_"
        assert np.array_equal(te.rows, z[key + "test_rows"]) and np.array_equal(te.cols, z[key + "test_cols"])
        assert np.array_equal(tr.entry_rows, z[key + "train_rows"])
        assert tr.nnz + len(te) == r.nnz
    with pytest.raises(ValueError):
        P.split_holdout(r, 1.0, 0)
    tt = P.transform_ratings(P.Triplets(np.array([0, 1, 2]), np.array([0, 1, 1]), np.array([0.0, 50.0, 100.0])),
                             zero_floor=0.5, scale=20.0)
    assert tt.values.tobytes() == z["transform_vals"].tobytes()
    with pytest.raises(ValueError):
        P.transform_ratings(tt, scale=0.0)


def test_pairwise_plan_combines_to_numpy():
    """The host half of pairwise_sum_device: numpy's pairwise tree cut into nodes of <= 65,536
    elements, each node summed by numpy itself (what the device kernel restates) and combined
    back up the same tree, equals np.add.reduce of the whole array bit for bit."""
    from paper_2111_11682_b200.data import _pairwise_combine, _pairwise_plan
    rng = np.random.default_rng(3)
    for n in (1, 9, 65536, 65537, 131075, 1_000_003):
        x = rng.standard_normal(n) * 10.0 ** rng.integers(-5, 5, n)
        offs, lens = _pairwise_plan(n)
        assert sum(lens) == n and max(lens) <= 65536
        sums = [float(np.add.reduce(x[o:o + m])) for o, m in zip(offs, lens)]
        assert _pairwise_combine(n, sums) == float(np.add.reduce(x))


def test_model_dims_bounds():
    """Exact kernels take F <= 512 and K <= 128 (four mask words, the top-K kernels' bound);
    the fp32 Hogwild mode F <= 256, K <= 64; the reference has no bound (factorization.py:75-82)."""
    import pytest
    from paper_2111_11682_b200.factorization import MAX_K, _check_model_dims, _mask_words
    from paper_2111_11682_b200.hogwild import hogwild_supported
    assert MAX_K == 128
    _check_model_dims(256, 128)
    with pytest.raises(ValueError, match="K=129"):
        _check_model_dims(8, 129)
    _check_model_dims(512, 8)
    with pytest.raises(ValueError, match="F=513"):
        _check_model_dims(513, 8)
    assert [_mask_words(k) for k in (0, 32, 33, 64, 65, 128)] == [1, 1, 2, 2, 4, 4]
    assert hogwild_supported(128, 64) and not hogwild_supported(128, 65)


def _seq_sum_by_binade_runs(x, chunk=64):
    """Host restatement of rmse.cu's exact parallel serial sum (seq_chunk_fn_kernel /
    seq_walk_kernel): per chunk, the function b -> (D_b, b') on the grid of the chunk's
    approximate starting sum; a chunk on S's grid that stays in S's binade is applied as one
    integer step, any other chunk term by term."""
    import math
    n = len(x)
    csum = [math.fsum(x[c:c + chunk]) for c in range(0, n, chunk)]
    approx = np.concatenate([[0.0], np.cumsum(csum)[:-1]])

    def grid(S):
        return max(math.frexp(S)[1] - 53, -1074)

    fns = []
    for ci, c in enumerate(range(0, n, chunk)):
        A = approx[ci]
        ok = A > 0 and math.isfinite(A)
        ue = grid(A) if ok else 0
        d0, d1, o0, o1 = 0, 0, 0, 1
        for v in x[c:c + chunk]:
            try:
                y = math.ldexp(v, -ue)
            except OverflowError:   # the device's ldexp gives inf: not on this grid
                y = math.inf
            if not (0.0 <= y < 2.0 ** 53):
                ok = False
                break
            fl = math.floor(y)
            fr = y - fl
            if fr == 0.5:
                e0, e1, p0, p1 = fl + (fl & 1), fl + ((fl & 1) ^ 1), 0, 0
            else:
                d = fl + (1 if fr > 0.5 else 0)
                e0, e1, p0, p1 = d, d, d & 1, (d & 1) ^ 1
            d0, o0 = d0 + (e1 if o0 else e0), (p1 if o0 else p0)
            d1, o1 = d1 + (e1 if o1 else e0), (p1 if o1 else p0)
        fns.append((ok, ue, d0, d1))
    S = 0.0
    for ci, c in enumerate(range(0, n, chunk)):
        ok, ue, d0, d1 = fns[ci]
        if ok and S > 0 and math.isfinite(S) and grid(S) == ue:
            Si = int(math.ldexp(S, -ue))
            D = d1 if Si & 1 else d0
            if Si + D < 2 ** 53:
                S = math.ldexp(float(Si + D), ue)
                continue
        for v in x[c:c + chunk]:
            S = S + v
    return S


def test_sequential_sum_algebra_matches_accumulate():
    """The binade-run algebra behind culsh_sequential_sum equals numpy's sequential
    accumulate bit for bit: normal squares, exact ties (to even), binade changes, leading
    zeros and subnormals (the CUDA kernels are checked the same way on the GPU)."""
    rng = np.random.default_rng(7)
    e = rng.standard_normal(6000)
    u = 2.0 ** -52
    ties = rng.choice(np.array([0.5, 1.5, 2.5, 1.0, 0.0]) * u, 3000)
    ties[0] = 1.0
    cases = [e * e, ties, 2.0 ** (np.arange(3000) / 60.0),
             np.concatenate([np.zeros(300), rng.random(500) * 1e-310, rng.random(800)])]
    for x in cases:
        assert _seq_sum_by_binade_runs(list(map(float, x))) == np.add.accumulate(x)[-1]
