"""Small invocations of every kernel family, for compute-sanitizer (SURVEY §5 race detection):

  compute-sanitizer --tool memcheck  python tools/sanitize_kernels.py all
  compute-sanitizer --tool racecheck python tools/sanitize_kernels.py deterministic
  compute-sanitizer --tool synccheck python tools/sanitize_kernels.py deterministic

"deterministic" = the bit-exact kernels (hashing, top-K, exact SGD / DSGD stages, online
passes, GSM, RMSE); "all" adds the Hogwild epoch, which races on purpose (lock-free updates,
SURVEY §5: racy modes are excluded from determinism claims) and is checked for memory errors
only.  Each case also compares against the oracle, so a sanitizer-perturbed schedule that
changed a result would fail here too.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_11682_b200 as P  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def ratings(M, N, dens, seed, lo=1, hi=6):
    rng = np.random.default_rng(seed)
    rows, cols = np.nonzero(rng.random((M, N)) < dens)
    return P.SparseRatings(M, N, rows, cols, rng.integers(lo, hi, len(rows)).astype(np.float64))


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "deterministic"
    torch.cuda.set_device(0)
    r = ratings(400, 150, 0.06, 0)
    cfg = P.LshConfig(G=8, p=3, q=12, psi_exponent=2, seed=3)
    tbl, hs = P.simlsh_topk(r, cfg, 8)
    ref = orc.simlsh_topk(r.col_ptr, r.col_rows, r.col_vals, r.M, 8, 3, 12, 2, 3, 8)
    assert hs.acc.tobytes() == ref.acc.tobytes() and tbl.entries.tobytes() == ref.entries.tobytes()
    rr = P.SparseRatings(r.M, r.N, r.entry_rows, r.entry_cols, r.entry_values * 0.37)   # ordered fp64 path
    hs2 = P.compute_hash_state(rr, cfg)
    ref2 = orc.simlsh_topk(rr.col_ptr, rr.col_rows, rr.col_vals, rr.M, 8, 3, 12, 2, 3, None)
    assert hs2.acc.tobytes() == ref2.acc.tobytes()
    tc = P.TrainConfig(F=16, K=8, epochs=2, seed=0)
    p = P.train_full(r, tbl, tc)
    d, mu = orc.build_csr(r.M, r.N, r.entry_rows, r.entry_cols, r.entry_values)
    m = orc.train_full(d, mu, ref.entries, 16, 8, 2, 0, tc.rates_at, tc.regs)
    assert p.U.tobytes() == m.U.tobytes()
    pp = P.parallel_train(r, tbl, tc, 3)
    assert np.isfinite(pp.U).all()
    base, batch, _, _ = P.holdback_variables(r, 20, 10, seed=1)
    t0, s0 = P.simlsh_topk(base, cfg, 8)
    p0 = P.train_full(base, t0, tc)
    P.absorb_increment(p0, s0, base, batch, tc)
    P.rmse(p, r.triplets(), r)
    # the exact parallel serial sum (chunk sums / prefix / functions / scanned walk), with a
    # binade change and ties inside, against numpy's sequential accumulate
    from paper_2111_11682_b200 import _native as nat
    xs = np.random.default_rng(5).random(70_000) ** 4
    xs[:300] = 2.0 ** -53
    xs[0] = 1.0
    xd, sd = nat.to_dev(xs), nat.empty((1,), "float64")
    nat.call("culsh_sequential_sum", nat.ptr(xd), len(xs), nat.ptr(sd), nat.stream_ptr())
    assert float(sd.item()) == np.add.accumulate(xs)[-1]
    # K above two mask words (exact column kernel with four words)
    tw, _ = P.simlsh_topk(r, cfg, 70)
    pw = P.train_full(r, tw, P.TrainConfig(F=16, K=70, epochs=1, seed=2))
    dw, muw = orc.build_csr(r.M, r.N, r.entry_rows, r.entry_cols, r.entry_values)
    mw = orc.train_full(dw, muw, tw.entries, 16, 70, 1, 2, P.TrainConfig(F=16, K=70).rates_at,
                        P.TrainConfig(F=16, K=70).regs)
    assert pw.U.tobytes() == mw.U.tobytes() and pw.W.tobytes() == mw.W.tobytes()
    P.gsm_topk(r, P.SimilarityConfig(K=6), method="count")
    P.gsm_topk(r, P.SimilarityConfig(K=6), method="merge")
    if which == "all":
        ph = P.train_full(r, tbl, P.TrainConfig(F=32, K=8, epochs=2, seed=0), mode="hogwild")
        assert ph.all_finite()
    torch.cuda.synchronize()
    print(f"sanitize cases ({which}) ok")


if __name__ == "__main__":
    main()
