"""Calibrate bench.py's CPU baseline (the oracle port, cpu_baseline.kind = "port") against
the unmodified reference (numba) on the SAME sample and the same host threads.  Runs in
the build container only (it imports /root/reference, which does not travel to the GPU
box); writes profiles/r2_cpu_calibration.json, which bench.py quotes next to the port's
numbers so the reported CPU baseline can be read in reference units.

Sample = bench.py's cpu_baseline sample: 2 % of the C3 rows at the workload's density.
  simLSH top-K  : lshmf.simlsh_topk            vs oracle.simlsh_topk     (entries compared)
  DSGD epoch    : lshmf.parallel_train(D, 1 ep) vs oracle.parallel_epoch (D = threads)

  python tools/calibrate_cpu_baseline.py
"""
import json
import os
import shutil
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
REF_SRC = "/tmp/culsh_refpkg/src"
if not os.path.isdir(REF_SRC):
    shutil.copytree("/root/reference/pkg/src", REF_SRC)   # numba writes caches next to sources
sys.path.insert(0, REF_SRC)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba")

import lshmf  # noqa: E402

from oracle import oracle as orc  # noqa: E402

RATES = dict(alpha_b=0.02, alpha_b_hat=0.02, alpha_u=0.02, alpha_v=0.02, alpha_w=0.001, alpha_c=0.001,
             lambda_b=0.01, lambda_b_hat=0.01, lambda_u=0.01, lambda_v=0.01, lambda_w=0.05, lambda_c=0.05,
             beta=0.3)


def best_of(n, fn):
    ts = []
    out = None
    for _ in range(n):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return out, min(ts)


def main():
    M, N, nnz, F, K = 480189, 17770, 100480507, 128, 32
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(0)                     # bench.py cpu_baseline's sample
    Ms = int(M * 0.02)
    counts = np.maximum(1, rng.binomial(N, nnz / (M * N), Ms))
    key = np.unique(np.repeat(np.arange(Ms, dtype=np.int64), counts) * N +
                    rng.integers(0, N, int(counts.sum())))
    rows, cols = (key // N).astype(np.int32), (key % N).astype(np.int32)
    vals = rng.integers(1, 6, len(key)).astype(np.float64)
    r = lshmf.SparseRatings(Ms, N, rows, cols, vals)
    lc = lshmf.LshConfig(G=8, p=3, q=100, psi_exponent=2, seed=0)
    lshmf.simlsh_topk(r, lc, K)                        # numba JIT warm-up
    (tb, _), ref_lsh = best_of(2, lambda: lshmf.simlsh_topk(r, lc, K))
    hs, port_lsh = best_of(2, lambda: orc.simlsh_topk(r.col_ptr, r.col_rows, r.col_vals, Ms, 8, 3, 100, 2, 0,
                                                        K, threads))
    same = bool(np.array_equal(hs.entries, tb.entries))

    D = threads
    cfg1 = lshmf.TrainConfig(F=F, K=K, epochs=1, seed=0, **RATES)
    lshmf.parallel_train(r, tb, lshmf.TrainConfig(F=F, K=K, epochs=1, seed=0, **RATES), D)   # warm
    t0 = time.perf_counter()
    lshmf.parallel_train(r, tb, cfg1, D)
    ref_1 = time.perf_counter() - t0
    cfg3 = lshmf.TrainConfig(F=F, K=K, epochs=3, seed=0, **RATES)
    t0 = time.perf_counter()
    lshmf.parallel_train(r, tb, cfg3, D)
    ref_3 = time.perf_counter() - t0
    ref_epoch = (ref_3 - ref_1) / 2                    # per-epoch, init / partition excluded
    csr, mu = orc.build_csr(Ms, N, rows, cols, vals)
    m = orc.init_model(Ms, N, F, K, hs.entries, mu, csr.base_b, csr.base_bhat, 0)
    rates = orc.make_rates((0.02, 0.02, 0.02, 0.02, 0.001, 0.001), (0.01, 0.01, 0.01, 0.01, 0.05, 0.05))
    part = orc.partition(csr, D)
    orc.parallel_epoch(csr, m, rates, D, part, threads)
    _, port_epoch = best_of(2, lambda: orc.parallel_epoch(csr, m, rates, D, part, threads))
    out = {
        "what": "oracle port vs unmodified reference (numba) on bench.py's cpu_baseline sample, same host",
        "host_threads": threads, "sample": {"rows": Ms, "cols": N, "ratings": int(len(rows))},
        "simlsh_topk_s": {"reference": ref_lsh, "port": port_lsh, "port_over_reference_time": port_lsh / ref_lsh,
                          "entries_identical": same},
        "dsgd_epoch_s": {"reference": ref_epoch, "port": port_epoch, "D": D,
                         "port_over_reference_time": port_epoch / ref_epoch},
        "reading": "port_over_reference_time < 1: the port is faster than the reference, so GPU/CPU "
                   "ratios quoted against the port understate the speed-up over the reference",
    }
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "r2_cpu_calibration.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
