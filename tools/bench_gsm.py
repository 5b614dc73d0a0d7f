"""GSM exact top-K at scale: device time of gsm_topk's count
route (densify + 4 int8 tensor-core GEMMs + fp64 selection) on the C2 / C3 shapes,
the oracle (reference algorithm, all host threads) timed on a bounded sample of
target columns and extrapolated, and a bit-exactness check of the sampled rows.

  python tools/bench_gsm.py [c2|c3] [--sample 48]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_11682_b200 import _native as nat, synth  # noqa: E402
from paper_2111_11682_b200.similarity import SimilarityConfig, gsm_topk  # noqa: E402


def main():
    cfgname = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c2"
    sample = int(sys.argv[sys.argv.index("--sample") + 1]) if "--sample" in sys.argv else 48
    M, N, nnz, F, K, e = synth.SHAPES[cfgname]
    dm = synth.random_sparse_device(M, N, nnz, seed=0)
    d = dm.dev
    cfg = SimilarityConfig(K=K)
    gsm_topk(d, cfg)                       # warm (allocations)
    torch.cuda.synchronize()
    runs = []
    for _ in range(3):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        t0 = time.perf_counter()
        tbl = gsm_topk(d, cfg)
        ev[1].record()
        torch.cuda.synchronize()
        runs.append((ev[0].elapsed_time(ev[1]) / 1e3, time.perf_counter() - t0))
    dev_s = float(np.median([r[0] for r in runs]))
    # int8 work of the four products: 2 * N^2 * M each
    ops = 4 * 2.0 * N * N * M
    # the reference algorithm (oracle port, all host threads) on a sample of target
    # columns against all N candidates, extrapolated to N targets
    from oracle import oracle as orc
    cp = nat.to_host(d.col_ptr)
    cr = nat.to_host(d.col_rows)
    cv = nat.to_host(d.col_vals)
    pick = np.sort(np.random.default_rng(0).choice(N, size=min(sample, N), replace=False))
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    sub = orc.gsm_topk_targets(cp, cr, cv, N, pick, K, 100.0, threads)
    cpu_s = time.perf_counter() - t0
    ok = bool(np.array_equal(sub, tbl.entries[pick]))
    line = {"metric": "GSM exact top-K build time", "config": cfgname, "M": M, "N": N, "nnz": int(dm.nnz),
            "K": K, "runs_s": [r[0] for r in runs], "route": "count (culsh_gsm_stats_tc: tcgen05 kind::i8, TMEM)", "device_s": dev_s,
            "wall_s": float(np.median([r[1] for r in runs])), "int8_tops": ops / dev_s / 1e12,
            "cpu_oracle": {"threads": threads, "sample_targets": len(pick), "sample_s": cpu_s,
                           "extrapolated_s": cpu_s * N / len(pick)},
            "sample_rows_bit_exact": ok}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
