"""Cost of the drop-in SparseRatings(M, N, rows, cols, values) on C3-sized host numpy
triplets (100M ratings): the device build (stable device sorts + device baselines in numpy's
order, host views lazy) against the reference's host lexsort build, plus baselines().

  python tools/ingest_cost.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_11682_b200 as P  # noqa: E402
import paper_2111_11682_b200.data as D  # noqa: E402
from paper_2111_11682_b200 import _native as nat, synth  # noqa: E402


def main():
    torch.cuda.set_device(0)
    M, N, nnz, F, K, e = synth.SHAPES["c3"]
    d = synth.random_sparse_device(M, N, nnz, seed=0).dev
    cols = torch.repeat_interleave(torch.arange(N, device="cuda", dtype=torch.int32), d.col_ptr[1:] - d.col_ptr[:-1])
    perm = torch.randperm(d.nnz, device="cuda")               # arbitrary entry order
    rows = nat.to_host(d.col_rows[perm]).copy()
    cols = nat.to_host(cols[perm]).copy()
    vals = nat.to_host(d.col_vals[perm]).copy()
    del d
    out = {"nnz": int(len(rows))}
    P.SparseRatings(M, N, rows[:2_000_000], cols[:2_000_000], vals[:2_000_000])   # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = P.SparseRatings(M, N, rows, cols, vals)
    b = r.baselines()
    torch.cuda.synchronize()
    out["device_build_plus_baselines_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    _ = r.col_rows, r.row_ptr
    out["first_host_view_reads_s"] = time.perf_counter() - t0
    D._DEVICE_BUILD_MIN = 1 << 62
    t0 = time.perf_counter()
    h = P.SparseRatings(M, N, rows, cols, vals)
    out["host_lexsort_build_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    hb = h.baselines()
    out["host_baselines_s"] = time.perf_counter() - t0
    out["same_views"] = bool(h.col_rows.tobytes() == r.col_rows.tobytes() and h.row_ptr.tobytes() == r.row_ptr.tobytes())
    out["same_baselines"] = bool(hb.mu == b.mu and hb.b.tobytes() == b.b.tobytes() and hb.b_hat.tobytes() == b.b_hat.tobytes())
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
