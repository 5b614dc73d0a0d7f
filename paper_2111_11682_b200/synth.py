"""Synthetic workloads of BASELINE.json's configs, generated directly in HBM.

The reference's ``random_sparse`` (datasets.py:147-164) draws a Binomial(M,
density) count per column and that many distinct rows, with integer stars
1..5.  Generating 100M ratings that way on the host takes ~100 s,
so the bench builds the same distribution on the device: per-column Binomial
counts (numpy, seeded), uniform rows drawn with replacement then de-duplicated
(~0.6% duplicates at Netflix shape), stars uniform in 1..5.  Both index views
and the (integer-exact) baselines are built in HBM; this is setup, never timed.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .data import DeviceRatings

SHAPES = {
    # name: (M, N, nnz, F, K, psi_exponent)
    "c1": (943, 1682, 100_000, 32, 16, 2),
    "c2": (138_493, 26_744, 20_000_263, 64, 32, 2),
    "c3": (480_189, 17_770, 100_480_507, 128, 32, 2),
    "c5": (1_000_990, 624_961, 262_810_175, 128, 64, 4),
}


@dataclass
class DeviceMatrix:
    dev: DeviceRatings
    M: int
    N: int
    nnz: int


def random_sparse_device(M: int, N: int, nnz_target: int, seed: int = 0) -> DeviceMatrix:
    t = nat.torch()
    d = nat.device()
    rng = np.random.default_rng(seed)
    per_col = np.maximum(rng.binomial(M, nnz_target / (M * N), size=N), 1).astype(np.int64)
    total = int(per_col.sum())
    g = t.Generator(device=d)
    g.manual_seed(seed)
    cols = t.repeat_interleave(t.arange(N, device=d, dtype=t.int64), t.from_numpy(per_col).to(d))
    rows = t.randint(0, M, (total,), generator=g, device=d, dtype=t.int64)
    key = cols * M + rows
    key, _ = t.sort(key)
    key = t.unique_consecutive(key)
    del rows, cols
    nnz = int(key.numel())
    col = (key // M).to(t.int32)
    row = (key % M).to(t.int32)
    vals = t.randint(1, 6, (nnz,), generator=g, device=d, dtype=t.int64).to(t.float64)
    col_ptr = t.zeros(N + 1, dtype=t.int64, device=d)
    col_ptr[1:] = t.cumsum(t.bincount(col, minlength=N), 0)
    # CSR: stable order by (row, col)
    rkey = row.to(t.int64) * N + col.to(t.int64)
    order = t.argsort(rkey, stable=True)
    del rkey
    row_cols = col[order].contiguous()
    row_vals = vals[order].contiguous()
    del order
    row_ptr = t.zeros(M + 1, dtype=t.int64, device=d)
    row_cnt = t.bincount(row, minlength=M)
    row_ptr[1:] = t.cumsum(row_cnt, 0)
    # baselines (integer data: every summation order is exact)
    mu = float(vals.sum().item()) / nnz
    rs = t.zeros(M, dtype=t.float64, device=d).index_add_(0, row.to(t.int64), vals)
    cs = t.zeros(N, dtype=t.float64, device=d).index_add_(0, col.to(t.int64), vals)
    cc = (col_ptr[1:] - col_ptr[:-1]).to(t.float64)
    rc = row_cnt.to(t.float64)
    base_b = t.where(rc > 0, rs / rc.clamp(min=1) - mu, t.zeros_like(rs))
    base_bhat = t.where(cc > 0, cs / cc.clamp(min=1) - mu, t.zeros_like(cs))
    del col
    dev = DeviceRatings.from_device(M, N, col_ptr, row.contiguous(), vals, row_ptr, row_cols,
                                    row_vals, mu, base_b, base_bhat)
    dev.exact_baselines = True            # integer stars: every sum above is exact
    dev._integer_valued = True
    return DeviceMatrix(dev, M, N, nnz)


def random_sparse_ratings(M: int, N: int, nnz_target: int, seed: int = 0):
    """The same matrix as a drop-in ``SparseRatings`` (device-built; entry order = column
    major), for driving the public API at full scale without a host build."""
    from .data import SparseRatings
    t = nat.torch()
    dm = random_sparse_device(M, N, nnz_target, seed)
    d = dm.dev
    cols = t.repeat_interleave(t.arange(N, device=d.col_ptr.device, dtype=t.int32),
                               d.col_ptr[1:] - d.col_ptr[:-1])
    return SparseRatings._from_device(d, (d.col_rows, cols, d.col_vals))


def structured_triplets_device(M: int, N: int, nnz_target: int, seed: int = 0, rank: int = 6):
    """Skewed, low-rank-plus-noise integer ratings (the survey's "perf-stress"
    generator; same recipe as the reference's synthetic_movielens_100k,
    datasets.py:37-102, without the series structure): lognormal row activity and
    column popularity, rating = clip(round(3.6 + b_u + b_i + u.v + N(0, 0.7)), 1, 5).
    Returns device (rows, cols, vals) in random order, duplicates removed."""
    t = nat.torch()
    d = nat.device()
    g = t.Generator(device=d)
    g.manual_seed(seed)
    act = t.exp(t.randn(M, generator=g, device=d))
    pop = t.exp(1.2 * t.randn(N, generator=g, device=d))
    r = t.multinomial(act, nnz_target, replacement=True, generator=g)
    c = t.multinomial(pop, nnz_target, replacement=True, generator=g)
    key = t.unique(c * M + r)
    perm = t.randperm(key.numel(), generator=g, device=d)
    key = key[perm]
    rows, cols = (key % M).to(t.int32), (key // M).to(t.int32)
    bu = 0.35 * t.randn(M, generator=g, device=d, dtype=t.float64)
    bi = 0.45 * t.randn(N, generator=g, device=d, dtype=t.float64)
    U = 0.35 * t.randn(M, rank, generator=g, device=d, dtype=t.float64)
    V = 0.35 * t.randn(N, rank, generator=g, device=d, dtype=t.float64)
    score = (3.6 + bu[rows.long()] + bi[cols.long()] + (U[rows.long()] * V[cols.long()]).sum(1)
             + 0.7 * t.randn(rows.numel(), generator=g, device=d, dtype=t.float64))
    vals = t.clamp(t.round(score), 1.0, 5.0)
    return rows, cols, vals


def host_row_sample(dm: DeviceMatrix, n_rows: int):
    """Host copy (for the CPU baseline) of rows [0, n_rows): full CSR rows, the CSC
    restricted to those rows, and the baselines -- every row keeps all its ratings
    so neighbour lookups cost what they cost on the full matrix."""
    d = dm.dev
    t = nat.torch()
    row_ptr = nat.to_host(d.row_ptr)
    hi = int(row_ptr[n_rows])
    rows = np.repeat(np.arange(n_rows, dtype=np.int32), np.diff(row_ptr[:n_rows + 1]))
    cols = nat.to_host(d.row_cols[:hi])
    vals = nat.to_host(d.row_vals[:hi])
    return rows, cols, vals, float(d.mu), nat.to_host(d.base_b), nat.to_host(d.base_bhat)
