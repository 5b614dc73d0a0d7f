"""Synthetic workloads of BASELINE.json's configs, generated directly in HBM.

The reference's ``random_sparse`` (datasets.py:147-164) draws a Binomial(M,
density) count per column and that many distinct rows, with integer stars
1..5.  Generating 100M ratings that way on the host takes ~100 s,
so the bench builds the same distribution on the device: per-column counts (a
seeded multinomial split of exactly the config's rating count), distinct rows per
column from a keyed permutation of [0, M), stars 1..5 from a hash -- all a pure
function of (seed, column), so every rank of a multi-GPU run generates exactly its
own shard of the same matrix (csrc/init.cu culsh_synth_columns).  Both index views
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


def column_counts(M: int, N: int, nnz_target: int, seed: int = 0) -> np.ndarray:
    """Per-column rating counts: a multinomial split of exactly nnz_target ratings over
    the N columns (each column ~Binomial(M, density) as in datasets.py:147-164, but the
    total is the config's exact count), at least 1 and at most M per column."""
    rng = np.random.default_rng(seed)
    c = rng.multinomial(nnz_target, np.full(N, 1.0 / N))
    return np.clip(c, 1, M).astype(np.int64)


def hashed_shard(M: int, N: int, nnz_target: int, seed: int = 0, cols: tuple | None = None,
                 rows: tuple | None = None, chunk: int = 1 << 25):
    """Device triplets (rows i32, cols i32, vals f64), sorted by (col, row), of the
    synthetic matrix restricted to a column range and/or a row range; the same seed gives
    the same matrix for any shard (csrc/init.cu culsh_synth_columns).  Also returns the
    global column pointer (host int64)."""
    t = nat.torch()
    dev = nat.device()
    cnt = column_counts(M, N, nnz_target, seed)
    cp = np.zeros(N + 1, np.int64)
    np.cumsum(cnt, out=cp[1:])
    cp_d = t.from_numpy(cp).to(dev)
    c0, c1 = cols if cols is not None else (0, N)
    parts_r, parts_c, parts_v = [], [], []
    j = c0
    while j < c1:   # column chunks of ~chunk entries (bounded scratch)
        j2 = int(np.searchsorted(cp, cp[j] + chunk, side="right")) - 1
        j2 = min(max(j2, j + 1), c1)
        n = int(cp[j2] - cp[j])
        r = nat.empty((max(n, 1),), "int32")
        v = nat.empty((max(n, 1),), "float64")
        nat.call("culsh_synth_columns", M, j, j2, nat.ptr(cp_d), int(seed) & ((1 << 64) - 1), nat.ptr(r),
                 nat.ptr(v), nat.stream_ptr())
        r, v = r[:n], v[:n]
        c = t.repeat_interleave(t.arange(j, j2, device=dev, dtype=t.int32), cp_d[j + 1:j2 + 1] - cp_d[j:j2])
        if rows is not None:
            keep = (r >= rows[0]) & (r < rows[1])
            r, c, v = r[keep], c[keep], v[keep]
        key = c.to(t.int64) * M + r.to(t.int64)
        key, order = t.sort(key)
        parts_r.append(r[order])
        parts_c.append(c[order])
        parts_v.append(v[order])
        j = j2
    if not parts_r:
        z = t.zeros(0, dtype=t.int32, device=dev)
        return z, z.clone(), t.zeros(0, dtype=t.float64, device=dev), cp
    return t.cat(parts_r), t.cat(parts_c), t.cat(parts_v), cp


def device_ratings_from_sorted(M: int, N: int, rows, cols, vals, baselines: bool = True):
    """DeviceRatings from device triplets already sorted by (col, row): CSC directly, CSR by
    a device sort; baselines from the two views' exact segment sums (integer stars)."""
    from .data import device_baselines
    t = nat.torch()
    d = rows.device
    nnz = int(rows.numel())
    col_ptr = t.zeros(N + 1, dtype=t.int64, device=d)
    col_ptr[1:] = t.cumsum(t.bincount(cols, minlength=N), 0)
    order = t.argsort(rows.to(t.int64) * N + cols.to(t.int64))
    row_cols = cols[order].contiguous()
    row_vals = vals[order].contiguous()
    del order
    row_ptr = t.zeros(M + 1, dtype=t.int64, device=d)
    row_ptr[1:] = t.cumsum(t.bincount(rows, minlength=M), 0)
    if baselines and nnz:
        mu, bb, bh = device_baselines(M, N, col_ptr, vals, row_ptr, row_vals, nnz)
    else:
        mu, bb, bh = 0.0, t.zeros(M, dtype=t.float64, device=d), t.zeros(N, dtype=t.float64, device=d)
    dev = DeviceRatings.from_device(M, N, col_ptr, rows.contiguous(), vals.contiguous(), row_ptr, row_cols,
                                    row_vals, mu, bb, bh)
    dev.exact_baselines = bool(baselines)
    dev._integer_valued = True
    return dev


def random_sparse_device(M: int, N: int, nnz_target: int, seed: int = 0) -> DeviceMatrix:
    """The whole synthetic matrix in HBM (hashed_shard over all columns)."""
    rows, cols, vals, _ = hashed_shard(M, N, nnz_target, seed)
    dev = device_ratings_from_sorted(M, N, rows, cols, vals)
    return DeviceMatrix(dev, M, N, dev.nnz)


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
