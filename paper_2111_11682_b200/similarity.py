"""Neighbour table J^K (reference similarity.py:14-48) and the
exact column-similarity search (similarity.py:51-213): shrunk
Pearson over co-rated rows, the all-pairs GSM top-K and the random control.

GSM runs on the GPU (csrc/similarity.cu), bit-identical to the reference:
  * count route (integer ratings in [-11, 11], the usual stars): dense int8
    panels X (indicator), R (values), Q (squares) and four int8 tensor-core
    GEMMs with exact int32 accumulation give n = X'X, s1 = R'X, s12 = R'R,
    q1 = Q'X (s2, q2 by transposition); every statistic is then the exact
    integer the reference's fp64 sums produce;
  * merge route (any values): thread per pair, ascending-row merge in fp64,
    the reference's own summation order.
Both feed one selection kernel: the reference's fp64 expression tree for the
shrunk similarity (-fmad=false) and the (similarity desc, index asc) top-K that
_topk_insert's strict comparisons produce.
"""

from __future__ import annotations

import os
import sys

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat


@dataclass
class NeighborTable:
    """Per-column Top-K neighbour indices, one row of K entries per column."""

    N: int
    K: int
    entries: np.ndarray  # (N, K) int32

    def validate(self) -> None:
        if self.entries.shape != (self.N, self.K):
            raise ValueError(f"entries shape {self.entries.shape} != ({self.N}, {self.K})")
        e = np.asarray(self.entries)
        if self.K:
            s = np.sort(e, axis=1)
            dup = (s[:, 1:] == s[:, :-1]).any(axis=1) if self.K > 1 else np.zeros(self.N, bool)
            if dup.any():
                raise ValueError(f"duplicate neighbor in row {int(np.flatnonzero(dup)[0])}")
            selfn = (e == np.arange(self.N)[:, None]).any(axis=1)
            if selfn.any():
                raise ValueError(f"self-neighbor in row {int(np.flatnonzero(selfn)[0])}")
            bad = ((e < 0) | (e >= self.N)).any(axis=1)
            if bad.any():
                raise ValueError(f"neighbor index out of range in row {int(np.flatnonzero(bad)[0])}")

    def device_entries(self):
        """(N*K,) int32 copy of ``entries`` in HBM.  Cached against a host snapshot, so an
        in-place edit of ``entries`` (a plain array, as in the reference) is picked up."""
        e = np.ascontiguousarray(self.entries, dtype=np.int32)
        cache = self.__dict__.get("_dev_cache")
        if cache is not None and cache[1].shape == e.shape and np.array_equal(cache[1], e):
            return cache[0]
        dev = nat.to_dev(e.reshape(-1) if e.size else np.zeros(1, np.int32), np.int32)
        self.__dict__["_dev_cache"] = (dev, e.copy())
        return dev

    def write_csv(self, path) -> None:
        with open(path, "w") as fh:
            fh.write("j,rank,neighbor\n")
            for j in range(self.N):
                for rank in range(self.K):
                    fh.write(f"{j},{rank},{self.entries[j, rank]}\n")

    @classmethod
    def read_csv(cls, path) -> "NeighborTable":
        data = np.loadtxt(path, delimiter=",", skiprows=1, dtype=np.int64, ndmin=2)
        N = int(data[:, 0].max()) + 1
        K = int(data[:, 1].max()) + 1
        entries = np.zeros((N, K), dtype=np.int32)
        entries[data[:, 0], data[:, 1]] = data[:, 2]
        return cls(N=N, K=K, entries=entries)


@dataclass
class SimilarityConfig:
    """similarity.py:51-54"""

    K: int
    lambda_rho: float = 100.0


def _csc(ratings):
    """Device CSC of a SparseRatings / DeviceSparseRatings / DeviceRatings."""
    return ratings.device() if hasattr(ratings, "device") else ratings


def _pair(ratings, j1: int, j2: int, lambda_rho: float) -> np.ndarray:
    if not (0 <= j1 < ratings.N and 0 <= j2 < ratings.N):
        raise ValueError("column index out of range")
    d = _csc(ratings)
    out = nat.empty((3,), "float64")
    nat.call("culsh_pair_similarity", nat.ptr(d.col_ptr), nat.ptr(d.col_rows), nat.ptr(d.col_vals),
             int(j1), int(j2), float(lambda_rho), nat.ptr(out), nat.stream_ptr())
    return nat.to_host(out)


def pearson(ratings, j1: int, j2: int) -> float:
    """Pearson correlation of two columns over their co-rated rows (similarity.py:110-121)."""
    if j1 == j2:
        raise ValueError("pearson requires two distinct columns")
    return float(_pair(ratings, j1, j2, 100.0)[0])


def shrunk_similarity(ratings, j1: int, j2: int, lambda_rho: float = 100.0) -> float:
    """n/(n+lambda) * rho over the co-rated rows (similarity.py:124-135)."""
    if j1 == j2:
        raise ValueError("shrunk_similarity requires two distinct columns")
    return float(_pair(ratings, j1, j2, lambda_rho)[1])


_GSM_MAX_K = 128


def _gsm_count(d, K: int, lambda_rho: float, entries) -> bool:
    """Count route; False (nothing written) when a value is not an integer in [-11, 11].
    The statistics of all pairs are four int8 products of dense column panels, computed
    by one tensor-core kernel (culsh_gsm_stats_tc) per pass over rating-row chunks."""
    t = nat.torch()
    N, M = d.N, d.M
    ld = max(128, (N + 127) // 128 * 128)
    free = t.cuda.mem_get_info()[0]
    prod_bytes = 6 * ld * ld * 4
    # rows of the dense panels per pass (int32 products accumulate exactly across passes)
    budget = max(int(0.5 * free) - prod_bytes, 3 * ld * 64)
    mc = max(64, min((M + 63) // 64 * 64, budget // (3 * ld) // 64 * 64))
    g = t.empty((6, ld, ld), dtype=t.int32, device=nat.device())   # + transposes of R X', Q X' 
    st = nat.zeros((1,), "int32")
    if os.environ.get("CULSH_GSM_DEBUG"):
        print(f"_gsm_count: free={free / 2**30:.1f} GiB rows/pass={mc} passes={-(-M // mc)}", file=sys.stderr)
    for m0 in range(0, M, mc):
        m1 = min(M, m0 + mc)
        w = (m1 - m0 + 63) // 64 * 64
        pan = t.zeros((3 * ld * w,), dtype=t.int8, device=nat.device())
        nat.call("culsh_gsm_densify_tiled", nat.ptr(d.col_ptr), nat.ptr(d.col_rows), nat.ptr(d.col_vals),
                 N, m0, m1, ld, w, nat.ptr(pan), nat.ptr(st), nat.stream_ptr())
        if int(st.item()):
            return False
        nat.call("culsh_gsm_stats_tc", nat.ptr(pan), ld, w, int(m0 > 0), nat.ptr(g[0]), nat.ptr(g[1]),
                 nat.ptr(g[2]), nat.ptr(g[3]), nat.ptr(g[4]), nat.ptr(g[5]), nat.stream_ptr())
        del pan
    nat.call("culsh_gsm_count_select", nat.ptr(g[0]), nat.ptr(g[1]), nat.ptr(g[2]), nat.ptr(g[3]),
             nat.ptr(g[4]), nat.ptr(g[5]), ld, N, 0, N, K, float(lambda_rho), nat.ptr(entries), nat.stream_ptr())
    return True


def gsm_topk(ratings, config: SimilarityConfig, method: str = "auto") -> NeighborTable:
    """Exact top-K neighbours of every column by shrunk Pearson similarity
    (similarity.py:188-200): all N*(N-1) pairs, ties to the lower index, rows by
    descending similarity.  method: "auto" (count route when the ratings allow it,
    else merge), "count" or "merge" -- every route gives the same bytes."""
    N = ratings.N
    K = config.K
    if K > N - 1:
        raise ValueError(f"K={K} exceeds N-1={N - 1}")
    if K < 1:
        raise ValueError("K must be positive")
    if K > _GSM_MAX_K:
        raise ValueError(f"the GPU GSM keeps at most {_GSM_MAX_K} neighbours per column")
    if method not in ("auto", "count", "merge"):
        raise ValueError(f"unknown method {method!r}")
    d = _csc(ratings)
    entries = nat.empty((N * K,), "int32")
    done = False
    if method in ("auto", "count") and d.nnz:
        done = _gsm_count(d, K, config.lambda_rho, entries)
        if not done and method == "count":
            raise ValueError("the count route needs integer ratings in [-11, 11]")
    if not done:
        nat.call("culsh_gsm_merge_topk", nat.ptr(d.col_ptr), nat.ptr(d.col_rows), nat.ptr(d.col_vals), N, 0,
                 N, K, float(config.lambda_rho), nat.ptr(entries), nat.stream_ptr())
    return NeighborTable(N=N, K=K, entries=nat.to_host(entries).reshape(N, K).astype(np.int32))


def random_topk(N: int, K: int, seed: int) -> NeighborTable:
    """Uniform random neighbour selection without replacement, excluding self
    (similarity.py:203-213).  The values are defined by numpy's PCG64 stream
    (rng.choice per column), so they are drawn on the host like init_params."""
    if K > N - 1:
        raise ValueError(f"K={K} exceeds N-1={N - 1}")
    rng = np.random.default_rng(seed)
    entries = np.empty((N, K), dtype=np.int32)
    for j in range(N):
        picks = rng.choice(N - 1, size=K, replace=False)
        picks[picks >= j] += 1
        entries[j] = picks
    return NeighborTable(N=N, K=K, entries=entries)
