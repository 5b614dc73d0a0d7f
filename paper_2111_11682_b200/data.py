"""Sparse rating data: the input type of the hot path.

Host side mirrors the reference's ``SparseRatings`` (data.py:166-257): the
triplets in input order plus CSR (sorted by (row, col)) and CSC (sorted by
(col, row)) numpy views, read-only, and the data baselines mu, b, b_hat
(data.py:289-309) which the model uses as fixed residual statistics.

Device side (``SparseRatings.device()``): the same two views resident in HBM as
int64 pointers / int32 indices / fp64 values, the CSC->CSR position map used by
the exact SGD schedule, and the baselines; exposed to the C ABI as a
``CulshData`` struct.  Parsing, text I/O and holdout splitting of the reference
are ingest, not hot path (SURVEY §2 Table A), and are not rebuilt here.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat


@dataclass
class Triplets:
    """A batch of rating triplets in dense index space (data.py:40-71)."""

    rows: np.ndarray
    cols: np.ndarray
    values: np.ndarray
    row_ids: list | None = None
    col_ids: list | None = None

    def __len__(self) -> int:
        return len(self.rows)

    @property
    def M(self) -> int:
        if self.row_ids is not None:
            return len(self.row_ids)
        return int(self.rows.max()) + 1 if len(self.rows) else 0

    @property
    def N(self) -> int:
        if self.col_ids is not None:
            return len(self.col_ids)
        return int(self.cols.max()) + 1 if len(self.cols) else 0


@dataclass
class BaselineStats:
    """Global mean plus per-row and per-column deviations (data.py:260-266)."""

    mu: float
    b: np.ndarray
    b_hat: np.ndarray


_HOST_VIEWS = ("entry_rows", "entry_cols", "entry_values", "row_ptr", "row_cols", "row_vals",
               "col_ptr", "col_rows", "col_vals")

# SparseRatings of at least this many entries build their index views on the device (when a
# GPU is present): the same arrays as the host lexsorts, orders of magnitude faster.
_DEVICE_BUILD_MIN = 1 << 20


def _gpu_present() -> bool:
    try:
        t = nat.torch()
        if not t.cuda.is_available():
            return False
        nat.load_library()
        return True
    except Exception:   # no GPU / no libculsh.so: the host build (the reference's own)
        return False


class SparseRatings:
    """Dual-indexed sparse matrix, immutable after construction (data.py:166-207).

    Built from host triplets (the reference's constructor: two lexsorts), or -- by
    ``extend_ratings`` and other device producers -- directly in HBM
    (``_from_device``); the host views of a device-built matrix (entry arrays, CSR,
    CSC) are downloaded on first access, read-only like the reference's."""

    def __init__(self, M: int, N: int, rows: np.ndarray, cols: np.ndarray, values: np.ndarray,
                 row_ids: list | None = None, col_ids: list | None = None):
        self.M = int(M)
        self.N = int(N)
        self.entry_rows = np.ascontiguousarray(rows, dtype=np.int32)
        self.entry_cols = np.ascontiguousarray(cols, dtype=np.int32)
        self.entry_values = np.ascontiguousarray(values, dtype=np.float64)
        self.row_ids = row_ids
        self.col_ids = col_ids
        nnz = len(self.entry_rows)
        if len(self.entry_cols) != nnz or len(self.entry_values) != nnz:
            raise ValueError("triplet arrays must have equal length")
        self._nnz = nnz
        self._baselines = None
        self._dev = None
        self._dev_entries = None
        for arr in (self.entry_rows, self.entry_cols, self.entry_values):
            arr.flags.writeable = False
        if nnz >= _DEVICE_BUILD_MIN and _gpu_present():
            self._device_build()
            return
        order = np.lexsort((self.entry_cols, self.entry_rows))
        self.row_ptr = np.zeros(self.M + 1, dtype=np.int64)
        np.cumsum(np.bincount(self.entry_rows, minlength=self.M), out=self.row_ptr[1:])
        self.row_cols = self.entry_cols[order]
        self.row_vals = self.entry_values[order]
        order = np.lexsort((self.entry_rows, self.entry_cols))
        self.col_ptr = np.zeros(self.N + 1, dtype=np.int64)
        np.cumsum(np.bincount(self.entry_cols, minlength=self.N), out=self.col_ptr[1:])
        self.col_rows = self.entry_rows[order]
        self.col_vals = self.entry_values[order]
        for arr in (self.row_ptr, self.row_cols, self.row_vals, self.col_ptr, self.col_rows, self.col_vals):
            arr.flags.writeable = False

    def _device_build(self) -> None:
        """Large matrices: both index views built in HBM by stable device sorts of the
        composite keys (the same permutations as the two lexsorts -- (row, col) order and
        (col, row) order, ties in entry order), the baselines on the device in numpy's
        summation order; the host views (row_ptr, col_rows, ...) are materialised on first
        read.  C3 (100M ratings): ~0.1 s instead of ~25 s of host lexsorts + np.add.at."""
        t = nat.torch()
        er, ec, ev = self.device_entries()
        M, N = self.M, self.N
        ckey, o = t.sort(ec.long() * M + er.long(), stable=True)
        col_ptr = t.searchsorted(ckey, t.arange(N + 1, device=ckey.device, dtype=t.int64) * M)
        del ckey
        crow, cval = er[o].contiguous(), ev[o].contiguous()
        del o
        rkey, o2 = t.sort(er.long() * N + ec.long(), stable=True)
        row_ptr = t.searchsorted(rkey, t.arange(M + 1, device=rkey.device, dtype=t.int64) * N)
        del rkey
        rcol, rval = ec[o2].contiguous(), ev[o2].contiguous()
        del o2
        mu, bb, bh = exact_baselines_device(M, N, er, ec, ev)
        dev = DeviceRatings.from_device(M, N, col_ptr, crow, cval, row_ptr, rcol, rval, mu, bb, bh)
        dev.exact_baselines = True
        self._dev = dev
        self._baselines = BaselineStats(float(mu), nat.to_host(bb)[:M].copy(), nat.to_host(bh)[:N].copy())

    @classmethod
    def _from_device(cls, dev: "DeviceRatings", entries, row_ids=None, col_ids=None,
                     baselines: "BaselineStats | None" = None) -> "SparseRatings":
        """A matrix whose index views already live in HBM (``dev``) together with its
        entry-order triplets ``entries`` = (rows i32, cols i32, values f64) tensors."""
        self = cls.__new__(cls)
        self.M, self.N, self._nnz = dev.M, dev.N, dev.nnz
        self.row_ids, self.col_ids = row_ids, col_ids
        self._dev = dev
        self._dev_entries = entries
        self._baselines = baselines
        return self

    def __getattr__(self, name):
        # host views of a device-built matrix, materialised on first access
        if name in _HOST_VIEWS and self.__dict__.get("_dev") is not None:
            d, (er, ec, ev) = self._dev, self._dev_entries
            n = self._nnz
            src = {"entry_rows": (er, n), "entry_cols": (ec, n), "entry_values": (ev, n),
                   "row_ptr": (d.row_ptr, self.M + 1), "row_cols": (d.row_cols, n),
                   "row_vals": (d.row_vals, n), "col_ptr": (d.col_ptr, self.N + 1),
                   "col_rows": (d.col_rows, n), "col_vals": (d.col_vals, n)}[name]
            a = np.ascontiguousarray(nat.to_host(src[0])[:src[1]])
            a.flags.writeable = False
            self.__dict__[name] = a
            return a
        raise AttributeError(name)

    @property
    def nnz(self) -> int:
        return self._nnz

    def triplets(self) -> Triplets:
        t = Triplets(self.entry_rows, self.entry_cols, self.entry_values, self.row_ids,
                     self.col_ids)
        t._source = self        # rmse() evaluates the training set on its device copy
        return t

    def device_entries(self):
        """The entry-order triplets (rows i32, cols i32, values f64) in HBM (cached;
        the matrix is immutable)."""
        if self._dev_entries is None:
            self._dev_entries = (nat.to_dev(self.entry_rows, np.int32), nat.to_dev(self.entry_cols, np.int32),
                                 nat.to_dev(self.entry_values, np.float64))
        return self._dev_entries

    def csc_entry_perm(self):
        """Entry index of every CSC position (int64, device), or None when the entries
        are already in CSC order.  The CSC is sorted by (col, row) and (row, col) pairs
        are unique, so this is the argsort of col * M + row (cached)."""
        if self.__dict__.get("_csc_perm_done"):
            return self._csc_perm
        t = nat.torch()
        er, ec, _ = self.device_entries()
        n = self._nnz
        key = ec[:n].to(t.int64) * self.M + er[:n].to(t.int64)
        perm = t.argsort(key)
        ident = bool(t.equal(perm, t.arange(n, device=perm.device))) if n else True
        self._csc_perm = None if ident else perm
        self._csc_perm_done = True
        return self._csc_perm

    def csr_entry_index(self):
        """Entry index of every CSR position (int32, device), or None when the entries
        are in CSR order: the CSC entry permutation carried through csc2csr (cached)."""
        if self.__dict__.get("_csr_entry_done"):
            return self._csr_entry
        t = nat.torch()
        n = self._nnz
        dev = self.device()
        perm = self.csc_entry_perm()
        src = perm.to(t.int32) if perm is not None else t.arange(n, dtype=t.int32, device=dev.csc2csr.device)
        ce = t.empty(max(n, 1), dtype=t.int32, device=src.device)
        if n:
            ce.scatter_(0, dev.csc2csr[:n].to(t.int64), src)
        ident = bool(t.equal(ce[:n], t.arange(n, dtype=t.int32, device=ce.device))) if n else True
        self._csr_entry = None if ident else ce
        self._csr_entry_done = True
        return self._csr_entry

    def row_slice(self, i: int):
        lo, hi = self.row_ptr[i], self.row_ptr[i + 1]
        return self.row_cols[lo:hi], self.row_vals[lo:hi]

    def col_slice(self, j: int):
        lo, hi = self.col_ptr[j], self.col_ptr[j + 1]
        return self.col_rows[lo:hi], self.col_vals[lo:hi]

    def rating(self, i: int, j: int) -> float | None:
        cols, vals = self.row_slice(i)
        k = np.searchsorted(cols, j)
        if k < len(cols) and cols[k] == j:
            return float(vals[k])
        return None

    def baselines(self) -> BaselineStats:
        if self._baselines is None:
            d = self._dev
            if d is not None and getattr(d, "exact_baselines", False):
                # integer-valued data: the device sums are exact, hence the reference's bytes
                self._baselines = BaselineStats(d.mu, nat.to_host(d.base_b)[:self.M].copy(),
                                                nat.to_host(d.base_bhat)[:self.N].copy())
            else:
                self._baselines = compute_baselines(self)
        return self._baselines

    def device(self) -> "DeviceRatings":
        """HBM-resident copy of both views (built once, cached)."""
        if self._dev is None:
            self._dev = DeviceRatings(self)
        return self._dev

    def save(self, path) -> None:
        """LSHMF-R v1 text matrix (data.py:238-243): header, then one ``row col value``
        line per entry in entry order, values as Python float repr."""
        with open(path, "w") as fh:
            fh.write(f"{RATINGS_MAGIC} {RATINGS_VERSION} {self.M} {self.N} {self.nnz}\n")
            fh.writelines(f"{i} {j} {v!r}\n" for i, j, v in
                          zip(self.entry_rows.tolist(), self.entry_cols.tolist(), self.entry_values.tolist()))

    @classmethod
    def load(cls, path) -> "SparseRatings":
        """Read an LSHMF-R v1 file (data.py:245-257); ValueError on a foreign header."""
        with open(path) as fh:
            header = fh.readline().split()
            if len(header) != 5 or header[0] != RATINGS_MAGIC or header[1] != RATINGS_VERSION:
                raise ValueError(f"{path}: not a {RATINGS_MAGIC} {RATINGS_VERSION} file")
            M, N, nnz = int(header[2]), int(header[3]), int(header[4])
            rows = np.empty(nnz, dtype=np.int32)
            cols = np.empty(nnz, dtype=np.int32)
            vals = np.empty(nnz, dtype=np.float64)
            for k in range(nnz):
                fields = fh.readline().split()
                rows[k], cols[k], vals[k] = int(fields[0]), int(fields[1]), float(fields[2])
        return build_indices(Triplets(rows, cols, vals), M=M, N=N)


RATINGS_MAGIC = "LSHMF-R"
RATINGS_VERSION = "v1"


def build_indices(triplets: Triplets, M: int | None = None, N: int | None = None) -> SparseRatings:
    """Index triplets, rejecting out-of-range, non-finite and duplicate entries (data.py:269-286)."""
    rows, cols, vals = triplets.rows, triplets.cols, triplets.values
    M = triplets.M if M is None else M
    N = triplets.N if N is None else N
    if len(rows) and (rows.min() < 0 or rows.max() >= M):
        raise ValueError("row index out of range")
    if len(cols) and (cols.min() < 0 or cols.max() >= N):
        raise ValueError("column index out of range")
    if len(vals) and not np.all(np.isfinite(vals)):
        raise ValueError("non-finite rating value")
    if len(rows) >= _DEVICE_BUILD_MIN and _gpu_present():
        # the same first duplicate as the host lexsort below: stable device sort of row*N+col
        t = nat.torch()
        key = nat.to_dev(np.asarray(rows, np.int64)) * int(N) + nat.to_dev(np.asarray(cols, np.int64))
        sk, order = t.sort(key, stable=True)
        same = t.nonzero(sk[1:] == sk[:-1])
        if same.numel():
            k = int(order[int(same[0, 0].item())].item())
            raise ValueError(f"duplicate entry at (row={rows[k]}, col={cols[k]})")
    elif len(rows):
        order = np.lexsort((cols, rows))
        same = (np.diff(rows[order]) == 0) & (np.diff(cols[order]) == 0)
        if same.any():
            k = order[int(np.flatnonzero(same)[0])]
            raise ValueError(f"duplicate entry at (row={rows[k]}, col={cols[k]})")
    return SparseRatings(M, N, rows, cols, vals, triplets.row_ids, triplets.col_ids)


def compute_baselines(ratings: SparseRatings) -> BaselineStats:
    """mu and per-row / per-column mean deviations, 0 where empty (data.py:289-309).

    Host numpy with the reference's summation order (np.mean pairwise sum,
    np.add.at in entry order) so the residual statistics are bit-identical.
    """
    if ratings.nnz == 0:
        raise ValueError("cannot compute baselines of an empty matrix")
    mu = float(ratings.entry_values.mean())
    row_counts = np.diff(ratings.row_ptr)
    col_counts = np.diff(ratings.col_ptr)
    row_sums = np.zeros(ratings.M)
    np.add.at(row_sums, ratings.entry_rows, ratings.entry_values)
    col_sums = np.zeros(ratings.N)
    np.add.at(col_sums, ratings.entry_cols, ratings.entry_values)
    b = np.zeros(ratings.M)
    nz = row_counts > 0
    b[nz] = row_sums[nz] / row_counts[nz] - mu
    b_hat = np.zeros(ratings.N)
    nz = col_counts > 0
    b_hat[nz] = col_sums[nz] / col_counts[nz] - mu
    return BaselineStats(mu=mu, b=b, b_hat=b_hat)


class DeviceSparseRatings:
    """A SparseRatings built directly in HBM from device triplets (large inputs).

    Same role as SparseRatings for the GPU entry points (``device()``,
    ``baselines()``, ``M``/``N``/``nnz``); both index views are built by device
    sorts.  Baselines are computed on the device in the reference's summation order
    (exact_baselines_device), so they are bit-identical to compute_baselines of the same
    triplets for any values.
    """

    def __init__(self, M: int, N: int, rows, cols, vals):
        t = nat.torch()
        d = rows.device
        self.M, self.N, self.nnz = int(M), int(N), int(rows.numel())
        rows = rows.to(t.int32)
        cols = cols.to(t.int32)
        vals = vals.to(t.float64)
        ckey = cols.long() * M + rows.long()
        ckey, o = t.sort(ckey)
        crow, cval = rows[o].contiguous(), vals[o].contiguous()
        col_ptr = t.searchsorted(ckey, t.arange(N + 1, device=d, dtype=t.int64) * M)
        rkey, o2 = t.sort(rows.long() * N + cols.long())
        row_ptr = t.searchsorted(rkey, t.arange(M + 1, device=d, dtype=t.int64) * N)
        del ckey, rkey
        if self.nnz:
            mu, bb, bh = exact_baselines_device(M, N, rows, cols, vals)
        else:
            mu, bb, bh = 0.0, t.zeros(M, dtype=t.float64, device=d), t.zeros(N, dtype=t.float64, device=d)
        self._dev = DeviceRatings.from_device(M, N, col_ptr, crow, cval, row_ptr,
                                              cols[o2].contiguous(), vals[o2].contiguous(), mu, bb, bh)
        self._stats = BaselineStats(mu, nat.to_host(bb), nat.to_host(bh))

    def device(self) -> "DeviceRatings":
        return self._dev

    def baselines(self) -> BaselineStats:
        return self._stats


class DeviceRatings:
    """Both views of a SparseRatings in HBM plus the CulshData view for the C ABI.

    Layout: col_ptr/row_ptr int64 (N+1 / M+1), col_rows/row_cols int32 (nnz),
    col_vals/row_vals float64 (nnz), csc2csr int32 (nnz), base_b (M) and
    base_bhat (N) float64.  About 36 bytes per rating.
    """

    @classmethod
    def from_device(cls, M: int, N: int, col_ptr, col_rows, col_vals, row_ptr, row_cols, row_vals,
                    mu: float, base_b, base_bhat, csc2csr=None, map_out=None) -> "DeviceRatings":
        """Wrap index arrays that already live in HBM (e.g. built by synth.py).

        csc2csr: a callable(DeviceRatings) that fills self.csc2csr, default the
        full binary-search map; map_out: preallocated int32 storage (>= nnz) for it."""
        self = cls.__new__(cls)
        self.M, self.N, self.nnz = int(M), int(N), int(col_rows.numel())
        self.col_ptr, self.col_rows, self.col_vals = col_ptr, col_rows, col_vals
        self.row_ptr, self.row_cols, self.row_vals = row_ptr, row_cols, row_vals
        self.mu, self.base_b, self.base_bhat = float(mu), base_b, base_bhat
        self.csc2csr = map_out if map_out is not None else nat.empty((max(self.nnz, 1),), "int32")
        self.struct = self._make_struct()
        if csc2csr is not None:
            csc2csr(self)
        else:
            nat.call("culsh_csc_to_csr_map", ctypes.byref(self.struct), nat.ptr(self.csc2csr),
                     nat.stream_ptr())
        return self

    def __init__(self, r: SparseRatings, with_baselines: bool = True):
        self.M, self.N, self.nnz = r.M, r.N, r.nnz
        self.col_ptr = nat.to_dev(r.col_ptr, np.int64)
        self.col_rows = nat.to_dev(r.col_rows, np.int32)
        self.col_vals = nat.to_dev(r.col_vals, np.float64)
        self.row_ptr = nat.to_dev(r.row_ptr, np.int64)
        self.row_cols = nat.to_dev(r.row_cols, np.int32)
        self.row_vals = nat.to_dev(r.row_vals, np.float64)
        self.csc2csr = nat.empty((max(r.nnz, 1),), "int32")
        self.exact_baselines = False
        if r.nnz and with_baselines and r._baselines is None and self.integer_valued():
            # every sum exact: device statistics are the reference's bytes (data.py:289-309)
            self.mu, self.base_b, self.base_bhat = device_baselines(
                r.M, r.N, self.col_ptr, self.col_vals, self.row_ptr, self.row_vals, r.nnz)
            self.exact_baselines = True
        elif r.nnz and with_baselines:
            st = r.baselines()
            self.mu = st.mu
            self.base_b = nat.to_dev(st.b, np.float64)
            self.base_bhat = nat.to_dev(st.b_hat, np.float64)
        else:
            self.mu = 0.0
            self.base_b = nat.zeros((max(r.M, 1),), "float64")
            self.base_bhat = nat.zeros((max(r.N, 1),), "float64")
        self.struct = self._make_struct()
        nat.call("culsh_csc_to_csr_map", ctypes.byref(self.struct), nat.ptr(self.csc2csr),
                 nat.stream_ptr())

    def _make_struct(self) -> nat.CulshData:
        p = nat.ptr
        return nat.CulshData(self.M, self.N, self.nnz, p(self.col_ptr), p(self.col_rows),
                             p(self.col_vals), p(self.row_ptr), p(self.row_cols), p(self.row_vals),
                             p(self.csc2csr), p(self.base_b), p(self.base_bhat))

    def integer_valued(self) -> bool:
        """Whether every rating is an integer (then every baseline sum is exact and
        device-side statistics equal the reference's bit for bit).  Cached."""
        v = self.__dict__.get("_integer_valued")
        if v is None:
            t = nat.torch()
            vals = self.col_vals[:self.nnz]
            v = bool(t.all(vals == t.round(vals)).item()) if self.nnz else True
            self._integer_valued = v
        return v

    def set_baselines(self, mu: float, b: np.ndarray, b_hat: np.ndarray) -> None:
        self.mu = float(mu)
        self.base_b = nat.to_dev(b, np.float64)
        self.base_bhat = nat.to_dev(b_hat, np.float64)
        self.struct = self._make_struct()


_PW_CHUNK = 1 << 16


def _pairwise_plan(n: int):
    """Nodes of numpy's pairwise split tree over n elements (halves rounded down to multiples
    of 8) of at most _PW_CHUNK elements, left to right: (offsets, lengths)."""
    offs, lens = [], []

    def split(o, m):
        if m <= _PW_CHUNK:
            offs.append(o)
            lens.append(m)
            return
        m2 = m // 2
        m2 -= m2 % 8
        split(o, m2)
        split(o + m2, m - m2)

    if n:
        split(0, n)
    return offs, lens


def _pairwise_combine(n: int, node_sums) -> float:
    """numpy's sum of the whole array from the sums of _pairwise_plan(n)'s nodes, combined
    up the same tree (left + right, IEEE double)."""
    vals = iter(node_sums)

    def combine(m):
        if m <= _PW_CHUNK:
            return next(vals)
        m2 = m // 2
        m2 -= m2 % 8
        left = combine(m2)
        return left + combine(m - m2)

    return combine(n) if n else 0.0


def pairwise_sum_device(x) -> float:
    """numpy's np.add.reduce of a device float64 vector, bit for bit: the top of numpy's
    pairwise split tree is walked on the host down to nodes of <= 65,536 elements
    (_pairwise_plan), culsh_pairwise_chunks sums each node on the device (thread per node,
    the same tree below), and the node sums are combined back up in the same order."""
    n = int(x.numel())
    if n == 0:
        return 0.0
    offs, lens = _pairwise_plan(n)
    part = nat.empty((len(offs),), "float64")
    d_off = nat.to_dev(np.asarray(offs, np.int64))      # keep both alive until the kernel ran
    d_len = nat.to_dev(np.asarray(lens, np.int64))
    nat.call("culsh_pairwise_chunks", nat.ptr(x), nat.ptr(d_off), nat.ptr(d_len), len(offs), nat.ptr(part),
             nat.stream_ptr())
    return _pairwise_combine(n, nat.to_host(part).tolist())


def _ordered_sums(n_seg: int, keys, vals, init=None):
    """Per-segment sums of vals grouped by keys (int32 device, 0 <= key < n_seg), each in
    entry order (a stable sort), as np.add.at(zeros, keys, vals) + init."""
    t = nat.torch()
    sk, order = t.sort(keys.to(t.int64), stable=True)
    ptr = t.searchsorted(sk, t.arange(n_seg + 1, device=sk.device, dtype=t.int64))
    out = nat.empty((max(n_seg, 1),), "float64")
    nat.call("culsh_ordered_segment_sums", n_seg, nat.ptr(ptr), nat.ptr(order), nat.ptr(vals), nat.ptr(init),
             nat.ptr(out), nat.stream_ptr())
    cnt = (ptr[1:] - ptr[:-1]).to(t.float64)
    return out[:n_seg], cnt


def exact_baselines_device(M: int, N: int, rows, cols, vals):
    """compute_baselines (data.py:289-309) on the device for ANY values, bit-identical to
    the host numpy: mu by numpy's pairwise mean, row / column sums sequential in entry order
    (np.add.at), then sum / count - mu.  rows / cols / vals: device triplets in ENTRY order.
    Returns (mu, b, b_hat) with b, b_hat device float64."""
    t = nat.torch()
    n = int(vals.numel())
    mu = pairwise_sum_device(vals) / n
    rs, rc = _ordered_sums(M, rows, vals)
    cs, cc = _ordered_sums(N, cols, vals)
    bb = t.where(rc > 0, rs / rc.clamp(min=1) - mu, t.zeros_like(rs))
    bh = t.where(cc > 0, cs / cc.clamp(min=1) - mu, t.zeros_like(cs))
    return mu, bb, bh


def device_baselines(M: int, N: int, col_ptr, col_vals, row_ptr, row_vals, nnz: int):
    """compute_baselines (data.py:289-309) from the two views' segment sums (exact,
    hence bit-identical, for integer-valued ratings)."""
    t = nat.torch()
    cs = nat.empty((max(N, 1),), "float64")
    rs = nat.empty((max(M, 1),), "float64")
    nat.call("culsh_segment_sums", N, nat.ptr(col_ptr), nat.ptr(col_vals), nat.ptr(cs), nat.stream_ptr())
    nat.call("culsh_segment_sums", M, nat.ptr(row_ptr), nat.ptr(row_vals), nat.ptr(rs), nat.stream_ptr())
    cs, rs = cs[:N], rs[:M]
    mu = float(cs.sum().item()) / max(nnz, 1)
    cnt_c = (col_ptr[1:] - col_ptr[:-1]).to(t.float64)
    rc = (row_ptr[1:] - row_ptr[:-1]).to(t.float64)
    bb = t.where(rc > 0, rs / rc.clamp(min=1) - mu, t.zeros_like(rs))
    bh = t.where(cnt_c > 0, cs / cnt_c.clamp(min=1) - mu, t.zeros_like(cs))
    return mu, bb, bh


def transform_ratings(triplets: Triplets, zero_floor: float | None = None,
                      scale: float | None = None) -> Triplets:
    """Replace exact-zero values by ``zero_floor``, then divide by ``scale``
    (data.py:150-163); the inverse scale is applied at evaluation time."""
    if scale is not None and scale <= 0:
        raise ValueError(f"scale must be positive, got {scale}")
    values = np.array(triplets.values, dtype=np.float64, copy=True)
    if zero_floor is not None:
        values[values == 0.0] = zero_floor
    if scale is not None:
        values = values / scale
    return Triplets(triplets.rows, triplets.cols, values, triplets.row_ids, triplets.col_ids)


def split_holdout(ratings: SparseRatings, test_fraction: float, seed: int):
    """Deterministic holdout split (data.py:312-346): returns (train SparseRatings over
    the same index space, test Triplets).  Entries move to the test side in the order of
    numpy's PCG64 permutation (the reference's stream, drawn here) while their row and
    column keep a training entry; the sequential decisions run natively
    (culsh_split_holdout) instead of as an interpreted loop."""
    import ctypes
    if not (0 <= test_fraction < 1):
        raise ValueError(f"test_fraction must be in [0, 1), got {test_fraction}")
    nnz = ratings.nnz
    n_test = int(round(test_fraction * nnz))
    in_test = np.zeros(nnz, dtype=np.uint8)
    if n_test > 0:
        perm = np.ascontiguousarray(np.random.default_rng(seed).permutation(nnz), dtype=np.int64)
        rows = np.ascontiguousarray(ratings.entry_rows, dtype=np.int32)
        cols = np.ascontiguousarray(ratings.entry_cols, dtype=np.int32)
        p = lambda a: ctypes.c_void_p(a.ctypes.data)
        nat.call("culsh_split_holdout", p(rows), p(cols), nnz, ratings.M, ratings.N, p(perm), n_test,
                 p(in_test))
    mask = in_test.astype(bool)
    keep = ~mask
    train = SparseRatings(ratings.M, ratings.N, ratings.entry_rows[keep], ratings.entry_cols[keep],
                          ratings.entry_values[keep], ratings.row_ids, ratings.col_ids)
    test = Triplets(ratings.entry_rows[mask].copy(), ratings.entry_cols[mask].copy(),
                    ratings.entry_values[mask].copy(), ratings.row_ids, ratings.col_ids)
    return train, test
