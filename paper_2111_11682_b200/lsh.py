"""simLSH signatures, buckets and frequency Top-K on the GPU.

Same public surface and semantics as the reference module lshmf.lsh
(lsh.py:30-438); every array result is bit-identical to it.  The compute runs
in libculsh.so (csrc/lsh.cu, csrc/topk.cu):

  assign_row_hashes  -> culsh_row_hash_table   (lsh.py:68-114)
  compute_hash_state -> culsh_hash_accumulate  (lsh.py:161-183, 231-239, 246-260 fused)
  simlsh_topk        -> + culsh_topk           (lsh.py:263-374, 401-438)

Host objects (RowHashes, HashState) keep their device tensors and materialise
numpy views lazily, so a device pipeline never round-trips through the host.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .data import SparseRatings
from .similarity import NeighborTable

HASHSTATE_MAGIC = "LSHMF-H"
HASHSTATE_VERSION = "v1"


@dataclass
class LshConfig:
    """Signature parameters: G bits per map, p maps per group, q groups (lsh.py:30-50)."""

    G: int = 8
    p: int = 3
    q: int = 100
    psi_exponent: int = 2
    seed: int = 0

    def validate(self) -> None:
        if not (1 <= self.G <= 64):
            raise ValueError(f"G must be in [1, 64], got {self.G}")
        if self.p < 1 or self.q < 1:
            raise ValueError("p and q must be >= 1")
        if self.p * self.G > 64:
            raise ValueError(f"p*G = {self.p * self.G} exceeds the 64-bit bucket key")
        if self.psi_exponent not in (1, 2, 4):
            raise ValueError(f"psi_exponent must be 1, 2 or 4, got {self.psi_exponent}")
        if self.seed < 0:
            raise ValueError("seed must be nonnegative")


def _ns(G: int) -> int:
    return (G + 7) // 8


class RowHashes:
    """Random G-bit row hashes for all p*q maps, keyed by (seed, group, map, row).

    ``bits`` is the reference's (M, q, p, G) uint8 tensor (lsh.py:81-105); on the
    device the same bits are a packed (M, q, p, ceil(G/8)) byte table.
    """

    def __init__(self, bits: np.ndarray | None = None, seed: int = 0, *, _table=None,
                 _shape=None):
        self.seed = int(seed)
        self._bits = None if bits is None else np.ascontiguousarray(bits, dtype=np.uint8)
        self._table = _table
        self._shape = tuple(_shape) if _shape is not None else tuple(self._bits.shape)

    @property
    def bits(self) -> np.ndarray:
        if self._bits is None:
            M, q, p, G = self._shape
            out = nat.empty((max(M * q * p * G, 1),), "uint8")
            nat.call("culsh_unpack_bits", nat.ptr(self._table), M, q, p, G, nat.ptr(out),
                     nat.stream_ptr())
            self._bits = nat.to_host(out)[:M * q * p * G].reshape(M, q, p, G)
        return self._bits

    @property
    def M(self) -> int:
        return self._shape[0]

    def map_bits(self, g: int, m: int) -> np.ndarray:
        return self.bits[:, g, m, :]

    def table(self):
        """Packed device table (packs injected host bits on first use)."""
        if self._table is None:
            M, q, p, G = self._shape
            src = nat.to_dev(self._bits.reshape(-1) if self._bits.size else np.zeros(1, np.uint8))
            t = _table_alloc(M, q, p, G)
            nat.call("culsh_pack_bits", nat.ptr(src), M, q, p, G, nat.ptr(t), nat.stream_ptr())
            self._table = t
        return self._table

    def extended(self, M_new: int) -> "RowHashes":
        if M_new < self.M:
            raise ValueError("cannot shrink row hashes")
        _, q, p, G = self._shape
        return _device_row_hashes(M_new, q, p, G, self.seed)


def _table_alloc(M: int, q: int, p: int, G: int):
    """Packed table storage: M rows + one all-zero padding row (read by the
    bit-count kernel for group tails)."""
    rec = (q * p * _ns(G) + 15) // 16 * 16   # row record padded to the 16-byte bulk-copy unit
    t = nat.empty(((M + 1) * rec,), "uint8")
    t[M * rec:].zero_()
    return t


def _device_row_hashes(M: int, q: int, p: int, G: int, seed: int) -> RowHashes:
    t = _table_alloc(M, q, p, G)
    nat.call("culsh_row_hash_table", ctypes.c_uint64(seed), q, p, G, 0, M, nat.ptr(t),
             nat.stream_ptr())
    return RowHashes(None, seed, _table=t, _shape=(M, q, p, G))


def assign_row_hashes(M: int, config: LshConfig) -> RowHashes:
    """Independent uniform G-bit hashes for every (group, map, row) (lsh.py:108-114)."""
    config.validate()
    if M < 0:
        raise ValueError("M must be nonnegative")
    return _device_row_hashes(M, config.q, config.p, config.G, config.seed)


class HashState:
    """Per-column signed accumulators and signatures (lsh.py:186-228).

    ``acc`` (N, q, p, G) float64 and ``sig`` (N, q, p, G) uint8.  One side is the
    source of truth:

    * a state built by the device pipeline (``simlsh_topk``, ``update_hashes_incremental``)
      keeps acc / sig / the packed group keys (q, N) u64 resident on the device; the host
      arrays are read-only copies materialised on first access, so an in-place edit of
      them fails loudly instead of silently diverging from the device copy;
    * a state built from host arrays (the constructor, ``load``, or assigning ``.acc`` /
      ``.sig``) is owned by the host, as in the reference dataclass: every device use
      re-reads those arrays (acc uploaded, group keys packed from ``sig``, as
      ``_state_group_keys`` does at lsh.py:417-423), so edits made to them are seen.
    """

    def __init__(self, acc: np.ndarray | None = None, sig: np.ndarray | None = None,
                 config: LshConfig | None = None, *, _dev_acc=None, _dev_sig=None,
                 _dev_keys=None, _shape=None):
        self.config = config
        self._acc = acc
        self._sig = sig
        self._dev_acc = _dev_acc
        self._dev_sig = _dev_sig
        self._dev_keys = _dev_keys
        self._host_truth = _dev_acc is None
        self._shape = tuple(_shape) if _shape is not None else tuple(np.shape(acc))

    def __eq__(self, other):
        if not isinstance(other, HashState):
            return NotImplemented
        return (self.config == other.config and np.array_equal(self.acc, other.acc)
                and np.array_equal(self.sig, other.sig))

    @staticmethod
    def _readonly(a: np.ndarray) -> np.ndarray:
        a.flags.writeable = False
        return a

    @property
    def acc(self) -> np.ndarray:
        if self._acc is None:
            self._acc = self._readonly(nat.to_host(self._dev_acc).reshape(self._shape))
        return self._acc

    @acc.setter
    def acc(self, value):
        self._to_host_truth()
        self._acc = value
        self._shape = tuple(np.shape(value))

    @property
    def sig(self) -> np.ndarray:
        if self._sig is None:
            if self._dev_sig is not None:
                self._sig = self._readonly(nat.to_host(self._dev_sig).reshape(self._shape))
            else:
                self._sig = (self.acc >= 0.0).astype(np.uint8)
                if not self._host_truth:
                    self._readonly(self._sig)
        return self._sig

    @sig.setter
    def sig(self, value):
        self._to_host_truth()
        self._sig = value

    def _to_host_truth(self) -> None:
        """Switch ownership to the host arrays (materialising the other one first)."""
        if not self._host_truth:
            acc, sig = self.acc, self.sig
            self._acc = np.array(acc)
            self._sig = np.array(sig)
        self._host_truth = True
        self._dev_acc = self._dev_sig = self._dev_keys = None

    @property
    def N(self) -> int:
        return self._shape[0]

    def acc_map(self, g: int, m: int) -> np.ndarray:
        return self.acc[:, g, m, :]

    def sig_map(self, g: int, m: int) -> np.ndarray:
        return self.sig[:, g, m, :]

    def device_acc(self):
        """acc (N*q*p*G,) f64 on the device: the resident copy, or a fresh upload of the
        host array when the host owns the state."""
        if self._host_truth:
            return nat.to_dev(np.ascontiguousarray(self._acc, dtype=np.float64).reshape(-1)
                              if np.size(self._acc) else np.zeros(1))
        return self._dev_acc

    def device_keys(self):
        """(q, N) uint64 group keys on the device: resident, or packed from the host
        ``sig`` when the host owns the state (lsh.py:417-423 derives keys from sig)."""
        if not self._host_truth and self._dev_keys is not None:
            return self._dev_keys
        c = self.config
        N = self.N
        keys = nat.empty((c.q * max(N, 1),), "uint64")
        if N:
            if self._host_truth:
                sig = self._sig if self._sig is not None else (self._acc >= 0.0)
                sig_dev = nat.to_dev(np.ascontiguousarray(sig, dtype=np.uint8).reshape(-1))
                nat.call("culsh_pack_keys", nat.ptr(sig_dev), N, c.q, c.p, c.G, nat.ptr(keys),
                         nat.stream_ptr())
            else:
                _keys_from_acc(self._dev_acc, N, c, keys)
        if not self._host_truth:
            self._dev_keys = keys
        return keys

    def save(self, path) -> None:
        c = self.config
        with open(path, "wb") as fh:
            header = (f"{HASHSTATE_MAGIC} {HASHSTATE_VERSION} {self.N} {c.G} "
                      f"{c.p} {c.q} {c.psi_exponent} {c.seed}\n")
            fh.write(header.encode())
            blob = np.ascontiguousarray(self.acc.transpose(1, 2, 0, 3))
            fh.write(blob.astype("<f8").tobytes())

    @classmethod
    def load(cls, path) -> "HashState":
        with open(path, "rb") as fh:
            header = fh.readline().decode().split()
            if len(header) != 8 or header[0] != HASHSTATE_MAGIC or header[1] != HASHSTATE_VERSION:
                raise ValueError(f"{path}: not a {HASHSTATE_MAGIC} {HASHSTATE_VERSION} file")
            N, G, p, q, e, seed = (int(x) for x in header[2:])
            blob = np.frombuffer(fh.read(), dtype="<f8")
        acc = blob.reshape(q, p, N, G).transpose(2, 0, 1, 3).copy()
        config = LshConfig(G=G, p=p, q=q, psi_exponent=e, seed=seed)
        return cls(acc=acc, sig=(acc >= 0.0).astype(np.uint8), config=config)


def _keys_from_acc(acc_dev, N: int, c: LshConfig, keys_out) -> None:
    """Group keys of an existing accumulator state: threshold + pack on the device.

    Runs the accumulation kernel in `into` mode over empty columns, which leaves
    acc unchanged and re-emits sig-derived keys (lsh.py:246-260, 417-423).
    """
    empty_ptr = nat.zeros((N + 1,), "int64")
    dummy_rows = nat.zeros((1,), "int32")
    dummy_vals = nat.zeros((1,), "float64")
    table = nat.zeros((max(c.q * c.p * _ns(c.G), 1),), "uint8")
    nat.call("culsh_hash_accumulate", nat.ptr(empty_ptr), nat.ptr(dummy_rows), nat.ptr(dummy_vals),
             0, N, None, nat.ptr(table), c.q, c.p, c.G, c.psi_exponent, 1, 0, nat.ptr(acc_dev),
             None, nat.ptr(keys_out), N, nat.stream_ptr())


def _int_path_ok(dev, col_begin: int, n_cols: int, col_list, e: int) -> bool:
    bad = nat.zeros((1,), "int32")
    nat.call("culsh_psi_int_check", nat.ptr(dev.col_ptr), nat.ptr(dev.col_vals), col_begin, n_cols,
             nat.ptr(col_list), e, nat.ptr(bad), nat.stream_ptr())
    return int(bad.item()) == 0


_MAX_CLASSES = 16
_SLICE_MB = int(__import__("os").environ.get("CULSH_HASH_SLICE_MB", "0"))   # 0 = one pass
_COUNT_VARIANT = 1   # 0: bulk-copy (TMA engine) staging, 1: register double buffering (faster)


def _value_classes(dev):
    """Distinct rating values of the matrix if there are at most 16 (cached per
    DeviceRatings; the ratings are immutable), else None."""
    if hasattr(dev, "_value_classes"):
        return dev._value_classes
    nb = 1184   # 148 SMs x 8: enough loads in flight to stream the values at HBM speed
    out = nat.empty((nb * (_MAX_CLASSES + 1),), "float64")
    nat.call("culsh_value_set", nat.ptr(dev.col_vals), dev.nnz, nat.ptr(out), nb, nat.stream_ptr())
    o = nat.to_host(out).reshape(nb, _MAX_CLASSES + 1)
    if (o[:, 0] < 0).any():
        classes = None
    else:
        have = np.arange(_MAX_CLASSES)[None, :] < o[:, :1]
        vals = np.unique(o[:, 1:][have])
        classes = vals if len(vals) <= _MAX_CLASSES else None
    dev._value_classes = classes
    return classes


def _class_partition(dev, classes: np.ndarray):
    """Row indices of every column grouped by value class (cached per DeviceRatings)."""
    if getattr(dev, "_class_part", None) is None:
        NC = len(classes)
        cv = nat.to_dev(np.asarray(classes, np.float64))
        rows_bc = nat.empty((max(dev.nnz, 1),), "int32")
        off = nat.empty(((NC + 1) * max(dev.N, 1),), "int32")
        nat.call("culsh_class_partition", nat.ptr(dev.col_ptr), nat.ptr(dev.col_rows),
                 nat.ptr(dev.col_vals), dev.N, nat.ptr(cv), NC, nat.ptr(rows_bc), nat.ptr(off),
                 nat.stream_ptr())
        dev._class_part = (rows_bc, off)
    return dev._class_part


def _psi_int(v: float, e: int):
    p = v if e == 1 else (v * v if e == 2 else (v * v) * (v * v))
    return int(p) if float(p).is_integer() and abs(p) < 2 ** 20 else None


def _count_path(dev, table, c: LshConfig, acc, sig, keys, col_begin, n_cols, keys_ld,
                table_ready=None) -> bool:
    """Harley-Seal bit-count kernel (exact integers) when the data allow it."""
    W8 = c.q * c.p * _ns(c.G)
    if W8 % 4 or W8 > 512 or dev.nnz == 0:
        return False
    classes = _value_classes(dev)
    if classes is None:
        return False
    psi = [_psi_int(float(v), c.psi_exponent) for v in classes]
    if any(x is None for x in psi):
        return False
    cpsi = nat.to_dev(np.asarray(psi, np.int32))

    def count(c0, nc):
        nat.call("culsh_hash_count", nat.ptr(dev.col_ptr), nat.ptr(rows_bc), nat.ptr(off), len(classes),
                 nat.ptr(cpsi), dev.M, int(_SLICE_MB), int(_COUNT_VARIANT), c0, nc, nat.ptr(table),
                 c.q, c.p, c.G, nat.ptr(acc), nat.ptr(sig), nat.ptr(keys),
                 dev.N if keys_ld is None else keys_ld, nat.stream_ptr())

    # (pipelining the class partition by column chunks on a side stream under the bit-count
    # kernel was measured slower: 10.7 vs 10.1 ms at C3 -- the concurrent partition slows the
    # gather-bound count kernel more than it hides)
    rows_bc, off = _class_partition(dev, classes)
    if table_ready is not None:
        nat.torch().cuda.current_stream().wait_event(table_ready)
    count(col_begin, n_cols)
    return True


def _accumulate(dev, table, c: LshConfig, acc, sig, keys, col_begin: int, n_cols: int,
                col_list=None, into: bool = False, keys_ld: int | None = None,
                allow_count: bool = True, table_ready=None) -> None:
    if not into and col_list is None and allow_count and _count_path(dev, table, c, acc, sig, keys, col_begin,
                                                                     n_cols, keys_ld, table_ready):
        return   # (its value classes all have integer psi: no separate integer check needed)
    int_path = (not into) and _int_path_ok(dev, col_begin, n_cols, col_list, c.psi_exponent)
    if table_ready is not None:
        nat.torch().cuda.current_stream().wait_event(table_ready)
    nat.call("culsh_hash_accumulate", nat.ptr(dev.col_ptr), nat.ptr(dev.col_rows),
             nat.ptr(dev.col_vals), col_begin, n_cols, nat.ptr(col_list), nat.ptr(table), c.q, c.p,
             c.G, c.psi_exponent, int(into), int(int_path), nat.ptr(acc), nat.ptr(sig),
             nat.ptr(keys), dev.N if keys_ld is None else keys_ld, nat.stream_ptr())


def compute_hash_state(ratings: SparseRatings, config: LshConfig,
                       hashes: RowHashes | None = None) -> HashState:
    """Encode every column under all p*q maps (lsh.py:231-239)."""
    config.validate()
    if hashes is None:
        hashes = assign_row_hashes(ratings.M, config)
    else:
        _, q, p, G = hashes._shape
        if (q, p, G) != (config.q, config.p, config.G):
            raise ValueError("row hashes do not match the configuration")
        if hashes.M < ratings.M:
            raise ValueError("row hashes do not cover every row")
    return hash_state_device(ratings.device(), config, hashes)


def hash_state_device(dev, config: LshConfig, hashes: RowHashes | None = None) -> HashState:
    """compute_hash_state on HBM-resident ratings (a DeviceRatings)."""
    config.validate()
    t = nat.torch()
    table_ready = None
    if hashes is None:
        # the row-hash table depends only on (seed, M): generate it on a side stream under the
        # value-set / class-partition passes; the accumulate waits for it
        main = t.cuda.current_stream()
        side = nat.side_stream("row_hashes")
        side.wait_stream(main)
        with t.cuda.stream(side):
            hashes = assign_row_hashes(dev.M, config)
            table_ready = t.cuda.Event()
            table_ready.record(side)
        hashes.table().record_stream(main)
    N, c = dev.N, config
    W = c.q * c.p * c.G
    acc = nat.empty((max(N * W, 1),), "float64")
    sig = nat.empty((max(N * W, 1),), "uint8")
    keys = nat.empty((c.q * max(N, 1),), "uint64")
    if N:
        _accumulate(dev, hashes.table(), c, acc, sig, keys, 0, N, table_ready=table_ready)
    elif table_ready is not None:
        t.cuda.current_stream().wait_event(table_ready)
    return HashState(config=config, _dev_acc=acc, _dev_sig=sig, _dev_keys=keys,
                     _shape=(N, c.q, c.p, c.G))


def simlsh_signature(j: int, ratings: SparseRatings, H: np.ndarray, psi_exponent: int = 1):
    """Encode column j against one M x G hash map (lsh.py:126-158, Fig. 3)."""
    H = np.ascontiguousarray(H, dtype=np.uint8)
    M, G = H.shape
    if not (1 <= G <= 64):
        raise ValueError("G must be in [1, 64]")
    if psi_exponent not in (1, 2, 4):
        raise ValueError(f"psi_exponent must be 1, 2 or 4, got {psi_exponent}")
    hashes = RowHashes(H.reshape(M, 1, 1, G), 0)
    cfg = LshConfig(G=G, p=1, q=1, psi_exponent=psi_exponent, seed=0)
    dev = ratings.device()
    acc = nat.zeros((ratings.N * G,), "float64")
    sig = nat.zeros((ratings.N * G,), "uint8")
    col = nat.to_dev(np.array([j], np.int32))
    _accumulate(dev, hashes.table(), cfg, acc, sig, None, 0, 1, col_list=col)
    a = nat.to_host(acc).reshape(ratings.N, G)[j].copy()
    s = nat.to_host(sig).reshape(ratings.N, G)[j].copy()
    return a, s


def _topk_device(keys, q: int, N_total: int, key_bits: int, j_base: int, n_cols: int, K: int,
                 seed: int):
    entries = nat.empty((max(n_cols * K, 1),), "int32")
    ncand = ctypes.c_int64(0)
    nat.call("culsh_topk", nat.ptr(keys), q, N_total, key_bits, j_base, n_cols, K,
             ctypes.c_uint64(seed), nat.ptr(entries), ctypes.byref(ncand), nat.stream_ptr())
    return entries, int(ncand.value)


def coarse_candidates(signatures) -> list[np.ndarray]:
    """Bucket columns that agree on all p maps of one group (lsh.py:290-305).

    ``signatures`` is a sequence of p arrays of shape (N, G); returns, per column,
    the sorted int32 array of the other columns sharing its bucket key.
    """
    sig_group = np.stack([np.asarray(s, dtype=np.uint8) for s in signatures], axis=1)
    N, p, G = sig_group.shape
    if p * G > 64:
        raise ValueError("p*G exceeds the 64-bit bucket key")
    if N == 0:
        return []
    sig = nat.to_dev(np.ascontiguousarray(sig_group.reshape(N, 1, p, G)).reshape(-1))
    keys = nat.empty((N,), "uint64")
    nat.call("culsh_pack_keys", nat.ptr(sig), N, 1, p, G, nat.ptr(keys), nat.stream_ptr())
    offsets = nat.empty((N + 1,), "int64")
    total = ctypes.c_int64(0)
    nat.call("culsh_candidates", nat.ptr(keys), 1, N, p * G, 0, N, nat.ptr(offsets), None, 0,
             ctypes.byref(total), nat.stream_ptr())
    cand = nat.empty((max(total.value, 1),), "int32")
    nat.call("culsh_candidates", nat.ptr(keys), 1, N, p * G, 0, N, nat.ptr(offsets), nat.ptr(cand),
             max(total.value, 1), ctypes.byref(total), nat.stream_ptr())
    off = nat.to_host(offsets)
    c = nat.to_host(cand)[:total.value]
    return [c[off[j]:off[j + 1]].astype(np.int32) for j in range(N)]


def fine_topk(candidate_sets, K: int, N: int, seed: int) -> NeighborTable:
    """Top-K by occurrence frequency across the q groups, seeded supplement
    (lsh.py:377-398); ``candidate_sets`` is q per-group lists of per-column arrays."""
    if K > N - 1:
        raise ValueError(f"K={K} exceeds N-1={N - 1}")
    counts = np.zeros(N + 1, dtype=np.int64)
    for group in candidate_sets:
        for j in range(N):
            counts[j + 1] += len(group[j])
    offsets = np.cumsum(counts)
    cand = np.empty(max(int(offsets[N]), 1), dtype=np.int32)
    fill = offsets[:N].copy()
    for group in candidate_sets:
        for j in range(N):
            k = len(group[j])
            cand[fill[j]:fill[j] + k] = group[j]
            fill[j] += k
    entries = nat.empty((max(N * K, 1),), "int32")
    cand_d, off_d = nat.to_dev(cand), nat.to_dev(offsets)   # keep alive across the call
    nat.call("culsh_select_topk", nat.ptr(cand_d), nat.ptr(off_d), int(offsets[N]), 0, N, K,
             ctypes.c_uint64(seed), N, nat.ptr(entries), nat.stream_ptr())
    return NeighborTable(N=N, K=K, entries=nat.to_host(entries)[:N * K].reshape(N, K).copy())


def simlsh_topk(ratings: SparseRatings, config: LshConfig, K: int):
    """Approximate Top-K neighbours of every column (lsh.py:426-438).

    Returns (NeighborTable, HashState).
    """
    config.validate()
    if K > ratings.N - 1:
        raise ValueError(f"K={K} exceeds N-1={ratings.N - 1}")
    state = compute_hash_state(ratings, config)
    N = ratings.N
    entries, _ = _topk_device(state.device_keys(), config.q, N, config.p * config.G, 0, N, K,
                              config.seed)
    ent = nat.to_host(entries)[:N * K].reshape(N, K).astype(np.int32, copy=False)
    return NeighborTable(N=N, K=K, entries=ent), state


def simlsh_topk_device(dev, config: LshConfig, K: int):
    """simlsh_topk on HBM-resident ratings; returns (entries (N*K) int32 device tensor,
    HashState, candidate count) without any host round trip of the arrays."""
    config.validate()
    if K > dev.N - 1:
        raise ValueError(f"K={K} exceeds N-1={dev.N - 1}")
    state = hash_state_device(dev, config)
    entries, ncand = _topk_device(state.device_keys(), config.q, dev.N, config.p * config.G, 0,
                                  dev.N, K, config.seed)
    return entries, state, ncand
