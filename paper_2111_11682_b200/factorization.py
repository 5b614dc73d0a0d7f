"""Nonlinear-neighbourhood model: prediction, SGD training and RMSE on the GPU.

Same public surface as the reference module lshmf.factorization
(factorization.py:34-601).  Two training modes:

  mode="exact"   (default) deterministic serial-order fp64 schedule on the GPU,
                 bit-identical to the reference's train_full
                 (csrc/sgd_exact.cu: _full_pass_block, factorization.py:332-363)
  mode="hogwild" fp32 warp-per-column Hogwild epochs, the performance mode
                 (csrc/sgd_hogwild.cu; paper Alg. 3), RMSE-equivalent within 0.005

Host numpy is used only where the reference defines a host-side numpy stream
that parity depends on: parameter initialisation (PCG64 uniform draws,
factorization.py:196-211) and the learning-rate schedule.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass, replace

import numpy as np

from . import _native as nat
from .data import BaselineStats, SparseRatings, Triplets
from .similarity import NeighborTable

MODEL_MAGIC = "LSHMF-M"
MODEL_VERSION = "v1"


class TrainingDivergedError(RuntimeError):
    """Raised when a non-finite value appears during training (factorization.py:34-39)."""

    def __init__(self, epoch: int):
        super().__init__(f"training diverged at epoch {epoch}")
        self.epoch = epoch


def learning_rate(alpha: float, beta: float, t: int) -> float:
    """alpha / (1 + beta * t^1.5) at epoch t (factorization.py:42-44)."""
    return alpha / (1.0 + beta * t ** 1.5)


@dataclass
class TrainConfig:
    """Rank, neighbour count, per-parameter rates/regularisers and schedule (factorization.py:47-99)."""

    F: int = 32
    K: int = 32
    alpha_b: float = 0.035
    alpha_b_hat: float = 0.035
    alpha_u: float = 0.035
    alpha_v: float = 0.035
    alpha_w: float = 0.002
    alpha_c: float = 0.002
    beta: float = 0.3
    lambda_b: float = 0.02
    lambda_b_hat: float = 0.02
    lambda_u: float = 0.02
    lambda_v: float = 0.02
    lambda_w: float = 0.002
    lambda_c: float = 0.002
    epochs: int = 50
    init_scale: float | None = None
    seed: int = 0
    clamp_range: tuple[float, float] | None = None

    def validate(self) -> None:
        for name in ("alpha_b", "alpha_b_hat", "alpha_u", "alpha_v", "alpha_w", "alpha_c"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")
        for name in ("lambda_b", "lambda_b_hat", "lambda_u", "lambda_v",
                     "lambda_w", "lambda_c", "beta"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be nonnegative")

    def rates_at(self, t: int) -> tuple:
        return (learning_rate(self.alpha_b, self.beta, t),
                learning_rate(self.alpha_b_hat, self.beta, t),
                learning_rate(self.alpha_u, self.beta, t),
                learning_rate(self.alpha_v, self.beta, t),
                learning_rate(self.alpha_w, self.beta, t),
                learning_rate(self.alpha_c, self.beta, t))

    @property
    def regs(self) -> tuple:
        return (self.lambda_b, self.lambda_b_hat, self.lambda_u,
                self.lambda_v, self.lambda_w, self.lambda_c)

    @property
    def effective_init_scale(self) -> float:
        return self.init_scale if self.init_scale is not None else 1.0 / np.sqrt(self.F)


def _rates_struct(rates, regs) -> nat.CulshRates:
    return nat.CulshRates(*[float(x) for x in tuple(rates) + tuple(regs)])


@dataclass
class ModelParams:
    """All trainable state plus the neighbour table (factorization.py:105-185)."""

    mu: float
    b: np.ndarray
    b_hat: np.ndarray
    U: np.ndarray
    V: np.ndarray
    W: np.ndarray
    C: np.ndarray
    neighbors: NeighborTable | None = None

    @property
    def M(self) -> int:
        return len(self.b)

    @property
    def N(self) -> int:
        return len(self.b_hat)

    @property
    def F(self) -> int:
        return self.U.shape[1]

    @property
    def K(self) -> int:
        return self.W.shape[1]

    def nbr_entries(self) -> np.ndarray:
        if self.neighbors is None:
            return np.zeros((self.N, 0), dtype=np.int32)
        return self.neighbors.entries

    def copy(self) -> "ModelParams":
        nbr = None
        if self.neighbors is not None:
            nbr = NeighborTable(self.neighbors.N, self.neighbors.K, self.neighbors.entries.copy())
        return ModelParams(self.mu, self.b.copy(), self.b_hat.copy(), self.U.copy(),
                           self.V.copy(), self.W.copy(), self.C.copy(), nbr)

    def all_finite(self) -> bool:
        return bool(np.isfinite(self.mu)
                    and np.isfinite(self.b).all() and np.isfinite(self.b_hat).all()
                    and np.isfinite(self.U).all() and np.isfinite(self.V).all()
                    and np.isfinite(self.W).all() and np.isfinite(self.C).all())

    def save(self, path) -> None:
        with open(path, "wb") as fh:
            fh.write(f"{MODEL_MAGIC} {MODEL_VERSION} {self.M} {self.N} "
                     f"{self.F} {self.K}\n".encode())
            fh.write(struct.pack("<d", self.mu))
            for arr in (self.b, self.b_hat, self.U, self.V, self.W, self.C):
                fh.write(np.ascontiguousarray(arr, dtype="<f8").tobytes())
            fh.write(np.ascontiguousarray(self.nbr_entries(), dtype="<u4").tobytes())

    @classmethod
    def load(cls, path) -> "ModelParams":
        with open(path, "rb") as fh:
            header = fh.readline().decode().split()
            if len(header) != 6 or header[0] != MODEL_MAGIC or header[1] != MODEL_VERSION:
                raise ValueError(f"{path}: not a {MODEL_MAGIC} {MODEL_VERSION} file")
            M, N, F, K = (int(x) for x in header[2:])
            mu = struct.unpack("<d", fh.read(8))[0]

            def read_f8(*shape):
                n = int(np.prod(shape))
                return np.frombuffer(fh.read(8 * n), dtype="<f8").reshape(shape).copy()

            b = read_f8(M)
            b_hat = read_f8(N)
            U = read_f8(M, F)
            V = read_f8(N, F)
            W = read_f8(N, K)
            C = read_f8(N, K)
            entries = np.frombuffer(fh.read(4 * N * K), dtype="<u4").reshape(N, K).astype(np.int32)
        neighbors = NeighborTable(N=N, K=K, entries=entries) if K > 0 else None
        return cls(mu, b, b_hat, U, V, W, C, neighbors)


@dataclass
class NeighborSplit:
    """Positions k of a column's neighbour list split by whether row i rated them."""

    explicit: np.ndarray
    implicit: np.ndarray


def init_params(M: int, N: int, F: int, K: int, neighbors: NeighborTable | None,
                baselines: BaselineStats, config: TrainConfig) -> ModelParams:
    """Biases from the baselines, U/V uniform in [0, init_scale], W/C zero (factorization.py:196-211)."""
    if neighbors is not None and (neighbors.N != N or neighbors.K != K):
        raise ValueError("neighbor table does not match N, K")
    rng = np.random.default_rng(config.seed)
    scale = config.effective_init_scale
    U = rng.uniform(0.0, scale, size=(M, F))
    V = rng.uniform(0.0, scale, size=(N, F))
    return ModelParams(mu=baselines.mu, b=baselines.b.copy(), b_hat=baselines.b_hat.copy(),
                       U=U, V=V, W=np.zeros((N, K)), C=np.zeros((N, K)), neighbors=neighbors)


# ------------------------------------------------------------ device model ---

class DeviceModel64:
    """fp64 ModelParams resident in HBM, exposed to the C ABI as CulshModel64."""

    def __init__(self, p: ModelParams):
        self.mu = float(p.mu)
        self.F, self.K = p.F, p.K
        self.b = nat.to_dev(p.b, np.float64)
        self.bhat = nat.to_dev(p.b_hat, np.float64)
        self.U = nat.to_dev(p.U.reshape(-1) if p.U.size else np.zeros(1), np.float64)
        self.V = nat.to_dev(p.V.reshape(-1) if p.V.size else np.zeros(1), np.float64)
        self.W = nat.to_dev(p.W.reshape(-1) if p.W.size else np.zeros(1), np.float64)
        self.C = nat.to_dev(p.C.reshape(-1) if p.C.size else np.zeros(1), np.float64)
        ent = p.nbr_entries()
        self.nbr = nat.to_dev(ent.reshape(-1) if ent.size else np.zeros(1, np.int32), np.int32)
        self.struct = nat.CulshModel64(self.mu, nat.ptr(self.b), nat.ptr(self.bhat), nat.ptr(self.U),
                                       nat.ptr(self.V), nat.ptr(self.W), nat.ptr(self.C),
                                       nat.ptr(self.nbr), self.F, self.K)

    def download(self, p: ModelParams) -> None:
        """Copy the device state back into p's numpy arrays (in place)."""
        p.b[...] = nat.to_host(self.b)[:p.M]
        p.b_hat[...] = nat.to_host(self.bhat)[:p.N]
        if p.U.size:
            p.U[...] = nat.to_host(self.U).reshape(p.U.shape)
        if p.V.size:
            p.V[...] = nat.to_host(self.V).reshape(p.V.shape)
        if p.W.size:
            p.W[...] = nat.to_host(self.W).reshape(p.W.shape)
            p.C[...] = nat.to_host(self.C).reshape(p.C.shape)


class _Scratch:
    """Per-pass device scratch of the exact schedule (row_last, ticket, status, plan)."""

    def __init__(self, M: int, N: int):
        self.row_last = nat.empty((max(M, 1),), "int32")
        self.ticket = nat.zeros((1,), "int32")
        self.status = nat.zeros((1,), "int32")
        self.seg = nat.zeros((2 * max(N, 1),), "int64")
        self.chain = nat.zeros((max(N, 1),), "int32")

    def status_value(self) -> int:
        v = int(self.status.item())
        if v & 2:
            raise nat.NativeError("exact SGD schedule stalled: a row predecessor never published "
                                  "(inconsistent pass plan)")
        return v


def _plan_full(dev, sc: _Scratch, col_lo, col_hi, row_lo, row_hi) -> None:
    nat.call("culsh_pass_plan", nat.ptr(dev.col_ptr), nat.ptr(dev.col_rows), dev.N, 0, col_lo,
             col_hi, row_lo, row_hi, None, None, 1, 0, nat.ptr(sc.seg), nat.ptr(sc.chain),
             nat.stream_ptr())


def _colpass(dev, dm: DeviceModel64, sc: _Scratch, rates: nat.CulshRates, col_lo, col_hi,
             row_mode: int, M_old: int = 0, variant: int = 0, pre=None) -> None:
    """One exact column pass; ``pre`` = _exact_lookups(...) of the same columns."""
    if pre is not None:
        mask, rv, base = pre
        nat.call("culsh_sgd_exact_colpass_pre", ctypes.byref(dev.struct), ctypes.byref(dm.struct),
                 ctypes.byref(rates), nat.ptr(sc.seg), nat.ptr(sc.chain), col_lo, col_hi, row_mode,
                 M_old, variant, nat.ptr(sc.row_last), nat.ptr(sc.ticket), nat.ptr(sc.status),
                 nat.ptr(mask), nat.ptr(rv), base, nat.stream_ptr())
        return
    nat.call("culsh_sgd_exact_colpass", ctypes.byref(dev.struct), ctypes.byref(dm.struct),
             ctypes.byref(rates), nat.ptr(sc.seg), nat.ptr(sc.chain), col_lo, col_hi, row_mode,
             M_old, variant, nat.ptr(sc.row_last), nat.ptr(sc.ticket), nat.ptr(sc.status),
             nat.stream_ptr())


def _exact_lookups(dev, dm: DeviceModel64, col_lo: int, col_hi: int, mem_fraction: float = 1.0):
    """Neighbour lookups of columns [col_lo, col_hi) for _colpass's ``pre``: the K
    dependent binary searches of every update leave the update chain (which is what
    bounds a pass on long columns / hot rows).  None when K == 0, the range is empty, or
    the arrays (entries x K x 8 B) would exceed ``mem_fraction`` of the free memory."""
    K = dm.struct.K
    if K == 0 or col_hi <= col_lo:
        return None
    cp = dev.col_ptr
    base = int(cp[col_lo].item())
    n = int(cp[col_hi].item()) - base
    t = nat.torch()
    if n * K * 8.5 > mem_fraction * t.cuda.mem_get_info()[0]:
        return None
    kpl = 1 if K <= 32 else 2
    mask = nat.empty((max(n * kpl, 1),), "int32")
    rv = nat.empty((max(n * K, 1),), "float64")
    nat.call("culsh_exact_lookup", ctypes.byref(dev.struct), ctypes.byref(dm.struct), col_lo, col_hi,
             nat.ptr(mask), nat.ptr(rv), nat.stream_ptr())
    return mask, rv, base


def _check_model_dims(F: int, K: int) -> None:
    if not (1 <= F <= 256):
        raise ValueError(f"F={F} outside the supported range [1, 256]")
    if not (0 <= K <= 64):
        raise ValueError(f"K={K} outside the supported range [0, 64]")


# ------------------------------------------------------------- public ops ---

def _residual_baselines(ratings: SparseRatings):
    stats = ratings.baselines()
    return stats.b, stats.b_hat


def split_neighbors(i: int, j: int, neighbors: NeighborTable,
                    ratings: SparseRatings) -> NeighborSplit:
    """Partition column j's neighbour positions by whether row i rated them (factorization.py:421-433)."""
    explicit, implicit = [], []
    for k in range(neighbors.K):
        if ratings.rating(i, int(neighbors.entries[j, k])) is not None:
            explicit.append(k)
        else:
            implicit.append(k)
    return NeighborSplit(explicit=np.asarray(explicit, dtype=np.int64),
                         implicit=np.asarray(implicit, dtype=np.int64))


def _predict_pairs(params: ModelParams, ratings: SparseRatings, rows, cols) -> np.ndarray:
    dev = ratings.device()
    dm = DeviceModel64(params)
    rows = nat.to_dev(np.asarray(rows, np.int32).reshape(-1))
    cols = nat.to_dev(np.asarray(cols, np.int32).reshape(-1))
    n = rows.numel()
    out = nat.empty((max(n, 1),), "float64")
    nat.call("culsh_predict", ctypes.byref(dev.struct), ctypes.byref(dm.struct), nat.ptr(rows),
             nat.ptr(cols), n, nat.ptr(out), nat.stream_ptr())
    return nat.to_host(out)[:n]


def predict(i: int, j: int, params: ModelParams, ratings: SparseRatings,
            clamp: tuple[float, float] | None = None) -> float:
    """Predicted value at (i, j) (factorization.py:436-448)."""
    if not (0 <= i < params.M and 0 <= j < params.N):
        raise IndexError(f"index ({i}, {j}) out of range for {params.M}x{params.N} model")
    _check_model_dims(max(params.F, 1), params.K)
    pred = float(_predict_pairs(params, ratings, [i], [j])[0])
    if clamp is not None:
        pred = min(max(pred, clamp[0]), clamp[1])
    return float(pred)


def sgd_update(i: int, j: int, params: ModelParams, rates: tuple, regs: tuple,
               ratings: SparseRatings) -> float:
    """All six update rules at sample (i, j) in place; returns the error (factorization.py:451-473)."""
    r = ratings.rating(i, j)
    if r is None:
        raise ValueError(f"no rating at ({i}, {j})")
    _check_model_dims(params.F, params.K)
    e = r - float(_predict_pairs(params, ratings, [i], [j])[0])
    dev = ratings.device()
    dm = DeviceModel64(params)
    sc = _Scratch(ratings.M, ratings.N)
    lo = int(ratings.col_ptr[j])
    idx = lo + int(np.searchsorted(ratings.col_slice(j)[0], i))
    seg = np.zeros(2 * ratings.N, np.int64)
    seg[2 * j], seg[2 * j + 1] = idx, idx + 1
    sc.seg = nat.to_dev(seg)
    chain = np.zeros(ratings.N, np.int32)
    chain[j] = j                      # the pass holds this one sample: no row predecessor
    sc.chain = nat.to_dev(chain)
    _colpass(dev, dm, sc, _rates_struct(rates, regs), j, j + 1, 1)
    dm.download(params)
    if not np.isfinite(e) or sc.status_value():
        raise TrainingDivergedError(epoch=0)
    return float(e)


def _transposed_device(r: SparseRatings):
    """The ratings with rows and columns swapped, in HBM (row-major passes run the
    column-pass kernels on it)."""
    from .data import DeviceRatings
    dev = r.device()
    return DeviceRatings.from_device(r.N, r.M, dev.row_ptr, dev.row_cols, dev.row_vals, dev.col_ptr,
                                     dev.col_rows, dev.col_vals, 0.0, nat.zeros((max(r.N, 1),), "float64"),
                                     nat.zeros((max(r.M, 1),), "float64"))


def train_basic(ratings: SparseRatings, config: TrainConfig, with_biases: bool = False,
                sort_rows_by_count: bool = False, racy_workers: int = 0,
                epoch_callback=None) -> ModelParams:
    """Basic MF (U, V, optional biases), row-major SGD (factorization.py:476-527; the
    paper's CUSGD++, Alg. 2).

    racy_workers == 0: the exact serial row-major order, bit-identical to the
    reference, run by the exact kernel on the transposed matrix (rows take the role
    of columns; the wavefront waits on the previous updater of each column).
    racy_workers > 0: lock-free (Hogwild on V) fp32 on the GPU, like the reference's
    racy mode nondeterministic; the worker count itself is not meaningful here.
    """
    config.validate()
    M, N = ratings.M, ratings.N
    rng = np.random.default_rng(config.seed)
    scale = config.effective_init_scale
    U = rng.uniform(0.0, scale, size=(M, config.F))
    V = rng.uniform(0.0, scale, size=(N, config.F))
    if with_biases:
        stats = ratings.baselines()
        mu, b, bhat = stats.mu, stats.b.copy(), stats.b_hat.copy()
    else:
        mu, b, bhat = 0.0, np.zeros(M), np.zeros(N)
    params = ModelParams(mu=mu, b=b, b_hat=bhat, U=U, V=V, W=np.zeros((N, 0)), C=np.zeros((N, 0)),
                         neighbors=None)
    if config.epochs == 0 or ratings.nnz == 0:
        return params
    _check_model_dims(config.F, 0)
    if sort_rows_by_count:   # process rows in that order == relabel rows by rank
        counts = np.diff(ratings.row_ptr)
        order = np.argsort(-counts, kind="stable").astype(np.int64)
    else:
        order = np.arange(M, dtype=np.int64)
    rank = np.empty(M, dtype=np.int64)
    rank[order] = np.arange(M)
    work = ratings if not sort_rows_by_count else SparseRatings(
        M, N, rank[ratings.entry_rows], ratings.entry_cols, ratings.entry_values)
    # transposed model: the kernel's (row side, column side) = (columns, rows) of the data
    tp = ModelParams(mu=mu, b=params.b_hat, b_hat=params.b[order], U=params.V, V=params.U[order],
                     W=np.zeros((M, 0)), C=np.zeros((M, 0)), neighbors=None)
    if racy_workers > 0:
        from .hogwild import HogwildTrainer
        tdev = _transposed_device(work)
        tcfg = replace(config, K=0, alpha_b=config.alpha_b_hat, alpha_b_hat=config.alpha_b,
                       alpha_u=config.alpha_v, alpha_v=config.alpha_u,
                       lambda_b=config.lambda_b_hat, lambda_b_hat=config.lambda_b,
                       lambda_u=config.lambda_v, lambda_v=config.lambda_u)
        # rotated visiting order: the row-major transpose has short "columns" (a user's ~200
        # ratings) swept in near lock-step by every resident warp, so without it many warps
        # update the same item row from one stale copy at once (diverged at C3, 1 run in 2)
        tr = HogwildTrainer(None, None, tcfg, dev=tdev, params=tp, rotate=True, train_biases=with_biases)
        for t in range(config.epochs):
            tr.epoch(t)
            if epoch_callback is not None:
                _basic_from_transposed(tr.to_params(), params, order)
                epoch_callback(t, params)
        _basic_from_transposed(tr.to_params(), params, order)
        return params
    tdev = _transposed_device(work)
    dm = DeviceModel64(tp)
    sc = _Scratch(N, M)
    _plan_full(tdev, sc, 0, M, 0, N)
    for t in range(config.epochs):
        gb, gbh, gu, gv, _, _ = config.rates_at(t)
        if not with_biases:
            gb = gbh = 0.0
        rates = _rates_struct((gbh, gb, gv, gu, 0.0, 0.0),
                              (config.lambda_b_hat, config.lambda_b, config.lambda_v, config.lambda_u,
                               0.0, 0.0))
        _colpass(tdev, dm, sc, rates, 0, M, 1, 0, variant=3)
        if sc.status_value():
            dm.download(tp)
            _basic_from_transposed(tp, params, order)
            raise TrainingDivergedError(epoch=t)
        if epoch_callback is not None:
            dm.download(tp)
            _basic_from_transposed(tp, params, order)
            epoch_callback(t, params)
            tp = ModelParams(mu=mu, b=params.b_hat, b_hat=params.b[order], U=params.V,
                             V=params.U[order], W=np.zeros((M, 0)), C=np.zeros((M, 0)))
            dm = DeviceModel64(tp)
    dm.download(tp)
    _basic_from_transposed(tp, params, order)
    return params


def _basic_from_transposed(tp: ModelParams, params: ModelParams, order: np.ndarray) -> None:
    params.b_hat[...] = tp.b
    params.V[...] = tp.U
    params.b[order] = tp.b_hat
    params.U[order] = tp.V


def train_full(ratings: SparseRatings, neighbors: NeighborTable | None,
               config: TrainConfig, epoch_callback=None, mode: str = "exact") -> ModelParams:
    """Full neighbourhood model, column-major SGD over all six parameter classes
    (factorization.py:530-556).  mode="exact" is bit-identical to the reference;
    mode="hogwild" is the fp32 performance mode (see hogwild.py)."""
    config.validate()
    K = neighbors.K if neighbors is not None else 0
    if K != config.K:
        config = replace(config, K=K)
    if mode == "hogwild":
        from .hogwild import HogwildTrainer
        tr = HogwildTrainer(ratings, neighbors, config)
        for t in range(config.epochs):
            tr.epoch(t)
            if epoch_callback is not None:
                epoch_callback(t, tr.to_params())
        return tr.to_params()
    if mode != "exact":
        raise ValueError(f"unknown mode {mode!r}")
    stats = ratings.baselines()
    params = init_params(ratings.M, ratings.N, config.F, K, neighbors, stats, config)
    if config.epochs == 0 or ratings.nnz == 0:
        return params
    _check_model_dims(config.F, K)
    dev = ratings.device()
    dm = DeviceModel64(params)
    sc = _Scratch(ratings.M, ratings.N)
    _plan_full(dev, sc, 0, ratings.N, 0, ratings.M)
    pre = _exact_lookups(dev, dm, 0, ratings.N, 0.25)   # once per fit, reused every epoch
    for t in range(config.epochs):
        _colpass(dev, dm, sc, _rates_struct(config.rates_at(t), config.regs), 0, ratings.N, 1, pre=pre)
        if sc.status_value():
            dm.download(params)
            raise TrainingDivergedError(epoch=t)
        if epoch_callback is not None:
            dm.download(params)
            epoch_callback(t, params)
            dm = DeviceModel64(params)   # the callback may have edited params
    dm.download(params)
    return params


def rmse(params: ModelParams, testset: Triplets, ratings: SparseRatings,
         unscale: float | None = None, clamp: tuple[float, float] | None = None) -> float:
    """Root-mean-square error over held-out triplets (factorization.py:559-579)."""
    if len(testset) == 0:
        raise ValueError("empty test set")
    _check_model_dims(max(params.F, 1), params.K)
    dev = ratings.device()
    dm = DeviceModel64(params)
    n = len(testset)
    tr = nat.to_dev(np.asarray(testset.rows, np.int32))
    tc = nat.to_dev(np.asarray(testset.cols, np.int32))
    tv = nat.to_dev(np.asarray(testset.values, np.float64))
    scratch = nat.empty((n + 256,), "float64")
    out = nat.empty((1,), "float64")
    lo, hi = clamp if clamp is not None else (0.0, 0.0)
    nat.call("culsh_rmse", ctypes.byref(dev.struct), ctypes.byref(dm.struct), nat.ptr(tr),
             nat.ptr(tc), nat.ptr(tv), n, int(clamp is not None), float(lo), float(hi),
             1.0 if unscale is None else float(unscale), nat.ptr(scratch), nat.ptr(out),
             nat.stream_ptr())
    return float(out.item())


def objective_value(params: ModelParams, ratings: SparseRatings, regs: tuple) -> float:
    """Full-batch regularised squared-error objective (factorization.py:582-601)."""
    pred = _predict_pairs(params, ratings, ratings.entry_rows, ratings.entry_cols)
    d = ratings.entry_values - pred
    total = float(np.add.accumulate(d * d)[-1]) if len(d) else 0.0
    lb, lbh, lu, lv, lw, lc = regs
    total += lb * float(np.sum(params.b ** 2))
    total += lbh * float(np.sum(params.b_hat ** 2))
    total += lu * float(np.sum(params.U ** 2))
    total += lv * float(np.sum(params.V ** 2))
    total += lw * float(np.sum(params.W ** 2))
    total += lc * float(np.sum(params.C ** 2))
    return total
