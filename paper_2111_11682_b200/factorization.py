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


_FIELDS = ("b", "b_hat", "U", "V", "W", "C")


class ModelParams:
    """All trainable state plus the neighbour table (factorization.py:105-185).

    Same fields as the reference dataclass (mu, b, b_hat, U, V, W, C, neighbors), with
    one addition: the arrays may live in HBM.  A model produced by training (or by
    ``extend_params``) is backed by its device copy and each host array is materialised
    only when it is first read, so an epoch callback that only calls ``rmse``/``predict``
    never moves the model across PCIe.  Per array the newest copy is tracked:

    * ``D`` -- the device copy is newer (host array absent or stale);
    * ``S`` -- both copies are equal and the host array was only read internally;
    * ``H`` -- the host array is the truth: it was passed in, assigned, or handed out by an
      attribute read (the caller may edit it in place, as with the reference's live
      arrays), so every device use uploads it first.
    """

    def __init__(self, mu: float, b: np.ndarray, b_hat: np.ndarray, U: np.ndarray,
                 V: np.ndarray, W: np.ndarray, C: np.ndarray,
                 neighbors: NeighborTable | None = None):
        self.mu = mu
        self.neighbors = neighbors
        self._h = {"b": b, "b_hat": b_hat, "U": U, "V": V, "W": W, "C": C}
        self._state = dict.fromkeys(_FIELDS, "H")
        self._dims = (len(b), len(b_hat), int(np.shape(U)[1]), int(np.shape(W)[1]))
        self._dev = None

    @classmethod
    def _from_device(cls, mu: float, dev, M: int, N: int, neighbors: NeighborTable | None):
        """A model whose only copy is the device model ``dev`` (DeviceModel64/32)."""
        self = cls.__new__(cls)
        self.mu = float(mu)
        self.neighbors = neighbors
        self._h = dict.fromkeys(_FIELDS)
        self._state = dict.fromkeys(_FIELDS, "D")
        self._dims = (int(M), int(N), int(dev.F), int(dev.K))
        self._dev = dev
        return self

    # -- host views ----------------------------------------------------------
    def _peek(self, name: str) -> np.ndarray:
        """Current host value of one array for an internal read-only use."""
        if self._state[name] == "D":
            self._h[name] = self._dev.download(name, self._h[name])
            self._state[name] = "S"
        return self._h[name]

    def _get(self, name: str) -> np.ndarray:
        a = self._peek(name)
        self._state[name] = "H"
        return a

    def _set(self, name: str, value) -> None:
        self._h[name] = value
        self._state[name] = "H"
        if name in ("b", "b_hat", "U", "W"):
            M, N, F, K = self._dims
            sh = np.shape(value)
            self._dims = {"b": (sh[0], N, F, K), "b_hat": (M, sh[0], F, K),
                          "U": (M, N, sh[1], K), "W": (M, N, F, sh[1])}[name]

    b = property(lambda s: s._get("b"), lambda s, v: s._set("b", v))
    b_hat = property(lambda s: s._get("b_hat"), lambda s, v: s._set("b_hat", v))
    U = property(lambda s: s._get("U"), lambda s, v: s._set("U", v))
    V = property(lambda s: s._get("V"), lambda s, v: s._set("V", v))
    W = property(lambda s: s._get("W"), lambda s, v: s._set("W", v))
    C = property(lambda s: s._get("C"), lambda s, v: s._set("C", v))

    # -- device copy ---------------------------------------------------------
    def _device(self, precision: int = 64):
        """The device model with every array current (host-truth arrays uploaded first).

        precision=0 returns the backing as it is (DeviceModel64, or the fp32 DeviceModel32
        of a Hogwild fit); precision=64 always returns a DeviceModel64 -- for an fp32
        backing a widened temporary copy (the backing itself stays the trainer's)."""
        if self._dev is None:
            self._dev = DeviceModel64(self)
        else:
            for n in _FIELDS:
                if self._state[n] == "H":
                    self._dev.upload(n, self._h[n])
        dev = self._dev
        nbr = self.nbr_entries_device()
        if dev.nbr is not nbr:
            dev.nbr = nbr
            dev._restruct()
        if precision == 64 and not isinstance(dev, DeviceModel64):
            return dev.widen()
        return dev

    def _own(self) -> None:
        """Mark host arrays created internally (never seen by a caller) as synced, so
        they are not re-uploaded on every device use."""
        for n in _FIELDS:
            if self._state[n] == "H":
                self._state[n] = "S"

    def _device_updated(self) -> None:
        """Kernels changed the device copy: it is now the newest for every array."""
        for n in _FIELDS:
            self._state[n] = "D"

    def nbr_entries_device(self):
        if self.neighbors is None or self.K == 0:
            return nat.zeros((1,), "int32")
        return self.neighbors.device_entries()

    @property
    def M(self) -> int:
        return self._dims[0]

    @property
    def N(self) -> int:
        return self._dims[1]

    @property
    def F(self) -> int:
        return self._dims[2]

    @property
    def K(self) -> int:
        return self._dims[3]

    def nbr_entries(self) -> np.ndarray:
        if self.neighbors is None:
            return np.zeros((self.N, 0), dtype=np.int32)
        return self.neighbors.entries

    def copy(self) -> "ModelParams":
        nbr = None
        if self.neighbors is not None:
            nbr = NeighborTable(self.neighbors.N, self.neighbors.K, self.neighbors.entries.copy())
        return ModelParams(self.mu, *[self._peek(n).copy() for n in _FIELDS], nbr)

    def all_finite(self) -> bool:
        if not np.isfinite(self.mu):
            return False
        if self._dev is not None and all(s != "H" for s in self._state.values()):
            return self._dev.all_finite(self.M, self.N)
        return all(bool(np.isfinite(self._peek(n)).all()) for n in _FIELDS)

    def save(self, path) -> None:
        with open(path, "wb") as fh:
            fh.write(f"{MODEL_MAGIC} {MODEL_VERSION} {self.M} {self.N} "
                     f"{self.F} {self.K}\n".encode())
            fh.write(struct.pack("<d", self.mu))
            for n in _FIELDS:
                fh.write(np.ascontiguousarray(self._peek(n), dtype="<f8").tobytes())
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


_M64 = (1 << 64) - 1


def pcg64_uniform_device(seed, skip: int, n: int, scale: float, dtype: str = "float64"):
    """``np.random.default_rng(seed).uniform(0, scale, skip + n)[skip:]`` generated in
    HBM (csrc/init.cu: the PCG64 stream jumped ahead per thread), bit for bit."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    out = nat.empty((max(int(n), 1),), dtype)
    nat.call("culsh_pcg64_uniform", s >> 64, s & _M64, inc >> 64, inc & _M64, int(skip), int(n),
             float(scale), int(dtype == "float32"), nat.ptr(out), nat.stream_ptr())
    return out


def _dev_bias(a, n: int, dtype: str):
    """A device copy of a baseline vector (host array or device tensor)."""
    t = nat.torch()
    if isinstance(a, t.Tensor):
        v = a[:n].to(getattr(t, dtype)).clone()
    else:
        v = nat.to_dev(np.asarray(a, np.float64)[:n]).to(getattr(t, dtype))
    return v if n else nat.zeros((1,), dtype)


def init_params(M: int, N: int, F: int, K: int, neighbors: NeighborTable | None,
                baselines: BaselineStats, config: TrainConfig, *, _dtype: str = "float64",
                _dev_baselines=None) -> ModelParams:
    """Biases from the baselines, U/V uniform in [0, init_scale], W/C zero
    (factorization.py:196-211).  Generated in HBM: U and V are the reference's
    ``default_rng(seed).uniform`` draws in the same order (U's M*F values, then V's),
    bit for bit (csrc/init.cu); the host arrays are materialised on first read."""
    if neighbors is not None and (neighbors.N != N or neighbors.K != K):
        raise ValueError("neighbor table does not match N, K")
    scale = config.effective_init_scale
    U = pcg64_uniform_device(config.seed, 0, M * F, scale, _dtype)
    V = pcg64_uniform_device(config.seed, M * F, N * F, scale, _dtype)
    bb, bh = (_dev_baselines if _dev_baselines is not None else (baselines.b, baselines.b_hat))
    arrays = {"b": _dev_bias(bb, M, _dtype), "b_hat": _dev_bias(bh, N, _dtype), "U": U, "V": V,
              "W": nat.zeros((max(N * K, 1),), _dtype), "C": nat.zeros((max(N * K, 1),), _dtype)}
    nbr = neighbors.device_entries() if (neighbors is not None and K) else None
    if _dtype == "float32":
        from .hogwild import DeviceModel32
        dm = DeviceModel32.from_arrays(arrays, baselines.mu, M, N, F, K, nbr)
    else:
        dm = DeviceModel64(arrays=arrays, mu=baselines.mu, M=M, N=N, F=F, K=K, nbr=nbr)
    return ModelParams._from_device(baselines.mu, dm, M, N, neighbors)


# ------------------------------------------------------------ device model ---

_DEV_NAME = {"b": "b", "b_hat": "bhat", "U": "U", "V": "V", "W": "W", "C": "C"}


class DeviceModel64:
    """fp64 ModelParams resident in HBM, exposed to the C ABI as CulshModel64."""

    def __init__(self, p: ModelParams | None = None, *, arrays: dict | None = None,
                 mu: float = 0.0, M: int = 0, N: int = 0, F: int = 0, K: int = 0, nbr=None):
        if p is not None:
            mu, M, N, F, K = float(p.mu), p.M, p.N, p.F, p.K
            arrays = {}
            for n in _FIELDS:
                a = p._peek(n)
                arrays[n] = nat.to_dev(a.reshape(-1) if a.size else np.zeros(1), np.float64)
            nbr = p.nbr_entries_device()
        self.mu = float(mu)
        self.M, self.N, self.F, self.K = M, N, F, K
        for n, a in arrays.items():
            setattr(self, _DEV_NAME[n], a)
        self.nbr = nbr if nbr is not None else nat.zeros((1,), "int32")
        self._restruct()

    def _restruct(self) -> None:
        self.struct = nat.CulshModel64(self.mu, nat.ptr(self.b), nat.ptr(self.bhat), nat.ptr(self.U),
                                       nat.ptr(self.V), nat.ptr(self.W), nat.ptr(self.C),
                                       nat.ptr(self.nbr), self.F, self.K)

    def _shape(self, name: str, M: int, N: int):
        return {"b": (M,), "b_hat": (N,), "U": (M, self.F), "V": (N, self.F),
                "W": (N, self.K), "C": (N, self.K)}[name]

    def download(self, name, out=None):
        """Host fp64 copy of one array (``name`` a ModelParams field); with the legacy
        form ``download(params)`` every array is copied into params (in place)."""
        if isinstance(name, ModelParams):
            p = name
            for n in _FIELDS:
                p._h[n] = self.download(n, p._h[n])
                p._state[n] = "H"
            return None
        d = getattr(self, _DEV_NAME[name])
        shape = self._shape(name, self.M, self.N)
        n = int(np.prod(shape))
        host = nat.to_host(d[:n]).reshape(shape) if n else np.zeros(shape)
        if out is not None and out.shape == shape and out.dtype == np.float64 and out.flags.writeable:
            out[...] = host
            return out
        return np.asarray(host, dtype=np.float64)   # a fresh array already (no second copy)

    def upload(self, name: str, host: np.ndarray) -> None:
        d = getattr(self, _DEV_NAME[name])
        a = np.ascontiguousarray(host, dtype=np.float64).reshape(-1)
        if a.size:
            nat.copy_to_device(d[:a.size], a)

    def all_finite(self, M: int, N: int) -> bool:
        t = nat.torch()
        F, K = self.F, self.K
        parts = [self.b[:M], self.bhat[:N], self.U[:M * F], self.V[:N * F], self.W[:N * K], self.C[:N * K]]
        return all(bool(t.isfinite(x).all().item()) for x in parts if x.numel())


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


def _exact_lookups(dev, dm: DeviceModel64, col_lo: int, col_hi: int, mem_fraction: float = 0.5):
    """Neighbour lookups of columns [col_lo, col_hi) for _colpass's ``pre``: the K
    dependent binary searches of every update leave the update chain (which is what
    bounds a pass on long columns / hot rows).  None when K == 0, the range is empty, or
    the arrays (entries x (8K + 4 ceil(K/32)) B) would exceed ``mem_fraction`` of the free memory."""
    K = dm.struct.K
    if K == 0 or col_hi <= col_lo:
        return None
    cp = dev.col_ptr
    base = int(cp[col_lo].item())
    n = int(cp[col_hi].item()) - base
    t = nat.torch()
    kpl = _mask_words(K)
    if n * (8 * K + 4 * kpl) > mem_fraction * t.cuda.mem_get_info()[0]:   # rv f64 + mask words
        return None
    mask = nat.empty((max(n * kpl, 1),), "int32")
    rv = nat.empty((max(n * K, 1),), "float64")
    nat.call("culsh_exact_lookup", ctypes.byref(dev.struct), ctypes.byref(dm.struct), col_lo, col_hi,
             nat.ptr(mask), nat.ptr(rv), nat.stream_ptr())
    return mask, rv, base


# the largest K of the exact (reference-order) kernels, the online path and rmse / predict:
# four 32-bit explicit-neighbour mask words per rating, the top-K kernels' bound (topk.cu).
# The fp32 Hogwild mode keeps two (K <= 64, hogwild.hogwild_supported).
MAX_K = 128
# the largest F of the same kernels (16 fp64 factors per lane); the Hogwild mode keeps 256
MAX_F = 512


def _mask_words(K: int) -> int:
    """Mask words per rating of the exact kernels (sgd_exact.cu exact_kpl)."""
    return 1 if K <= 32 else 2 if K <= 64 else 4


def _check_model_dims(F: int, K: int) -> None:
    # the reference accepts any F and K (factorization.py:75-82); the kernels keep up to
    # MAX_F factors per row and MAX_K neighbours per column
    if not (1 <= F <= MAX_F):
        raise ValueError(f"F={F} outside the supported range [1, {MAX_F}] (the reference has no bound)")
    if not (0 <= K <= MAX_K):
        raise ValueError(f"K={K} outside the supported range [0, {MAX_K}] (the reference has no bound)")


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
    dm = params._device(64)
    rows = np.asarray(rows, np.int32).reshape(-1)
    cols = np.asarray(cols, np.int32).reshape(-1)
    if len(rows) and (rows.min() < 0 or rows.max() >= ratings.M or cols.min() < 0 or cols.max() >= ratings.N):
        raise IndexError(f"pair outside the ratings' {ratings.M} x {ratings.N} index space")
    rows, cols = nat.to_dev(rows), nat.to_dev(cols)
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
    dm = params._device(0)
    if not isinstance(dm, DeviceModel64):   # an fp32 (Hogwild) backing: update in fp64
        params._dev = dm = params._device(64)
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
    params._device_updated()
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
    mode="hogwild" is the fp32 performance mode (see hogwild.py).

    The model stays in HBM for the whole fit: ``epoch_callback(t, params)`` receives the
    live ModelParams backed by the device copy, so ``rmse``/``predict`` inside it run on
    the resident model, host arrays are copied down only if the callback reads them,
    and edits it makes to them are uploaded before the next epoch (the reference passes
    its live arrays)."""
    config.validate()
    K = neighbors.K if neighbors is not None else 0
    if K != config.K:
        config = replace(config, K=K)
    if mode == "hogwild":
        from .hogwild import HogwildTrainer
        tr = HogwildTrainer(ratings, neighbors, config)
        params = ModelParams._from_device(tr.model.mu, tr.model, ratings.M, ratings.N, neighbors)
        for t in range(config.epochs):
            tr.epoch(t)
            params._device_updated()
            if epoch_callback is not None:
                epoch_callback(t, params)
                params._device(0)        # upload whatever the callback edited
        return params
    if mode != "exact":
        raise ValueError(f"unknown mode {mode!r}")
    if ratings.nnz == 0:
        return init_params(ratings.M, ratings.N, config.F, K, neighbors, ratings.baselines(), config)
    dev = ratings.device()
    params = init_params(ratings.M, ratings.N, config.F, K, neighbors, BaselineStats(dev.mu, None, None),
                         config, _dev_baselines=(dev.base_b, dev.base_bhat))
    if config.epochs == 0:
        return params
    _check_model_dims(config.F, K)
    dm = params._device(64)
    sc = _Scratch(ratings.M, ratings.N)
    _plan_full(dev, sc, 0, ratings.N, 0, ratings.M)
    pre = _exact_lookups(dev, dm, 0, ratings.N, 0.25)   # once per fit, reused every epoch
    for t in range(config.epochs):
        _colpass(dev, dm, sc, _rates_struct(config.rates_at(t), config.regs), 0, ratings.N, 1, pre=pre)
        params._device_updated()
        if sc.status_value():
            raise TrainingDivergedError(epoch=t)
        if epoch_callback is not None:
            epoch_callback(t, params)
            dm = params._device(64)      # uploads whatever the callback edited
    return params


def _test_device(testset: Triplets, ratings: SparseRatings):
    """Device (rows, cols, values) of a test set.  The training set itself
    (``ratings.triplets()``) and split_holdout's test sets are immutable and keep one
    device copy; any other Triplets is uploaded per call."""
    src = getattr(testset, "_source", None)
    if src is not None and src is ratings:
        return ratings.device_entries()
    dev = getattr(testset, "_dev", None)
    cached = dev is not None
    if not cached:
        dev = (nat.to_dev(np.asarray(testset.rows, np.int32)), nat.to_dev(np.asarray(testset.cols, np.int32)),
               nat.to_dev(np.asarray(testset.values, np.float64)))
        if all(not np.asarray(a).flags.writeable for a in (testset.rows, testset.cols, testset.values)):
            testset._dev = dev
            cached = True
    # the kernels index b / U / V / the CSR with these: out-of-range pairs raise here
    # (the reference's numba loop would read out of bounds); once per immutable test set
    key = (ratings.M, ratings.N)
    n = len(testset)
    if n and getattr(testset, "_dev_checked", None) != key:
        t = nat.torch()
        lo_r, hi_r = t.aminmax(dev[0][:n])
        lo_c, hi_c = t.aminmax(dev[1][:n])
        r0, r1, c0, c1 = t.stack([lo_r, hi_r, lo_c, hi_c]).tolist()
        if r0 < 0 or r1 >= ratings.M or c0 < 0 or c1 >= ratings.N:
            raise IndexError(f"test triplet outside the ratings' {ratings.M} x {ratings.N} index space")
        if cached:
            testset._dev_checked = key
    return dev


def _test_rows(testset: Triplets, ratings: SparseRatings):
    """The test set grouped by row on the device: (ptr (M+1) int64, cols int32, values f64,
    position in the test set int32).  A stable sort keeps each row's targets in test-set
    order; cached next to the device copy when the test set is immutable."""
    cache = getattr(testset, "_dev_rows", None)
    if cache is not None and cache[0] is ratings:
        return cache[1]
    t = nat.torch()
    tr, tc, tv = _test_device(testset, ratings)
    n = len(testset)
    M = ratings.M
    order = t.sort(tr[:n], stable=True)[1]
    ptr = t.zeros(M + 1, dtype=t.int64, device=tr.device)
    t.cumsum(t.bincount(tr[:n].to(t.int64), minlength=M), 0, out=ptr[1:])
    rows = (ptr, tc[:n][order].contiguous(), tv[:n][order].contiguous(), order.to(t.int32))
    if getattr(testset, "_dev", None) is not None:
        testset._dev_rows = (ratings, rows)
    return rows


def _train_lookup(dev, nbr, K: int):
    """Per-(ratings, J^K) lookup cache for rmse over the training set: the explicit-
    neighbour mask of every CSC entry and the CSC position of each explicit pair (built
    once with the Hogwild stream's intersection kernel, ~0.5 GB at C3; cached on the
    device ratings, keyed by the neighbour table's device copy)."""
    key = (nbr.data_ptr(), K)
    cache = dev.__dict__.setdefault("_train_lookup", {})
    if key in cache and cache[key][0] is nbr:
        return cache[key][1:]
    cache.clear()
    t = nat.torch()
    MW = 1 if K <= 32 else 2
    mask = nat.zeros((max(dev.nnz * MW, 1),), "int32")
    nexpl = nat.zeros((max(dev.N, 1),), "int64")
    nat.call("culsh_explicit_stream", ctypes.byref(dev.struct), float(dev.mu), nat.ptr(nbr), K,
             nat.ptr(mask), nat.ptr(nexpl), None, None, nat.stream_ptr())
    ng = (dev.nnz + 31) // 32
    cnt = nat.zeros((max(ng, 1),), "int64")
    nat.call("culsh_train_lookup", ctypes.byref(dev.struct), nat.ptr(nbr), K, nat.ptr(mask), nat.ptr(cnt),
             None, None, nat.stream_ptr())
    base = t.zeros(max(ng, 1), dtype=t.int64, device=cnt.device)
    if ng > 1:
        t.cumsum(cnt[:ng - 1], 0, out=base[1:ng])
    total = int((base[ng - 1] + cnt[ng - 1]).item()) if ng else 0
    pos = nat.empty((max(total, 1),), "int32")
    nat.call("culsh_train_lookup", ctypes.byref(dev.struct), nat.ptr(nbr), K, nat.ptr(mask), None,
             nat.ptr(base), nat.ptr(pos), nat.stream_ptr())
    cache[key] = (nbr, mask, base, pos)
    return mask, base, pos


_ROWS_RMSE_MAX_N = 65536   # per-warp row bitmap of the row-order rmse kernel
_ROWS_RMSE_MIN_TEST = 4096  # smaller test sets: the ungrouped kernel (no sort)


def rmse(params: ModelParams, testset: Triplets, ratings: SparseRatings,
         unscale: float | None = None, clamp: tuple[float, float] | None = None) -> float:
    """Root-mean-square error over held-out triplets (factorization.py:559-579).

    Runs on the resident model (no host copy of the parameters).  When ``testset`` is the
    training set itself (``ratings.triplets()``, as the CLI's per-epoch callback passes
    it, cli.py:204-210) the ratings' device views and a cached neighbour-lookup table are
    used; other test sets are uploaded and their neighbour values binary-searched."""
    if len(testset) == 0:
        raise ValueError("empty test set")
    _check_model_dims(max(params.F, 1), params.K)
    dev = ratings.device()
    dm = params._device(0)
    m32 = not isinstance(dm, DeviceModel64)   # a Hogwild fit's fp32 backing: read as is, fp64 math
    n = len(testset)
    scratch = nat.empty((n + 256,), "float64")
    out = nat.empty((1,), "float64")
    lo, hi = clamp if clamp is not None else (0.0, 0.0)
    us = 1.0 if unscale is None else float(unscale)
    head = ((ctypes.byref(dev.struct), ctypes.byref(dm.struct), float(dm.mu), int(dm.F), nat.ptr(dm.nbr))
            if m32 else (ctypes.byref(dev.struct), ctypes.byref(dm.struct)))
    wide_k = dm.K > 64   # beyond the two mask words of the row / lookup-cache kernels
    if getattr(testset, "_source", None) is ratings and n == dev.nnz and dev.N <= _ROWS_RMSE_MAX_N and not wide_k:
        # CSR order, one warp per row (U read once per row; no lookup cache)
        ce = ratings.csr_entry_index()
        if m32:
            nat.call("culsh_rmse_train_rows_m32", *head, nat.ptr(ce), int(clamp is not None), float(lo),
                     float(hi), us, nat.ptr(scratch), nat.ptr(out), nat.stream_ptr())
        else:
            nat.call("culsh_rmse_train_rows", *head, nat.ptr(ce), int(clamp is not None), float(lo), float(hi),
                     us, nat.ptr(scratch), nat.ptr(out), nat.stream_ptr())
        return float(out.item())
    if getattr(testset, "_source", None) is ratings and n == dev.nnz and not wide_k:
        K = dm.K
        mask = base = pos = None
        if K:
            mask, base, pos = _train_lookup(dev, dm.nbr, K)
        perm = ratings.csc_entry_perm()
        nat.call("culsh_rmse_train_m32" if m32 else "culsh_rmse_train", *head, nat.ptr(mask),
                 nat.ptr(base), nat.ptr(pos), nat.ptr(perm), int(clamp is not None), float(lo), float(hi),
                 us, nat.ptr(scratch), nat.ptr(out), nat.stream_ptr())
        return float(out.item())
    if dev.N <= _ROWS_RMSE_MAX_N and n >= _ROWS_RMSE_MIN_TEST and not wide_k:
        # grouped by row: one warp per row against the row's bitmap (the ungrouped kernel
        # binary-searches every neighbour and gathers U and V per target)
        tp, tcol, tval, tix = _test_rows(testset, ratings)
        if m32:
            nat.call("culsh_rmse_rows_m32", *head, nat.ptr(tp), nat.ptr(tcol), nat.ptr(tval), nat.ptr(tix), n,
                     int(clamp is not None), float(lo), float(hi), us, nat.ptr(scratch), nat.ptr(out),
                     nat.stream_ptr())
        else:
            nat.call("culsh_rmse_rows", *head, nat.ptr(tp), nat.ptr(tcol), nat.ptr(tval), nat.ptr(tix), n,
                     int(clamp is not None), float(lo), float(hi), us, nat.ptr(scratch), nat.ptr(out),
                     nat.stream_ptr())
        return float(out.item())
    tr, tc, tv = _test_device(testset, ratings)
    nat.call("culsh_rmse_m32" if m32 else "culsh_rmse", *head, nat.ptr(tr),
             nat.ptr(tc), nat.ptr(tv), n, int(clamp is not None), float(lo), float(hi), us,
             nat.ptr(scratch), nat.ptr(out), nat.stream_ptr())
    return float(out.item())


def objective_value(params: ModelParams, ratings: SparseRatings, regs: tuple) -> float:
    """Full-batch regularised squared-error objective (factorization.py:582-601)."""
    pred = _predict_pairs(params, ratings, ratings.entry_rows, ratings.entry_cols)
    d = ratings.entry_values - pred
    total = float(np.add.accumulate(d * d)[-1]) if len(d) else 0.0
    lb, lbh, lu, lv, lw, lc = regs
    total += lb * float(np.sum(params._peek("b") ** 2))
    total += lbh * float(np.sum(params._peek("b_hat") ** 2))
    total += lu * float(np.sum(params._peek("U") ** 2))
    total += lv * float(np.sum(params._peek("V") ** 2))
    total += lw * float(np.sum(params._peek("W") ** 2))
    total += lc * float(np.sum(params._peek("C") ** 2))
    return total
