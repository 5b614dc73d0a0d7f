"""fp32 Hogwild training -- the performance mode of train_full.

Per fit (once): upload fp32 parameters (same PCG64 initial values as the
reference's init_params, factorization.py:196-211), build the explicit-neighbour
stream (a K-bit mask per rating + compact residuals, csrc/sgd_hogwild.cu), and
order columns longest-first.  Per epoch: ONE kernel launch
(culsh_sgd_hogwild_epoch) that updates all six parameter classes.

HBM traffic per update (the roofline's algorithmic bytes):
  B_upd = 8 (row, value) + 8F (u_i read+write) + 8 (b_i read+write)
          + K/8 (mask) + 4*E (residuals, E = mean explicit count)
plus per column per epoch 2(4F + 8K + 4) bytes of v/w/c/b_hat.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .data import BaselineStats
from .factorization import (ModelParams, TrainConfig, TrainingDivergedError, _rates_struct,
                            init_params)
from .similarity import NeighborTable


_DEV_NAME = {"b": "b", "b_hat": "bhat", "U": "U", "V": "V", "W": "W", "C": "C"}


class DeviceModel32:
    """fp32 model of a Hogwild fit in HBM (CulshModel32); also the device backing of
    the ModelParams that train_full(mode="hogwild") returns (host views widened to
    fp64 on first read)."""

    def __init__(self, p: ModelParams):
        t = nat.torch()
        dev = nat.device()
        f32 = lambda a: t.from_numpy(np.ascontiguousarray(a, np.float32).reshape(-1)).to(dev)
        self.M, self.N, self.F, self.K = p.M, p.N, p.F, p.K
        self.mu = float(p.mu)
        self.b = f32(p._peek("b"))
        self.bhat = f32(p._peek("b_hat"))
        self.U = f32(p._peek("U"))
        self.V = f32(p._peek("V"))
        W, C = p._peek("W"), p._peek("C")
        self.W = f32(W) if W.size else nat.zeros((1,), "float32")
        self.C = f32(C) if C.size else nat.zeros((1,), "float32")
        self.nbr = p.nbr_entries_device()
        self.Fp = self.F
        self._pad()
        self._restruct()

    @classmethod
    def from_arrays(cls, arrays: dict, mu: float, M: int, N: int, F: int, K: int, nbr=None,
                    padded: bool = False):
        """``arrays`` hold U / V as (M, F) / (N, F) rows, or already in the padded
        storage layout when ``padded``."""
        self = cls.__new__(cls)
        self.M, self.N, self.F, self.K, self.mu = M, N, F, K, float(mu)
        for n, a in arrays.items():
            setattr(self, _DEV_NAME[n], a)
        self.nbr = nbr if nbr is not None else nat.zeros((1,), "int32")
        self.Fp = hogwild_width(F) if padded else F
        self._pad()
        self._restruct()
        return self

    def _pad(self) -> None:
        """Store U / V with the kernel's row width Fp = hogwild_width(F): the extra
        features are zero and stay zero (their update is gamma*(e*0 - lambda*0)), so
        the model is the F-feature model; host views drop them."""
        Fp = hogwild_width(self.F)
        if Fp == self.Fp:
            return
        t = nat.torch()
        for name, rows in (("U", self.M), ("V", self.N)):
            old = getattr(self, name)
            new = t.zeros((max(rows * Fp, 1),), dtype=t.float32, device=old.device)
            if rows:
                new[:rows * Fp].view(rows, Fp)[:, :self.F] = old[:rows * self.F].view(rows, self.F)
            setattr(self, name, new)
        self.Fp = Fp

    def _logical(self, name: str):
        """Device view of parameter ``name`` in the logical (unpadded) shape, flattened."""
        a = getattr(self, _DEV_NAME[name])
        if name in ("U", "V") and self.Fp != self.F:
            rows = self.M if name == "U" else self.N
            return a[:rows * self.Fp].view(rows, self.Fp)[:, :self.F].reshape(-1)
        return a

    @classmethod
    def from_params(cls, p: ModelParams):
        """fp32 copy of a ModelParams: converted on the device when p is device-backed
        and current there, else from the host arrays."""
        dev = p._dev
        if dev is not None and all(s != "H" for s in p._state.values()):
            t = nat.torch()
            if isinstance(dev, cls):
                arrays = {n: getattr(dev, _DEV_NAME[n]).clone() for n in _DEV_NAME}
                return cls.from_arrays(arrays, p.mu, p.M, p.N, p.F, p.K, p.nbr_entries_device(),
                                       padded=True)
            arrays = {n: getattr(dev, _DEV_NAME[n]).to(t.float32) for n in _DEV_NAME}
            return cls.from_arrays(arrays, p.mu, p.M, p.N, p.F, p.K, p.nbr_entries_device())
        return cls(p)

    def _restruct(self) -> None:
        self.struct = nat.CulshModel32(self.mu, nat.ptr(self.b), nat.ptr(self.bhat), nat.ptr(self.U),
                                       nat.ptr(self.V), nat.ptr(self.W), nat.ptr(self.C), self.Fp,
                                       self.K)

    def _shape(self, name: str):
        M, N, F, K = self.M, self.N, self.F, self.K
        return {"b": (M,), "b_hat": (N,), "U": (M, F), "V": (N, F), "W": (N, K), "C": (N, K)}[name]

    def download(self, name: str, out=None) -> np.ndarray:
        shape = self._shape(name)
        n = int(np.prod(shape))
        # widen on the device, then one staged copy (no host-side fp32 -> fp64 pass)
        host = (nat.to_host(self._logical(name)[:n].to(nat.torch().float64)).reshape(shape)
                if n else np.zeros(shape))
        if out is not None and out.shape == shape and out.dtype == np.float64 and out.flags.writeable:
            out[...] = host
            return out
        return host

    def upload(self, name: str, host: np.ndarray) -> None:
        a = np.ascontiguousarray(host, dtype=np.float64).reshape(-1)
        if a.size:
            src = nat.to_dev(a).to(nat.torch().float32)   # staged fp64 upload, narrowed on the device
            if name in ("U", "V") and self.Fp != self.F:
                rows = a.size // self.F
                getattr(self, name)[:rows * self.Fp].view(rows, self.Fp)[:, :self.F].copy_(src.view(rows, self.F))
            else:
                getattr(self, _DEV_NAME[name])[:a.size].copy_(src)

    def all_finite(self, M: int, N: int) -> bool:
        t = nat.torch()
        F, K = self.Fp, self.K
        parts = [self.b[:M], self.bhat[:N], self.U[:M * F], self.V[:N * F], self.W[:N * K], self.C[:N * K]]
        return all(bool(t.isfinite(x).all().item()) for x in parts if x.numel())

    def widen(self):
        """An fp64 DeviceModel64 copy (device-side conversion)."""
        from .factorization import DeviceModel64
        t = nat.torch()
        arrays = {n: self._logical(n).to(t.float64) for n in _DEV_NAME}
        return DeviceModel64(arrays=arrays, mu=self.mu, M=self.M, N=self.N, F=self.F, K=self.K,
                             nbr=self.nbr)

    def to_params(self, neighbors: NeighborTable | None, M: int, N: int) -> ModelParams:
        h = lambda n: self.download(n)
        return ModelParams(mu=self.mu, b=h("b"), b_hat=h("b_hat"), U=h("U"), V=h("V"), W=h("W"),
                           C=h("C"), neighbors=neighbors)


def hogwild_width(F: int) -> int:
    """Row width the Hogwild kernels run for F features: F itself for F <= 32 or
    F in (64, 128, 256), else the next of 64 / 128 / 256 (zero-padded features)."""
    if F <= 32 or F in (64, 128, 256):
        return F
    return 64 if F <= 64 else 128 if F <= 128 else 256


def hogwild_supported(F: int, K: int) -> bool:
    return 1 <= F <= 256 and 0 <= K <= 64


class HogwildTrainer:
    """Device-resident fp32 training state for one fit.

    ``dev`` may be a DeviceRatings (data.py) or any object with the same
    attributes (bench.py builds one directly in HBM).
    """

    def __init__(self, ratings, neighbors: NeighborTable | None, config: TrainConfig,
                 dev=None, params: ModelParams | None = None, rotate: bool = False,
                 max_warps: int | None = None, atomic_rows: bool = True,
                 packed: bool = True, split: bool = True, split_cap: int | None = None,
                 p16: bool = True, train_biases: bool = True):
        config.validate()
        self.rotate = rotate
        self.atomic_rows = atomic_rows
        self.config = config
        self.neighbors = neighbors
        K = neighbors.K if neighbors is not None else 0
        if not hogwild_supported(config.F, K):
            raise ValueError(f"Hogwild mode supports 1 <= F <= 256 and K <= 64 (the reference takes any "
                             f"F and K, factorization.py:75-82); got F={config.F}, K={K}")
        t = nat.torch()
        self.dev = dev if dev is not None else ratings.device()
        d = self.dev
        self.M, self.N, self.nnz = d.M, d.N, d.nnz
        # Hogwild staleness grows with (concurrently updated columns) / (rows): keep at
        # most one active column warp per `rows_per_warp` rows (no cap at C2/C3 scale).
        self.max_warps = max(32, d.M // 16) if max_warps is None else max_warps
        if params is None:   # the reference's initial values, drawn directly as fp32 in HBM
            stats = BaselineStats(d.mu, None, None)
            params = init_params(d.M, d.N, config.F, K, neighbors, stats, config, _dtype="float32",
                                 _dev_baselines=(d.base_b, d.base_bhat))
            self.model = params._dev
        else:
            self.model = DeviceModel32.from_params(params)
        self.K = K
        MW = 1 if K <= 32 else 2
        self.MW = MW
        # explicit-neighbour stream (data + J^K only; once per fit)
        self.nbr = neighbors.device_entries() if K else nat.zeros((1,), "int32")
        self.model.nbr = self.nbr
        self.mask = nat.zeros((max(d.nnz * MW, 1),), "int32")
        nexpl = nat.zeros((max(d.N, 1),), "int64")
        self.resid_ptr = nat.zeros((d.N + 1,), "int64")
        if K and d.nnz:
            nat.call("culsh_explicit_stream", ctypes.byref(d.struct), float(d.mu), nat.ptr(self.nbr),
                     K, nat.ptr(self.mask), nat.ptr(nexpl), None, None, nat.stream_ptr())
            t.cumsum(nexpl[:d.N], 0, out=self.resid_ptr[1:])
        n_res = int(self.resid_ptr[-1].item()) if d.N else 0
        self.resid = nat.zeros((max(n_res, 1),), "float32")
        if K and n_res:
            nat.call("culsh_explicit_stream", ctypes.byref(d.struct), float(d.mu), nat.ptr(self.nbr),
                     K, nat.ptr(self.mask), nat.ptr(nexpl), nat.ptr(self.resid_ptr),
                     nat.ptr(self.resid), nat.stream_ptr())
        self.n_explicit = n_res
        self.vals32 = d.col_vals.to(t.float32)
        counts = d.col_ptr[1:] - d.col_ptr[:-1]
        self.col_order = t.argsort(counts, descending=True, stable=True).to(t.int32)
        self.ticket = nat.zeros((1,), "int32")
        self.status = nat.zeros((1,), "int32")
        self.loss = nat.zeros((1,), "float64")
        self.train_biases = train_biases
        self.use_p16 = p16   # 2-byte records when deltas and values fit (not with rotation)
        self.packed = self._build_packed() if packed else None
        self.work = self._build_work_list(split_cap) if split else None

    def _build_packed(self):
        """Packed rating stream (culsh_pack_stream): 4 B per rating + mask words of the
        ratings with explicit neighbours only.  None when the data do not fit it
        (more than 16 distinct values or M >= 2^27); the wide stream is used then."""
        from .lsh import _value_classes
        d = self.dev
        t = nat.torch()
        if d.nnz == 0 or d.M >= (1 << 27):
            return None
        classes = _value_classes(d)
        if classes is None:
            return None
        lut = nat.to_dev(np.unique(np.asarray(classes, np.float32)), np.float32)
        mcount = nat.zeros((max(d.N, 1),), "int64")
        mptr = nat.zeros((d.N + 1,), "int64")
        st = nat.zeros((1,), "int32")
        nat.call("culsh_pack_stream", d.N, nat.ptr(d.col_ptr), nat.ptr(d.col_rows), nat.ptr(self.vals32),
                 nat.ptr(self.mask), self.MW, nat.ptr(lut), int(lut.numel()), None, nat.ptr(mcount), None,
                 None, nat.ptr(st), nat.stream_ptr())
        t.cumsum(mcount[:d.N], 0, out=mptr[1:])
        n_m = int(mptr[-1].item())
        words = nat.zeros((max(d.nnz, 1),), "int32")
        cmask = nat.zeros((max(n_m * self.MW, 1),), "int32")
        nat.call("culsh_pack_stream", d.N, nat.ptr(d.col_ptr), nat.ptr(d.col_rows), nat.ptr(self.vals32),
                 nat.ptr(self.mask), self.MW, nat.ptr(lut), int(lut.numel()), nat.ptr(words), None,
                 nat.ptr(mptr), nat.ptr(cmask), nat.ptr(st), nat.stream_ptr())
        if int(st.item()):
            return None
        pk = {"words": words, "cmask": cmask, "mptr": mptr, "lut": lut, "w16": None, "first_row": None}
        if self.use_p16 and not self.rotate and lut.numel() <= 8:
            w16 = nat.zeros((max(d.nnz, 1),), "int16")
            first = nat.zeros((max(d.N, 1),), "int32")
            st.zero_()
            nat.call("culsh_pack16", d.N, nat.ptr(d.col_ptr), nat.ptr(d.col_rows), nat.ptr(self.vals32),
                     nat.ptr(self.mask), self.MW, nat.ptr(lut), int(lut.numel()), nat.ptr(w16), nat.ptr(first),
                     nat.ptr(st), nat.stream_ptr())
            if not int(st.item()):
                pk["w16"], pk["first_row"] = w16, first
        return pk

    def _build_work_list(self, cap: int | None = None):
        """Work segments for skewed data: a column longer than the average work of a
        resident warp (nnz / warps) would bound the epoch by its sequential chain, so it is
        split into S segments of at most that length, run by different warps concurrently,
        each from the column's current parameters; each adds 1/S of its change to the
        column parameters (parameter averaging: a plain sum would apply every segment's
        pull on v_j at full strength and overshoot).  None when no column is that long."""
        d = self.dev
        if d.N == 0 or d.nnz == 0:
            return None
        t = nat.torch()
        if cap is None:
            warps = 32 * t.cuda.get_device_properties(nat.device()).multi_processor_count
            # cap = 2 x the mean per-warp work.  Shorter segments are faster but average more
            # (tools/skew_cap_sweep.py, skewed data): C3 6 epochs 15.3 -> 9.7 ms/epoch at 1x
            # with unchanged held-out RMSE, but C2 8 epochs +0.0017 (2x) -> +0.0049 (1x) from
            # the exact fit, at the 0.005 bar; split_cap overrides
            cap = max(1024, 2 * -(-d.nnz // warps))
        col_ptr = nat.to_host(d.col_ptr).astype(np.int64)
        cnt = np.diff(col_ptr)
        if cnt.max() <= cap:
            return None
        nseg = np.maximum(1, -(-cnt // cap))
        col = np.repeat(np.arange(d.N, dtype=np.int64), nseg)
        first = np.repeat(np.cumsum(nseg) - nseg, nseg)
        part = np.arange(len(col)) - first                   # segment index within its column
        ns = nseg[col]
        lo = col_ptr[col] + (cnt[col] * part) // ns
        hi = col_ptr[col] + (cnt[col] * (part + 1)) // ns
        order = np.argsort(-(hi - lo), kind="stable")       # longest first
        # segment end carries the column's segment count S in bits 40-63 (1/S-averaged merge)
        seg = np.stack([lo[order], hi[order] | (ns[order].astype(np.int64) << 40)], axis=1).reshape(-1)
        return {"n": len(order), "col": nat.to_dev(col[order].astype(np.int32), np.int32),
                "seg": nat.to_dev(seg.astype(np.int64), np.int64), "cap": int(cap),
                "split_cols": int((nseg > 1).sum())}

    def block_work(self, seg, cols) -> dict:
        """Per-ticket work list of one DSGD block (multi-GPU stage): column j of ``cols``
        runs entries [seg[2j], seg[2j+1]).  When the block has fewer columns than the GPU has
        resident warps (D = 8 at C3: 2,221 columns for 4,736 warps), each column's range is
        cut into S segments of about total / warps entries, merged like the work segments of
        _build_work_list (1/S-averaged column parameters), so the stage fills the GPU;
        otherwise S = 1 everywhere.  Launched with launch_work (packed stream when built)."""
        t = nat.torch()
        cols_h = nat.to_host(cols).astype(np.int64)
        seg_h = nat.to_host(seg).astype(np.int64).reshape(-1, 2)[cols_h]
        lo, hi = seg_h[:, 0], seg_h[:, 1]
        cnt = hi - lo
        warps = 32 * t.cuda.get_device_properties(nat.device()).multi_processor_count
        if len(cols_h) >= warps or cnt.sum() == 0:
            nseg = np.ones(len(cols_h), np.int64)
        else:
            L = max(64, -(-int(cnt.sum()) // warps))
            nseg = np.maximum(1, -(-cnt // L))
        idx = np.repeat(np.arange(len(cols_h)), nseg)
        first = np.repeat(np.cumsum(nseg) - nseg, nseg)
        part = np.arange(len(idx)) - first
        ns = nseg[idx]
        s_lo = lo[idx] + (cnt[idx] * part) // ns
        s_hi = lo[idx] + (cnt[idx] * (part + 1)) // ns
        order = np.argsort(-(s_hi - s_lo), kind="stable")   # longest first
        sg = np.stack([s_lo[order], s_hi[order] | (ns[order] << 40)], axis=1).reshape(-1)
        return {"n": int(len(order)), "col": nat.to_dev(cols_h[idx][order].astype(np.int32), np.int32),
                "seg": nat.to_dev(sg.astype(np.int64), np.int64), "split_cols": int((nseg > 1).sum())}

    def _seg_cursors(self, work: dict):
        """The work list with each segment's stream cursors at its start (culsh_segment_cursors,
        once per list, resident stream): [lo, hi | S << 40, mask slot, residual offset] per
        ticket.  The epoch kernel (flags bit 4) then starts every segment without scanning its
        column from the beginning -- the scan grew with the segment's depth in its column (late
        DSGD stages, the tails of split columns)."""
        if "seg4" not in work:
            d = self.dev
            seg4 = nat.empty((4 * max(work["n"], 1),), "int64")
            pk = self.packed
            if pk is not None:
                nat.call("culsh_segment_cursors", work["n"], nat.ptr(d.col_ptr), nat.ptr(work["col"]),
                         nat.ptr(work["seg"]), nat.ptr(pk["words"]), None, None, nat.ptr(pk["mptr"]),
                         nat.ptr(pk["cmask"]), self.MW, nat.ptr(seg4), nat.stream_ptr())
            else:
                nat.call("culsh_segment_cursors", work["n"], nat.ptr(d.col_ptr), nat.ptr(work["col"]),
                         nat.ptr(work["seg"]), None, None, None, None, nat.ptr(self.mask), self.MW,
                         nat.ptr(seg4), nat.stream_ptr())
            work["seg4"] = seg4
        return work["seg4"]

    def launch_work(self, t_epoch: int, work: dict) -> None:
        """Enqueue one block_work list (no host synchronisation)."""
        rates = self._rates(t_epoch)
        seg4 = self._seg_cursors(work)
        if self.packed is not None:
            self._launch_packed(work["n"], self._stream_buffers(resident=True), work["col"], rates, self.loss,
                                seg4, cursors=True)
            return
        d = self.dev
        nat.call("culsh_sgd_hogwild_epoch", work["n"], nat.ptr(d.col_ptr), nat.ptr(seg4),
                 nat.ptr(d.col_rows), nat.ptr(self.vals32), nat.ptr(self.mask), nat.ptr(self.resid_ptr),
                 nat.ptr(self.resid), nat.ptr(work["col"]), ctypes.byref(self.model.struct),
                 ctypes.byref(rates), int(self.rotate) | (2 if self.atomic_rows else 0) | 8 | 16,
                 int(self.max_warps), nat.ptr(self.ticket), nat.ptr(self.loss), nat.ptr(self.status),
                 nat.stream_ptr())

    def _rates(self, t_epoch: int):
        """Epoch t's rates (factorization.py:99); with train_biases False the two bias
        rates are 0, so b and b_hat keep their values (basic MF without biases)."""
        r = list(self.config.rates_at(t_epoch))
        if not self.train_biases:
            r[0] = r[1] = 0.0
        return _rates_struct(tuple(r), self.config.regs)

    def kernel_name(self) -> str:
        """The epoch kernel a whole-matrix launch_epoch (device-resident stream) runs."""
        F, K = hogwild_width(self.config.F), self.K
        at = str(bool(self.atomic_rows)).lower()
        fv = 1 if F <= 32 else F // 32
        return "hogwild_kernel<%d,%d,%s,%s,false>" % (fv, self.MW, at, str(self.packed is not None).lower())

    def bytes_per_update(self) -> float:
        """Algorithmic HBM bytes per rating update (SURVEY §8(d) B_upd) + per-column share."""
        F, K = self.config.F, self.K
        E = self.n_explicit / max(self.nnz, 1)
        b_upd = 8 + 8 * F + 8 + K / 8 + 4 * E
        b_col = 2 * (4 * F + 8 * K + 4) + 4 * K
        return b_upd + b_col * self.N / max(self.nnz, 1)

    def launch_epoch(self, t_epoch: int, seg=None, col_order=None, n_cols: int | None = None) -> None:
        """Enqueue one epoch (no host synchronisation).  With ``seg`` / ``col_order``
        it runs one DSGD block: the listed columns, entry ranges from seg."""
        c = self.config
        rates = self._rates(t_epoch)
        d = self.dev
        order = self.col_order if col_order is None else col_order
        n = d.N if n_cols is None else n_cols
        wflag = 0
        if seg is None and col_order is None and self.work is not None:
            order, seg, n, wflag = self.work["col"], self._seg_cursors(self.work), self.work["n"], 8 | 16
        if self.packed is not None and (seg is None or wflag):
            self._launch_packed(n, self._stream_buffers(resident=True), order, rates, self.loss, seg,
                                cursors=bool(wflag & 16))
            return
        nat.call("culsh_sgd_hogwild_epoch", n, nat.ptr(d.col_ptr), nat.ptr(seg), nat.ptr(d.col_rows),
                 nat.ptr(self.vals32), nat.ptr(self.mask), nat.ptr(self.resid_ptr),
                 nat.ptr(self.resid), nat.ptr(order), ctypes.byref(self.model.struct),
                 ctypes.byref(rates),
                 int(self.rotate) | (2 if self.atomic_rows else 0) | wflag,
                 int(self.max_warps), nat.ptr(self.ticket),
                 nat.ptr(self.loss),
                 nat.ptr(self.status), nat.stream_ptr())

    def _launch_packed(self, n, bufs, order, rates, loss, seg=None, cursors: bool = False) -> None:
        """Packed-stream epoch over ``bufs`` (the _stream_buffers() layout); ``cursors``: seg is
        a _seg_cursors list (4-byte records only)."""
        pk, d = self.packed, self.dev
        flags = (int(self.rotate) | (2 if self.atomic_rows else 0) | (8 if seg is not None else 0) |
                 (16 if cursors else 0))
        if len(bufs) == 4:   # 2-byte records
            if cursors:
                raise ValueError("segment cursors are built for the resident 4-byte records")
            w16, first_row, cmask, resid = bufs
            nat.call("culsh_sgd_hogwild_epoch_packed16", n, nat.ptr(d.col_ptr), nat.ptr(seg), nat.ptr(w16),
                     nat.ptr(first_row), nat.ptr(pk["lut"]), nat.ptr(pk["mptr"]), nat.ptr(cmask),
                     nat.ptr(self.resid_ptr), nat.ptr(resid), nat.ptr(order), ctypes.byref(self.model.struct),
                     ctypes.byref(rates), flags, int(self.max_warps), nat.ptr(self.ticket), nat.ptr(loss),
                     nat.ptr(self.status), nat.stream_ptr())
            return
        words, cmask, resid = bufs
        nat.call("culsh_sgd_hogwild_epoch_packed", n, nat.ptr(d.col_ptr), nat.ptr(seg), nat.ptr(words),
                 nat.ptr(pk["lut"]), nat.ptr(pk["mptr"]), nat.ptr(cmask), nat.ptr(self.resid_ptr), nat.ptr(resid),
                 nat.ptr(order), ctypes.byref(self.model.struct), ctypes.byref(rates), flags,
                 int(self.max_warps), nat.ptr(self.ticket), nat.ptr(loss), nat.ptr(self.status),
                 nat.stream_ptr())

    def epoch(self, t_epoch: int) -> None:
        self.launch_epoch(t_epoch)
        if int(self.status.item()):
            raise TrainingDivergedError(epoch=t_epoch)

    def pinned_stream(self) -> dict:
        """Pinned host copy of the per-epoch rating stream: every per-rating array the
        epoch reads -- the packed words, the compact explicit masks and residuals when
        the packed stream is in use, else CSC rows, fp32 values, masks and residuals."""
        names = {4: ("w16", "first_row", "cmask", "resid")} if (self.packed is not None and
                                                               self.packed["w16"] is not None) else {}
        bufs = self._stream_buffers()
        if not names:
            names = {3: ("words", "cmask", "resid"), 4: ("rows", "vals", "mask", "resid")}
        return {k: v.cpu().pin_memory() for k, v in zip(names[len(bufs)], bufs)}

    def _stream_buffers(self, resident: bool = False):
        """Device arrays one epoch reads.  Streamed from the host: 2-byte records + first
        rows + compact masks + residuals when they fit (the smallest transfer); resident:
        4-byte records + masks + residuals (the fastest to decode: no per-chunk prefix
        sum, 13.2 vs 13.6 ms at C3); else the wide (rows, vals, masks, residuals)."""
        pk = self.packed
        if pk is not None and pk["w16"] is not None and not resident:
            return (pk["w16"], pk["first_row"], pk["cmask"], self.resid)
        if pk is not None:
            return (pk["words"], pk["cmask"], self.resid)
        return (self.dev.col_rows, self.vals32, self.mask, self.resid)

    def _launch_stream(self, bufs, t_epoch, loss, launch=None) -> None:
        """One epoch (or, with ``launch`` = (order, seg, n), part of one) over the stream
        buffers ``bufs``."""
        c = self.config
        rates = self._rates(t_epoch)
        d = self.dev
        order, seg, n, wflag = self.col_order, None, d.N, 0
        if self.work is not None:
            order, seg, n, wflag = self.work["col"], self.work["seg"], self.work["n"], 8
        if launch is not None:
            order, seg, n = launch
            wflag = 8 if seg is not None else 0
        if self.packed is not None:
            self._launch_packed(n, bufs, order, rates, loss, seg)
            return
        rows_b, vals_b, mask_b, resid_b = bufs
        nat.call("culsh_sgd_hogwild_epoch", n, nat.ptr(d.col_ptr), nat.ptr(seg), nat.ptr(rows_b),
                 nat.ptr(vals_b), nat.ptr(mask_b), nat.ptr(self.resid_ptr), nat.ptr(resid_b),
                 nat.ptr(order), ctypes.byref(self.model.struct), ctypes.byref(rates),
                 int(self.rotate) | (2 if self.atomic_rows else 0) | wflag,
                 int(self.max_warps), nat.ptr(self.ticket), nat.ptr(loss),
                 nat.ptr(self.status), nat.stream_ptr())

    def _chunk_plan(self, n_chunks: int):
        """Column ranges of ~equal rating count for a pipelined first epoch: per chunk the
        element range of every stream array and the chunk's launch list (its columns, or
        its work segments, in the epoch's longest-first order)."""
        key = ("chunks", n_chunks)
        if getattr(self, "_plan_key", None) == key:
            return self._plan
        t = nat.torch()
        d = self.dev
        col_ptr = nat.to_host(d.col_ptr).astype(np.int64)
        rptr = nat.to_host(self.resid_ptr).astype(np.int64)
        cb = np.unique(np.searchsorted(col_ptr, np.linspace(0, d.nnz, n_chunks + 1), side="left"))
        cb[0], cb[-1] = 0, d.N
        if self.work is not None:
            wcol = nat.to_host(self.work["col"]).astype(np.int64)
            wseg = nat.to_host(self.work["seg"]).reshape(-1, 2)
        else:
            order = nat.to_host(self.col_order).astype(np.int64)
        mptr = nat.to_host(self.packed["mptr"]).astype(np.int64) if self.packed is not None else None
        plan = []
        for c0, c1 in zip(cb[:-1], cb[1:]):
            if c1 <= c0:
                continue
            e0, e1 = int(col_ptr[c0]), int(col_ptr[c1])
            if self.packed is not None and self.packed["w16"] is not None:
                ranges = [(e0, e1), (int(c0), int(c1)), (int(mptr[c0]) * self.MW, int(mptr[c1]) * self.MW),
                          (int(rptr[c0]), int(rptr[c1]))]
            elif self.packed is not None:
                ranges = [(e0, e1), (int(mptr[c0]) * self.MW, int(mptr[c1]) * self.MW),
                          (int(rptr[c0]), int(rptr[c1]))]
            else:
                ranges = [(e0, e1), (e0, e1), (e0 * self.MW, e1 * self.MW), (int(rptr[c0]), int(rptr[c1]))]
            if self.work is not None:
                sel = (wcol >= c0) & (wcol < c1)
                launch = (nat.to_dev(wcol[sel].astype(np.int32), np.int32),
                          nat.to_dev(np.ascontiguousarray(wseg[sel]).reshape(-1), np.int64), int(sel.sum()))
            else:
                sel = order[(order >= c0) & (order < c1)]
                launch = (nat.to_dev(sel.astype(np.int32), np.int32), None, len(sel))
            plan.append((ranges, launch))
        self._plan_key, self._plan = key, plan
        return plan

    def epoch_from_host(self, host: dict, t_epoch: int):
        """One epoch whose rating stream comes from pinned host memory: H2D copy of
        the stream, the epoch kernel, D2H of the epoch's summed squared error.
        Returns (sum of e^2 over the epoch, h2d bytes, d2h bytes)."""
        bufs = self._stream_buffers()
        for dst, src in zip(bufs, host.values()):
            dst.copy_(src, non_blocking=True)
        self.loss.zero_()
        self._launch_stream(bufs, t_epoch, self.loss)
        loss = float(self.loss.item())
        if int(self.status.item()):
            raise TrainingDivergedError(epoch=t_epoch)
        h2d = sum(int(v.numel() * v.element_size()) for v in host.values())
        return loss, h2d, 8 + 4

    def train_from_host(self, host: dict, t_start: int, n_epochs: int, first_chunks: int = 4):
        """Epochs whose rating stream comes from pinned host memory every epoch, with
        the H2D copy of epoch e+1 (copy stream, double buffer) overlapping the
        kernel of epoch e, and each epoch's loss copied back (D2H) as it finishes.
        The first epoch, which has no earlier kernel to hide its copy behind, is
        pipelined in ``first_chunks`` column ranges: range c's kernel runs while range
        c+1 is copied (Hogwild order within an epoch is free).
        Returns (per-epoch sum of e^2, h2d bytes per epoch, d2h bytes per epoch)."""
        t = nat.torch()
        comp = t.cuda.current_stream()
        cstream = t.cuda.Stream()
        first = self._stream_buffers()
        bufs = [first, tuple(t.empty_like(x) for x in first)]
        src = tuple(host.values())
        copied = [t.cuda.Event(), t.cuda.Event()]
        used = [t.cuda.Event(), t.cuda.Event()]
        loss_dev = t.zeros(n_epochs, dtype=t.float64, device=self.loss.device)
        loss_host = t.zeros(n_epochs, dtype=t.float64).pin_memory()

        def fill(b):
            with t.cuda.stream(cstream):
                cstream.wait_event(used[b])
                for dst, s_ in zip(bufs[b], src):
                    dst.copy_(s_, non_blocking=True)
                copied[b].record(cstream)

        for b in (0, 1):
            used[b].record(comp)
        plan = self._chunk_plan(first_chunks) if first_chunks > 1 and n_epochs > 0 else None
        if plan is None:
            fill(0)
        else:   # epoch 0: chunk c's copy on the copy stream, its kernel after it on comp
            evs = []
            with t.cuda.stream(cstream):
                for ranges, _ in plan:
                    for dst, s_, (a, z) in zip(bufs[0], src, ranges):
                        dst[a:z].copy_(s_[a:z], non_blocking=True)
                    ev = t.cuda.Event()
                    ev.record(cstream)
                    evs.append(ev)
        for e in range(n_epochs):
            b = e % 2
            if plan is not None and e == 0:
                if n_epochs > 1:
                    fill(1)
                for ev, (_, launch) in zip(evs, plan):
                    comp.wait_event(ev)
                    self._launch_stream(bufs[0], t_start, loss_dev[0:], launch)
                used[0].record(comp)
                loss_host[0:1].copy_(loss_dev[0:1], non_blocking=True)
                continue
            comp.wait_event(copied[b])
            if e + 1 < n_epochs:
                fill(1 - b)
            self._launch_stream(bufs[b], t_start + e, loss_dev[e:])
            used[b].record(comp)
            loss_host[e:e + 1].copy_(loss_dev[e:e + 1], non_blocking=True)
        comp.synchronize()
        if int(self.status.item()):
            raise TrainingDivergedError(epoch=t_start + n_epochs - 1)
        h2d = sum(int(v.numel() * v.element_size()) for v in src)
        return loss_host.numpy().copy(), h2d, 8

    def to_params(self) -> ModelParams:
        return self.model.to_params(self.neighbors, self.M, self.N)

    def rmse(self, t_rows, t_cols, t_vals) -> float:
        """Test RMSE of the current fp32 model (predictions evaluated in fp64)."""
        n = len(t_rows)
        if n == 0:
            raise ValueError("empty test set")
        tr = nat.to_dev(np.asarray(t_rows, np.int32))
        tc = nat.to_dev(np.asarray(t_cols, np.int32))
        tv = nat.to_dev(np.asarray(t_vals, np.float64))
        scratch = nat.empty((n + 256,), "float64")
        out = nat.empty((1,), "float64")
        nat.call("culsh_rmse32", ctypes.byref(self.dev.struct), ctypes.byref(self.model.struct),
                 nat.ptr(self.nbr), nat.ptr(tr), nat.ptr(tc), nat.ptr(tv), n, nat.ptr(scratch),
                 nat.ptr(out), nat.stream_ptr())
        return float(out.item())
