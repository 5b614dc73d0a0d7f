"""Device-resident online updates at scale.

``OnlineSession`` keeps the ratings (both index views), the simLSH accumulators
and group keys, J^K and the fp64 model in HBM across increments and absorbs an
IncrementBatch with the same semantics as the reference's absorb_increment
(online.py:317-332), stage by stage:

  row hashes      the packed table for M-hat rows (a pure function of (seed, g, m, i))
  hash update     culsh_hash_accumulate `into` touched old columns + new columns
  top-K for new   culsh_topk over all N-hat keys, selection for the new columns only
  extend ratings  culsh_append_segments on the CSC and the CSR (the reference
                  rebuilds the whole SparseRatings with two lexsorts, 82% of its time)
  extend params   new rows of U/V from the reference's PCG64 stream (seed, 0x0B1),
                  new biases from the batch means (online.py:187-227), appended in HBM
  train           exact row pass + exact column pass (online.py:230-314)

Baselines of the extended data are recomputed on the device; they are
bit-identical to compute_baselines for integer-valued ratings (all sums exact).
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _native as nat
from .data import DeviceRatings
from .factorization import (DeviceModel64, ModelParams, TrainConfig, TrainingDivergedError,
                            _Scratch, _colpass, _exact_lookups, _plan_full, _rates_struct)
from .lsh import HashState, LshConfig, RowHashes, _ns, _table_alloc, _topk_device
from .online import IncrementBatch, append_device


class _Reserve:
    """A 1-D HBM buffer with spare capacity: view(n) returns its first n elements,
    regrowing by `grow` (keeping the first `keep` elements) only when n exceeds it,
    so a stream of increments does not hit cudaMalloc on every batch."""

    def __init__(self, dtype: str, grow: float):
        self.dtype, self.grow, self.buf = dtype, grow, None

    def view(self, n: int, keep: int = 0):
        n = max(int(n), 1)
        if self.buf is None or self.buf.numel() < n:
            nb = nat.empty((int(n * self.grow) + 1,), self.dtype)
            if keep and self.buf is not None:
                nb[:keep] = self.buf[:keep]
            self.buf = nb
        return self.buf[:n]


_VIEW_FIELDS = (("col_ptr", "int64", "N1"), ("col_rows", "int32", "nnz"), ("col_vals", "float64", "nnz"),
                ("row_ptr", "int64", "M1"), ("row_cols", "int32", "nnz"), ("row_vals", "float64", "nnz"),
                ("csc2csr", "int32", "nnz"))


class OnlineSession:
    """HBM-resident state for a stream of increments (paper Alg. 4).

    Memory: the two index views live in a ping-pong pair of reserved buffer sets
    (the append reads set s and writes set 1-s); the row-hash table and the model
    arrays grow in place inside reserved buffers.  `reserve` is the headroom factor
    (default 1.25: ~25% growth before the first reallocation)."""

    def __init__(self, dev: DeviceRatings, state: HashState, entries, K: int, params: ModelParams,
                 config: TrainConfig, reserve: float = 1.25):
        t = nat.torch()
        if dev.nnz and not bool(t.all(dev.col_vals == t.round(dev.col_vals)).item()):
            raise ValueError("OnlineSession keeps every sum exact and needs integer-valued ratings; "
                             "use absorb_increment for other values")
        self.dev = dev
        self.state = state
        self.lsh: LshConfig = state.config
        self.K = K
        self.entries = entries            # (N*K,) int32 device
        self.config = config
        self.mu = float(params.mu)
        self.model = DeviceModel64(params)
        self.M, self.N = dev.M, dev.N
        self.reserve = float(reserve)
        self._sets = [{f: _Reserve(dt, self.reserve) for f, dt, _ in _VIEW_FIELDS} for _ in range(2)]
        self._cur = 1                     # the next append writes set 0
        self._table = _Reserve("uint8", self.reserve)
        self._table_rows = 0
        m = self.model
        self._model = {k: _Reserve(dt, self.reserve) for k, dt in
                       (("b", "float64"), ("bhat", "float64"), ("U", "float64"), ("V", "float64"),
                        ("W", "float64"), ("C", "float64"), ("nbr", "int32"))}
        for k, r in self._model.items():
            src = getattr(m, k)
            r.view(src.numel())[:] = src
            setattr(m, k, r.buf[:src.numel()])

    def _extend_row_hashes(self, M_hat: int) -> RowHashes:
        c = self.lsh
        rec = (c.q * c.p * _ns(c.G) + 15) // 16 * 16
        lo = self._table_rows if self._table_rows <= M_hat else 0
        table = self._table.view((M_hat + 1) * rec, keep=lo * rec)
        table[M_hat * rec:].zero_()      # the all-zero padding row
        nat.call("culsh_row_hash_table", ctypes.c_uint64(c.seed), c.q, c.p, c.G, lo, M_hat,
                 nat.ptr(table), nat.stream_ptr())
        self._table_rows = M_hat
        return RowHashes(None, c.seed, _table=table, _shape=(M_hat, c.q, c.p, c.G))

    def _grow_model(self, name: str, n_keep: int, new):
        r = self._model[name]
        v = r.view(n_keep + new.numel(), keep=n_keep)
        if new.numel():
            v[n_keep:] = new
        return v

    def absorb(self, batch: IncrementBatch) -> dict:
        t = nat.torch()
        if batch.base_M != self.M or batch.base_N != self.N:
            raise ValueError("increment base shape does not match the session")
        batch.validate()
        if len(batch.values) and not np.all(np.asarray(batch.values) == np.round(batch.values)):
            raise ValueError("OnlineSession needs integer-valued ratings; use absorb_increment")
        c = self.lsh
        tm = {}

        def mark(name, t0):
            t.cuda.synchronize()
            tm[name] = time.perf_counter() - t0
            return time.perf_counter()

        t.cuda.synchronize()
        t0 = time.perf_counter()
        M_hat, N_hat, N_old, M_old = batch.M_hat, batch.N_hat, self.N, self.M
        # (1) row hashes for the extended row space: old rows copied, new rows hashed
        hashes = self._extend_row_hashes(M_hat)
        t0 = mark("row_hashes", t0)
        # (2) incremental hash state (online.py:120-149)
        from .online import update_hashes_incremental
        self.state = update_hashes_incremental(self.state, batch, hashes)
        t0 = mark("hash_update", t0)
        # (3) top-K for the new columns (online.py:152-184)
        n_new = N_hat - N_old
        if self.entries.data_ptr() != self._model["nbr"].buf.data_ptr():
            self._model["nbr"].view(N_old * self.K)[:] = self.entries[:N_old * self.K]
        ent = self._model["nbr"].view(N_hat * self.K, keep=N_old * self.K)
        if n_new > 0:
            e_new, _ = _topk_device(self.state.device_keys(), c.q, N_hat, c.p * c.G, N_old, n_new,
                                    self.K, c.seed)
            ent[N_old * self.K:] = e_new[:n_new * self.K]
        self.entries = ent
        t0 = mark("topk_new", t0)
        # (4) extend both index views in HBM (online.py:84-93)
        d = self.dev
        br = nat.to_dev(np.asarray(batch.rows, np.int32))
        bcl = nat.to_dev(np.asarray(batch.cols, np.int32))
        bv = nat.to_dev(np.asarray(batch.values, np.float64))
        self._cur ^= 1
        sets = self._sets[self._cur]
        d._integer_valued = True          # checked at construction and per batch
        self.dev, (rptr_d, rval_d, cptr_d, cval_d) = append_device(
            d, M_hat, N_hat, br, bcl, bv, alloc=lambda f, dt, n: sets[f].view(n))
        t0 = mark("extend_ratings", t0)
        # (5) extend the model (online.py:187-227), same PCG64 stream as the reference
        cfg = self.config
        F = self.model.F
        rng = np.random.default_rng((cfg.seed, 0x0B1))
        scale = cfg.effective_init_scale
        U_new = rng.uniform(0.0, scale, size=(batch.new_row_count, F))
        V_new = rng.uniform(0.0, scale, size=(batch.new_col_count, F))
        # new biases: batch means of the new variables minus mu (online.py:205-215); the
        # batch's own row / column segments (rptr_d, cptr_d) give exact integer sums
        def batch_means(ptr, vals, first, count):
            if count == 0:
                return t.zeros(0, dtype=t.float64, device=nat.device())
            sums = nat.empty((count,), "float64")
            nat.call("culsh_segment_sums", count, nat.ptr(ptr[first:]), nat.ptr(vals), nat.ptr(sums),
                     nat.stream_ptr())
            cnt = (ptr[first + 1:first + count + 1] - ptr[first:first + count]).to(t.float64)
            return t.where(cnt > 0, sums / cnt.clamp(min=1) - self.mu, t.zeros_like(sums))
        b_new = batch_means(rptr_d, rval_d, M_old, batch.new_row_count)
        bh_new = batch_means(cptr_d, cval_d, N_old, batch.new_col_count)
        m = self.model
        K = self.K
        m.b = self._grow_model("b", M_old, b_new)
        m.bhat = self._grow_model("bhat", N_old, bh_new)
        m.U = self._grow_model("U", M_old * F, nat.to_dev(U_new.reshape(-1)))
        m.V = self._grow_model("V", N_old * F, nat.to_dev(V_new.reshape(-1)))
        if K:
            m.W = self._grow_model("W", N_old * K, nat.zeros((n_new * K,), "float64"))
            m.C = self._grow_model("C", N_old * K, nat.zeros((n_new * K,), "float64"))
        m.nbr = self.entries
        m.struct = nat.CulshModel64(m.mu, nat.ptr(m.b), nat.ptr(m.bhat), nat.ptr(m.U), nat.ptr(m.V),
                                    nat.ptr(m.W), nat.ptr(m.C), nat.ptr(m.nbr), F, K)
        t0 = mark("extend_params", t0)
        # (6) train the new variables (online.py:274-314)
        dv = self.dev
        sc = _Scratch(M_hat, N_hat)
        _plan_full(dv, sc, N_old, N_hat, 0, M_hat)
        pre = _exact_lookups(dv, m, N_old, N_hat)   # the new columns' neighbour lookups, once
        t_plan = time.perf_counter()
        t.cuda.synchronize()
        t_row = 0.0
        for ep in range(cfg.epochs):
            rates = _rates_struct(cfg.rates_at(ep), cfg.regs)
            t1 = time.perf_counter()
            nat.call("culsh_sgd_exact_rowpass", ctypes.byref(dv.struct), ctypes.byref(m.struct),
                     ctypes.byref(rates), M_old, M_hat, N_old, nat.ptr(sc.status), nat.stream_ptr())
            t.cuda.synchronize()
            t_row += time.perf_counter() - t1
            if not sc.status_value():
                _colpass(dv, m, sc, rates, N_old, N_hat, 2, M_old, pre=pre)
            if sc.status_value():
                raise TrainingDivergedError(epoch=ep)
        tm["inc_plan_lookups"] = t_plan - t0
        tm["inc_rowpass"] = t_row
        t0 = mark("train_incremental", t0)
        self.M, self.N = M_hat, N_hat
        tm["total"] = sum(v for k, v in tm.items() if not k.startswith("inc_"))
        tm["batch_ratings"] = int(len(batch.rows))
        return tm

    def to_params(self) -> ModelParams:
        """Download the current model (fp64) as a ModelParams."""
        from .similarity import NeighborTable
        m = self.model
        F, K = m.F, self.K
        M, N = self.M, self.N
        h = nat.to_host
        return ModelParams(mu=self.mu, b=h(m.b)[:M].copy(), b_hat=h(m.bhat)[:N].copy(),
                           U=h(m.U)[:M * F].reshape(M, F).copy(), V=h(m.V)[:N * F].reshape(N, F).copy(),
                           W=h(m.W)[:N * K].reshape(N, K).copy() if K else np.zeros((N, 0)),
                           C=h(m.C)[:N * K].reshape(N, K).copy() if K else np.zeros((N, 0)),
                           neighbors=NeighborTable(N, K, h(self.entries)[:N * K].reshape(N, K).copy())
                           if K else None)
