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
                            _Scratch, _colpass, _plan_full, _rates_struct)
from .lsh import HashState, LshConfig, RowHashes, _ns, _table_alloc, _topk_device
from .online import IncrementBatch, device_segments


def _device_baselines(M: int, N: int, col_ptr, col_rows, col_vals):
    t = nat.torch()
    nnz = col_rows.numel()
    mu = float(col_vals.sum().item()) / max(nnz, 1)
    cnt_c = (col_ptr[1:] - col_ptr[:-1]).to(t.float64)
    col_of = t.repeat_interleave(t.arange(N, device=col_rows.device), col_ptr[1:] - col_ptr[:-1])
    cs = t.zeros(N, dtype=t.float64, device=col_rows.device).index_add_(0, col_of, col_vals)
    rs = t.zeros(M, dtype=t.float64, device=col_rows.device).index_add_(0, col_rows.long(), col_vals)
    rc = t.bincount(col_rows, minlength=M).to(t.float64)
    bb = t.where(rc > 0, rs / rc.clamp(min=1) - mu, t.zeros_like(rs))
    bh = t.where(cnt_c > 0, cs / cnt_c.clamp(min=1) - mu, t.zeros_like(cs))
    return mu, bb, bh


class OnlineSession:
    """HBM-resident state for a stream of increments (paper Alg. 4)."""

    def __init__(self, dev: DeviceRatings, state: HashState, entries, K: int, params: ModelParams,
                 config: TrainConfig):
        self.dev = dev
        self.state = state
        self.lsh: LshConfig = state.config
        self.K = K
        self.entries = entries            # (N*K,) int32 device
        self.config = config
        self.mu = float(params.mu)
        self.model = DeviceModel64(params)
        self.M, self.N = dev.M, dev.N

    def _extend_row_hashes(self, M_hat: int) -> RowHashes:
        c = self.lsh
        rec = (c.q * c.p * _ns(c.G) + 15) // 16 * 16
        table = _table_alloc(M_hat, c.q, c.p, c.G)
        old = getattr(self, "_table", None)
        if old is not None and self._table_rows <= M_hat:
            table[:self._table_rows * rec] = old[:self._table_rows * rec]
            lo = self._table_rows
        else:
            lo = 0
        nat.call("culsh_row_hash_table", ctypes.c_uint64(c.seed), c.q, c.p, c.G, lo, M_hat,
                 nat.ptr(table), nat.stream_ptr())
        self._table, self._table_rows = table, M_hat
        return RowHashes(None, c.seed, _table=table, _shape=(M_hat, c.q, c.p, c.G))

    def absorb(self, batch: IncrementBatch) -> dict:
        t = nat.torch()
        if batch.base_M != self.M or batch.base_N != self.N:
            raise ValueError("increment base shape does not match the session")
        batch.validate()
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
        ent = nat.empty((N_hat * self.K,), "int32")
        ent[:N_old * self.K] = self.entries[:N_old * self.K]
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
        cptr_d, crow_d, cval_d = device_segments(N_hat, bcl, br, bv)
        rptr_d, rcol_d, rval_d = device_segments(M_hat, br, bcl, bv)
        nnz_hat = d.nnz + len(batch.rows)
        new_col_ptr = nat.empty((N_hat + 1,), "int64")
        new_col_rows = nat.empty((max(nnz_hat, 1),), "int32")
        new_col_vals = nat.empty((max(nnz_hat, 1),), "float64")
        new_row_ptr = nat.empty((M_hat + 1,), "int64")
        new_row_cols = nat.empty((max(nnz_hat, 1),), "int32")
        new_row_vals = nat.empty((max(nnz_hat, 1),), "float64")
        nat.call("culsh_append_segments", N_old, N_hat, nat.ptr(d.col_ptr), nat.ptr(d.col_rows),
                 nat.ptr(d.col_vals), nat.ptr(cptr_d), nat.ptr(crow_d), nat.ptr(cval_d),
                 nat.ptr(new_col_ptr), nat.ptr(new_col_rows), nat.ptr(new_col_vals), nat.stream_ptr())
        nat.call("culsh_append_segments", M_old, M_hat, nat.ptr(d.row_ptr), nat.ptr(d.row_cols),
                 nat.ptr(d.row_vals), nat.ptr(rptr_d), nat.ptr(rcol_d), nat.ptr(rval_d),
                 nat.ptr(new_row_ptr), nat.ptr(new_row_cols), nat.ptr(new_row_vals), nat.stream_ptr())
        mu_x, bb, bh = _device_baselines(M_hat, N_hat, new_col_ptr, new_col_rows[:nnz_hat],
                                         new_col_vals[:nnz_hat])
        self.dev = DeviceRatings.from_device(M_hat, N_hat, new_col_ptr, new_col_rows[:nnz_hat],
                                             new_col_vals[:nnz_hat], new_row_ptr, new_row_cols[:nnz_hat],
                                             new_row_vals[:nnz_hat], mu_x, bb, bh)
        t0 = mark("extend_ratings", t0)
        # (5) extend the model (online.py:187-227), same PCG64 stream as the reference
        cfg = self.config
        F = self.model.F
        rng = np.random.default_rng((cfg.seed, 0x0B1))
        scale = cfg.effective_init_scale
        U_new = rng.uniform(0.0, scale, size=(batch.new_row_count, F))
        V_new = rng.uniform(0.0, scale, size=(batch.new_col_count, F))
        b_new = np.zeros(batch.new_row_count)
        bh_new = np.zeros(batch.new_col_count)
        if len(batch.rows):
            rs = np.zeros(M_hat)
            rc = np.zeros(M_hat)
            np.add.at(rs, batch.rows, batch.values)
            np.add.at(rc, batch.rows, 1.0)
            sel = rc[M_old:] > 0
            b_new[sel] = rs[M_old:][sel] / rc[M_old:][sel] - self.mu
            cs = np.zeros(N_hat)
            cc = np.zeros(N_hat)
            np.add.at(cs, batch.cols, batch.values)
            np.add.at(cc, batch.cols, 1.0)
            sel = cc[N_old:] > 0
            bh_new[sel] = cs[N_old:][sel] / cc[N_old:][sel] - self.mu
        m = self.model
        K = self.K
        m.b = t.cat([m.b[:M_old], nat.to_dev(b_new)])
        m.bhat = t.cat([m.bhat[:N_old], nat.to_dev(bh_new)])
        m.U = t.cat([m.U[:M_old * F], nat.to_dev(U_new.reshape(-1))])
        m.V = t.cat([m.V[:N_old * F], nat.to_dev(V_new.reshape(-1))])
        if K:
            m.W = t.cat([m.W[:N_old * K], nat.zeros((n_new * K,), "float64")])
            m.C = t.cat([m.C[:N_old * K], nat.zeros((n_new * K,), "float64")])
        m.nbr = self.entries
        m.struct = nat.CulshModel64(m.mu, nat.ptr(m.b), nat.ptr(m.bhat), nat.ptr(m.U), nat.ptr(m.V),
                                    nat.ptr(m.W), nat.ptr(m.C), nat.ptr(m.nbr), F, K)
        t0 = mark("extend_params", t0)
        # (6) train the new variables (online.py:274-314)
        dv = self.dev
        sc = _Scratch(M_hat, N_hat)
        _plan_full(dv, sc, N_old, N_hat, 0, M_hat)
        for ep in range(cfg.epochs):
            rates = _rates_struct(cfg.rates_at(ep), cfg.regs)
            nat.call("culsh_sgd_exact_rowpass", ctypes.byref(dv.struct), ctypes.byref(m.struct),
                     ctypes.byref(rates), M_old, M_hat, N_old, nat.ptr(sc.status), nat.stream_ptr())
            if not sc.status_value():
                _colpass(dv, m, sc, rates, N_old, N_hat, 2, M_old)
            if sc.status_value():
                raise TrainingDivergedError(epoch=ep)
        t0 = mark("train_incremental", t0)
        self.M, self.N = M_hat, N_hat
        tm["total"] = sum(tm.values())
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
