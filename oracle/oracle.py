"""ctypes front-end for the CPU oracle (culsh_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, as the checker.  The product
package never imports this module.

Each wrapper takes the same arguments as the reference function it restates
(cited per function) and returns numpy arrays.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liborcl.so")
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_vp = ctypes.c_void_p


def build() -> str:
    """Compile liborcl.so with the committed Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.orc_splitmix64.restype = ctypes.c_uint64
        _lib.orc_splitmix64.argtypes = [ctypes.c_uint64]
        _lib.orc_map_key.restype = ctypes.c_uint64
        _lib.orc_map_key.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64]
        _lib.orc_topk_from_group_keys.restype = ctypes.c_int64
        _lib.orc_rmse.restype = ctypes.c_double
        _lib.orc_predict.restype = ctypes.c_double
        for name in ("orc_full_pass_block", "orc_stage_pass", "orc_parallel_epoch",
                     "orc_online_row_pass", "orc_online_col_pass"):
            getattr(_lib, name).restype = ctypes.c_int
        _lib.orc_set_threads(os.cpu_count() or 1)   # hash-stage threads; outputs do not depend on it
    return _lib


def _p(a: np.ndarray):
    assert a.flags.c_contiguous
    return ctypes.c_void_p(a.ctypes.data)


def n_threads() -> int:
    return os.cpu_count() or 1


# ------------------------------------------------------------------ LSH ----

def splitmix64(x: int) -> int:
    """lsh.py:53-58"""
    return int(lib().orc_splitmix64(ctypes.c_uint64(x & 0xFFFFFFFFFFFFFFFF)))


def assign_bits(seed: int, q: int, p: int, M: int, G: int) -> np.ndarray:
    """lsh.py:68-78 -> (M, q, p, G) uint8"""
    bits = np.empty((M, q, p, G), dtype=np.uint8)
    lib().orc_assign_bits(ctypes.c_uint64(seed), q, p, ctypes.c_int64(M), G, _p(bits))
    return bits


def accumulate_all(col_ptr, col_rows, col_vals, bits, e, nthreads=None) -> np.ndarray:
    """lsh.py:161-179 -> acc (N, q, p, G) float64"""
    col_ptr = np.ascontiguousarray(col_ptr, dtype=np.int64)
    col_rows = np.ascontiguousarray(col_rows, dtype=np.int32)
    col_vals = np.ascontiguousarray(col_vals, dtype=np.float64)
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    N = len(col_ptr) - 1
    _, q, p, G = bits.shape
    acc = np.empty((N, q, p, G), dtype=np.float64)
    lib().orc_accumulate_all(_p(col_ptr), _p(col_rows), _p(col_vals), ctypes.c_int64(N),
                             _p(bits), q, p, G, e, _p(acc),
                             n_threads() if nthreads is None else nthreads)
    return acc


def accumulate_into(acc, col_ptr, col_rows, col_vals, bits, e) -> None:
    """online.py:96-117 (in place)"""
    col_ptr = np.ascontiguousarray(col_ptr, dtype=np.int64)
    col_rows = np.ascontiguousarray(col_rows, dtype=np.int32)
    col_vals = np.ascontiguousarray(col_vals, dtype=np.float64)
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    _, q, p, G = bits.shape
    lib().orc_accumulate_into(_p(acc), _p(col_ptr), _p(col_rows), _p(col_vals),
                              ctypes.c_int64(len(col_ptr) - 1), _p(bits), q, p, G, e)


def threshold(acc) -> np.ndarray:
    """lsh.py:182-183"""
    acc = np.ascontiguousarray(acc)
    sig = np.empty(acc.shape, dtype=np.uint8)
    lib().orc_threshold(_p(acc), ctypes.c_int64(acc.size), _p(sig))
    return sig


def group_keys(sig) -> np.ndarray:
    """lsh.py:246-260 + 417-423 -> (q, N) uint64"""
    sig = np.ascontiguousarray(sig, dtype=np.uint8)
    N, q, p, G = sig.shape
    keys = np.empty((q, N), dtype=np.uint64)
    lib().orc_pack_group_keys(_p(sig), ctypes.c_int64(N), q, p, G, _p(keys))
    return keys


def topk_from_group_keys(keys, K: int, seed: int, j_base: int = 0, n_cols: int | None = None):
    """lsh.py:401-414 (and online.py:152-184 with j_base) -> (entries, n_candidates)"""
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    q, N = keys.shape
    if n_cols is None:
        n_cols = N - j_base
    entries = np.empty((n_cols, K), dtype=np.int32)
    total = lib().orc_topk_from_group_keys(_p(keys), q, ctypes.c_int64(N), ctypes.c_int64(j_base),
                                           ctypes.c_int64(n_cols), K, ctypes.c_uint64(seed),
                                           _p(entries))
    return entries, int(total)


@dataclass
class HashResult:
    acc: np.ndarray
    sig: np.ndarray
    keys: np.ndarray
    entries: np.ndarray | None


def simlsh_topk(col_ptr, col_rows, col_vals, M, G, p, q, e, seed, K, nthreads=None) -> HashResult:
    """lsh.py:426-438 composed from the stage restatements."""
    if nthreads:
        lib().orc_set_threads(int(nthreads))
    bits = assign_bits(seed, q, p, M, G)
    acc = accumulate_all(col_ptr, col_rows, col_vals, bits, e, nthreads)
    sig = threshold(acc)
    keys = group_keys(sig)
    entries = topk_from_group_keys(keys, K, seed)[0] if K is not None else None
    return HashResult(acc, sig, keys, entries)


# ------------------------------------------------------------------ SGD ----

class Rates(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in
                ("gb", "gbh", "gu", "gv", "gw", "gc", "lb", "lbh", "lu", "lv", "lw", "lc")]


def make_rates(rates, regs) -> Rates:
    return Rates(*[float(x) for x in tuple(rates) + tuple(regs)])


@dataclass
class Model:
    """Mutable fp64 model state (factorization.py:105-185 ModelParams fields)."""
    mu: float
    b: np.ndarray
    bhat: np.ndarray
    U: np.ndarray
    V: np.ndarray
    W: np.ndarray
    C: np.ndarray
    nbr: np.ndarray

    def copy(self) -> "Model":
        return Model(self.mu, self.b.copy(), self.bhat.copy(), self.U.copy(), self.V.copy(),
                     self.W.copy(), self.C.copy(), self.nbr.copy())


@dataclass
class Csr:
    """Both index views plus the residual baselines (data.py:166-309)."""
    M: int
    N: int
    row_ptr: np.ndarray
    row_cols: np.ndarray
    row_vals: np.ndarray
    col_ptr: np.ndarray
    col_rows: np.ndarray
    col_vals: np.ndarray
    base_b: np.ndarray
    base_bhat: np.ndarray


def build_csr(M, N, rows, cols, vals) -> Csr:
    """data.py:189-201 index build + data.py:289-309 baselines."""
    rows = np.asarray(rows, np.int32)
    cols = np.asarray(cols, np.int32)
    vals = np.asarray(vals, np.float64)
    o = np.lexsort((cols, rows))
    row_ptr = np.zeros(M + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=M), out=row_ptr[1:])
    o2 = np.lexsort((rows, cols))
    col_ptr = np.zeros(N + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=N), out=col_ptr[1:])
    mu = float(vals.mean())
    rc = np.diff(row_ptr)
    cc = np.diff(col_ptr)
    rs = np.zeros(M)
    np.add.at(rs, rows, vals)
    cs = np.zeros(N)
    np.add.at(cs, cols, vals)
    bb = np.zeros(M)
    nz = rc > 0
    bb[nz] = rs[nz] / rc[nz] - mu
    bh = np.zeros(N)
    nz = cc > 0
    bh[nz] = cs[nz] / cc[nz] - mu
    return Csr(M, N, row_ptr, np.ascontiguousarray(cols[o]), np.ascontiguousarray(vals[o]),
               col_ptr, np.ascontiguousarray(rows[o2]), np.ascontiguousarray(vals[o2]), bb, bh), mu


def _model_args(d: Csr, m: Model):
    F = m.U.shape[1]
    K = m.W.shape[1]
    return [_p(d.row_ptr), _p(d.row_cols), _p(d.row_vals), ctypes.c_double(m.mu),
            _p(m.b), _p(m.bhat), _p(m.U), _p(m.V), _p(m.W), _p(m.C),
            _p(m.nbr), F, K, _p(d.base_b), _p(d.base_bhat)]


def full_pass(d: Csr, m: Model, rates: Rates, col_lo=0, col_hi=None, row_lo=0, row_hi=None,
              update_row=True, update_col=True) -> int:
    """factorization.py:332-363 _full_pass_block (in place)"""
    col_hi = d.N if col_hi is None else col_hi
    row_hi = d.M if row_hi is None else row_hi
    return lib().orc_full_pass_block(
        ctypes.c_int64(col_lo), ctypes.c_int64(col_hi), ctypes.c_int64(row_lo),
        ctypes.c_int64(row_hi), ctypes.c_int64(d.M), _p(d.col_ptr), _p(d.col_rows),
        _p(d.col_vals), *_model_args(d, m), ctypes.byref(rates), int(update_row), int(update_col))


def partition(d: Csr, D: int):
    """parallel.py:99-107 make_partition -> (row_bounds, col_bounds, block_ptr)"""
    row_bounds = np.array([(k * d.M) // D for k in range(D + 1)], np.int64)
    col_bounds = np.array([(k * d.N) // D for k in range(D + 1)], np.int64)
    bp = np.empty((d.N, D + 1), np.int64)
    lib().orc_block_pointers(_p(d.col_ptr), _p(d.col_rows), ctypes.c_int64(d.N),
                             _p(row_bounds), D + 1, _p(bp))
    return row_bounds, col_bounds, bp


def parallel_epoch(d: Csr, m: Model, rates: Rates, D: int, part=None, nthreads=None) -> int:
    """parallel.py:186-215, one epoch of the D x D rotation (in place)"""
    if part is None:
        part = partition(d, D)
    _, col_bounds, bp = part
    return lib().orc_parallel_epoch(D, _p(col_bounds), _p(bp), _p(d.col_rows), _p(d.col_vals),
                                    *_model_args(d, m), ctypes.byref(rates),
                                    n_threads() if nthreads is None else nthreads)


def online_row_pass(d: Csr, m: Model, rates: Rates, row_lo, row_hi, N_old) -> int:
    """online.py:230-250"""
    return lib().orc_online_row_pass(ctypes.c_int64(row_lo), ctypes.c_int64(row_hi),
                                     ctypes.c_int64(N_old), *_model_args(d, m), ctypes.byref(rates))


def online_col_pass(d: Csr, m: Model, rates: Rates, col_lo, col_hi, M_old) -> int:
    """online.py:253-271"""
    return lib().orc_online_col_pass(ctypes.c_int64(col_lo), ctypes.c_int64(col_hi),
                                     ctypes.c_int64(M_old), _p(d.col_ptr), _p(d.col_rows),
                                     _p(d.col_vals), *_model_args(d, m), ctypes.byref(rates))


def rmse(d: Csr, m: Model, t_rows, t_cols, t_vals, clamp=None, unscale=None) -> float:
    """factorization.py:394-409 + 559-579"""
    t_rows = np.ascontiguousarray(t_rows, np.int32)
    t_cols = np.ascontiguousarray(t_cols, np.int32)
    t_vals = np.ascontiguousarray(t_vals, np.float64)
    lo, hi = clamp if clamp is not None else (0.0, 0.0)
    F = m.U.shape[1]
    K = m.W.shape[1]
    return float(lib().orc_rmse(
        _p(t_rows), _p(t_cols), _p(t_vals), ctypes.c_int64(len(t_rows)),
        _p(d.row_ptr), _p(d.row_cols), _p(d.row_vals), ctypes.c_double(m.mu),
        _p(m.b), _p(m.bhat), _p(m.U), _p(m.V), _p(m.W), _p(m.C), _p(m.nbr), F, K,
        _p(d.base_b), _p(d.base_bhat), int(clamp is not None), ctypes.c_double(lo),
        ctypes.c_double(hi), ctypes.c_double(1.0 if unscale is None else float(unscale))))


def learning_rate(alpha, beta, t):
    """factorization.py:42-44"""
    return alpha / (1.0 + beta * t ** 1.5)


def init_model(M, N, F, K, nbr, mu, base_b, base_bhat, seed, init_scale=None) -> Model:
    """factorization.py:196-211 (numpy PCG64 stream, same draw order)"""
    rng = np.random.default_rng(seed)
    scale = init_scale if init_scale is not None else 1.0 / np.sqrt(F)
    U = rng.uniform(0.0, scale, size=(M, F))
    V = rng.uniform(0.0, scale, size=(N, F))
    nbr = np.zeros((N, 0), np.int32) if nbr is None else np.ascontiguousarray(nbr, np.int32)
    return Model(mu, base_b.copy(), base_bhat.copy(), U, V, np.zeros((N, K)), np.zeros((N, K)), nbr)


# --------------------------------------------------------------- Online ----

def train_full(d: Csr, mu, nbr, F, K, epochs, seed, rates_fn, regs, init_scale=None,
               callback=None) -> Model:
    """factorization.py:530-556 train_full (serial column-major epochs)."""
    m = init_model(d.M, d.N, F, K, nbr, mu, d.base_b, d.base_bhat, seed, init_scale)
    for t in range(epochs):
        bad = full_pass(d, m, make_rates(rates_fn(t), regs))
        if bad:
            raise FloatingPointError(f"diverged at epoch {t}")
        if callback is not None:
            callback(t, m)
    return m


def parallel_train(d: Csr, mu, nbr, F, K, epochs, seed, rates_fn, regs, D, init_scale=None,
                   nthreads=None) -> Model:
    """parallel.py:166-227 parallel_train (D x D rotation, deterministic for fixed D)."""
    m = init_model(d.M, d.N, F, K, nbr, mu, d.base_b, d.base_bhat, seed, init_scale)
    part = partition(d, D)
    for t in range(epochs):
        if parallel_epoch(d, m, make_rates(rates_fn(t), regs), D, part, nthreads):
            raise FloatingPointError(f"diverged at epoch {t}")
    return m


def absorb_increment(m: Model, acc, lsh_cfg, orig: Csr, orig_triplets, batch, F, K, epochs,
                     seed, rates_fn, regs, init_scale=None):
    """online.py:317-332 absorb_increment, composed from the restated stages.

    lsh_cfg = (G, p, q, e, lsh_seed); orig_triplets = (rows, cols, vals) of the
    original matrix in entry order; batch = (base_M, base_N, n_rows, n_cols,
    rows, cols, vals).  Returns (model_ext, acc_ext, entries_ext, csr_ext).
    """
    G, p, q, e, lseed = lsh_cfg
    base_M, base_N, nr_, nc_, brows, bcols, bvals = batch
    brows = np.asarray(brows, np.int32)
    bcols = np.asarray(bcols, np.int32)
    bvals = np.asarray(bvals, np.float64)
    M_hat, N_hat = base_M + nr_, base_N + nc_
    # online.py:324 + 120-149 update_hashes_incremental
    bits = assign_bits(lseed, q, p, M_hat, G)
    acc_ext = np.zeros((N_hat, q, p, G))
    acc_ext[:base_N] = acc
    order = np.lexsort((brows, bcols))
    cp = np.zeros(N_hat + 1, np.int64)
    np.cumsum(np.bincount(bcols, minlength=N_hat), out=cp[1:])
    accumulate_into(acc_ext, cp, brows[order], bvals[order], bits, e)
    sig = threshold(acc_ext)
    # online.py:152-184 topk_for_new
    keys = group_keys(sig)
    entries = np.empty((N_hat, K), np.int32)
    entries[:base_N] = m.nbr
    if N_hat > base_N:
        entries[base_N:] = topk_from_group_keys(keys, K, lseed, base_N, N_hat - base_N)[0]
    # online.py:84-93 extend_ratings
    r0, c0, v0 = orig_triplets
    d_ext, mu_ext = build_csr(M_hat, N_hat, np.concatenate([r0, brows]),
                              np.concatenate([c0, bcols]), np.concatenate([v0, bvals]))
    # online.py:187-227 extend_params
    rng = np.random.default_rng((seed, 0x0B1))
    scale = init_scale if init_scale is not None else 1.0 / np.sqrt(F)
    b = np.zeros(M_hat)
    b[:base_M] = m.b
    bhat = np.zeros(N_hat)
    bhat[:base_N] = m.bhat
    if len(brows):
        rs = np.zeros(M_hat)
        rc = np.zeros(M_hat)
        np.add.at(rs, brows, bvals)
        np.add.at(rc, brows, 1.0)
        new = (np.arange(M_hat) >= base_M) & (rc > 0)
        b[new] = rs[new] / rc[new] - m.mu
        cs = np.zeros(N_hat)
        cc = np.zeros(N_hat)
        np.add.at(cs, bcols, bvals)
        np.add.at(cc, bcols, 1.0)
        new = (np.arange(N_hat) >= base_N) & (cc > 0)
        bhat[new] = cs[new] / cc[new] - m.mu
    U = np.vstack([m.U, rng.uniform(0.0, scale, size=(nr_, F))])
    V = np.vstack([m.V, rng.uniform(0.0, scale, size=(nc_, F))])
    W = np.vstack([m.W, np.zeros((nc_, K))])
    C = np.vstack([m.C, np.zeros((nc_, K))])
    me = Model(m.mu, b, bhat, np.ascontiguousarray(U), np.ascontiguousarray(V),
               np.ascontiguousarray(W), np.ascontiguousarray(C), entries)
    # online.py:274-314 train_incremental (baselines of the EXTENDED data)
    for t in range(epochs):
        rt = make_rates(rates_fn(t), regs)
        bad = online_row_pass(d_ext, me, rt, base_M, M_hat, base_N)
        if not bad:
            bad = online_col_pass(d_ext, me, rt, base_N, N_hat, base_M)
        if bad:
            raise FloatingPointError(f"diverged at epoch {t}")
    return me, acc_ext, entries, d_ext


def stage_pass(d: Csr, m: Model, rates: Rates, col_lo: int, col_hi: int, rb: int,
               block_ptr: np.ndarray) -> int:
    """parallel.py:110-128 _stage_pass: one worker's (row block rb) x (columns) block."""
    nb = block_ptr.shape[1]
    return lib().orc_stage_pass(ctypes.c_int64(col_lo), ctypes.c_int64(col_hi), rb,
                                _p(block_ptr), nb, _p(d.col_rows), _p(d.col_vals),
                                *_model_args(d, m), ctypes.byref(rates))


def train_basic(d: Csr, mu_data, F, epochs, seed, rates_fn, regs, with_biases=False,
                sort_rows_by_count=False, init_scale=None) -> Model:
    """factorization.py:476-527 train_basic, serial (racy_workers=0)."""
    rng = np.random.default_rng(seed)
    scale = init_scale if init_scale is not None else 1.0 / np.sqrt(F)
    U = rng.uniform(0.0, scale, size=(d.M, F))
    V = rng.uniform(0.0, scale, size=(d.N, F))
    if with_biases:
        mu, b, bh = mu_data, d.base_b.copy(), d.base_bhat.copy()
    else:
        mu, b, bh = 0.0, np.zeros(d.M), np.zeros(d.N)
    if sort_rows_by_count:
        order = np.argsort(-np.diff(d.row_ptr), kind="stable").astype(np.int64)
    else:
        order = np.arange(d.M, dtype=np.int64)
    lib().orc_basic_pass.restype = ctypes.c_int
    for t in range(epochs):
        rt = make_rates(rates_fn(t), regs)
        bad = lib().orc_basic_pass(_p(order), ctypes.c_int64(d.M), _p(d.row_ptr), _p(d.row_cols),
                                   _p(d.row_vals), ctypes.c_double(mu), _p(b), _p(bh), _p(U), _p(V), F,
                                   int(with_biases), ctypes.byref(rt))
        if bad:
            raise FloatingPointError(f"diverged at epoch {t}")
    return Model(mu, b, bh, U, V, np.zeros((d.N, 0)), np.zeros((d.N, 0)), np.zeros((d.N, 0), np.int32))


# ----------------------------------------------------------- similarity ----

def pair_stats(r1, v1, r2, v2) -> np.ndarray:
    """similarity.py:57-90 -> [n, s1, s2, s12, q1, q2]"""
    r1, r2 = np.ascontiguousarray(r1, np.int32), np.ascontiguousarray(r2, np.int32)
    v1, v2 = np.ascontiguousarray(v1, np.float64), np.ascontiguousarray(v2, np.float64)
    out = np.zeros(6)
    lib().orc_pair_stats(_p(r1), _p(v1), ctypes.c_int64(len(r1)), _p(r2), _p(v2),
                         ctypes.c_int64(len(r2)), _p(out))
    return out


def pearson_from_stats(st) -> float:
    """similarity.py:93-107"""
    f = lib().orc_pearson_from_stats
    f.restype = ctypes.c_double
    st = np.ascontiguousarray(st, np.float64)
    return float(f(_p(st)))


def gsm_topk(col_ptr, col_rows, col_vals, N, K, lambda_rho=100.0, nthreads=None) -> np.ndarray:
    """similarity.py:164-185 -> (N, K) int32"""
    ent = np.zeros((N, K), dtype=np.int32)
    cp = np.ascontiguousarray(col_ptr, np.int64)
    cr = np.ascontiguousarray(col_rows, np.int32)
    cv = np.ascontiguousarray(col_vals, np.float64)
    lib().orc_gsm_topk(_p(cp), _p(cr), _p(cv), ctypes.c_int64(N), K, ctypes.c_double(lambda_rho),
                       _p(ent), nthreads or n_threads())
    return ent


def gsm_topk_targets(col_ptr, col_rows, col_vals, N, targets, K, lambda_rho=100.0, nthreads=None):
    """similarity.py:164-185 for the listed target columns only -> (len(targets), K) int32"""
    tg = np.ascontiguousarray(targets, np.int64)
    ent = np.zeros((len(tg), K), dtype=np.int32)
    cp = np.ascontiguousarray(col_ptr, np.int64)
    cr = np.ascontiguousarray(col_rows, np.int32)
    cv = np.ascontiguousarray(col_vals, np.float64)
    lib().orc_gsm_topk_targets(_p(cp), _p(cr), _p(cv), ctypes.c_int64(N), _p(tg), ctypes.c_int64(len(tg)), K,
                               ctypes.c_double(lambda_rho), _p(ent), nthreads or n_threads())
    return ent
