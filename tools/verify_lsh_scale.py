"""Full-scale simLSH parity evidence (GPU vs the oracle, itself pinned to the reference):
C3 integer stars (bit-count path) and a C2-shape matrix with non-integer values (ordered
fp64 path).  Prints one JSON line per case with sha256 digests and the comparison.

  python tools/verify_lsh_scale.py
"""
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as orc  # noqa: E402
from paper_2111_11682_b200 import _native as nat, lsh, synth  # noqa: E402
from paper_2111_11682_b200.data import DeviceSparseRatings  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def case(name, dev, M, N, K, e):
    cfg = lsh.LshConfig(psi_exponent=e, seed=0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ent, state, _ = lsh.simlsh_topk_device(dev, cfg, K)
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t0
    cp, cr, cv = nat.to_host(dev.col_ptr), nat.to_host(dev.col_rows), nat.to_host(dev.col_vals)
    t0 = time.perf_counter()
    ref = orc.simlsh_topk(cp, cr, cv, M, 8, 3, 100, e, 0, K)
    cpu_s = time.perf_counter() - t0
    g_ent = nat.to_host(ent)[:N * K].reshape(N, K)
    out = {"case": name, "M": M, "N": N, "nnz": int(dev.nnz), "K": K, "psi_exponent": e,
           "gpu_s": gpu_s, "oracle_s": cpu_s, "oracle_threads": orc.n_threads(),
           "acc_sha_gpu": sha(state.acc), "acc_sha_oracle": sha(ref.acc),
           "acc_equal": state.acc.tobytes() == ref.acc.tobytes(),
           "sig_equal": state.sig.tobytes() == ref.sig.tobytes(),
           "entries_equal": bool(np.array_equal(g_ent, ref.entries)),
           "zero_acc_count": int((ref.acc == 0).sum())}
    print(json.dumps(out), flush=True)


def main():
    M, N, nnz, F, K, e = synth.SHAPES["c3"]
    dm = synth.random_sparse_device(M, N, nnz, seed=0)
    case("c3_integer_stars", dm.dev, M, N, K, e)
    del dm
    torch.cuda.empty_cache()
    M, N, nnz, F, K, e = synth.SHAPES["c2"]
    dm = synth.random_sparse_device(M, N, nnz, seed=1)
    d = dm.dev
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    vals = d.col_vals * 0.37 + 0.2 * torch.randn(d.col_vals.shape, generator=g, device="cuda",
                                                  dtype=torch.float64)
    col = torch.repeat_interleave(torch.arange(N, device="cuda"), d.col_ptr[1:] - d.col_ptr[:-1]).to(torch.int32)
    r = DeviceSparseRatings(M, N, d.col_rows, col, vals)
    case("c2_real_values", r.device(), M, N, K, e)


if __name__ == "__main__":
    main()
