"""Per-stage CUDA-event timing of the simLSH top-K build at a BASELINE shape (GPU).

  python tools/lsh_stages.py [c3]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2111_11682_b200 import _native as nat, lsh, synth

shape = sys.argv[1] if len(sys.argv) > 1 else "c3"
M, N, nnz, F, K, e = synth.SHAPES[shape]
dm = synth.random_sparse_device(M, N, nnz, seed=0)
dev = dm.dev
c = lsh.LshConfig(psi_exponent=e)


def timed(fn, reps=3):
    out = None
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return out, min(ts)


W = c.q * c.p * c.G
acc = nat.empty((N * W,), "float64")
sig = nat.empty((N * W,), "uint8")
keys = nat.empty((c.q * N,), "uint64")


def clear():
    for a in ("_value_classes", "_class_part"):
        if hasattr(dev, a):
            delattr(dev, a)


h, t_hash = timed(lambda: lsh.assign_row_hashes(M, c))
print(f"row-hash table        {t_hash:8.3f} ms")
_, t_chk = timed(lambda: lsh._int_path_ok(dev, 0, N, None, e))
print(f"psi int check         {t_chk:8.3f} ms")
_, t_vs = timed(lambda: (clear(), lsh._value_classes(dev)))
print(f"value classes         {t_vs:8.3f} ms  -> {dev._value_classes}")
_, t_cp = timed(lambda: (setattr(dev, "_class_part", None), lsh._class_partition(dev, dev._value_classes)))
print(f"class partition       {t_cp:8.3f} ms")
for var in (0, 1):
    for mb in (0, 96, 48):
        lsh._SLICE_MB = mb
        lsh._COUNT_VARIANT = var
        _, t_cnt = timed(lambda: lsh._count_path(dev, h.table(), c, acc, sig, keys, 0, N, None))
        print(f"hash_count variant={var} slice={mb:3d}MB {t_cnt:8.3f} ms")
lsh._SLICE_MB = 0
lsh._COUNT_VARIANT = 1
print(f"hash_count kernel     {t_cnt:8.3f} ms  ({nnz * W / t_cnt / 1e9:.1f} G signed adds/ms equiv.)")
_, t_acc = timed(lambda: lsh._accumulate(dev, h.table(), c, acc, sig, keys, 0, N, allow_count=False))
print(f"int accumulate kernel {t_acc:8.3f} ms (previous path, for comparison)")
ent, t_topk = timed(lambda: lsh._topk_device(keys, c.q, N, c.p * c.G, 0, N, K, c.seed))
print(f"buckets + top-K       {t_topk:8.3f} ms  (candidates {ent[1]})")
clear()
_, t_all = timed(lambda: (clear(), lsh.simlsh_topk_device(dev, c, K)), reps=3)
print(f"simlsh_topk_device    {t_all:8.3f} ms (end to end, caches cleared)")
