"""Per-entry-point GPU time of one C3 simLSH top-K build (CUDA events around every C call).

  python tools/lsh_breakdown.py
"""
import sys, json, collections
sys.path.insert(0, ".")
import torch
from paper_2111_11682_b200 import _native as nat, lsh, synth
M, N, nnz, F, K, e = synth.SHAPES["c3"]
dm = synth.random_sparse_device(M, N, nnz, seed=0)
cfg = lsh.LshConfig(psi_exponent=e)
for _ in range(2):
    lsh.simlsh_topk_device(dm.dev, cfg, K)
torch.cuda.synchronize()
orig = nat.call
times = collections.defaultdict(float)
evs = []
def timed_call(name, *a):
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); r = orig(name, *a); t.record(); evs.append((name, s, t)); return r
nat.call = timed_call
for attr in ("_value_classes", "_class_part"):   # time the data-dependent prep too (as bench.py)
    if hasattr(dm.dev, attr):
        delattr(dm.dev, attr)
import time
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); t0 = time.perf_counter(); a.record()
lsh.simlsh_topk_device(dm.dev, cfg, K)
b.record(); torch.cuda.synchronize(); wall = time.perf_counter() - t0
for name, s, t in evs:
    times[name] += s.elapsed_time(t)
print(json.dumps({"wall_ms": wall * 1e3, "gpu_span_ms": a.elapsed_time(b), "per_call_ms": dict(times)}, indent=1))
