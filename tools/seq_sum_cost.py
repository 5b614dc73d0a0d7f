"""Time culsh_sequential_sum (the exact parallel form of the reference's serial fp64 sum)
against the one-thread loop and the pairwise tree, 1M and 100M squared errors (GPU)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_11682_b200 import _native as nat  # noqa: E402

out = {}
for n in (1_000_000, 100_000_000):
    e = torch.randn(n, dtype=torch.float64, device="cuda") * 0.9
    x = e * e
    res = nat.empty((1,), "float64")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        nat.call("culsh_sequential_sum", nat.ptr(x), n, nat.ptr(res), nat.stream_ptr())
    ts = []
    for _ in range(5):
        ev0.record()
        nat.call("culsh_sequential_sum", nat.ptr(x), n, nat.ptr(res), nat.stream_ptr())
        ev1.record()
        torch.cuda.synchronize()
        ts.append(ev0.elapsed_time(ev1))
    ref = np.add.accumulate(x.cpu().numpy())[-1]
    out[f"n{n}"] = {"ms_median": sorted(ts)[2], "bit_exact_vs_numpy_accumulate": bool(float(res.item()) == ref),
                    "one_thread_loop_ms_extrapolated": n * 4.4e-6}
print(json.dumps(out))
