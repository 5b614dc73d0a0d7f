"""Host materialisation of a C3-sized fp32 device matrix (U: 480,189 x 128) as a fresh fp64
numpy array -- the dominant per-fit cost after the epochs (tools/fit_breakdown.py).
Strategies timed (device sync on both sides, fresh destination each run):

  cpu_astype      U.cpu().numpy().astype(float64)                   (round-1 path)
  f64_copy        U.double() on the device, copy_ into np.empty (torch.from_numpy)
  f64_copy_thr    the same split over T host threads (parallel page faults / copies)
  staged_thr      U.double() -> a reusable pinned staging buffer in chunks, T threads
                  copying chunks out into np.empty while the next chunk streams

  python tools/d2h_bench.py
"""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402


def timed(fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def main():
    torch.cuda.set_device(0)
    M, F = 480189, 128
    U = torch.rand(M * F, device="cuda", dtype=torch.float32)
    n = U.numel()
    T = min(16, os.cpu_count() or 1)
    pool = ThreadPoolExecutor(T)
    out = {"n": n, "threads": T, "thp": open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip()}

    out["cpu_astype"] = timed(lambda: U.cpu().numpy().astype(np.float64))

    def f64_copy():
        dst = np.empty(n, np.float64)
        torch.from_numpy(dst).copy_(U.double())
        return dst
    out["f64_copy"] = timed(f64_copy)

    def f64_copy_thr():
        dst = np.empty(n, np.float64)
        d64 = U.double()
        torch.cuda.synchronize()
        step = -(-n // T)
        def part(k):
            lo, hi = k * step, min(n, (k + 1) * step)
            torch.from_numpy(dst[lo:hi]).copy_(d64[lo:hi])
        list(pool.map(part, range(T)))
        return dst
    out["f64_copy_thr"] = timed(f64_copy_thr)

    CH = 8 << 20                                  # doubles per chunk (64 MB)
    stage = [torch.empty(CH, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    copy_stream = torch.cuda.Stream()

    def staged_thr():
        dst = np.empty(n, np.float64)
        d64 = U.double()
        ev = [torch.cuda.Event() for _ in range(2)]
        futs = [None, None]
        cur = torch.cuda.current_stream()
        copy_stream.wait_stream(cur)
        for c, lo in enumerate(range(0, n, CH)):
            b = c & 1
            if futs[b] is not None:
                for f in futs[b]:
                    f.result()
            hi = min(n, lo + CH)
            with torch.cuda.stream(copy_stream):
                stage[b][:hi - lo].copy_(d64[lo:hi], non_blocking=True)
                ev[b].record(copy_stream)
            ev[b].synchronize()
            sub = -(-(hi - lo) // T)
            src = stage[b].numpy()
            futs[b] = [pool.submit(np.copyto, dst[lo + k * sub:min(hi, lo + (k + 1) * sub)],
                                   src[k * sub:min(hi - lo, (k + 1) * sub)]) for k in range(T)]
        for fs in futs:
            for f in fs or []:
                f.result()
        return dst
    out["staged_thr"] = timed(staged_thr)
    ref = U.double().cpu().numpy()
    assert np.array_equal(staged_thr(), ref) and np.array_equal(f64_copy_thr(), ref)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
