"""GSM count route phase timings at C2 / C3 (CUDA events per phase, several runs): densify into
the tiled panels, the tcgen05 statistics kernel, the fp64 select.  For run-to-run variance.

  python tools/gsm_phases.py c3 [runs]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_11682_b200 import _native as nat, synth  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    runs = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    M, N, nnz, F, K, e = synth.SHAPES[name]
    d = synth.random_sparse_device(M, N, nnz, seed=0).dev
    ld = (N + 127) // 128 * 128
    w = (M + 63) // 64 * 64
    pan = torch.zeros((3 * ld * w,), dtype=torch.int8, device="cuda")
    g = torch.empty((6, ld, ld), dtype=torch.int32, device="cuda")
    st = nat.zeros((1,), "int32")
    entries = nat.empty((N * K,), "int32")
    for r in range(runs):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        pan.zero_()
        nat.call("culsh_gsm_densify_tiled", nat.ptr(d.col_ptr), nat.ptr(d.col_rows), nat.ptr(d.col_vals), N, 0, M,
                 ld, w, nat.ptr(pan), nat.ptr(st), nat.stream_ptr())
        ev[1].record()
        nat.call("culsh_gsm_stats_tc", nat.ptr(pan), ld, w, 0, nat.ptr(g[0]), nat.ptr(g[1]), nat.ptr(g[2]),
                 nat.ptr(g[3]), nat.ptr(g[4]), nat.ptr(g[5]), nat.stream_ptr())
        ev[2].record()
        nat.call("culsh_gsm_count_select", nat.ptr(g[0]), nat.ptr(g[1]), nat.ptr(g[2]), nat.ptr(g[3]),
                 nat.ptr(g[4]), nat.ptr(g[5]), ld, N, 0, N,
                 K, 100.0, nat.ptr(entries), nat.stream_ptr())
        ev[3].record()
        torch.cuda.synchronize()
        t = [ev[i].elapsed_time(ev[i + 1]) / 1e3 for i in range(3)]
        print(json.dumps({"run": r, "densify_s": t[0], "stats_s": t[1], "select_s": t[2]}), flush=True)


if __name__ == "__main__":
    main()
