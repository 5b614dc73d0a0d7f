"""Summarise gpurun_out/b_quick.log (bench line) and gpurun_out/ncu_quick.csv."""
import csv
import json
import os
import sys

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
b = os.path.join(out, "b_quick.log")
if os.path.exists(b):
    lines = [x for x in open(b) if x.startswith("{")]
    if lines:
        d = json.loads(lines[-1])
        print("ms/epoch %.3f  value %.3fe9  e2e %.3fe9  h2d %.0f MB  rmse %.5f  frac %.3f  lsh %.3fs" % (
            d["ms_per_step"], d["value"] / 1e9, d["e2e"]["value"] / 1e9,
            d["e2e"]["h2d_bytes_per_step"] / 1e6, d["train_rmse_running"], d["roofline"]["frac"],
            d["lsh_build_s"]))
    else:
        print(open(b).read()[-3000:])
c = os.path.join(out, "ncu_quick.csv")
if os.path.exists(c):
    rows = list(csv.reader(open(c)))
    hs = [r for r in rows if r and r[0] == "ID"]
    if hs:
        h = hs[0]
        for r in rows:
            if r and r[0] == "0" and len(r) == len(h):
                print("  ", r[h.index("Metric Name")], r[h.index("Metric Value")])
