"""Summarise ncu captures (run here, no GPU needed) into profiles/.

  python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r1_launches.md
  python tools/ncu_summary.py full gpurun_out/prof_hogwild.ncu-rep profiles/r1_ncu_hogwild.md \
         [--traffic-json profiles/ncu_traffic_c3.json]
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "lts__t_bytes.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed.sum",
    "smsp__inst_executed.avg.per_cycle_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_per_inst_issued.ratio",
]


def _to_ms(v: float, unit: str) -> float:
    return {"nsecond": v / 1e6, "ns": v / 1e6, "usecond": v / 1e3, "us": v / 1e3,
            "msecond": v, "ms": v, "second": v * 1e3, "s": v * 1e3}.get(unit, v / 1e6)


def launches(src: str, dst: str) -> None:
    rows = list(csv.reader(open(src)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += _to_ms(float(r[vi].replace(",", "")), r[ui])
    tot = sum(t for _, t in agg.values())
    out = io.StringIO()
    out.write(f"# Launch list (ncu gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n\n")
    out.write(f"source: `{src}`; compare SHARES, not absolutes.\n\n")
    out.write("| kernel | launches | total ms | ms/launch | share |\n|---|---:|---:|---:|---:|\n")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.write(f"| `{k}` | {n} | {t:.3f} | {t / n:.3f} | {100 * t / tot:.1f}% |\n")
    out.write(f"\ntotal {tot:.3f} ms over {sum(n for n, _ in agg.values())} launches\n")
    open(dst, "w").write(out.getvalue())
    print(out.getvalue())


def full(rep: str, dst: str, traffic_json: str | None = None) -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    out = io.StringIO()
    summaries = []
    for v in rows[2:]:
        name = v[h.index("Kernel Name")]
        d = {}
        for k in KEYS:
            for i, n in enumerate(h):
                if n == k:
                    d[k] = (v[i], u[i])
        summaries.append((name, d))
        out.write(f"## `{name[:140]}`\n\n| metric | value | unit |\n|---|---:|---|\n")
        for k, (val, unit) in d.items():
            out.write(f"| {k} | {val} | {unit} |\n")
        try:
            rd = float(d["dram__bytes_read.sum"][0].replace(",", ""))
            wr = float(d["dram__bytes_write.sum"][0].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = rd * scale[d["dram__bytes_read.sum"][1]] + wr * scale[d["dram__bytes_write.sum"][1]]
            out.write(f"\nDRAM traffic per launch: {tot / 1e9:.3f} GB\n\n")
            if traffic_json:
                json.dump({"kernel": name.split("(")[0], "dram_bytes_per_launch": tot, "source": rep},
                          open(traffic_json, "w"), indent=1)
        except (KeyError, ValueError):
            pass
    hdr = f"# ncu --set full summary ({rep})\n\n--clock-control none; one launch per kernel; numbers under the profiler are not bench values.\n\n"
    open(dst, "w").write(hdr + out.getvalue())
    print(hdr + out.getvalue())


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        tj = None
        if "--traffic-json" in sys.argv:
            tj = sys.argv[sys.argv.index("--traffic-json") + 1]
        full(sys.argv[2], sys.argv[3], tj)
