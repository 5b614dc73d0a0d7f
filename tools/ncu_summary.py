"""Summarise ncu captures (run here, no GPU needed) into profiles/.

  python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r1_launches.md
  python tools/ncu_summary.py full gpurun_out/prof_hogwild.ncu-rep profiles/r1_ncu_hogwild.md \
         [--roofline-json profiles/ncu_roofline_c3.json --lib paper_2111_11682_b200/_lib/libculsh.so]
  python tools/ncu_summary.py sass paper_2111_11682_b200/_lib/libculsh.so profiles/r2_sass.md \
         hogwild_kernel hash_count_kernel ...

--roofline-json writes what bench.py's `roofline.measured` quotes: the kernel's DRAM bytes
and unit utilisations from this capture, with the build identity of the tree it profiled
(bench.build_sha256: CUDA sources + header + Makefile; bench.py marks the numbers
`same_build` only when its own tree has that identity).  Run it on the tree that was
profiled, before changing any CUDA source.
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
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_l1tex2xbar_write_bytes.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
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


def _num(d, k):
    v, unit = d[k]
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1.0)


def _build_sha256() -> str:
    """bench.py's build identity (sources + header + Makefile of the profiled tree)."""
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    return bench.build_sha256()


def _opt(d, key):
    """A metric that older captures may lack (None then)."""
    return _num(d, key) if key in d else None


def full(rep: str, dst: str, traffic_json: str | None = None, lib: str | None = None) -> None:
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
                ms = _to_ms(_num(d, "gpu__time_duration.sum") / 1.0, d["gpu__time_duration.sum"][1])
                rec = {"kernel": name.split("(")[0], "source": rep.split("/")[-1],
                       "ncu": "--set full --clock-control none (cold-ish, one launch)",
                       "duration_ms": ms, "dram_bytes_per_launch": tot,
                       "dram_read_bytes": _num(d, "dram__bytes_read.sum"),
                       "dram_write_bytes": _num(d, "dram__bytes_write.sum"),
                       "dram_gbs": tot / (ms * 1e-3) / 1e9,
                       "l2_hit_pct": _num(d, "lts__t_sector_hit_rate.pct"),
                       "l2_throughput_pct": _num(d, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                       "l1tex_throughput_pct": _num(d, "l1tex__throughput.avg.pct_of_peak_sustained_active"),
                       "sm_throughput_pct": _num(d, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                       "issue_ipc": (_num(d, "smsp__inst_executed.avg.per_cycle_active")
                                     if "smsp__inst_executed.avg.per_cycle_active" in d else None),
                       "warps_active_pct": _num(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
                       "issue_active_pct": _opt(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                       # L1 -> L2 request interface (RED data + read requests) and its write bytes
                       "l1_to_l2_req_pct": _opt(d, "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                       "l1_to_l2_write_bytes_pct": _opt(d, "l1tex__m_l1tex2xbar_write_bytes.sum.pct_of_peak_sustained_elapsed"),
                       "shared_wavefronts_pct": _opt(d, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
                       "registers": _num(d, "launch__registers_per_thread"),
                       "build_sha256": _build_sha256() if lib else None}
                json.dump(rec, open(traffic_json, "w"), indent=1)
        except (KeyError, ValueError):
            pass
    hdr = f"# ncu --set full summary ({rep})\n\n--clock-control none; one launch per kernel; numbers under the profiler are not bench values.\n\n"
    open(dst, "w").write(hdr + out.getvalue())
    print(hdr + out.getvalue())


def sass(lib: str, dst: str, kernels) -> None:
    """Per-kernel SASS opcode histogram (cuobjdump -sass): the instruction mix behind the
    ncu numbers, and proof of which units a kernel uses (UTCIMMA / UTMALDG = tcgen05 MMA /
    TMA; FFMA2 / FMUL2 = paired fp32; REDG / REDUX = reductions; LDGSTS = cp.async)."""
    import re
    txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    funcs = re.split(r"\n\s+Function : ", txt)
    out = io.StringIO()
    out.write(f"# SASS opcode mix per hot kernel (`cuobjdump -sass {lib.split('/')[-1]}`, sm_100a)\n\n")
    for k in kernels:
        out.write(f"## kernels matching `{k}`\n\n")
        for f in funcs[1:]:
            fname = f.split("\n", 1)[0].strip()
            if k not in fname:
                continue
            ops = defaultdict(int)
            for line in f.split("\n"):
                m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
                if m:
                    ops[m.group(2)] += 1
            tot = sum(ops.values())
            top = sorted(ops.items(), key=lambda x: -x[1])
            out.write(f"`{fname[:160]}` -- {tot} instructions\n\n")
            out.write(", ".join(f"{o} {n}" for o, n in top[:40]) + "\n\n")
            keyfam = ("UTCIMMA", "UTCHMMA", "UTCBAR", "UBLKCP", "UTMALDG", "LDTM", "LDGSTS", "REDG", "REDUX",
                      "FFMA2", "FMUL2", "SHFL", "VOTE", "POPC", "ATOMS", "DADD", "DFMA", "DMUL")
            fam = {k: sum(n for o, n in ops.items() if o.startswith(k)) for k in keyfam}
            out.write("key families: " + ", ".join(f"{k} {v}" for k, v in fam.items() if v) + "\n\n")
    open(dst, "w").write(out.getvalue())
    print(out.getvalue()[:4000])


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    elif mode == "sass":
        sass(sys.argv[2], sys.argv[3], sys.argv[4:])
    else:
        tj = lib = None
        for flag in ("--traffic-json", "--roofline-json"):
            if flag in sys.argv:
                tj = sys.argv[sys.argv.index(flag) + 1]
        if "--lib" in sys.argv:
            lib = sys.argv[sys.argv.index("--lib") + 1]
        full(sys.argv[2], sys.argv[3], tj, lib)
