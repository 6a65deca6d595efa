#!/usr/bin/env python3
"""Summarise ncu outputs into committed profile notes.

  tools/ncu_summary.py launches <launches.csv>          per-kernel totals of a
        `ncu --metrics gpu__time_duration.sum --csv` launch list (markdown table)
  tools/ncu_summary.py full <report.ncu-rep> [...]      key metrics of `--set full`
        captures (markdown table), incl. dram bytes per launch
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "Duration", "Elapsed Cycles", "SM Frequency", "Grid Size", "Block Size", "Registers Per Thread",
    "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "Achieved Occupancy",
    "Issue Slots Busy", "Executed Ipc Active", "Executed Instructions", "No Eligible",
    "Active Warps Per Scheduler", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
    "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64.sum",
       "smsp__inst_executed_pipe_fp64.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed.sum", "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]


def launches(path: str) -> None:
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi = h.index("Kernel Name"), h.index("Metric Value")
    per = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > mi:
            per[r[ki].split("(")[0].replace("(anonymous namespace)::", "")].append(float(r[mi].replace(",", "")))
    tot = sum(sum(v) for v in per.values())
    print(f"| kernel | launches | total ms | share | avg us |\n|---|---|---|---|---|")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k}` | {len(v)} | {sum(v) / 1e6:.3f} | {100 * sum(v) / tot:.1f}% | {sum(v) / len(v) / 1e3:.2f} |")
    print(f"| **all** | {sum(len(v) for v in per.values())} | {tot / 1e6:.3f} | 100% | |")


def full(paths: list[str]) -> None:
    cols = []
    for p in paths:
        det = subprocess.run(["ncu", "-i", p, "--page", "details", "--csv"], capture_output=True, text=True).stdout
        raw = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        d = {}
        name = ""
        for row in csv.DictReader(io.StringIO(det)):
            name = row.get("Kernel Name", name)
            if row.get("Metric Name") in KEYS and row["Metric Name"] not in d:
                d[row["Metric Name"]] = f"{row['Metric Value']} {row['Metric Unit']}".strip()
        rr = list(csv.reader(io.StringIO(raw)))
        if len(rr) >= 3:
            h, units, vals = rr[0], rr[1], rr[2]
            for k in RAW:
                if k in h:
                    i = h.index(k)
                    d[k] = f"{vals[i]} {units[i]}".strip()
        cols.append((p.split("/")[-1], name.split("(")[0].replace("(anonymous namespace)::", ""), d))
    print("| metric | " + " | ".join(f"{c[0]} (`{c[1]}`)" for c in cols) + " |")
    print("|---" * (len(cols) + 1) + "|")
    for k in KEYS + RAW:
        if any(k in c[2] for c in cols):
            print(f"| {k} | " + " | ".join(c[2].get(k, "") for c in cols) + " |")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2:])
