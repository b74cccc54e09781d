#!/usr/bin/env python
"""Summarise an ncu --set full report of one kernel launch as a markdown table
(the rows profiles/r1_ncu_summary.md quotes) plus the top stall sites.

    python tools/ncu_summary.py gpurun_out/r1c_k2_cfg2.ncu-rep [--alg-bytes B]

--alg-bytes: algorithmic bytes per launch to compare with DRAM
traffic (traffic well above it means re-reads).
"""
from __future__ import annotations

import argparse
import csv
import io
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes.sum.per_second", "DRAM throughput"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("gpc__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers"),
]

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def ncu_csv(rep: str, page: str) -> list[list[str]]:
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], check=True, capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--alg-bytes", type=float, default=0.0)
    ap.add_argument("--top", type=int, default=8)
    a = ap.parse_args()
    rows = ncu_csv(a.report, "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    print("| metric | value |\n|---|---|")
    traffic = 0.0
    for key, label in METRICS:
        if key in hdr:
            i = hdr.index(key)
            print(f"| {label} (`{key}`) | {vals[i]} {units[i]} |")
            if key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                traffic += float(vals[i].replace(",", "")) * UNIT.get(units[i], 1)
    if traffic:
        print(f"| DRAM traffic per launch | {traffic:.6g} B |")
        if a.alg_bytes:
            print(f"| traffic / algorithmic bytes | {traffic / a.alg_bytes:.4f} |")
    src = ncu_csv(a.report, "source")
    h = src[1]
    data = src[2:]
    si, ti = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    tot = sum(float(r[si] or 0) for r in data) or 1.0
    print(f"\nTop stall sites ({int(tot)} samples):\n")
    for r in sorted(data, key=lambda r: -float(r[si] or 0))[: a.top]:
        print(f"* {100 * float(r[si]) / tot:5.1f} %  `{r[ti].strip()[:80]}`")


if __name__ == "__main__":
    main()
