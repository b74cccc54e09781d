"""Summarise bench.py JSON lines (one file per run) into a markdown table.

usage: python tools/scaling_table.py gpurun_out/s_n{1,2,4}_cfg*.log
"""
import json
import re
import sys
from collections import defaultdict


def load(path):
    for line in open(path):
        line = line.strip()
        if line.startswith("{"):
            return json.loads(line)
    return None


def main(paths):
    rows = defaultdict(dict)
    for p in paths:
        j = load(p)
        if not j:
            continue
        m = re.search(r"cfg(\d)", p)
        rows[m.group(1) if m else "?"][j["n_gpus"]] = j
    print("| config | GPUs | tokens/s | ms/step | KV TB/s (aggregate) | speed-up vs 1 GPU | MA kernel ms per rank | exchange ms per rank | clocks |")
    print("|---|---|---|---|---|---|---|---|---|")
    for cfg in sorted(rows):
        base = rows[cfg].get(1)
        for n in sorted(rows[cfg]):
            j = rows[cfg][n]
            sp = j["value"] / base["value"] if base else float("nan")
            pr = j.get("per_rank_ms", {})
            ma = ", ".join(f"{x:.3f}" for x in pr.get("ma", []))
            ex = ", ".join("-" if x is None else f"{x:.3f}" for x in pr.get("exchange", []))
            clk = j.get("clocks", {})
            print(f"| {cfg} | {n} | {j['value']:.0f} | {j['ms_per_step']:.4f} | {j['kv_gbs'] / 1000:.2f} | "
                  f"{sp:.2f}x | {ma} | {ex} | {clk.get('sm_mhz')} MHz {','.join(clk.get('reasons', []))} |")


if __name__ == "__main__":
    main(sys.argv[1:])
