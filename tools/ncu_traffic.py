#!/usr/bin/env python
"""Record the DRAM traffic of the dominant kernel from an ncu --set full
report into profiles/ncu_traffic.json, stamped with the library build it was
measured on (sha256 of paper_2401_02669_b200/_lib/libdattn.so) and the git
head. bench.py reports ``roofline.traffic`` only when the stamp matches the
library it runs (compared by the hash of its device code, which survives a
rebuild of the same sources), so a capture of other kernel code can never feed
a bench line.

    python tools/ncu_traffic.py KEY REPORT.ncu-rep [--kernel REGEX]

KEY is the bench config key, e.g. cfg2_n1 (config 2 on one GPU). With several
launches in the report, the matching launches are averaged.
"""
from __future__ import annotations

import argparse
import csv
import hashlib
import io
import json
import os
import re
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_traffic.json")
LIB = os.path.join(ROOT, "paper_2401_02669_b200", "_lib", "libdattn.so")
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}  # bytes; durations in ns


def launches(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True, capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        yield {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def num(cell) -> float:
    v, u = cell
    return float(v.replace(",", "")) * UNIT.get(u, 1)


sys.path.insert(0, ROOT)
from bench import kernel_code_sha256  # noqa: E402


def module_of(kernel: str) -> str:
    """The cubin (source module) holding a kernel: K2 in dattn_gqa_tc, the
    CUDA-core kernels in dattn_kernels. The stamp then covers that module's
    device code only, so a change to another module leaves it valid."""
    return "dattn_gqa_tc" if "gqa_tc_kernel" in kernel else "dattn_kernels"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("key")
    ap.add_argument("report")
    ap.add_argument("--kernel", default="gqa_tc_kernel|ma_decode_kernel")
    a = ap.parse_args()
    rx = re.compile(a.kernel)
    tr, dur, names = [], [], set()
    for ln in launches(a.report):
        name = ln.get("Kernel Name", ("", ""))[0]
        if not rx.search(name):
            continue
        names.add(name)
        tr.append(num(ln["dram__bytes_read.sum"]) + num(ln["dram__bytes_write.sum"]))
        if "gpu__time_duration.sum" in ln:
            dur.append(num(ln["gpu__time_duration.sum"]))
    if not tr:
        raise SystemExit(f"no launch of {a.kernel!r} in {a.report}")
    head = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"], capture_output=True,
                          text=True).stdout.strip()
    j = json.load(open(OUT)) if os.path.exists(OUT) else {}
    j = {k: v for k, v in j.items() if isinstance(v, dict)}  # drop unstamped entries
    j[a.key] = {"traffic": sum(tr) / len(tr), "launches": len(tr), "kernel": sorted(names)[0],
                "duration_ns": sum(dur) / len(dur) if dur else None,
                "lib_sha256": hashlib.sha256(open(LIB, "rb").read()).hexdigest(),
                "code_module": module_of(sorted(names)[0]),
                "code_sha256": kernel_code_sha256(LIB, module_of(sorted(names)[0])),
                "git_head": head, "report": os.path.basename(a.report),
                "recorded": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
                "metric": "dram__bytes_read.sum + dram__bytes_write.sum per launch (ncu --set full)"}
    with open(OUT, "w") as f:
        json.dump(j, f, indent=1, sort_keys=True)
        f.write("\n")
    print(a.key, j[a.key])


if __name__ == "__main__":
    main()
