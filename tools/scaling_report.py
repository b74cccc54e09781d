"""Per-run detail table of bench.py JSON lines (one file per run): parity,
decode-loop parity, e2e, placement bound, roofline fraction, the migration
sweep and the overflow-borrowing loop -- the second table of
profiles/r2_scaling.md (the first comes from tools/scaling_table.py).

usage: python tools/scaling_report.py profiles/r2_scaling_logs/n*_cfg*.json
"""
import json
import sys


def row(d):
    n = d["n_gpus"]
    cfg = d["config"]["workload"][3]
    mig = d.get("migration") or {}
    sweep = " / ".join(f"{e['pages_per_step']}:{100 * e['slowdown_vs_no_migration']:+.1f}%"
                       for e in mig.get("sweep", []) if e["pages_per_step"])
    o = d.get("overflow_decode_loop") or {}
    ov = (f"{o['ms_per_step']:.3f} ms, {o['borrowed_blocks']} blocks, "
          f"{'pass' if (o.get('parity') or {}).get('pass') else 'n/a'}") if o else "-"
    par, loop = d["parity"], d["parity_decode_loop"]
    e = d["e2e"]
    return (cfg, n, f"| {cfg} | {n} | {par['max_norm_err']:.1e} {'pass' if par['pass'] else 'FAIL'} | "
                    f"{'pass' if loop['pass'] else 'FAIL'} | {e['value']:.0f} (median step "
                    f"{e['step_ms_rank0']['median']:.3f} ms) | {d['e2e_static']['value']:.0f} | "
                    f"{d['placement']['bound_ms']:.3f} | {d['placement']['frac']:.2f} | "
                    f"{d['roofline']['frac']:.3f} | {sweep or '-'} | {ov} |")


def main(paths):
    rows = []
    for p in paths:
        with open(p) as f:
            line = next((x for x in f if x.strip().startswith("{")), None)
        if line:
            rows.append(row(json.loads(line)))
    print("| config | GPUs | parity (max err) | loop parity | e2e tok/s | e2e static tok/s | "
          "placement bound ms | frac | roofline frac | migration m:slowdown | overflow loop |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for _, _, text in sorted(rows, key=lambda r: (r[0], r[1])):
        print(text)


if __name__ == "__main__":
    main(sys.argv[1:])
