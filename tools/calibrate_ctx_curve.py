#!/usr/bin/env python
"""Measure the B200 attention rate g(S) for the reference's perf model
(SURVEY.md §8f row 4).

The reference models one decode layer as
    T(beta, S) = W(beta)/f(beta) + S_total * attn_work_per_ctx_token / g(S_total)
(proj/include/kvsched/perfmodel.hpp:6-14, layer_time perfmodel.cpp:105-113) and
ships a synthetic constant g (default_ctx_curve, perfmodel.cpp:58-60;
default_cluster_config config.cpp:83-84). This tool measures the real curve on
one B200 through the product decode path: for each total context S, a batch of
equal-length requests (LLaMA-7B MHA 32x128, bf16 paged KV) is decoded and
timed with CUDA events (median of --steps steps), and
    g(S) = S / t_attn(S)      [context tokens per second per layer]
so the curve plugs into the reference with attn_work_per_ctx_token = 1 (f must
then be in the same units: seconds per layer of non-attention work).

Writes the samples and the ctx_rate_curve as JSON (default
profiles/r1_ctx_rate_curve.json). tests/test_ctx_curve.py feeds the committed
curve through the reference's own config parser and layer_time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

POINTS = [4096, 16384, 65536, 262144, 1048576, 4194304]


def measure(S: int, steps: int, warmup: int):
    import torch

    import paper_2401_02669_b200 as pb

    hq = hkv = 32
    d, page = 128, 16
    batch = max(1, min(64, S // 4096))
    lens = [S // batch + (1 if i < S % batch else 0) for i in range(batch)]
    pages = sum(-(-L // page) for L in lens) + 16
    st = pb.Store(d, hq, hkv, pb.BF16, page, pages, max_seqs=batch + 2,
                  max_pages_per_seq=max(-(-L // page) for L in lens) + 2)
    stream = torch.cuda.Stream()
    st.set_stream(stream.cuda_stream)
    ranges = []
    for r, L in enumerate(lens):
        seq = st.seq_create(L)
        st.fill_synthetic(seq, 20261018, r, 0, 1.0, 2.0)
        ranges.append(pb.Range(seq, r, 0, L))
    q = torch.empty(batch, hq, st.padded_dim, dtype=torch.bfloat16, device="cuda")
    st.q_fill_synthetic(q, batch, 20261018)
    out = torch.empty_like(q)
    for _ in range(warmup):
        st.decode(ranges, batch, q, out)
    torch.cuda.synchronize()
    ms = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st.decode(ranges, batch, q, out)
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    st.close()
    t = statistics.median(ms)
    return {"S": S, "batch": batch, "ms": t, "rate": S / (t * 1e-3),
            "kv_gbs": S * 2 * hkv * d * 2 / (t * 1e-3) / 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_ctx_rate_curve.json"))
    a = ap.parse_args()
    import torch
    samples = [measure(S, a.steps, a.warmup) for S in POINTS]
    doc = {
        "what": "B200 attention rate g(S) for kvsched::perf (ctx_rate_curve), measured through dattn_decode",
        "device": torch.cuda.get_device_name(0),
        "model": {"name": "LLaMA-7B attention layer", "num_q_heads": 32, "num_kv_heads": 32, "head_dim": 128,
                  "dtype": "bf16", "page_tokens": 16, "n_layers": 32,
                  "kv_bytes_per_token_all_layers": 2 * 32 * 128 * 2 * 32},
        "units": "x = total context tokens on the instance; rate = context tokens per second per layer "
                 "(attn_work_per_ctx_token = 1)",
        "timing": f"CUDA events around one dattn_decode, median of {a.steps} after {a.warmup} warm-up",
        "samples": samples,
        "ctx_rate_curve": [[s["S"], s["rate"]] for s in samples],
    }
    with open(a.out, "w") as f:
        json.dump(doc, f, indent=1)
    for s in samples:
        print(f"S={s['S']:>8} batch={s['batch']:>3} {s['ms']:.4f} ms  g={s['rate']:.3e} tok/s  "
              f"{s['kv_gbs']:.0f} GB/s")


if __name__ == "__main__":
    main()
