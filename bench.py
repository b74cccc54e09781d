#!/usr/bin/env python
"""DistAttention decode benchmark (BASELINE.json metric) -- one JSON line.

Default workload: BASELINE config 2 (batch 64 decode, LLaMA2-7B MHA 32x128,
ragged 1K-32K contexts, bf16 paged KV) on 1 B200. With --gpus N (launched by
torch.distributed.run, one process per GPU) the SAME workload is
sequence-sharded: every request's blocks are split into N contiguous shares
(config 5: the gManager-policy placement), each rank runs the MA kernel over its
share and K5 merges the (m, e, ma) partials locally, exchanges one record per
(row, q head) over NVLink and merges across ranks (strong scaling, total work
fixed).

A step = one decode step of one attention layer for the whole batch.
  value       tokens/s = B / t_step, inputs resident in HBM, device-timed with
              CUDA events over exactly --steps steps (max over ranks).
  e2e         the same through the C ABI with HOST q/out buffers: pinned H2D of
              q + plan, D2H of the output inside every step (wall clock).
  roofline    the MA kernel (K1 or K2, the dominant launch) timed alone with
              CUDA events on its stream; achieved = algorithmic bytes / duration;
              frac against the measured copy bandwidth, frac_nominal against
              the north_star's 8 TB/s.
  placement   per-rank KV bytes, the makespan bound they imply (max rank bytes
              at the measured peak) and the step's fraction of it (config 5 is
              placement-limited).
  cpu_baseline the reference's own multi_head_attention (oracle/_ref, compiled
              from the unmodified sources) on all host cores, bounded sample;
              single_thread_value = the same on 1 core (as shipped).
  model_tps   B / (n_layers * t_step), the reference's TPS = beta/(n T_layer)
              (perfmodel.cpp:120-130) for the workload's model depth.
--impl reference times only that CPU reference (rank 0) and prints its line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode-attention tokens/s and KV GB/s (% HBM roofline) at 1/2/4/8 B200 vs CPU"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", default="2", help="BASELINE config number (1..5)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU baseline budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0, help="0: same as --steps")
    ap.add_argument("--chunk-tokens", type=int, default=0)
    return ap.parse_args()


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        j = json.load(open(p))
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i in range(4) if r[i].lower().startswith("active")})
        loaded = [c for c, _, _ in rows]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(m for _, m, _ in rows),
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------- CPU side

def cpu_reference_sample(w, budget_s: float, reps_fixed: int = 0, threads: int = 0):
    """Time the reference CPU path on a bounded sample of the workload.

    The sample is the first requests of the batch (all their heads), generated
    with the same counter-hash values the GPU consumes (bf16-rounded, then
    widened to fp64: the reference API is fp64-only). Generation is outside
    the timed region. Returns the full-workload-equivalent tokens/s and info.
    """
    import ctypes
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np

    import oracle

    threads = threads or os.cpu_count() or 1
    # sample: leading requests, <= 96K context tokens (<= ~6 GB of fp64 K/V at 32 heads)
    cap = max(4096, int(96 * 1024 * 32 // max(w.hkv, 1)))
    idx, tot = [], 0
    for r, L in enumerate(w.lens):
        if idx and tot + L > cap:
            break
        idx.append(r)
        tot += L
    if tot > cap:  # one request longer than the cap: take its leading tokens
        lens = [cap]
    else:
        lens = [w.lens[r] for r in idx]
    B = len(lens)
    kv = [None] * (B * w.hkv)

    def gen(i):
        r, h = divmod(i, w.hkv)
        kv[i] = oracle.synth_kv(w.seed, r, h, 0, lens[r], w.d, w.amp_k, w.amp_v, w.dtype)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(gen, range(B * w.hkv)))
    q = np.ascontiguousarray(np.stack([np.stack([oracle.synth_q(w.seed, r, h, w.d, 1.0, w.dtype)
                                                 for h in range(w.hq)]) for r in range(B)]))
    ptrs = (ctypes.c_void_p * (2 * B * w.hkv))()
    for i, (k, v) in enumerate(kv):
        ptrs[2 * i] = k.ctypes.data
        ptrs[2 * i + 1] = v.ctypes.data
    L = np.ascontiguousarray(lens, dtype=np.int64)
    out = np.zeros((B, w.hq, w.d))
    sec = np.zeros(1)
    kind = "reference" if oracle.ref_available() else "port"
    seg = max(w.lens[0] // w.rblocks, 1) if w.rblocks > 1 else 0

    def one():
        if kind == "reference":
            R = oracle.ref()
            rc = R.ref_decode_timed(B, L.ctypes.data, ptrs, q.ctypes.data, w.hq, w.hkv, w.d, 0.0, seg,
                                    threads, out.ctypes.data, sec.ctypes.data)
            assert rc == 0, R.ref_last_error()
            return float(sec[0])
        t0 = time.perf_counter()
        oracle.decode_batch(w.seed, lens, w.hq, w.hkv, w.d, dtype=w.dtype, amp_k=w.amp_k, amp_v=w.amp_v,
                            seg_tokens=seg, threads=threads)
        return time.perf_counter() - t0

    times = []
    t_start = time.perf_counter()
    while True:
        times.append(one())
        if reps_fixed and len(times) >= reps_fixed:
            break
        if not reps_fixed and time.perf_counter() - t_start >= budget_s:
            break
    per = statistics.median(times)
    sample_tok_heads = sum(lens) * w.hkv
    full_tok_heads = w.total_tokens * w.hkv
    full_t = per * full_tok_heads / sample_tok_heads
    info = {
        "kind": kind, "cores": threads, "reps": len(times), "sample_seconds_per_rep": per,
        "sample": (f"{B} leading request(s) of the batch, {sum(lens)} context tokens x {w.hkv} kv heads "
                   f"({sum(lens) * w.hkv * w.d * 16 / 1e9:.2f} GB fp64 K+V), kvsched::attn::multi_head_attention "
                   f"per (request, kv head) on {threads} threads; scaled to the full workload by K/V tokens "
                   f"({full_tok_heads / sample_tok_heads:.1f}x)"),
        "kv_gbs_fp64": sample_tok_heads * w.d * 16 / per / 1e9,
    }
    return w.batch / full_t, info


def run_reference_arm(args, rank, ws):
    from paper_2401_02669_b200 import workloads
    if rank != 0:
        return
    w = workloads.config(args.config)
    for _ in range(max(args.warmup, 0)):
        pass  # warm-up reps are counted inside cpu_reference_sample via reps_fixed below
    total_reps = max(args.steps, 1) + max(args.warmup, 0)
    # each step: one bounded-sample rep; keep the whole run to a few minutes
    value, info = cpu_reference_sample(w, budget_s=0.0, reps_fixed=min(total_reps, 60))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * w.batch / value,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (counter-hash K/V/q, bf16-rounded values widened to fp64)",
        "config": {"workload": w.name, "batch": w.batch, "total_kv_tokens": w.total_tokens,
                   "heads": [w.hq, w.hkv], "head_dim": w.d, **w.meta},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": info["cores"], "kind": info["kind"],
                         "sample": info["sample"] + f"; {info['reps']} reps (steps capped at 60)"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "kv_gbs_fp64": info["kv_gbs_fp64"],
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU side

def run_b200_arm(args, rank, ws, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2401_02669_b200 as pb
    from paper_2401_02669_b200 import workloads

    w = workloads.config(args.config)
    torch.cuda.set_device(local)
    page = w.page_tokens
    shares = workloads.rank_shares(w, ws)[rank]
    pages = sum(-(-rr.tokens // page) for rr in shares) + 16
    max_pps = max(-(-rr.tokens // page) for rr in shares) + 2
    st = pb.Store(w.d, w.hq, w.hkv, w.dtype, page, pages, max_seqs=w.batch + 4,
                  max_pages_per_seq=max(max_pps, 1), device=local)
    stream = torch.cuda.Stream(device=local)
    st.set_stream(stream.cuda_stream)
    ranges = []
    for rr in shares:
        seq = st.seq_create(rr.tokens)
        st.fill_synthetic(seq, w.seed, rr.request, rr.tok_begin, w.amp_k, w.amp_v)
        if rr.tokens == 0:
            ranges.append(pb.Range(seq, rr.request, 0, 0))
            continue
        nb = w.rblocks if ws == 1 else 1
        cuts = [rr.tokens * i // nb for i in range(nb + 1)]
        for a, b in zip(cuts[:-1], cuts[1:]):
            ranges.append(pb.Range(seq, rr.request, a, b))
    ranges = pb.range_array(ranges)  # packed once, reused by every step
    tdt = {0: torch.bfloat16, 1: torch.float32}[w.dtype]
    q = torch.empty(w.batch, w.hq, st.padded_dim, dtype=tdt, device=f"cuda:{local}")
    st.q_fill_synthetic(q, w.batch, w.seed, 0, 1.0)
    out = torch.empty_like(q)
    if ws > 1:
        uid = [pb.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        st.comm_init(uid[0], rank, ws)

    def step(mem=pb.MEM_DEVICE, qq=q, oo=out):
        if ws > 1:
            st.decode_sharded(ranges, w.batch, qq, oo, mem=mem, chunk_tokens=args.chunk_tokens)
        else:
            st.decode(ranges, w.batch, qq, oo, mem=mem, chunk_tokens=args.chunk_tokens)

    def barrier():
        if ws > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    torch.cuda.synchronize()
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    barrier()

    # ---- region A: the headline, inputs resident in HBM ----
    sampler = ClockSampler(local)
    sampler.start()
    pb.launch_count(reset=True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = pb.launch_count()
    clocks = sampler.stop()
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    ms_step = ms_total / args.steps

    # ---- region B: the MA kernel (K1/K2) alone, CUDA events around each launch on its stream ----
    st.stats(reset=True)
    st.set_timing(True)
    kb = max(10, min(args.steps, 100))
    for _ in range(kb):
        step()
    torch.cuda.synchronize()
    s = st.stats(reset=True)
    st.set_timing(False)
    ma_ms = s.ma_ms / max(s.ma_timed, 1)
    merge_ms = s.merge_ms / max(s.merge_timed, 1)
    comm_ms = s.comm_ms / max(s.comm_timed, 1) if s.comm_timed else None
    rank_times = [[ma_ms, comm_ms]]
    if ws > 1:
        rank_times = [None] * ws
        dist.all_gather_object(rank_times, [ma_ms, comm_ms])
    kernel_name = {1: "ma_decode_kernel (K1, CUDA cores)", 2: "gqa_tc_kernel (K2, tcgen05)"}.get(s.last_kernel, "?")

    # ---- region C: end to end through the C ABI with host buffers ----
    qh = q.cpu().pin_memory()
    oh = torch.empty_like(qh).pin_memory()
    ke = args.e2e_steps or args.steps
    for _ in range(3):
        step(pb.MEM_HOST, qh, oh)
    barrier()
    t0 = time.perf_counter()
    for _ in range(ke):
        step(pb.MEM_HOST, qh, oh)
    t_e2e = max_over_ranks(time.perf_counter() - t0) / ke
    plan_bytes = st.stats().last_plan_bytes
    qbytes = qh.numel() * qh.element_size()

    # parity spot check of the benchmarked output (one request, all heads) is
    # done by tests/; here only a sanity check that the output is finite
    assert torch.isfinite(out.float()).all().item()

    if rank != 0:
        return
    peak, peak_src = measured_peak()
    # per-rank algorithmic bytes of one MA launch (rank 0's share)
    kv_rank = sum(2 * w.hkv * w.d * rr.tokens * w.elem_bytes for rr in shares)
    kv_ranks = [sum(2 * w.hkv * w.d * rr.tokens * w.elem_bytes for rr in rs) for rs in workloads.rank_shares(w, ws)]
    bound_ms = max(kv_ranks) / (peak * 1e9) * 1e3
    alg_rank = kv_rank + w.batch * w.hq * w.d * 2 * w.elem_bytes
    achieved = alg_rank / (ma_ms * 1e-3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(f"cfg{args.config}_n{ws}")
        except Exception:
            traffic = None
    value = w.batch / (ms_step * 1e-3)
    line = {
        "impl": "b200", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16" if w.dtype == 0 else "f32",
        "data": "synthetic (counter-hash K/V/q generated on device, seeded; no checkpoints)",
        "config": {"workload": w.name, "batch": w.batch, "total_kv_tokens": w.total_tokens,
                   "heads": [w.hq, w.hkv], "head_dim": w.d, "page_tokens": page,
                   "kv_bytes_per_step": w.kv_bytes(), "parallelism": f"sequence-shard x{ws}",
                   "l2": "inputs larger than L2 (KV >> 126 MB), no flush" if w.kv_bytes() > 4 * 126e6
                   else "KV near L2 size: steps re-read it (L2-warm)",
                   "chunk_tokens": s.last_chunk_tokens, "ma_items": s.last_items, "ma_grid": s.ma_grid, **w.meta},
        "kv_gbs": w.kv_bytes() / (ms_step * 1e-3) / 1e9,
        "model_tps": {"value": value / w.n_layers, "n_layers": w.n_layers},
        "rank0_kv_bytes": kv_rank,
        "placement": {"per_rank_kv_bytes": kv_ranks, "bound_ms": bound_ms, "frac": bound_ms / ms_step,
                      "aggregate_frac": w.kv_bytes() / (ws * peak * 1e9) / (ms_step * 1e-3)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "frac_nominal": achieved / 8000.0,
                     "kernel": kernel_name, "kernel_ms": ma_ms, "merge_ms": merge_ms, "exchange_ms": comm_ms,
                     "alg_bytes_per_launch": alg_rank, "peak_source": peak_src},
        "e2e": {"value": w.batch / t_e2e, "unit": "tokens/s", "h2d_bytes_per_step": qbytes + plan_bytes,
                "d2h_bytes_per_step": qbytes, "ms_per_step": t_e2e * 1e3},
        "gpu_launches": launches,
        "per_rank_ms": {"ma": [round(t[0], 4) for t in rank_times],
                        "exchange": [None if t[1] is None else round(t[1], 4) for t in rank_times]},
        "clocks": clocks,
    }
    if ws == 1 and not args.no_cpu_baseline:
        cv, info = cpu_reference_sample(w, args.cpu_seconds)
        c1, info1 = cpu_reference_sample(w, min(args.cpu_seconds, 4.0), threads=1)
        line["cpu_baseline"] = {"value": cv, "unit": "tokens/s", "cores": info["cores"], "kind": info["kind"],
                                "sample": info["sample"] + f"; {info['reps']} reps",
                                "single_thread_value": c1, "single_thread_reps": info1["reps"],
                                "kv_gbs_fp64": info["kv_gbs_fp64"], "single_thread_kv_gbs_fp64": info1["kv_gbs_fp64"]}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, ws)
        return
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    try:
        run_b200_arm(args, rank, ws, local)
    finally:
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
