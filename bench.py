#!/usr/bin/env python
"""DistAttention decode benchmark (BASELINE.json metric) -- one JSON line.

Default workload: BASELINE config 2 (batch 64 decode, LLaMA2-7B MHA 32x128,
ragged 1K-32K contexts, bf16 paged KV) on 1 B200. ``--gpus N`` runs the SAME
workload on N GPUs of this box, one process per GPU: launched by
torch.distributed.run (the driver's way), or, when WORLD_SIZE is unset,
re-executed by this script under torch.distributed.run itself. Every request's
blocks are sequence-sharded (configs 1-4: equal block-aligned shares; config 5:
the reference control plane's gManager placement, tests/golden/
cfg5_placement.json); each rank runs the MA kernel over its share and K5 merges
the (m, e, ma) partials locally, exchanges one record per (row, q head) over
NVLink and merges across ranks (strong scaling: total work fixed).

A step = one decode step of one attention layer for the whole batch.
  value        tokens/s = B / t_step, inputs resident in HBM, device-timed with
               CUDA events over exactly --steps steps (max over ranks). The
               batch is the same every step (KV >> L2 for configs 2-5: no flush).
  e2e          a real decode loop through the C ABI with HOST buffers, timed
               on the host clock around every step (max over ranks): each step
               appends one token per request (dattn_kv_append: H2D of the new K/V
               rows, pages allocated at page boundaries), decodes over the grown
               contexts (the plan is rebuilt and uploaded because every range
               grew) with q copied H2D and the output copied D2H.
               e2e_static: the same without the append (fixed batch, plan cached).
  parity       outside every timed region: sampled (row, q head) outputs of the
               benchmarked step AND of the decode loop's last step against the
               CPU oracle (oracle/, pinned to the reference by tests/golden/) on
               identical inputs, normalised error (oracles.hpp:50-56) <= tol
               (north_star: 2e-2 bf16, 1e-3 fp32). A failing check exits 1.
  roofline     the MA kernel (K1 or K2, the dominant launch) timed alone with
               CUDA events on its stream; achieved = algorithmic bytes / duration;
               frac against the measured copy bandwidth (MEASURED_PEAKS.json),
               frac_nominal against the north_star's 8 TB/s; traffic = DRAM
               bytes per launch from the ncu capture of THIS library build
               (profiles/ncu_traffic.json, keyed by the library's sha256).
  placement    per-rank KV bytes, the makespan bound they imply (max rank bytes
               at the measured peak) and the step's fraction of it (config 5 is
               placement-limited).
  cpu_baseline the reference's own multi_head_attention (oracle/_ref, compiled
               from the unmodified sources) on all host cores, bounded sample;
               single_thread_value = the same on 1 core (as shipped).
  model_tps    B / (n_layers * t_step), the reference's TPS = beta/(n T_layer)
               (perfmodel.cpp:120-130) for the workload's model depth.
--impl reference times only that CPU reference (rank 0) and prints its line;
it never loads the product library.
"""
from __future__ import annotations

import argparse
import gc
import hashlib
import json
import os
import shutil
import socket
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode-attention tokens/s and KV GB/s (% HBM roofline) at 1/2/4/8 B200 vs CPU"
_JSON_OUT = sys.stdout  # main() points it at the real stdout; everything else goes to stderr


def emit(line: dict) -> None:
    _JSON_OUT.write(json.dumps(line) + "\n")
    _JSON_OUT.flush()
TOL = {0: 2e-2, 1: 1e-3}  # north_star: bf16 2e-2, fp32 1e-3 (normalised error)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", default="2", help="BASELINE config number (1..5)")
    ap.add_argument("--cfg5-queue", type=int, default=64,
                    help="config 5: debtor queue of the reference placement (0, 64 or 512)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU baseline budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0, help="decode-loop steps (0: min(--steps, 64))")
    ap.add_argument("--chunk-tokens", type=int, default=0)
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle check (profiling runs)")
    ap.add_argument("--no-overflow-loop", action="store_true", help="N>1: skip the overflow-borrowing decode loop")
    ap.add_argument("--overflow-steps", type=int, default=48)
    ap.add_argument("--migration-pages", default="1,16,128,512",
                    help="N>1: pages pulled per decode step in the migration-overlap sweep ('' skips it)")
    return ap.parse_args()


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        j = json.load(open(p))
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def repo_libs_loaded():
    """Shared objects of this repo mapped into the process (evidence of which
    library a measurement ran through)."""
    libs = set()
    try:
        for line in open("/proc/self/maps"):
            p = line.split()[-1]
            if p.endswith(".so") and p.startswith(ROOT):
                libs.add(os.path.relpath(p, ROOT))
    except OSError:
        pass
    return sorted(libs)


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
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
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
                rows.append((float(parts[1]), float(parts[2]), float(parts[3]), parts[5:9]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, _, r in rows for i in range(4) if r[i].lower().startswith("active")})
        # samples under load: power above the idle floor (the first and last
        # samples bracket the region and may be idle)
        pmax = max(p for _, _, p, _ in rows)
        loaded = [c for c, _, p, _ in rows if p >= 0.5 * pmax] or [c for c, _, _, _ in rows]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(m for _, m, _, _ in rows),
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(loaded),
                "power_w_max": pmax}


# ----------------------------------------------------------------- CPU side

def cpu_reference_sample(w, budget_s: float, reps_fixed: int = 0, threads: int = 0, warmup: int = 0):
    """Time the reference CPU path on a bounded sample of the workload.

    The sample is the first requests of the batch (all their heads), generated
    with the same counter-hash values the GPU consumes (bf16-rounded, then
    widened to fp64: the reference API is fp64-only). Generation is outside
    the timed region; ``warmup`` untimed reps precede the timed ones. Returns
    the full-workload-equivalent tokens/s and info.
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

    for _ in range(max(warmup, 0)):
        one()
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
        "kind": kind, "cores": threads, "reps": len(times), "warmup_reps": max(warmup, 0),
        "sample_seconds_per_rep": per, "cpu_model": cpu_model(),
        "sample": (f"{B} leading request(s) of the batch, {sum(lens)} context tokens x {w.hkv} kv heads "
                   f"({sum(lens) * w.hkv * w.d * 16 / 1e9:.2f} GB fp64 K+V), kvsched::attn::multi_head_attention "
                   f"per (request, kv head) on {threads} threads; scaled to the full workload by K/V tokens "
                   f"({full_tok_heads / sample_tok_heads:.1f}x)"),
        "kv_gbs_fp64": sample_tok_heads * w.d * 16 / per / 1e9,
    }
    return w.batch / full_t, info


def run_reference_arm(args, rank, ws):
    # workloads is pure host code: importing it does not map libdattn.so
    from paper_2401_02669_b200 import workloads
    if rank != 0:
        return
    w = workloads.config(args.config, args.cfg5_queue)
    # each step is one bounded-sample rep; keep the whole run to a few minutes
    reps = min(max(args.steps, 1), 60)
    value, info = cpu_reference_sample(w, budget_s=0.0, reps_fixed=reps, warmup=min(max(args.warmup, 0), 3))
    libs = repo_libs_loaded()
    assert not any("libdattn" in x for x in libs), libs  # the reference arm never maps the product
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * w.batch / value,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (counter-hash K/V/q, bf16-rounded values widened to fp64)",
        "config": {"workload": w.name, "batch": w.batch, "total_kv_tokens": w.total_tokens,
                   "heads": [w.hq, w.hkv], "head_dim": w.d, **w.meta},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": info["cores"], "kind": info["kind"],
                         "cpu_model": info["cpu_model"],
                         "sample": info["sample"] + f"; {info['warmup_reps']} untimed + {info['reps']} timed reps "
                                                    f"(timed reps capped at 60)"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "kv_gbs_fp64": info["kv_gbs_fp64"],
        "libs_loaded": libs,
    }
    emit(line)


# ----------------------------------------------------------------- parity

def sample_rows(w, max_rows: int = 8):
    """Rows checked against the oracle: all of a small batch, else the first,
    the last, the longest, the shortest and seeded picks."""
    import random
    B = w.batch
    if B <= max_rows:
        return list(range(B))
    rows = {0, B - 1, max(range(B), key=lambda r: w.lens[r]), min(range(B), key=lambda r: w.lens[r])}
    rng = random.Random(w.seed)
    while len(rows) < max_rows:
        rows.add(rng.randrange(B))
    return sorted(rows)


def parity_check(w, out_host, lens, budget_tok_heads: float = 4e6):
    """Sampled (row, kv head) groups of ``out_host`` [B][Hq][dp] (the output of
    the benchmarked step over contexts ``lens``) against the CPU oracle on the
    same inputs. Returns the JSON object (``pass`` false when over tol)."""
    import random

    import numpy as np

    import oracle
    t0 = time.perf_counter()
    rows = sample_rows(w)
    g = w.hq // w.hkv
    cost = 1.0 + g / 2.0  # K/V generation + g q heads of compute per token
    rng = random.Random(w.seed ^ 0x5A5A)
    # the oracle's batch index is the query row and the logical sequence, as
    # on the GPU: pass every row up to the last checked one, select only the
    # sampled (row, kv head) pairs (the others are skipped, not computed)
    nb = rows[-1] + 1
    sel = np.zeros((nb, w.hkv), dtype=bool)
    per_row = budget_tok_heads / len(rows)
    for r in rows:
        k = int(max(1, min(w.hkv, per_row // max(lens[r] * cost, 1))))
        for h in sorted(rng.sample(range(w.hkv), k)):
            sel[r, h] = True
    ref = oracle.decode_ranges(w.seed, [0] * nb, [lens[r] if r in rows else 0 for r in range(nb)], list(range(nb)),
                               w.hq, w.hkv, w.d, dtype=w.dtype, amp_k=w.amp_k, amp_v=w.amp_v, select=sel)
    err = 0.0
    heads = 0
    finite = True
    for r in rows:
        for kvh in np.nonzero(sel[r])[0]:
            for h in range(kvh * g, (kvh + 1) * g):
                got = np.asarray(out_host[r, h, :w.d], dtype=np.float64)
                finite &= bool(np.isfinite(got).all())
                err = max(err, oracle.rel_err(got, ref[r, h]))
                heads += 1
    tol = TOL[w.dtype]
    return {"max_norm_err": err, "tol": tol, "pass": bool(finite and err <= tol), "rows_checked": rows,
            "row_heads_checked": heads, "of_row_heads": w.batch * w.hq,
            "metric": "max |got-ref| / max |ref| per (row, q head) (proj/tests/oracles.hpp:50-56)",
            "oracle": "oracle/dattn_oracle.c fp64 (pinned to the reference: tests/golden/)",
            "seconds": round(time.perf_counter() - t0, 2)}


# ----------------------------------------------------------------- GPU side

def kernel_code_sha256(lib_path: str, module: str = ""):
    """sha256 over the device code of a library: the .text.* (SASS) and
    .nv.info* sections of every cubin embedded in it (cuobjdump -xelf all), or
    of the cubins whose file name starts with ``module`` (e.g. "dattn_gqa_tc":
    K2 alone). nvcc builds are not byte-reproducible -- the fatbin and the
    cubins' debug line tables carry per-build temporary names -- but this code
    hash is, so a capture stays valid across rebuilds of the same sources and
    nothing else."""
    import struct
    with tempfile.TemporaryDirectory() as td:
        tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
        try:
            r = subprocess.run([tool, "-xelf", "all", os.path.abspath(lib_path)], cwd=td,
                               capture_output=True, text=True)
        except OSError:
            return None
        if r.returncode != 0:
            return None
        h = hashlib.sha256()
        for fn in sorted(os.listdir(td)):
            if module and not fn.startswith(module):
                continue
            b = open(os.path.join(td, fn), "rb").read()
            if b[:4] != b"\x7fELF" or b[4] != 2:
                continue
            shoff, = struct.unpack_from("<Q", b, 0x28)
            shentsize, shnum, shstrndx = struct.unpack_from("<HHH", b, 0x3A)
            secs = [struct.unpack_from("<IIQQQQIIQQ", b, shoff + i * shentsize) for i in range(shnum)]
            stro = secs[shstrndx][4]

            def name(off):
                e = b.index(b"\0", stro + off)
                return b[stro + off:e].decode()
            for sh in sorted(secs, key=lambda x: name(x[0])):
                nm = name(sh[0])
                if nm.startswith(".text.") or nm.startswith(".nv.info"):
                    h.update(fn.encode() + nm.encode() + b[sh[4]:sh[4] + sh[5]])
        return h.hexdigest()


def traffic_for(key: str):
    """DRAM bytes per launch of the dominant kernel from profiles/ncu_traffic.json,
    only when that capture was made on this library's device code (same
    kernel_code_sha256; the whole-file hash of a rebuild differs)."""
    import paper_2401_02669_b200 as pb
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        j = json.load(open(tf))
        ent = j.get(key)
    except Exception:
        return None, "no capture"
    if not isinstance(ent, dict):
        return None, "no capture for this config"
    code = kernel_code_sha256(pb.LIB_PATH, ent.get("code_module", ""))
    if code is None or ent.get("code_sha256") != code:
        return None, f"capture of other device code ({ent.get('git_head', '?')}); not reported"
    return ent.get("traffic"), f"ncu --set full, {ent.get('kernel')}, build {ent.get('git_head', '?')}"


def run_b200_arm(args, rank, ws, local):
    t_start = time.time()

    def stage(name):
        print(f"[bench rank {rank}] {name} (+{time.time() - t_start:.1f} s)", file=sys.stderr, flush=True)
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2401_02669_b200 as pb
    from paper_2401_02669_b200 import workloads

    w = workloads.config(args.config, args.cfg5_queue)
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    page = w.page_tokens
    all_shares = workloads.rank_shares(w, ws)
    shares = all_shares[rank]
    # decode loop: every request grows by one token per e2e step, on the rank
    # that holds its last token (the tail)
    ke = args.e2e_steps or min(args.steps, 64)
    grow_total = ke + 3
    tail_rank = {}
    for r_, rs in enumerate(all_shares):
        for rr in rs:
            if rr.tokens and rr.tok_end == w.lens[rr.request]:
                tail_rank[rr.request] = r_
    mine = [rr.request in tail_rank and tail_rank[rr.request] == rank for rr in shares]
    cap_tokens = [rr.tokens + (grow_total if m else 0) for rr, m in zip(shares, mine)]
    mig_rates = [int(x) for x in args.migration_pages.split(",") if x.strip()] if ws > 1 else []
    mig_cap = max(mig_rates, default=0)  # destination pages of the migration sweep (a ring)
    pages = sum(-(-t // page) for t in cap_tokens) + 16 + mig_cap
    max_pps = max([-(-t // page) for t in cap_tokens] + [mig_cap]) + 2
    st = pb.Store(w.d, w.hq, w.hkv, w.dtype, page, pages, max_seqs=w.batch + 4,
                  max_pages_per_seq=max(max_pps, 1), device=local)
    stream = torch.cuda.Stream(device=local)
    st.set_stream(stream.cuda_stream)
    seqs, ranges = [], []
    for rr in shares:
        seq = st.seq_create(rr.tokens)
        seqs.append(seq)
        st.fill_synthetic(seq, w.seed, rr.request, rr.tok_begin, w.amp_k, w.amp_v)
        if rr.tokens == 0:
            ranges.append(pb.Range(seq, rr.request, 0, 0))
            continue
        nb = w.rblocks if ws == 1 else 1
        cuts = [rr.tokens * i // nb for i in range(nb + 1)]
        for a, b in zip(cuts[:-1], cuts[1:]):
            ranges.append(pb.Range(seq, rr.request, a, b))
    franges = pb.range_array(ranges)  # packed once, reused by every step
    tdt = {0: torch.bfloat16, 1: torch.float32}[w.dtype]
    q = torch.empty(w.batch, w.hq, st.padded_dim, dtype=tdt, device=dev)
    st.q_fill_synthetic(q, w.batch, w.seed, 0, 1.0)
    out = torch.empty_like(q)
    comm = None
    if ws > 1:
        uid = [pb.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        st.comm_init(uid[0], rank, ws)
        crank, cn, xmode = st.comm_info()
        comm = {"nccl_rank": crank, "nccl_nranks": cn,
                "exchange": {1: "ncclAllGather + K3", 2: "K5 NVLink exchange", 3: "K1/K2 push + K6"}[xmode]}
        print(f"[bench rank {rank}] NCCL communicator: rank {crank} of {cn} (ncclCommCount); "
              f"exchange: {comm['exchange']}", file=sys.stderr, flush=True)
        assert crank == rank and cn == ws, comm

    def step(rg=franges, mem=pb.MEM_DEVICE, qq=q, oo=out):
        if ws > 1:
            st.decode_sharded(rg, w.batch, qq, oo, mem=mem, chunk_tokens=args.chunk_tokens)
        else:
            st.decode(rg, w.batch, qq, oo, mem=mem, chunk_tokens=args.chunk_tokens)

    def barrier():
        if ws > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    torch.cuda.synchronize()
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    barrier()

    stage("region A")
    # no Python garbage collection inside the timed regions: a gen-2 pass over
    # torch's heap stalled one decode-loop step for ~0.5 s (r2z run)
    gc.collect()
    gc.disable()
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
    out_a = out.cpu()

    stage("region B")
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

    stage("region C")
    # ---- region C: static e2e (fixed batch) through the C ABI with host buffers ----
    qh = q.cpu().pin_memory()
    oh = torch.empty_like(qh).pin_memory()
    for _ in range(3):
        step(mem=pb.MEM_HOST, qq=qh, oo=oh)
    barrier()
    t0 = time.perf_counter()
    for _ in range(ke):
        step(mem=pb.MEM_HOST, qq=qh, oo=oh)
    t_static = max_over_ranks(time.perf_counter() - t0) / ke
    static_same = bool(torch.equal(oh, out_a))

    stage("region D")
    # ---- region D: the decode loop, end to end ----
    # inputs of every step, made before the region: the new token's K/V rows
    # (the generator's values at position L_r + t, so the oracle can check the
    # result) in pinned host memory, [step][my tail requests][Hkv][dp]
    app_idx = [i for i, m in enumerate(mine) if m]
    app_seqs = [seqs[i] for i in app_idx]
    n_app = len(app_idx)
    lens_now = list(w.lens)
    kh = vh = None
    if n_app:
        kd = torch.empty(grow_total, n_app, w.hkv, st.padded_dim, dtype=tdt, device=dev)
        vd = torch.empty_like(kd)
        for t in range(grow_total):
            st.synthetic_rows([shares[i].request for i in app_idx], [w.lens[shares[i].request] + t for i in app_idx],
                              w.seed, kd[t], vd[t], w.amp_k, w.amp_v)
        kh = kd.cpu().pin_memory()
        vh = vd.cpu().pin_memory()
        del kd, vd
    cur_end = [rr.tokens for rr in shares]

    brk = [0.0, 0.0, 0.0]  # host seconds in append / range build / decode call
    # the decode loop's ranges, packed once: the last range of every request
    # (the one that grows) is tok_end-updated in place through a numpy view
    loop_rg, grow_idx = [], []
    for i, rr in enumerate(shares):
        if ws > 1 or w.rblocks == 1:
            loop_rg.append(pb.Range(seqs[i], rr.request, 0, rr.tokens))
        else:
            cuts = [rr.tokens * j // w.rblocks for j in range(w.rblocks + 1)]
            loop_rg.extend(pb.Range(seqs[i], rr.request, a, b) for a, b in zip(cuts[:-1], cuts[1:]))
        grow_idx.append(len(loop_rg) - 1)
    loop_ra = pb.range_array(loop_rg)
    loop_view = np.ctypeslib.as_array(loop_ra.arr)
    grow_idx = np.asarray(grow_idx)

    class _Ends:  # loop_ends[:] = cur_end writes tok_end of the growing ranges
        def __setitem__(self, key, vals):
            loop_view["tok_end"][grow_idx] = vals
    loop_ends = _Ends()
    split_log = []  # per step: (t, append ms, range build ms, decode call ms)

    def loop_step(t):
        c0 = time.perf_counter()
        if n_app:
            st.kv_append(app_seqs, kh[t], vh[t], mem=pb.MEM_HOST)
            for i in app_idx:
                cur_end[i] += 1
        c1 = time.perf_counter()
        # every range of a request ends at its current length (ws > 1: one
        # range per request per rank; ws == 1: rBlock cuts, the last one grows):
        # the packed range array is updated in place
        loop_ends[:] = cur_end
        c2 = time.perf_counter()
        step(rg=loop_ra, mem=pb.MEM_HOST, qq=qh, oo=oh)
        c3 = time.perf_counter()
        brk[0] += c1 - c0
        brk[1] += c2 - c1
        brk[2] += c3 - c2
        split_log.append((t, 1e3 * (c1 - c0), 1e3 * (c2 - c1), 1e3 * (c3 - c2)))

    for t in range(3):  # warm-up steps grow the contexts too
        loop_step(t)
    st.stats(reset=True)
    brk[:] = [0.0, 0.0, 0.0]
    barrier()
    per_step = []
    t0 = time.perf_counter()
    for t in range(3, 3 + ke):
        c = time.perf_counter()
        loop_step(t)
        per_step.append(time.perf_counter() - c)
    t_loop = max_over_ranks(time.perf_counter() - t0) / ke
    slowest = sorted(split_log[3:], key=lambda x: -(x[1] + x[2] + x[3]))[:3]
    per_step.sort()
    plan_bytes = st.stats().last_plan_bytes
    lens_now = [L + grow_total for L in w.lens]
    out_d = oh.clone()
    qbytes = qh.numel() * qh.element_size()
    app_bytes = 2 * n_app * w.hkv * st.padded_dim * st.elem_bytes

    stage("region E")
    # ---- region E (N > 1): paced block migration overlapped with decode ----
    # Every rank pulls m whole pages (K+V, all kv heads) of its left
    # neighbour's pool per decode step (dattn_kv_pull: copy engines over
    # NVLink, migration stream) while it decodes the same batch; the step
    # joins its pulls, so a step costs max(decode, copies). m = 1 page is the
    # reference's pacing (MigrationConfig step_tokens 16, config.hpp:44-51).
    # The destination is a ring of m pages; sources are real pages the decode
    # also reads. Same device timing as region A (max over ranks).
    migration = None
    if mig_rates:
        src_seq = max(range(len(shares)), key=lambda i: shares[i].tokens)
        my_pages = st.block_table(seqs[src_seq])
        all_pages = [None] * ws
        dist.all_gather_object(all_pages, my_pages)
        left = (rank + ws - 1) % ws
        src_pages = all_pages[left][:-1]  # full pages only (a sequence's last page may be partial)
        # every rank runs the same rates (each step has collectives): the
        # smallest source any rank pulls from bounds them
        min_src = min(len(pg) - 1 for pg in all_pages)
        dst = st.seq_create(mig_cap * page)
        km = max(10, min(args.steps, 50))
        page_bytes = 2 * w.hkv * page * st.padded_dim * st.elem_bytes
        sweep = []
        if min_src > 0:  # the first pull maps the peer pool lazily: keep it out of the sweep
            st.kv_pull(dst, 0, left, src_pages[:1])
            st.migration_join(wait_host=True)
        for m in [0] + mig_rates:
            if m > min_src:
                continue
            pulls = [src_pages[(j * m) % (len(src_pages) - m + 1):][:m] for j in range(km + 3)]

            def mstep(j):
                if m:
                    st.kv_pull(dst, 0, left, pulls[j])
                step()
                if m:
                    st.migration_join()

            for j in range(3):
                mstep(j)
            torch.cuda.synchronize()
            barrier()
            m0 = torch.cuda.Event(enable_timing=True)
            m1 = torch.cuda.Event(enable_timing=True)
            m0.record(stream)
            for j in range(3, 3 + km):
                mstep(j)
            m1.record(stream)
            torch.cuda.synchronize()
            barrier()
            t_m = max_over_ranks(m0.elapsed_time(m1)) / km
            sweep.append({"pages_per_step": m, "tokens_per_step": m * page,
                          "bytes_per_step_per_rank": m * page_bytes, "ms_per_step": t_m,
                          "nvlink_gbs_per_rank": m * page_bytes / (t_m * 1e-3) / 1e9})
        # the last pull's first and last pages hold the generator's values of
        # the left neighbour's tokens, bit for bit (oracle, outside the timing)
        st.migration_join(wait_host=True)
        pulled_ok = None
        last = pulls[km + 2]
        if last and not args.no_parity:
            import oracle
            lsh = all_shares[left]
            lrr = lsh[max(range(len(lsh)), key=lambda i: lsh[i].tokens)]
            pulled_ok = True
            for slot in (0, len(last) - 1):
                p_idx = src_pages.index(last[slot])
                for h in (0, w.hkv - 1):
                    k_, v_ = st.kv_read(dst, h, slot * page, page)
                    rk, rv = oracle.synth_kv(w.seed, lrr.request, h, lrr.tok_begin + p_idx * page, page, w.d,
                                             w.amp_k, w.amp_v, w.dtype)
                    pulled_ok &= bool(np.array_equal(k_[:, :w.d], rk[:, :w.d]) and np.array_equal(v_[:, :w.d], rv[:, :w.d]))
        oks = [None] * ws
        dist.all_gather_object(oks, pulled_ok)
        base = sweep[0]["ms_per_step"]
        for e_ in sweep:
            e_["slowdown_vs_no_migration"] = e_["ms_per_step"] / base - 1.0
        migration = {"what": "each rank pulls m pages/step of its left neighbour's KV pool (dattn_kv_pull, copy "
                             "engines over NVLink) while decoding the batch; step = decode + join of its pulls",
                     "page_bytes": page_bytes, "sweep": sweep, "pulled_pages_bit_exact": oks,
                     "reference_model": "MigrationConfig: 16 tokens/step hidden (overlap_cap_tokens), then "
                                        "+0.086/16 step per extra token (config.hpp:44-51)"}

    # ---- NVLink bytes per step of the K5 exchange (algorithmic) ----
    # NVML's NVLink throughput counters (field ids 138-141) answer
    # NVML_ERROR_NOT_SUPPORTED on these boxes, and querying NVLink state
    # perturbed the timing of later steps (2-GPU config 2: 1.40 instead of
    # 1.18 ms per step), so the line carries the algorithmic bytes only
    # (profiles/r2_nvlink_counters_probe.txt).
    nvlink = None
    if ws > 1:
        live = sum(1 for rr in shares if rr.tokens) * w.hq
        mine_alg = (ws - 1) * (live * st.record_bytes + (w.batch * w.hq - live) * 16)
        per = [None] * ws
        dist.all_gather_object(per, mine_alg)
        nvlink = {"exchange_alg_bytes_per_rank": per,
                  "what": "bytes each rank pushes over NVLink per step in K5: one record per (row, q head) "
                          "to every peer, identity records only their 16-byte header"}

    stage("region G")
    # ---- region G (N > 1): decode loop whose KV outgrows its home GPU ----
    # The same batch with every request homed whole on one GPU (round robin),
    # each GPU's page pool sized to its requests plus headroom -- none on
    # GPU 0. As contexts grow, GPU 0's requests take their next blocks on
    # peers through the block ledger's ensure_slot (simengine.cpp:318-354,
    # dattn_ledger_*): the slot's GPU appends the token, every GPU decodes the
    # tokens it holds (decode_loop.ClusterDecodeLoop). Host clock per step
    # (slot decisions + append + sharded decode, synchronised), max over ranks;
    # parity of the last step against the oracle at the grown lengths.
    overflow = None
    if ws > 1 and not args.no_overflow_loop:
        from paper_2401_02669_b200.decode_loop import ClusterDecodeLoop
        kg = args.overflow_steps
        homes = [i % ws for i in range(w.batch)]
        need = [0] * ws
        for i, L in enumerate(w.lens):
            need[homes[i]] += pb.blocks_for_tokens(L, page)
        n0 = sum(1 for h in homes if h == 0)
        grow_blocks = -(-kg // page) + 1
        caps = [need[0]] + [need[r] + 2 * (w.batch // ws + n0) * grow_blocks for r in range(1, ws)]
        st2 = pb.Store(w.d, w.hq, w.hkv, w.dtype, page, caps[rank], max_seqs=w.batch + 4,
                       max_pages_per_seq=max(caps), device=local)
        st2.set_stream(stream.cuda_stream)
        uid2 = [pb.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid2, src=0)
        st2.comm_init(uid2[0], rank, ws)
        loop = ClusterDecodeLoop(st2, rank, ws, caps, w.seed, w.amp_k, w.amp_v)
        for i, L in enumerate(w.lens):
            assert loop.admit(i, i, L, home=homes[i])
        out2 = torch.empty_like(q)
        for _ in range(3):
            loop.step(w.batch, q, out2)
        torch.cuda.synchronize()
        barrier()
        per = []
        t0 = time.perf_counter()
        for _ in range(kg):
            c = time.perf_counter()
            loop.step(w.batch, q, out2)
            torch.cuda.synchronize()
            per.append(time.perf_counter() - c)
        t_g = max_over_ranks(time.perf_counter() - t0) / kg
        lens_g = [loop.led.request(i)[1] for i in range(w.batch)]
        pages_ok = st2.info().free_pages == loop.led.free_blocks(rank)
        oks2 = [None] * ws
        dist.all_gather_object(oks2, pages_ok)
        par_g = None
        if rank == 0 and not args.no_parity:
            par_g = parity_check(w, out2.float().cpu().numpy() if w.dtype == 0 else out2.cpu().numpy(), lens_g)
        hosted = sum(1 for i in range(w.batch) if len({s_[0] for s_ in loop.led.segments(i)}) > 1)
        per.sort()
        overflow = {"what": "decode loop, requests homed whole round robin, GPU 0's pool without headroom: its "
                            "requests borrow blocks on peers (ensure_slot) as they grow; host clock per step incl. "
                            "slot decisions, appends and the sharded decode (synchronised), max over ranks",
                    "ms_per_step": t_g * 1e3, "tokens_per_s": w.batch / t_g, "steps": kg,
                    "step_ms_rank0": {"median": 1e3 * per[len(per) // 2], "max": 1e3 * per[-1]},
                    "capacity_blocks": caps, "borrowed_blocks": loop.led.borrowed(),
                    "requests_spanning_gpus": hosted, "stalled_request_steps": loop.stalled,
                    "pages_equal_ledger_per_rank": oks2, "parity": par_g}
        st2.close()

    gc.enable()
    stage("parity")
    # ---- parity of what was timed (outside every timed region) ----
    parity = parity_loop = None
    if rank == 0 and not args.no_parity:
        parity = parity_check(w, out_a.float().numpy() if w.dtype == 0 else out_a.numpy(), w.lens)
        parity["e2e_static_bitwise_equal"] = static_same
        parity["pass"] = parity["pass"] and static_same
        parity_loop = parity_check(w, out_d.float().numpy() if w.dtype == 0 else out_d.numpy(), lens_now)
        parity_loop["context_tokens_after_loop"] = sum(lens_now)

    if rank != 0:
        return 0
    peak, peak_src = measured_peak()
    # per-rank algorithmic bytes of one MA launch (rank 0's share)
    kv_rank = sum(2 * w.hkv * w.d * rr.tokens * w.elem_bytes for rr in shares)
    kv_ranks = [sum(2 * w.hkv * w.d * rr.tokens * w.elem_bytes for rr in rs) for rs in all_shares]
    bound_ms = max(kv_ranks) / (peak * 1e9) * 1e3
    alg_rank = kv_rank + w.batch * w.hq * w.d * 2 * w.elem_bytes
    achieved = alg_rank / (ma_ms * 1e-3) / 1e9
    traffic, traffic_src = traffic_for(f"cfg{args.config}_n{ws}")
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
                      "balanced_bound_ms": w.kv_bytes() / ws / (peak * 1e9) * 1e3,
                      "aggregate_frac": w.kv_bytes() / (ws * peak * 1e9) / (ms_step * 1e-3)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "frac_nominal": achieved / 8000.0,
                     "kernel": kernel_name, "kernel_ms": ma_ms, "merge_ms": merge_ms, "exchange_ms": comm_ms,
                     "alg_bytes_per_launch": alg_rank, "peak_source": peak_src},
        "e2e": {"value": w.batch / t_loop, "unit": "tokens/s",
                "h2d_bytes_per_step": qbytes + app_bytes + plan_bytes, "d2h_bytes_per_step": qbytes,
                "ms_per_step": t_loop * 1e3, "steps": ke,
                "what": "decode loop through the C ABI, host clock, max over ranks: per step dattn_kv_append of "
                        "one token per request (H2D of its K/V rows) + decode over the grown contexts "
                        "(plan rebuilt and uploaded) with H2D q and D2H output",
                "h2d_split": {"q": qbytes, "kv_rows_rank0": app_bytes, "plan_rank0": plan_bytes},
                "host_ms_rank0": {"kv_append_call": 1e3 * brk[0] / ke, "range_build": 1e3 * brk[1] / ke,
                                  "decode_call": 1e3 * brk[2] / ke},
                "step_ms_rank0": {"median": 1e3 * per_step[len(per_step) // 2],
                                  "p90": 1e3 * per_step[int(0.9 * (len(per_step) - 1))], "max": 1e3 * per_step[-1],
                                  "slowest": [{"step": t_, "append_ms": round(a_, 3), "ranges_ms": round(b_, 3),
                                               "decode_call_ms": round(c_, 3)} for t_, a_, b_, c_ in slowest]}},
        "e2e_static": {"value": w.batch / t_static, "unit": "tokens/s", "ms_per_step": t_static * 1e3,
                       "h2d_bytes_per_step": qbytes, "d2h_bytes_per_step": qbytes,
                       "what": "fixed batch repeated (plan cached), H2D q + D2H output"},
        "parity": parity, "parity_decode_loop": parity_loop,
        "gpu_launches": launches,
        "per_rank_ms": {"ma": [round(t[0], 4) for t in rank_times],
                        "exchange": [None if t[1] is None else round(t[1], 4) for t in rank_times]},
        "clocks": clocks,
        "libs_loaded": repo_libs_loaded(),
    }
    if comm:
        line["comm"] = comm
    if nvlink:
        line["nvlink"] = nvlink
    if migration:
        line["migration"] = migration
    if overflow:
        line["overflow_decode_loop"] = overflow
    if ws == 1 and not args.no_cpu_baseline:
        cv, info = cpu_reference_sample(w, args.cpu_seconds)
        c1, info1 = cpu_reference_sample(w, min(args.cpu_seconds, 4.0), threads=1)
        line["cpu_baseline"] = {"value": cv, "unit": "tokens/s", "cores": info["cores"], "kind": info["kind"],
                                "cpu_model": info["cpu_model"],
                                "sample": info["sample"] + f"; {info['reps']} reps",
                                "single_thread_value": c1, "single_thread_reps": info1["reps"],
                                "kv_gbs_fp64": info["kv_gbs_fp64"], "single_thread_kv_gbs_fp64": info1["kv_gbs_fp64"]}
    emit(line)
    ok = all(p is None or p["pass"] for p in (parity, parity_loop, (overflow or {}).get("parity")))
    if not ok:
        print("[bench] PARITY FAILED: " + json.dumps({"parity": parity, "parity_decode_loop": parity_loop}),
              file=sys.stderr, flush=True)
    return 0 if ok else 1


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(n: int) -> int:
    """Re-run this command as N ranks under torch.distributed.run (one process
    per GPU, rendezvous on 127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    print(f"[bench] launching {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd, stdout=_JSON_OUT)


def main():
    global _JSON_OUT
    args = parse()
    # stdout carries exactly the one JSON line: libraries that print to
    # stdout (NCCL's version banner, torch.distributed.run) go to stderr
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ws_env = os.environ.get("WORLD_SIZE")
    ws = int(ws_env or "1")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, ws)
        return 0
    if ws_env is None and args.gpus > 1:
        return self_launch(args.gpus)
    if ws != args.gpus:
        print(f"[bench] refusing: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr, flush=True)
        return 2
    # a rank stuck for BENCH_WATCHDOG_S seconds dumps every thread's stack
    # to stderr and exits, instead of holding the box until an outer timeout
    import faulthandler
    faulthandler.dump_traceback_later(float(os.environ.get("BENCH_WATCHDOG_S", "900")), exit=True)
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    try:
        rc = run_b200_arm(args, rank, ws, local)
    except BaseException:
        # the other ranks may sit in a collective: report and leave at once
        # (torch.distributed.run then stops them) instead of blocking in
        # destroy_process_group
        import traceback
        traceback.print_exc()
        sys.stderr.flush()
        os._exit(1)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
