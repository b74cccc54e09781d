"""TEST INFRASTRUCTURE ONLY -- ctypes bindings to the CPU oracle.

``liboracle.so`` is the plain-C restatement of the reference's DistAttention
math (dattn_oracle.c, every function citing /root/reference file:line).
``_ref/libkvsched_ref.so`` is the unmodified reference compiled by
oracle/Makefile (present when the reference was available at build time; it
travels to the GPU box as a prebuilt file).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this package, as the checker or as the timed
CPU baseline. The product package never does.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(_HERE, "liboracle.so")
REF_LIB = os.path.join(_HERE, "_ref", "libkvsched_ref.so")

D = ctypes.c_double
DP = ctypes.POINTER(ctypes.c_double)
I64 = ctypes.c_int64
U64 = ctypes.c_uint64
U32 = ctypes.c_uint32
VP = ctypes.c_void_p

BF16, F32, F64 = 0, 1, 2


def _load_oracle():
    lib = ctypes.CDLL(ORACLE_LIB)
    sig = {
        "or_effective_scale": (D, [ctypes.c_int, D]),
        "or_micro_attention": (I64, [VP, VP, VP, I64, ctypes.c_int, D, VP, VP, VP]),
        "or_naive_attention": (None, [VP, VP, VP, I64, ctypes.c_int, D, VP]),
        "or_combine": (None, [D, D, VP, I64, D, D, VP, I64, ctypes.c_int, VP, VP, VP, VP]),
        "or_aggregate": (ctypes.c_int, [ctypes.c_int, VP, VP, VP, VP, ctypes.c_int, VP]),
        "or_gqa_kv_head": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int]),
        "or_serialize_partial": (None, [D, D, VP, ctypes.c_int, VP]),
        "or_deserialize_seq_p": (I64, [VP]),
        "or_blocks_for_tokens": (I64, [I64, ctypes.c_int]),
        "or_attention_ld": (None, [VP, VP, VP, I64, ctypes.c_int, D, VP]),
        "or_rel_err": (D, [VP, VP, I64]),
        "or_rng_seed": (None, [VP, U64]),
        "or_rng_next_u64": (U64, [VP]),
        "or_rng_uniform01": (D, [VP]),
        "or_rng_uniform": (D, [VP, D, D]),
        "or_rng_uniform_int": (I64, [VP, I64, I64]),
        "or_rng_normal": (D, [VP]),
        "or_splitmix64": (U64, [U64]),
        "or_synth_value": (D, [U64, ctypes.c_int, U32, U32, U32, U32, ctypes.c_float, ctypes.c_int]),
        "or_synth_kv": (None, [U64, U32, U32, U32, I64, ctypes.c_int, ctypes.c_float, ctypes.c_float,
                               ctypes.c_int, VP, VP]),
        "or_synth_q": (None, [U64, U32, U32, ctypes.c_int, ctypes.c_float, ctypes.c_int, VP]),
        "or_f32_to_bf16_rne": (ctypes.c_uint16, [ctypes.c_float]),
        "or_decode_batch": (ctypes.c_int, [U64, ctypes.c_int, VP, VP, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, D, ctypes.c_int, ctypes.c_float,
                                           ctypes.c_float, ctypes.c_float, I64, ctypes.c_int, VP]),
        "or_decode_ranges": (ctypes.c_int, [U64, ctypes.c_int, VP, VP, VP, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int, D, ctypes.c_int, ctypes.c_float,
                                            ctypes.c_float, ctypes.c_float, ctypes.c_int, VP, VP, VP]),
        "or_decode_ranges_sel": (ctypes.c_int, [U64, ctypes.c_int, VP, VP, VP, ctypes.c_int, ctypes.c_int,
                                                ctypes.c_int, D, ctypes.c_int, ctypes.c_float,
                                                ctypes.c_float, ctypes.c_float, VP, ctypes.c_int, VP, VP,
                                                VP]),
    }
    for n, (r, a) in sig.items():
        f = getattr(lib, n)
        f.restype = r
        f.argtypes = a
    return lib


lib = _load_oracle()


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ---- reference math restated (distattention.cpp) ----
def effective_scale(d: int, scale: float = 0.0) -> float:
    return lib.or_effective_scale(d, scale)


def micro_attention(q, k, v, scale: float = 0.0):
    q, k, v = f64(q), f64(k), f64(v)
    d = q.shape[0]
    seq = k.shape[0] if k.size else 0
    m, e = np.zeros(1), np.zeros(1)
    ma = np.zeros(d)
    sp = lib.or_micro_attention(_p(q), _p(k), _p(v), seq, d, scale, _p(m), _p(e), _p(ma))
    return float(m[0]), float(e[0]), ma, int(sp)


def naive_attention(q, k, v, scale: float = 0.0):
    q, k, v = f64(q), f64(k), f64(v)
    out = np.zeros(q.shape[0])
    lib.or_naive_attention(_p(q), _p(k), _p(v), k.shape[0], q.shape[0], scale, _p(out))
    return out


def combine(a, b):
    (am, ae, ama, asq), (bm, be, bma, bsq) = a, b
    ama, bma = f64(ama), f64(bma)
    d = ama.shape[0]
    om, oe, osq = np.zeros(1), np.zeros(1), np.zeros(1, dtype=np.int64)
    oma = np.zeros(d)
    lib.or_combine(am, ae, _p(ama), asq, bm, be, _p(bma), bsq, d, _p(om), _p(oe), _p(oma), _p(osq))
    return float(om[0]), float(oe[0]), oma, int(osq[0])


def aggregate(parts):
    n = len(parts)
    d = len(parts[0][2])
    m = f64([p[0] for p in parts])
    e = f64([p[1] for p in parts])
    ma = f64(np.stack([np.asarray(p[2], dtype=np.float64) for p in parts]))
    sp = np.ascontiguousarray([p[3] for p in parts], dtype=np.int64)
    out = np.zeros(d)
    rc = lib.or_aggregate(n, _p(m), _p(e), _p(ma), _p(sp), d, _p(out))
    if rc != 0:
        raise ValueError("aggregate needs at least one covered token")
    return out


def attention_ld(q, k, v, scale: float):
    q, k, v = f64(q), f64(k), f64(v)
    out = np.zeros(q.shape[0])
    lib.or_attention_ld(_p(q), _p(k), _p(v), k.shape[0], q.shape[0], scale, _p(out))
    return out


def rel_err(got, ref) -> float:
    got, ref = f64(got).ravel(), f64(ref).ravel()
    return lib.or_rel_err(_p(got), _p(ref), ref.size)


def blocks_for_tokens(tokens: int, block: int) -> int:
    return lib.or_blocks_for_tokens(tokens, block)


def gqa_kv_head(h: int, hq: int, hkv: int) -> int:
    return lib.or_gqa_kv_head(h, hq, hkv)


class Rng:
    """sim::Rng restated (trace.cpp:14-53)."""

    def __init__(self, seed: int):
        self._buf = ctypes.create_string_buffer(312 * 8 + 16)
        lib.or_rng_seed(self._buf, seed)

    def next_u64(self) -> int:
        return lib.or_rng_next_u64(self._buf)

    def uniform01(self) -> float:
        return lib.or_rng_uniform01(self._buf)

    def uniform(self, lo, hi) -> float:
        return lib.or_rng_uniform(self._buf, lo, hi)

    def uniform_int(self, lo, hi) -> int:
        return lib.or_rng_uniform_int(self._buf, lo, hi)

    def normal(self) -> float:
        return lib.or_rng_normal(self._buf)


# ---- synthetic inputs (bit-identical to the CUDA fill kernels) ----
def synth_kv(seed: int, seq: int, head: int, tok0: int, n: int, d: int, amp_k=1.0, amp_v=2.0,
             dtype: int = BF16):
    k = np.zeros((max(n, 0), d))
    v = np.zeros((max(n, 0), d))
    lib.or_synth_kv(seed, seq, head, tok0, n, d, amp_k, amp_v, dtype, _p(k), _p(v))
    return k, v


def synth_q(seed: int, row: int, head: int, d: int, amp_q=1.0, dtype: int = BF16):
    q = np.zeros(d)
    lib.or_synth_q(seed, row, head, d, amp_q, dtype, _p(q))
    return q


def decode_ranges(seed: int, tok_lo: Sequence[int], tok_hi: Sequence[int], seq_ids: Sequence[int],
                  hq: int, hkv: int, d: int, scale: float = 0.0, dtype: int = BF16,
                  amp_q=1.0, amp_k=1.0, amp_v=2.0, threads: int = 0, want_me: bool = False,
                  select=None):
    """fp64 reference output [B, hq, d] of every request over [tok_lo, tok_hi).
    ``select``: optional boolean [B, hkv] -- compute only those (request, kv
    head) pairs (all q heads of each group); other outputs stay zero."""
    B = len(tok_lo)
    lo = np.ascontiguousarray(tok_lo, dtype=np.int64)
    hi = np.ascontiguousarray(tok_hi, dtype=np.int64)
    ids = np.ascontiguousarray(seq_ids, dtype=np.uint32)
    out = np.zeros((B, hq, d))
    m = np.zeros((B, hq)) if want_me else None
    e = np.zeros((B, hq)) if want_me else None
    threads = threads or (os.cpu_count() or 1)
    if select is None:
        lib.or_decode_ranges(seed, B, _p(lo), _p(hi), _p(ids), hq, hkv, d, scale, dtype, amp_q, amp_k,
                             amp_v, threads, _p(out), _p(m), _p(e))
    else:
        sel = np.ascontiguousarray(np.asarray(select, dtype=bool).reshape(B, hkv), dtype=np.uint8)
        lib.or_decode_ranges_sel(seed, B, _p(lo), _p(hi), _p(ids), hq, hkv, d, scale, dtype, amp_q, amp_k,
                                 amp_v, _p(sel), threads, _p(out), _p(m), _p(e))
    return (out, m, e) if want_me else out


def decode_batch(seed: int, lens: Sequence[int], hq: int, hkv: int, d: int, scale: float = 0.0,
                 dtype: int = BF16, amp_q=1.0, amp_k=1.0, amp_v=2.0, seg_tokens: int = 0,
                 threads: int = 0, seq_ids: Optional[Sequence[int]] = None):
    B = len(lens)
    L = np.ascontiguousarray(lens, dtype=np.int64)
    ids = np.ascontiguousarray(seq_ids if seq_ids is not None else range(B), dtype=np.uint32)
    out = np.zeros((B, hq, d))
    threads = threads or (os.cpu_count() or 1)
    lib.or_decode_batch(seed, B, _p(L), _p(ids), hq, hkv, d, scale, dtype, amp_q, amp_k, amp_v,
                        seg_tokens, threads, _p(out))
    return out


# ---- the compiled reference (oracle/_ref) ----
def ref_available() -> bool:
    return os.path.exists(REF_LIB)


_ref = None


def ref():
    """ctypes handle to the unmodified reference (oracle/_ref/libkvsched_ref.so)."""
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(REF_LIB)
        r = ctypes.CDLL(REF_LIB, mode=ctypes.RTLD_LOCAL)
        r.ref_last_error.restype = ctypes.c_char_p
        for n, a in {
            "ref_micro_attention": [VP, VP, VP, I64, ctypes.c_int, D, VP, VP, VP, VP],
            "ref_naive_attention": [VP, VP, VP, I64, ctypes.c_int, D, VP],
            "ref_combine": [D, D, VP, I64, D, D, VP, I64, ctypes.c_int, VP, VP, VP, VP],
            "ref_aggregate": [ctypes.c_int, VP, VP, VP, VP, ctypes.c_int, VP],
            "ref_gqa_kv_head": [ctypes.c_int, ctypes.c_int, ctypes.c_int, VP],
            "ref_serialize_partial": [D, D, VP, ctypes.c_int, VP, VP],
            "ref_deserialize_partial": [VP, I64, ctypes.c_int, VP, VP, VP, VP],
            "ref_multi_head_attention": [VP, VP, VP, I64, ctypes.c_int, ctypes.c_int, ctypes.c_int, D,
                                         VP, VP, VP],
            "ref_verify_attention": [ctypes.c_int, U64, D, VP, VP, VP],
            "ref_rng_draws": [U64, ctypes.c_int, VP, VP, VP, VP, I64, I64],
            "ref_decode_timed": [ctypes.c_int, VP, VP, VP, ctypes.c_int, ctypes.c_int, ctypes.c_int, D,
                                 I64, ctypes.c_int, VP, VP],
            "ref_default_config_json": [ctypes.c_int, I64, ctypes.POINTER(ctypes.c_void_p)],
            "ref_config_eval": [ctypes.c_char_p, ctypes.c_int, VP, VP, I64, VP, VP, VP],
            "ref_blocks_for_tokens": [I64, ctypes.c_int, VP],
            "ref_rmanager_trace": [I64, ctypes.c_int, VP, VP, VP, VP, VP, VP, VP, VP],
            "ref_cfg5_place": [ctypes.c_int, I64, I64, ctypes.c_int, ctypes.c_int, VP, VP, VP,
                               ctypes.c_int, VP, VP, VP],
            "ref_sim_log": [ctypes.c_int, VP, ctypes.c_int, ctypes.c_int, VP, VP, VP, D,
                            ctypes.POINTER(ctypes.c_void_p)],
        }.items():
            f = getattr(r, n)
            f.restype = ctypes.c_int
            f.argtypes = a
        _ref = r
    return _ref


# ---- the reference perf model / config ----
def ref_default_config(n_instances: int = 4, capacity_blocks: int = 256) -> str:
    """The reference's default cluster config (config.cpp:71-87) as JSON text."""
    r = ref()
    p = ctypes.c_void_p()
    rc = r.ref_default_config_json(n_instances, capacity_blocks, ctypes.byref(p))
    if rc != 0:
        raise RuntimeError(r.ref_last_error().decode())
    try:
        return ctypes.string_at(p).decode()
    finally:
        r.ref_string_free.argtypes = [ctypes.c_void_p]
        r.ref_string_free(p)


def ref_config_eval(text: str, xs: Sequence[float], ctx_lengths: Sequence[int]):
    """Parse ``text`` with the reference parser (which validates every curve)
    and return (g(xs), layer_time(load of ctx_lengths), n_layers). Raises
    ValueError with the reference's message when the config is rejected."""
    r = ref()
    x = np.ascontiguousarray(xs, dtype=np.float64)
    g = np.zeros(len(x))
    L = np.ascontiguousarray(ctx_lengths, dtype=np.int64)
    lt = np.zeros(1)
    nl = np.zeros(1, dtype=np.int32)
    rc = r.ref_config_eval(text.encode(), len(x), _p(x), _p(g), len(L), _p(L), _p(lt), _p(nl))
    if rc != 0:
        raise ValueError(r.ref_last_error().decode())
    return g, float(lt[0]), int(nl[0])


# ---- the reference ledger and control plane ----
def ref_blocks_for_tokens(tokens: int, block: int) -> int:
    """kvsched::perf::blocks_for_tokens (perfmodel.cpp:178-182), compiled."""
    r = ref()
    out = np.zeros(1, dtype=np.int64)
    if r.ref_blocks_for_tokens(tokens, block, _p(out)) != 0:
        raise ValueError(r.ref_last_error().decode())
    return int(out[0])


LEDGER_ALLOC_LOCAL, LEDGER_ALLOC_HOSTED, LEDGER_FREE = 0, 1, 2


def ref_rmanager_trace(capacity: int, ops):
    """Run ``ops`` = [(op, req, n, home)] through one reference RManager
    (controlplane.cpp:38-79). Returns per-op (result, used, free, local)."""
    r = ref()
    k = len(ops)
    op = np.ascontiguousarray([o[0] for o in ops], dtype=np.int32)
    req = np.ascontiguousarray([o[1] for o in ops], dtype=np.int64)
    n = np.ascontiguousarray([o[2] for o in ops], dtype=np.int64)
    n2 = np.ascontiguousarray([o[3] if len(o) > 3 else -1 for o in ops], dtype=np.int32)
    res, used, free, local = (np.zeros(max(k, 1), dtype=np.int64) for _ in range(4))
    rc = r.ref_rmanager_trace(capacity, k, _p(op), _p(req), _p(n), _p(n2), _p(res), _p(used), _p(free),
                              _p(local))
    if rc != 0:
        raise ValueError(r.ref_last_error().decode())
    return [(int(res[i]), int(used[i]), int(free[i]), int(local[i])) for i in range(k)]


def ref_cfg5_place(tokens: Sequence[int], n_inst: int, capacity_blocks: int, queued: int, rounds: int = 1):
    """Config-5 placement by the reference control plane (ref_bridge.cpp
    ref_cfg5_place): dispatch, heartbeats, GManager::plan + execute_move_sync.
    Returns (homes, blocks[req][inst], moves) with moves as dicts."""
    r = ref()
    n_req = len(tokens)
    t = np.ascontiguousarray(tokens, dtype=np.int64)
    home = np.zeros(n_req, dtype=np.int32)
    blocks = np.zeros(n_req * n_inst, dtype=np.int64)
    maxm = 256
    moves = np.zeros(6 * maxm, dtype=np.int64)
    gains = np.zeros(maxm)
    nm = np.zeros(1, dtype=np.int32)
    rc = r.ref_cfg5_place(n_inst, capacity_blocks, queued, rounds, n_req, _p(t), _p(home), _p(blocks), maxm,
                          _p(moves), _p(gains), _p(nm))
    if rc != 0:
        raise ValueError(r.ref_last_error().decode())
    mv = [dict(round=int(moves[6 * i]), req_id=int(moves[6 * i + 1]), src_instance=int(moves[6 * i + 2]),
               dst_instance=int(moves[6 * i + 3]), num_blocks=int(moves[6 * i + 4]),
               moved_blocks=int(moves[6 * i + 5]), est_gain=float(gains[i])) for i in range(min(int(nm[0]), maxm))]
    return [int(h) for h in home], blocks.reshape(n_req, n_inst).tolist(), mv


SIM_INFINITE, SIM_STRAWMAN, SIM_STATIC = 0, 1, 2


def ref_sim_log(capacities: Sequence[int], requests, policy: int = SIM_STRAWMAN, horizon_s: float = 1e5):
    """Run the reference cluster simulator (run_simulation, simengine.cpp) on
    ``requests`` = [(arrival_s, prompt_tokens, output_tokens)] (ids 0..n-1)
    over instances with the given block capacities, default model
    (config.cpp:71-87). Returns the parsed JSONL event log."""
    import json
    r = ref()
    caps = np.ascontiguousarray(capacities, dtype=np.int64)
    arr = np.ascontiguousarray([q[0] for q in requests], dtype=np.float64)
    pr = np.ascontiguousarray([q[1] for q in requests], dtype=np.int64)
    out = np.ascontiguousarray([q[2] for q in requests], dtype=np.int64)
    p = ctypes.c_void_p()
    rc = r.ref_sim_log(len(caps), _p(caps), policy, len(requests), _p(arr), _p(pr), _p(out), horizon_s,
                       ctypes.byref(p))
    if rc != 0:
        raise ValueError(r.ref_last_error().decode())
    text = ctypes.string_at(p.value).decode()
    r.ref_string_free.argtypes = [ctypes.c_void_p]
    r.ref_string_free(p)
    return [json.loads(line) for line in text.splitlines() if line.strip()]
