"""Generate tests/golden/reference_vectors.json from the REFERENCE itself.

Runs the unmodified reference (oracle/_ref/libkvsched_ref.so, compiled by
oracle/Makefile from /root/reference/proj/src/{distattention,verify,trace}.cpp)
on seeded inputs and records its outputs bit-exactly (float.hex). The
reference ships no stored golden vectors, so these fixtures
are the pin for the C restatement in oracle/dattn_oracle.c
(tests/test_oracle.py) and, through it, for the GPU parity tests.

Inputs are produced by the counter-hash generator (oracle.synth_kv/synth_q)
or by explicit small literal arrays; a digest of every generated input is
stored too so the generator itself is pinned.

Usage (in the container that has /root/reference):  python tests/golden/make_golden.py
"""
from __future__ import annotations

import ctypes
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_vectors.json")


def hexs(a):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).ravel()]


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def p(a):
    return a.ctypes.data


def main():
    R = oracle.ref()
    gold = {"generator": "tests/golden/make_golden.py", "reference": "oracle/_ref/libkvsched_ref.so"}

    # 1. compute_micro_attention / naive_attention over generated segments
    ma_cases = []
    for (seed, seq, d, scale, ak, dt) in [
        (1, 1, 1, 0.0, 1.0, oracle.F64), (2, 7, 3, 0.0, 1.0, oracle.F32), (3, 64, 16, 0.3, 1.0, oracle.BF16),
        (4, 300, 128, 0.0, 1.0, oracle.BF16), (5, 257, 64, 0.0, 30.0, oracle.BF16),
        (6, 1000, 128, 0.0, 5.0, oracle.F32), (7, 33, 129, 0.0, 1.0, oracle.F64),
        (8, 2048, 32, 1.5, 1.0, oracle.BF16),
    ]:
        k, v = oracle.synth_kv(seed, 0, 0, 0, seq, d, ak, 2.0, dt)
        q = oracle.synth_q(seed, 0, 0, d, 1.0, dt)
        m, e = np.zeros(1), np.zeros(1)
        ma = np.zeros(d)
        sp = np.zeros(1, dtype=np.int64)
        assert R.ref_micro_attention(p(q), p(k), p(v), seq, d, scale, p(m), p(e), p(ma), p(sp)) == 0
        out = np.zeros(d)
        assert R.ref_naive_attention(p(q), p(k), p(v), seq, d, scale, p(out)) == 0
        ma_cases.append({"seed": seed, "seq": seq, "d": d, "scale": scale, "amp_k": ak, "dtype": dt,
                         "input_digest": digest(q, k, v), "m": float(m[0]).hex(), "e": float(e[0]).hex(),
                         "ma": hexs(ma), "seq_p": int(sp[0]), "naive": hexs(out)})
    gold["micro_attention"] = ma_cases

    # 2. combine / aggregate over partials of disjoint cuts, incl. identities
    agg_cases = []
    for (seed, seq, d, cuts) in [(11, 50, 8, [0, 10, 10, 37, 50]), (12, 200, 64, [0, 1, 199, 200]),
                                 (13, 96, 24, [0, 96]), (14, 500, 128, [0, 0, 250, 250, 500, 500])]:
        k, v = oracle.synth_kv(seed, 1, 0, 0, seq, d, 25.0 if seed % 2 else 1.0, 2.0, oracle.F64)
        q = oracle.synth_q(seed, 0, 0, d, 1.0, oracle.F64)
        parts = []
        for a, b in zip(cuts[:-1], cuts[1:]):
            m, e = np.zeros(1), np.zeros(1)
            ma = np.zeros(d)
            sp = np.zeros(1, dtype=np.int64)
            kk, vv = np.ascontiguousarray(k[a:b]), np.ascontiguousarray(v[a:b])
            assert R.ref_micro_attention(p(q), p(kk), p(vv), b - a, d, 0.0, p(m), p(e), p(ma), p(sp)) == 0
            parts.append((float(m[0]), float(e[0]), ma.copy(), int(sp[0])))
        # pairwise left fold with combine_partials
        acc = parts[0]
        for nxt in parts[1:]:
            om, oe, osq = np.zeros(1), np.zeros(1), np.zeros(1, dtype=np.int64)
            oma = np.zeros(d)
            ama, bma = np.ascontiguousarray(acc[2]), np.ascontiguousarray(nxt[2])
            assert R.ref_combine(acc[0], acc[1], p(ama), acc[3], nxt[0], nxt[1], p(bma), nxt[3], d,
                                 p(om), p(oe), p(oma), p(osq)) == 0
            acc = (float(om[0]), float(oe[0]), oma.copy(), int(osq[0]))
        M = np.array([x[0] for x in parts])
        E = np.array([x[1] for x in parts])
        MA = np.ascontiguousarray(np.stack([x[2] for x in parts]))
        SP = np.array([x[3] for x in parts], dtype=np.int64)
        out = np.zeros(d)
        assert R.ref_aggregate(len(parts), p(M), p(E), p(MA), p(SP), d, p(out)) == 0
        agg_cases.append({"seed": seed, "seq": seq, "d": d, "cuts": cuts, "input_digest": digest(q, k, v),
                          "parts": [{"m": x[0].hex(), "e": x[1].hex(), "ma": hexs(x[2]), "seq_p": x[3]}
                                    for x in parts],
                          "fold": {"m": acc[0].hex(), "e": acc[1].hex(), "ma": hexs(acc[2]), "seq_p": acc[3]},
                          "aggregate": hexs(out)})
    gold["aggregate"] = agg_cases

    # 3. multi_head_attention with per-kv-head cut lists (GQA / MQA / MHA)
    mha_cases = []
    for (seed, seq, d, hq, hkv, cuts) in [
        (21, 40, 16, 4, 4, [[0, 40], [0, 5, 40], [0, 39, 40], [0, 0, 20, 40]]),
        (22, 64, 32, 4, 1, [[0, 16, 32, 48, 64]]),
        (23, 130, 128, 8, 2, [[0, 64, 130], [0, 1, 2, 130]]),
        (24, 300, 128, 64, 8, [[0, 100, 300]] * 8),
    ]:
        K = np.zeros((hkv, seq, d))
        V = np.zeros((hkv, seq, d))
        for h in range(hkv):
            K[h], V[h] = oracle.synth_kv(seed, 2, h, 0, seq, d, 1.0, 2.0, oracle.BF16)
        Q = np.stack([oracle.synth_q(seed, 0, h, d, 1.0, oracle.BF16) for h in range(hq)])
        flat = np.ascontiguousarray(np.concatenate([np.array(c, dtype=np.int64) for c in cuts]))
        ncuts = np.ascontiguousarray([len(c) - 1 for c in cuts], dtype=np.int32)
        out = np.zeros((hq, d))
        K, V, Q = map(np.ascontiguousarray, (K, V, Q))
        assert R.ref_multi_head_attention(p(Q), p(K), p(V), seq, hq, hkv, d, 0.0, p(flat), p(ncuts), p(out)) == 0
        mha_cases.append({"seed": seed, "seq": seq, "d": d, "hq": hq, "hkv": hkv, "cuts": cuts,
                          "input_digest": digest(Q, K, V), "out": hexs(out)})
    gold["multi_head_attention"] = mha_cases

    # 4. gqa_kv_head and wire format
    gq = []
    for (hq, hkv) in [(4, 4), (4, 1), (8, 2), (64, 8), (12, 4)]:
        row = []
        for h in range(hq):
            o = ctypes.c_int()
            assert R.ref_gqa_kv_head(h, hq, hkv, ctypes.byref(o)) == 0
            row.append(o.value)
        gq.append({"hq": hq, "hkv": hkv, "map": row})
    gold["gqa_kv_head"] = gq
    wire = []
    for d in (1, 3, 32, 64, 128):
        ma = np.arange(d, dtype=np.float64) * 0.25 - 1.0
        buf = np.zeros(d + 2)
        n = ctypes.c_int64()
        assert R.ref_serialize_partial(-1.5, 2.75, p(ma), d, p(buf), ctypes.byref(n)) == 0
        wire.append({"d": d, "nbytes": n.value, "payload": hexs(buf)})
    gold["wire"] = wire

    # 5. sim::Rng streams
    rng = []
    for seed in (1, 7, 20260816, 777001):
        n = 64
        u64 = np.zeros(n, dtype=np.uint64)
        u01, nor = np.zeros(n), np.zeros(n)
        ints = np.zeros(n, dtype=np.int64)
        assert R.ref_rng_draws(seed, n, p(u64), p(u01), p(nor), p(ints), -5, 2048) == 0
        rng.append({"seed": seed, "u64": [str(int(x)) for x in u64], "uniform01": hexs(u01),
                    "normal": hexs(nor), "uniform_int_m5_2048": [int(x) for x in ints]})
    gold["rng"] = rng

    # 6. the reference's randomized verifier (verify.cpp:170-186)
    ver = []
    for trials, seed in ((200, 7), (1000, 1)):
        mx, mean = np.zeros(1), np.zeros(1)
        ok = ctypes.c_int()
        assert R.ref_verify_attention(trials, seed, 1e-6, p(mx), p(mean), ctypes.byref(ok)) == 0
        ver.append({"trials": trials, "seed": seed, "max_rel_err": float(mx[0]), "mean_rel_err": float(mean[0]),
                    "pass": bool(ok.value)})
    gold["verify"] = ver

    # 7. a paged-decode batch in miniature (config-2 style, bf16 values):
    #    the reference's multi_head_attention per request, 64-token rBlocks
    lens = [1, 17, 300, 1000]
    hq = hkv = 4
    d = 128
    seed = 99
    outs = []
    for b, L in enumerate(lens):
        K = np.zeros((hkv, L, d))
        V = np.zeros((hkv, L, d))
        for h in range(hkv):
            K[h], V[h] = oracle.synth_kv(seed, b, h, 0, L, d, 1.0, 2.0, oracle.BF16)
        Q = np.stack([oracle.synth_q(seed, b, h, d, 1.0, oracle.BF16) for h in range(hq)])
        cuts = list(range(0, L, 64)) + [L]
        flat = np.ascontiguousarray(np.array(cuts * hkv, dtype=np.int64))
        ncuts = np.ascontiguousarray([len(cuts) - 1] * hkv, dtype=np.int32)
        out = np.zeros((hq, d))
        K, V, Q = map(np.ascontiguousarray, (K, V, Q))
        assert R.ref_multi_head_attention(p(Q), p(K), p(V), L, hq, hkv, d, 0.0, p(flat), p(ncuts), p(out)) == 0
        outs.append(hexs(out))
    gold["decode_batch"] = {"seed": seed, "lens": lens, "hq": hq, "hkv": hkv, "d": d, "seg_tokens": 64,
                            "dtype": oracle.BF16, "amp_q": 1.0, "amp_k": 1.0, "amp_v": 2.0, "out": outs}

    # 8. raw generator values (pins the CPU/GPU counter-hash generator)
    gen = []
    for (seed, tensor, seq, head, tok, dim, amp, dt) in [
        (1, 1, 0, 0, 0, 0, 1.0, 0), (1, 2, 3, 5, 1000, 127, 2.0, 0), (7, 1, 63, 31, 32767, 64, 30.0, 0),
        (7, 3, 15, 63, 0, 5, 1.0, 1), (123, 2, 1, 7, 1048575, 100, 2.0, 2), (5, 1, 0, 0, 12, 3, 5.0, 1)]:
        val = oracle.lib.or_synth_value(seed, tensor, seq, head, tok, dim, amp, dt)
        gen.append({"args": [seed, tensor, seq, head, tok, dim, amp, dt], "value": float(val).hex()})
    gold["generator_values"] = gen

    with open(OUT, "w") as f:
        json.dump(gold, f, indent=1)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
