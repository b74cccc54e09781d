"""CPU: pin the oracle (oracle/dattn_oracle.c) to the reference.

1. Against the golden vectors in tests/golden/reference_vectors.json, which
   tests/golden/make_golden.py produced by running the unmodified reference
   (oracle/_ref): bit-exact for every fp64 result, integer map and RNG draw.
2. Against the live reference build when oracle/_ref is present (random cases).
3. The reference's own hot-path test suite (proj/tests/test_distattention.cpp)
   compiled against the reference -- proves the build recipe and doctest shim.
"""
import hashlib
import json
import os
import subprocess

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "reference_vectors.json")))
ROOT = os.path.dirname(HERE)


def unhex(xs):
    return np.array([float.fromhex(x) for x in xs])


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def bits_equal(a, b):
    return np.array_equal(np.asarray(a, dtype=np.float64).view(np.uint64),
                          np.asarray(b, dtype=np.float64).view(np.uint64))


@pytest.mark.parametrize("case", GOLD["micro_attention"], ids=lambda c: f"seed{c['seed']}-L{c['seq']}-d{c['d']}")
def test_micro_attention_bit_exact(case):
    k, v = oracle.synth_kv(case["seed"], 0, 0, 0, case["seq"], case["d"], case["amp_k"], 2.0, case["dtype"])
    q = oracle.synth_q(case["seed"], 0, 0, case["d"], 1.0, case["dtype"])
    assert digest(q, k, v) == case["input_digest"], "generator drifted"
    m, e, ma, sp = oracle.micro_attention(q, k, v, case["scale"])
    assert m == float.fromhex(case["m"]) and e == float.fromhex(case["e"])
    assert bits_equal(ma, unhex(case["ma"]))
    assert sp == case["seq_p"]
    assert bits_equal(oracle.naive_attention(q, k, v, case["scale"]), unhex(case["naive"]))


@pytest.mark.parametrize("case", GOLD["aggregate"], ids=lambda c: f"seed{c['seed']}")
def test_combine_and_aggregate_bit_exact(case):
    d = case["d"]
    k, v = oracle.synth_kv(case["seed"], 1, 0, 0, case["seq"], d, 25.0 if case["seed"] % 2 else 1.0, 2.0,
                           oracle.F64)
    q = oracle.synth_q(case["seed"], 0, 0, d, 1.0, oracle.F64)
    assert digest(q, k, v) == case["input_digest"]
    cuts = case["cuts"]
    parts = [oracle.micro_attention(q, k[a:b], v[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
    for got, want in zip(parts, case["parts"]):
        assert got[0] == float.fromhex(want["m"]) and got[1] == float.fromhex(want["e"])
        assert bits_equal(got[2], unhex(want["ma"])) and got[3] == want["seq_p"]
    acc = parts[0]
    for nxt in parts[1:]:
        acc = oracle.combine(acc, nxt)
    f = case["fold"]
    assert acc[0] == float.fromhex(f["m"]) and acc[1] == float.fromhex(f["e"]) and acc[3] == f["seq_p"]
    assert bits_equal(acc[2], unhex(f["ma"]))
    assert bits_equal(oracle.aggregate(parts), unhex(case["aggregate"]))


@pytest.mark.parametrize("case", GOLD["multi_head_attention"], ids=lambda c: f"seed{c['seed']}-{c['hq']}x{c['hkv']}")
def test_multi_head_attention_bit_exact(case):
    d, hq, hkv, seq = case["d"], case["hq"], case["hkv"], case["seq"]
    K = np.zeros((hkv, seq, d))
    V = np.zeros((hkv, seq, d))
    for h in range(hkv):
        K[h], V[h] = oracle.synth_kv(case["seed"], 2, h, 0, seq, d, 1.0, 2.0, oracle.BF16)
    Q = np.stack([oracle.synth_q(case["seed"], 0, h, d, 1.0, oracle.BF16) for h in range(hq)])
    assert digest(Q, K, V) == case["input_digest"]
    want = unhex(case["out"]).reshape(hq, d)
    for h in range(hq):  # distattention.cpp:197-206, restated
        kvh = oracle.gqa_kv_head(h, hq, hkv)
        cuts = case["cuts"][kvh]
        parts = [oracle.micro_attention(Q[h], K[kvh, a:b], V[kvh, a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
        assert bits_equal(oracle.aggregate(parts), want[h])


def test_gqa_map_and_wire():
    for c in GOLD["gqa_kv_head"]:
        assert [oracle.gqa_kv_head(h, c["hq"], c["hkv"]) for h in range(c["hq"])] == c["map"]
    for w in GOLD["wire"]:
        d = w["d"]
        ma = np.arange(d, dtype=np.float64) * 0.25 - 1.0
        buf = np.zeros(d + 2)
        oracle.lib.or_serialize_partial(-1.5, 2.75, ma.ctypes.data, d, buf.ctypes.data)
        assert w["nbytes"] == (d + 2) * 8
        assert bits_equal(buf, unhex(w["payload"]))
        assert oracle.lib.or_deserialize_seq_p(buf.ctypes.data) == 1
    ident = np.array([-np.inf, 0.0, 0.0])
    assert oracle.lib.or_deserialize_seq_p(ident.ctypes.data) == 0


@pytest.mark.parametrize("case", GOLD["rng"], ids=lambda c: f"seed{c['seed']}")
def test_rng_streams_bit_exact(case):
    a, b, c, e = (oracle.Rng(case["seed"] + i) for i in range(4))
    assert [str(a.next_u64()) for _ in range(64)] == case["u64"]
    assert [b.uniform01() for _ in range(64)] == list(unhex(case["uniform01"]))
    assert bits_equal([c.normal() for _ in range(64)], unhex(case["normal"]))
    assert [e.uniform_int(-5, 2048) for _ in range(64)] == case["uniform_int_m5_2048"]


def test_decode_batch_bit_exact():
    g = GOLD["decode_batch"]
    out = oracle.decode_batch(g["seed"], g["lens"], g["hq"], g["hkv"], g["d"], dtype=g["dtype"],
                              amp_q=g["amp_q"], amp_k=g["amp_k"], amp_v=g["amp_v"], seg_tokens=g["seg_tokens"],
                              threads=4)
    for b in range(len(g["lens"])):
        assert bits_equal(out[b], unhex(g["out"][b]).reshape(g["hq"], g["d"]))


def test_generator_values():
    for c in GOLD["generator_values"]:
        assert oracle.lib.or_synth_value(*c["args"]) == float.fromhex(c["value"])


def test_generator_ranges_and_rounding():
    k, v = oracle.synth_kv(3, 0, 0, 0, 4096, 128, 1.0, 2.0, oracle.BF16)
    # bf16 rounding can reach the interval end
    assert k.min() >= -1.0 and k.max() <= 1.0 and v.min() >= -2.0 and v.max() <= 2.0
    # bf16-rounded: the low 16 bits of the fp32 image are zero
    assert np.all((k.astype(np.float32).view(np.uint32) & 0xFFFF) == 0)
    assert abs(k.mean()) < 0.01 and 0.3 < k.std() < 0.65


def test_blocks_for_tokens():
    for t, b in [(0, 16), (1, 16), (16, 16), (17, 16), (131072, 16), (1048576, 16), (5, 3)]:
        assert oracle.blocks_for_tokens(t, b) == -(-t // b)


@pytest.mark.skipif(not oracle.ref_available(), reason="reference build (oracle/_ref) not present")
def test_oracle_matches_live_reference_random():
    import ctypes
    R = oracle.ref()
    rng = np.random.default_rng(5)
    for _ in range(60):
        d = int(rng.integers(1, 140))
        seq = int(rng.integers(0, 400))
        amp = float(rng.choice([1.0, 30.0]))
        k = np.ascontiguousarray(rng.uniform(-amp, amp, (seq, d)))
        v = np.ascontiguousarray(rng.uniform(-2, 2, (seq, d)))
        q = np.ascontiguousarray(rng.uniform(-1, 1, d))
        scale = float(rng.choice([0.0, 0.7]))
        m, e = np.zeros(1), np.zeros(1)
        ma = np.zeros(d)
        sp = np.zeros(1, dtype=np.int64)
        assert R.ref_micro_attention(q.ctypes.data, k.ctypes.data, v.ctypes.data, seq, d, scale,
                                     m.ctypes.data, e.ctypes.data, ma.ctypes.data, sp.ctypes.data) == 0
        om, oe, oma, osp = oracle.micro_attention(q, k, v, scale)
        assert bits_equal([om, oe], [m[0], e[0]]) and bits_equal(oma, ma) and osp == sp[0]


REF_TEST = os.path.join(ROOT, "oracle", "_ref", "test_distattention_ref")


@pytest.mark.skipif(not os.path.exists(REF_TEST), reason="reference test binary not built")
def test_reference_own_suite_against_reference():
    r = subprocess.run([REF_TEST], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:]
    assert "10 passed | 0 failed" in r.stdout
