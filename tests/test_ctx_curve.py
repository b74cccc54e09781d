"""The B200-measured attention rate g(S) plugs into the reference perf model
(SURVEY.md §8f row 4).

profiles/r1_ctx_rate_curve.json is written on a B200 by
tools/calibrate_ctx_curve.py. Here (CPU) the curve is put into the reference's
default cluster config (config.cpp:71-87) and fed through the reference's own
parser (parse_cluster_config, which validates every curve) and layer_time
(perfmodel.cpp:105-113): the modelled attention share of a layer must equal the
measured B200 decode time at every sampled context size.
"""
import json
import os

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CURVE = os.path.join(ROOT, "profiles", "r1_ctx_rate_curve.json")

pytestmark = pytest.mark.skipif(not (oracle.ref_available() and os.path.exists(CURVE)),
                                reason="needs oracle/_ref and the measured curve")


def _config(doc):
    cfg = json.loads(oracle.ref_default_config(4, 40000))
    cfg["ctx_rate_curve"] = doc["ctx_rate_curve"]
    cfg["model"]["attn_work_per_ctx_token"] = 1.0
    cfg["model"]["n_layers"] = doc["model"]["n_layers"]
    cfg["model"]["kv_bytes_per_token"] = float(doc["model"]["kv_bytes_per_token_all_layers"])
    return cfg


def _f_default(beta):
    # default_batch_curve (perfmodel.cpp:50-56) at its sample points (powers of 2)
    return 2000.0 * beta / (beta + 8.0)


def test_curve_shape():
    doc = json.load(open(CURVE))
    xs = [x for x, _ in doc["ctx_rate_curve"]]
    assert len(xs) >= 2 and all(b > a for a, b in zip(xs, xs[1:]))
    assert all(r > 0 for _, r in doc["ctx_rate_curve"])
    # HBM-bound decode: the rate grows with S until the launch overhead is
    # amortised, then saturates near the copy bandwidth / KV bytes per token
    rates = [r for _, r in doc["ctx_rate_curve"]]
    assert rates[-1] > 3 * rates[0]
    peak_tok_s = 8.0e12 / (2 * 32 * 128 * 2)
    assert rates[-1] < peak_tok_s


def test_reference_parser_accepts_and_layer_time_matches():
    doc = json.load(open(CURVE))
    text = json.dumps(_config(doc))
    xs = [s["S"] for s in doc["samples"]]
    for s in doc["samples"]:
        beta, S = s["batch"], s["S"]
        lens = [S // beta + (1 if i < S % beta else 0) for i in range(beta)]
        g, lt, n_layers = oracle.ref_config_eval(text, xs, lens)
        assert n_layers == doc["model"]["n_layers"]
        assert g == pytest.approx([r for _, r in doc["ctx_rate_curve"]], rel=1e-12)
        attn = lt - 1.0 * beta / _f_default(beta)  # workload_per_token = 1
        assert attn == pytest.approx(s["ms"] * 1e-3, rel=1e-9)


def test_reference_parser_rejects_bad_curve():
    doc = json.load(open(CURVE))
    cfg = _config(doc)
    cfg["ctx_rate_curve"] = [[1.0, 5.0], [1.0, 6.0]]
    with pytest.raises(ValueError, match="strictly increasing"):
        oracle.ref_config_eval(json.dumps(cfg), [1.0], [1])
