"""CPU checks of the decode-plan builder (dattn_store::build_plan in
csrc/dattn_engine.cpp), run on the host without a GPU via tests/plan_probe.cpp
linked against libdattn.so: chunk rule, item counts, the longest-first claim
table, chunks per row, and the per-(row, kv head) completion counts that the
fused merge and K6 rely on."""
import json
import math
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2401_02669_b200", "_lib")
NCCL = "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl"
CUDA = "/usr/local/cuda"


@pytest.fixture(scope="module")
def plans(tmp_path_factory):
    if not (shutil.which("g++") and os.path.exists(os.path.join(LIB, "libdattn.so"))
            and os.path.isdir(os.path.join(NCCL, "include"))):
        pytest.skip("needs g++, the built libdattn.so and the NCCL headers")
    exe = str(tmp_path_factory.mktemp("probe") / "plan_probe")
    cmd = ["g++", "-std=c++20", "-O1", f"-I{ROOT}/include", f"-I{ROOT}/paper_2401_02669_b200/csrc",
           f"-I{NCCL}/include", f"-I{CUDA}/include", os.path.join(ROOT, "tests", "plan_probe.cpp"), "-o", exe,
           f"-L{LIB}", "-ldattn", f"-L{CUDA}/lib64", "-lcudart", f"-Wl,-rpath,{LIB}", f"-Wl,-rpath,{CUDA}/lib64",
           f"-Wl,-rpath,{NCCL}/lib"]
    subprocess.run(cmd, check=True, capture_output=True)
    out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    return {d["name"]: d for d in map(json.loads, out.splitlines())}


def _chunk_ok(c):
    return 512 <= c <= 8192 and c & (c - 1) == 0 and c % 16 == 0


def test_ragged_batch_claims_longest_first(plans):
    p = plans["ragged_k2"]
    lens = [1024, 32768, 5000, 17, 20000, 8192, 300, 12345]
    C = p["chunk"]
    assert _chunk_ok(C)
    assert p["items"] == sum(math.ceil(L / C) for L in lens) * 32
    assert p["table"]
    items = [i for i, _ in p["order"]]
    toks = [t for _, t in p["order"]]
    assert sorted(items) == list(range(p["items"]))  # a permutation
    assert all(a >= b for a, b in zip(toks, toks[1:]))  # longest first
    # equal lengths keep the natural order (kv heads of a chunk stay adjacent)
    for (i0, t0), (i1, t1) in zip(p["order"], p["order"][1:]):
        if t0 == t1:
            assert i1 > i0
    assert p["row_chunks"] == [math.ceil(L / C) for L in lens]
    assert p["expect"] == [math.ceil(L / C) for L in lens for _ in range(32)]


def test_uniform_batch_ends_on_quarter_chunks(plans):
    """Equal lengths: full chunks claimed in natural order (kv heads of a chunk
    adjacent), then each range's last chunk cut into four C/4 sub-ranges that
    run last, so the launch drains over a quarter chunk, not a full one; the
    sub-ranges tile the range exactly (partition invariance)."""
    p = plans["uniform_k2"]
    C = p["chunk"]
    assert C == 8192 and p["table"]
    per_range = 131072 // C  # 16 chunks per request
    full = 16 * (per_range - 1) * 8
    assert p["items"] == full + 16 * 4 * 8
    order = p["order"]
    assert [t for _, t in order[:full]] == [C] * full
    assert [i for i, _ in order[:full]] == sorted(i for i, _ in order[:full])
    assert [t for _, t in order[full:]] == [C // 4] * (16 * 4 * 8)
    assert sorted(i for i, _ in order) == list(range(p["items"]))
    for req in range(16):  # every request still covered exactly once, in order
        spans = [(lo, hi) for seq, row, kvh, lo, hi in p["ranges"] if row == req]
        assert spans[0][0] == 0 and spans[-1][1] == 131072
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert p["row_chunks"] == [per_range - 1 + 4] * 16
    assert p["expect"] == [per_range - 1 + 4] * (16 * 8)


def test_small_fp32_batch_uses_the_chunk_floor(plans):
    p = plans["cfg1_k1"]
    assert p["chunk"] == 512
    assert p["items"] == 4 * (1024 // 512) * 32
    assert p["row_chunks"] == [8]


def test_kv_head_ranges_empty_ranges_and_rows_without_ranges(plans):
    p = plans["kvh_empty"]
    C = p["chunk"]
    assert _chunk_ok(C)
    c0, c1, c3 = math.ceil(3000 / C), math.ceil(100 / C), math.ceil((9000 - 5) / C)
    assert p["row_chunks"] == [c0 + c1, 0, 0, c3]
    assert p["expect"] == [0, c0, 0, c1] + [0] * 4 + [0] * 4 + [c3] * 4
    assert p["items"] == c0 + c1 + 4 * c3
    assert sorted(i for i, _ in p["order"]) == list(range(p["items"]))
