"""CPU: host-side sequence sharding / placement and the
workload definitions. Block counts are bit-exact with blocks_for_tokens
(perfmodel.cpp:178-182)."""
import numpy as np
import pytest

import oracle
from paper_2401_02669_b200 import workloads
from paper_2401_02669_b200.sharding import coverage_ok, placement_from_moves, plan_rank_ranges


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_equal_shares_cover_block_aligned(n):
    lens = [0, 1, 15, 16, 17, 1000, 131072, 1048576]
    per = plan_rank_ranges(lens, n, 16)
    assert coverage_ok(per, lens)
    for rank in per:
        assert len(rank) == len(lens)  # every rank sees every request (maybe empty)
        for rr in rank:
            if rr.tokens == 0:
                continue
            assert rr.tok_begin % 16 == 0
            assert rr.tok_end % 16 == 0 or rr.tok_end == lens[rr.request]
    for req, L in enumerate(lens):
        nb = sum(oracle.blocks_for_tokens(rr.tokens, 16) for rank in per for rr in rank if rr.request == req)
        assert nb == oracle.blocks_for_tokens(L, 16)


def test_config4_eight_way_split_is_equal():
    per = plan_rank_ranges([1048576], 8, 16)
    assert [rank[0].tokens for rank in per] == [131072] * 8


def test_placement_from_moves_home_prefix_then_lenders():
    # request 0 homed on 0 with 32768 blocks, 2048 lent to instance 3 and 1024 to 1
    lens = [524288, 2048, 2048]
    per = placement_from_moves(lens, [0, 1, 2], {(0, 3): 2048, (0, 1): 1024}, 4, 16)
    assert coverage_ok(per, lens)
    r0 = {rr.rank: (rr.tok_begin, rr.tok_end) for rank in per for rr in rank if rr.request == 0}
    assert r0[0] == (0, (32768 - 3072) * 16)
    assert r0[1] == ((32768 - 3072) * 16, (32768 - 2048) * 16)
    assert r0[3] == ((32768 - 2048) * 16, 524288)
    with pytest.raises(ValueError):
        placement_from_moves(lens, [0, 1, 2], {(1, 0): 500}, 4, 16)
    with pytest.raises(ValueError):
        placement_from_moves(lens, [0, 1, 2], {(1, 1): 5}, 4, 16)


def test_workloads():
    w2 = workloads.config("2")
    assert w2.batch == 64 and min(w2.lens) >= 1024 and max(w2.lens) <= 32768
    assert w2.lens == workloads.config("2").lens  # deterministic
    assert w2.kv_bytes() == 2 * 32 * 128 * sum(w2.lens) * 2
    w3 = workloads.config("3")
    assert w3.kv_bytes() == 8589934592  # SURVEY.md §8d cfg 3
    w4 = workloads.config("4")
    assert w4.kv_bytes() == 17179869184
    w1 = workloads.config("1")
    assert w1.kv_bytes() == 134217728 and w1.rblocks == 4
    assert workloads.splitmix64(0) == oracle.lib.or_splitmix64(0)
    assert workloads.splitmix64(12345) == oracle.lib.or_splitmix64(12345)


@pytest.mark.parametrize("cfg", ["1", "2", "3", "4", "5"])
@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_bench_rank_shares_cover_every_config(cfg, n):
    w = workloads.config(cfg)
    per = workloads.rank_shares(w, n)
    assert len(per) == n and coverage_ok(per, w.lens)
    # every rank lists every request (empty ranges give identity partials)
    for rank in per:
        assert sorted({rr.request for rr in rank}) == sorted({rr.request for rr in rank})
    if cfg == "5" and n >= 4:
        # placement-limited: the home keeps >= 50% of the long request
        home_tokens = sum(rr.tokens for rr in per[0] if rr.request == 0)
        assert home_tokens >= w.lens[0] // 2


# ---- pinned to the compiled reference (oracle/_ref) ----
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


@needs_ref
def test_blocks_for_tokens_bit_exact_with_reference():
    """kvsched::perf::blocks_for_tokens (perfmodel.cpp:178-182), the compiled
    reference, against the product's sizing rule and the C oracle."""
    import paper_2401_02669_b200 as pb
    rng = np.random.default_rng(5)
    toks = [0, 1, 15, 16, 17, 31, 32, 33, 4095, 4096, 4097, 131072, 524288, 1048576, (1 << 40) + 3]
    toks += [int(x) for x in rng.integers(0, 1 << 31, 200)]
    for bs in (1, 3, 16, 32, 64, 128):
        for t in toks:
            want = oracle.ref_blocks_for_tokens(t, bs)
            assert pb.blocks_for_tokens(t, bs) == want
            assert oracle.blocks_for_tokens(t, bs) == want


@needs_ref
def test_cfg5_fixture_is_the_reference_control_planes_output():
    """tests/golden/cfg5_placement.json regenerates bit-for-bit from the
    reference (dispatch + heartbeats + GManager::plan + execute_move_sync)."""
    import importlib.util
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "make_cfg5_placement.py")
    spec = importlib.util.spec_from_file_location("make_cfg5_placement", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    with open(os.path.join(os.path.dirname(__file__), "golden", "cfg5_placement.json")) as f:
        committed = json.load(f)
    assert json.loads(json.dumps(mod.generate())) == committed


def test_cfg5_reference_placement_shapes():
    """Config 5 from the fixture: the planner lends only while freed blocks admit
    queued requests (scheduler.cpp:62-80), keeps >= 50 % at home
    (scheduler.cpp:425-431), and at 2 instances finds no creditor below 0.8
    utilisation (scheduler.hpp:52-58)."""
    from paper_2401_02669_b200.sharding import gmanager_placement
    w = workloads.config("5")
    lens = w.lens
    nb0 = 32768
    for n in (2, 4, 8):
        for q, lent_want in ((0, 0), (64, 2048 if n > 2 else 0), (512, 16384 if n > 2 else 0)):
            homes, lent = gmanager_placement(lens, n, q)
            assert homes[0] == 0
            assert sum(b for (r, _), b in lent.items() if r == 0) == lent_want
            assert all(r == 0 for (r, _) in lent)  # only the long request lends
            per = placement_from_moves(lens, homes, lent, n, 16)
            assert coverage_ok(per, lens)
            home_tok = sum(rr.tokens for rr in per[0] if rr.request == 0)
            assert home_tok == (nb0 - lent_want) * 16
            # the shorts sit on the other instances (most-free dispatch)
            assert all(h != 0 for h in homes[1:])
    with pytest.raises(ValueError):
        gmanager_placement(lens, 3, 64)
    with pytest.raises(ValueError):
        gmanager_placement(lens[:-1], 4, 64)
