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
