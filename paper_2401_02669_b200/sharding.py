"""Sequence sharding of rBlocks across the GPUs of one box.

DistAttention splits a request's KV along the sequence: every instance that
holds some of the request's blocks computes micro-attention partials over its
own tokens and only the (m, e, ma) partials travel. Partition
invariance (exhaustive test proj/tests/test_distattention.cpp:
107-131) makes any contiguous cover of [0, L) give the same output, so the
assignment below only has to be deterministic and block aligned.

Two placements:
  * ``plan_rank_ranges``: equal contiguous shares in whole blocks (configs 3, 4).
  * ``placement_from_moves``: the gManager's block counts per (request,
    instance) (MoveDirective, proj/include/kvsched/scheduler.hpp:68-75; the
    RManager ledgers controlplane.hpp:212-215) turned into token ranges: the
    home instance keeps the prefix, lenders take consecutive block ranges in
    ascending instance id (config 5). The counts for config 5 are the
    reference control plane's own output (tests/golden/cfg5_placement.json,
    made by tests/golden/make_cfg5_placement.py from oracle/_ref), read by
    ``gmanager_placement``.
"""
from __future__ import annotations

from dataclasses import dataclass
import json
import os
from typing import Dict, List, Sequence, Tuple


@dataclass(frozen=True)
class RankRange:
    request: int
    rank: int
    tok_begin: int
    tok_end: int

    @property
    def tokens(self) -> int:
        return self.tok_end - self.tok_begin


def _blocks(tokens: int, block: int) -> int:
    return (tokens + block - 1) // block  # perfmodel.cpp:178-182


def plan_rank_ranges(lens: Sequence[int], nranks: int, block_tokens: int) -> List[List[RankRange]]:
    """Split every request [0, L) into ``nranks`` contiguous block-aligned
    shares; rank r gets blocks [r*ceil(B/n), (r+1)*ceil(B/n)). Returns the
    ranges per rank (possibly empty, i.e. identity partials)."""
    if nranks < 1 or block_tokens < 1:
        raise ValueError("nranks and block_tokens must be >= 1")
    out: List[List[RankRange]] = [[] for _ in range(nranks)]
    for req, L in enumerate(lens):
        nb = _blocks(L, block_tokens)
        per = _blocks(nb, nranks) if nb else 0
        for r in range(nranks):
            b0, b1 = min(nb, r * per), min(nb, (r + 1) * per)
            lo, hi = min(L, b0 * block_tokens), min(L, b1 * block_tokens)
            out[r].append(RankRange(req, r, lo, hi))
    return out


def placement_from_moves(lens: Sequence[int], home: Sequence[int],
                         lent_blocks: Dict[Tuple[int, int], int], nranks: int,
                         block_tokens: int) -> List[List[RankRange]]:
    """Token ranges per rank from a block placement.

    ``home[req]`` is the request's home instance; ``lent_blocks[(req, inst)]``
    the blocks of ``req`` hosted on ``inst`` (the ``hosted_`` ledger of that
    instance's RManager). The home keeps the leading blocks; hosts take the
    following blocks in ascending instance order. Raises ``ValueError`` when
    more blocks are lent than the request has.
    """
    out: List[List[RankRange]] = [[] for _ in range(nranks)]
    for req, L in enumerate(lens):
        nb = _blocks(L, block_tokens)
        lenders = sorted((inst, n) for (r, inst), n in lent_blocks.items() if r == req and n > 0)
        lent = sum(n for _, n in lenders)
        if lent > nb:
            raise ValueError(f"request {req}: {lent} blocks lent but only {nb} exist")
        if any(inst == home[req] for inst, _ in lenders):
            raise ValueError("a request cannot be hosted on its own home instance")
        keep = nb - lent
        cur = 0
        spans = [(home[req], keep)] + lenders
        for inst, n in spans:
            lo, hi = min(L, cur * block_tokens), min(L, (cur + n) * block_tokens)
            out[inst].append(RankRange(req, inst, lo, hi))
            cur += n
    return out


def coverage_ok(per_rank: List[List[RankRange]], lens: Sequence[int]) -> bool:
    """Every request covered exactly once by disjoint contiguous ranges."""
    for req, L in enumerate(lens):
        spans = sorted((rr.tok_begin, rr.tok_end) for rank in per_rank for rr in rank
                       if rr.request == req and rr.tok_end > rr.tok_begin)
        cur = 0
        for lo, hi in spans:
            if lo != cur:
                return False
            cur = hi
        if cur != L:
            return False
    return True


CFG5_PLACEMENT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                              "cfg5_placement.json")


def gmanager_placement(lens: Sequence[int], nranks: int, queued: int, block_tokens: int = 16,
                       path: str = CFG5_PLACEMENT):
    """Config 5's (homes, lent_blocks) as the reference control plane placed
    them: dispatch to the most-free instance, heartbeats, GManager::plan +
    execute_move_sync until no move (see tests/golden/make_cfg5_placement.py).
    Returns inputs for ``placement_from_moves``. Raises ``ValueError`` when the
    fixture has no entry for (nranks, queued) or describes other lengths."""
    with open(path) as f:
        j = json.load(f)
    d = j["lens"]
    if list(lens) != [d["long"]] + [d["short"]] * d["n_short"] or block_tokens != j["block_tokens"]:
        raise ValueError("the config-5 placement fixture describes another batch")
    key = f"n{nranks}_q{queued}"
    if key not in j["placements"]:
        raise ValueError(f"no reference placement for {nranks} instances and queue {queued} "
                         f"(have {sorted(j['placements'])})")
    p = j["placements"][key]
    lent = {(r, i): b for r, i, b in p["hosted"]}
    return list(p["homes"]), lent
