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
    ascending instance id (config 5).
"""
from __future__ import annotations

from dataclasses import dataclass
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


def planner_placement(lens: Sequence[int], nranks: int, block_tokens: int,
                      retain_local_fraction: float = 0.5):
    """Config-5 placement, the reference policy restated on block counts.

    1. Dispatch: requests in order, each homed on the instance with the most
       free blocks, i.e. the least loaded (simengine.cpp:252-257); ties go to
       the lowest id.
    2. Lending (gManager plan_round, scheduler.cpp:215-295): an instance above
       the fair share ceil(total/N) lends blocks of its requests to instances
       below it, in ascending instance id, but every request keeps at least
       ceil(retain_local_fraction * blocks) at home (movable_blocks,
       scheduler.cpp:425-431; retain_local_fraction scheduler.hpp:56).
    Returns (homes, lent_blocks) for placement_from_moves.
    """
    nb = [_blocks(L, block_tokens) for L in lens]
    load = [0] * nranks
    homes = []
    for b in nb:
        h = min(range(nranks), key=lambda r: (load[r], r))
        homes.append(h)
        load[h] += b
    target = -(-sum(nb) // nranks)
    lent: Dict[Tuple[int, int], int] = {}
    for req, b in enumerate(nb):
        h = homes[req]
        keep_min = -(-int(retain_local_fraction * b * 1000) // 1000)
        movable = max(0, min(b - keep_min, load[h] - target))
        for r in range(nranks):
            if movable <= 0:
                break
            if r == h or load[r] >= target:
                continue
            take = min(movable, target - load[r])
            lent[(req, r)] = lent.get((req, r), 0) + take
            load[r] += take
            load[h] -= take
            movable -= take
    return homes, lent
