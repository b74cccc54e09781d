"""Host logic of the overflow-borrowing decode loop (decode_loop.ClusterDecodeLoop)
on CPU: every rank's replica of the loop drives a stand-in store that keeps
only page bookkeeping, so what is checked is what the loop asks the library
to do -- which rank appends each token, into which sequence, and the ranges
each rank decodes. Per step and request, the ranks' ranges must cover the
context exactly once, and each store's pages must match its instance's
ledger blocks."""
import random

import numpy as np

import paper_2401_02669_b200 as pb
from paper_2401_02669_b200.decode_loop import ClusterDecodeLoop


class PageStore:
    """The calls ClusterDecodeLoop makes on a pb.Store, with page accounting
    (blocks_for_tokens per sequence) and per-sequence token logs."""

    def __init__(self, rank, pages, page_tokens=16, hkv=2, dp=8):
        self.rank, self.capacity, self.page_tokens = rank, pages, page_tokens
        self.num_kv_heads, self.padded_dim, self.dtype, self.device = hkv, dp, pb.BF16, rank
        self.tokens = {}  # seq -> list of (request, position)
        self.next = 0
        self.decoded = []

    def used(self):
        return sum(pb.blocks_for_tokens(len(t), self.page_tokens) for t in self.tokens.values())

    def seq_create(self, tokens):
        s = self.next
        self.next += 1
        self.tokens[s] = [None] * tokens
        assert self.used() <= self.capacity
        return s

    def fill_synthetic(self, seq, seed, req, tok0, ak, av):
        self.tokens[seq] = [(req, tok0 + i) for i in range(len(self.tokens[seq]))]

    def synthetic_rows(self, reqs, pos, seed, k, v, ak, av):
        k[: len(reqs), 0, 0] = np.array(reqs) * 1_000_000 + np.array(pos)

    def kv_append(self, seqs, k, v, mem=0):
        for i, s in enumerate(seqs):
            code = int(k[i, 0, 0])
            self.tokens[s].append((code // 1_000_000, code % 1_000_000))
        assert self.used() <= self.capacity, "page pool overflow"

    def decode_sharded(self, ranges, rows, q, out, mem=0):
        self.decoded = [(r.seq, r.out_row, r.tok_begin, r.tok_end) for r in ranges]

    def seq_release(self, seq):
        del self.tokens[seq]


def run(world, caps, prompts, steps, seed):
    stores = [PageStore(r, caps[r]) for r in range(world)]
    loops = [ClusterDecodeLoop(stores[r], r, world, caps, seed) for r in range(world)]
    for lp in loops:
        lp.row_buffers = lambda n: (np.zeros((n, 2, 8), dtype=np.int64), np.zeros((n, 2, 8), dtype=np.int64))
    homes = {}
    for i, L in enumerate(prompts):
        h = 0 if i == 0 else -1
        oks = [lp.admit(i, i, L, home=h) for lp in loops]
        assert len(set(oks)) == 1
        homes[i] = loops[0].led.request(i)[0] if oks[0] else None
    for t in range(steps):
        parts = [lp.step(len(prompts), None, None) for lp in loops]
        assert all(p == parts[0] for p in parts)  # replicas agree
        for r in range(world):
            assert stores[r].used() == caps[r] - loops[r].led.free_blocks(r)
            for req in loops[r].running:  # the loop's incremental counts = the ledger's segments
                assert loops[r].local.get(req, 0) == loops[r].local_tokens(req)
                assert loops[r].ctx[req] == loops[r].led.request(req)[1]
        for req in loops[0].running:
            ctx = loops[0].led.request(req)[1]
            held = []
            for r in range(world):
                for seq, row, lo, hi in stores[r].decoded:
                    if row == req and hi > lo:
                        held += stores[r].tokens[seq][lo:hi]
            assert sorted(held) == [(req, p) for p in range(ctx)], (t, req)
    return loops


def test_overflow_loop_ranges_cover_every_context():
    for world in (2, 3, 4):
        loops = run(world, [46] + [80] * (world - 1), [700, 300, 200, 120, 40], 96, 5)
        assert loops[0].led.borrowed() > 0
        assert len({s[0] for s in loops[0].led.segments(0)}) > 1


def test_random_clusters_stall_instead_of_overflowing_pools():
    rng = random.Random(3)
    for _ in range(6):
        world = rng.randint(2, 4)
        caps = [rng.randint(20, 60) for _ in range(world)]
        prompts = [rng.randint(1, 16 * min(caps) // 2) for _ in range(rng.randint(2, 6))]
        loops = run(world, caps, prompts, 120, 9)
        total = sum(caps)
        used = sum(c - loops[0].led.free_blocks(i) for i, c in enumerate(caps))
        assert used <= total
