"""A sharded decode loop whose KV grows through the cluster block ledger
(DESIGN.md §5.5).

Every step each running request gets one new token. Where that token's K/V
goes is the reference simulator's ensure_slot (simengine.cpp:318-354),
evaluated by the block ledger of the C library (dattn_ledger_*): at the
request's home while the home has a free block, otherwise -- overflow
borrowing -- in a block on another GPU (an existing host first, then the
most-free instance none of whose own requests borrow, then any instance with
room). The ledger is replicated on every rank: all ranks apply the same
admissions, slot requests and advances in the same order, so their copies
stay identical without messages (the reference keeps one engine-wide view,
simengine.cpp:186-232). Each rank's page pool is sized to its instance's
capacity, so its free pages equal the ledger's free blocks at every step.

The rank that holds a request's next slot appends the token's K/V rows
(dattn_kv_append) to its sequence for that request -- the home sequence, or
a hosted sequence created at the first borrow -- and every rank decodes over
the tokens it holds (dattn_decode_sharded): the partials of home and hosted
blocks merge exactly as a sequence-sharded request's do (DistAttention,
PAPER.md:522-567). The new rows are the generator's values at the token's
position (K4), so the oracle can check any step.
"""
from __future__ import annotations

from typing import Dict, List, Sequence

from . import BF16, F32, MEM_DEVICE, Ledger, Range, Store


class ClusterDecodeLoop:
    def __init__(self, store: Store, rank: int, nranks: int, capacity_blocks: Sequence[int], seed: int,
                 amp_k: float = 1.0, amp_v: float = 2.0, allow_borrow: bool = True):
        if len(capacity_blocks) != nranks:
            raise ValueError("one capacity per rank")
        self.st, self.rank, self.nranks = store, rank, nranks
        self.led = Ledger(capacity_blocks, store.page_tokens)
        self.seed, self.amp_k, self.amp_v = seed, amp_k, amp_v
        self.allow_borrow = allow_borrow
        self.seqs: Dict[int, int] = {}  # request -> this rank's sequence (home or hosted)
        self.local: Dict[int, int] = {}  # request -> tokens of it this rank holds (= its segments here)
        self.ctx: Dict[int, int] = {}  # request -> context length (= the ledger's)
        self.rows: Dict[int, int] = {}  # request -> output row
        self.running: List[int] = []  # admission order, like the simulator's running list
        self.stalled = 0
        self._kbuf = self._vbuf = None
        self._none = store.seq_create(0)  # stands in for requests this rank holds nothing of

    # the dispatch of simengine.cpp:252-257: most free blocks, ties to the lowest id
    def dispatch_target(self) -> int:
        free = [self.led.free_blocks(i) for i in range(self.nranks)]
        return max(range(self.nranks), key=lambda i: (free[i], -i))

    def admit(self, req: int, row: int, tokens: int, home: int = -1) -> bool:
        """try_admit (simengine.cpp:262-268): the prompt's blocks at the home;
        the home rank fills them (prefill) with the generator's values."""
        home = self.dispatch_target() if home < 0 else home
        if not self.led.admit(req, home, tokens):
            return False
        self.rows[req] = row
        self.ctx[req] = tokens
        self.running.append(req)
        if home == self.rank:
            s = self.st.seq_create(tokens)
            self.st.fill_synthetic(s, self.seed, req, 0, self.amp_k, self.amp_v)
            self.seqs[req] = s
            self.local[req] = tokens
        return True

    def local_tokens(self, req: int) -> int:
        """Tokens of req on this rank, from the ledger's segments (the loop
        keeps the same count incrementally in self.local)."""
        return sum(hi - lo for inst, lo, hi in self.led.segments(req) if inst == self.rank)

    def ranges(self) -> List[Range]:
        """This rank's share of every running request (identity records for
        requests it holds nothing of)."""
        out = []
        for r in sorted(self.running, key=lambda r: self.rows[r]):
            n = self.local.get(r, 0)
            out.append(Range(self.seqs[r] if n else self._none, self.rows[r], 0, n))
        return out

    def grow(self) -> List[int]:
        """One token for every running request: ensure_slot, the K/V rows
        appended on the rank that holds the slot, ledger advance. Returns the
        participants (stalled requests -- no block anywhere -- skip the step,
        ensure_step simengine.cpp:356-371)."""
        inst = self.led.step(self.running, self.allow_borrow)  # ensure_slot + advance, one call
        where = dict(zip(self.running, inst))
        parts = [r for r in self.running if where[r] >= 0]
        self.stalled += len(self.running) - len(parts)
        mine = [r for r in parts if where[r] == self.rank]
        if mine:
            for r in mine:
                if r not in self.seqs:
                    self.seqs[r] = self.st.seq_create(0)  # first block hosted here
            if self._kbuf is None or self._kbuf.shape[0] < len(mine):
                self._kbuf, self._vbuf = self.row_buffers(len(mine))
            k, v = self._kbuf[: len(mine)], self._vbuf[: len(mine)]
            # a new token's position is its request's context length before the step
            self.st.synthetic_rows(mine, [self.ctx[r] for r in mine], self.seed, k, v, self.amp_k, self.amp_v)
            self.st.kv_append([self.seqs[r] for r in mine], k, v, mem=MEM_DEVICE)
            for r in mine:
                self.local[r] = self.local.get(r, 0) + 1
        for r in parts:
            self.ctx[r] += 1
        return parts

    def row_buffers(self, n: int):
        """Device buffers [n][num_kv_heads][padded_dim] for the new tokens' K/V rows."""
        import torch
        shape = (n, self.st.num_kv_heads, self.st.padded_dim)
        tdt = {BF16: torch.bfloat16, F32: torch.float32}.get(self.st.dtype, torch.float64)
        dev = f"cuda:{self.st.device}"
        return torch.empty(shape, dtype=tdt, device=dev), torch.empty(shape, dtype=tdt, device=dev)

    def step(self, num_rows: int, q, out, mem: int = MEM_DEVICE) -> List[int]:
        """grow(), then the sharded decode over every rank's tokens."""
        parts = self.grow()
        self.st.decode_sharded(self.ranges(), num_rows, q, out, mem=mem)
        return parts

    def release(self, req: int):
        """complete (simengine.cpp:300-303): free_request everywhere."""
        self.led.release(req)
        self.running.remove(req)
        self.local.pop(req, None)
        self.ctx.pop(req, None)
        s = self.seqs.pop(req, None)
        if s is not None:
            self.st.seq_release(s)
