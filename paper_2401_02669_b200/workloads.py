"""The BASELINE.json decode workloads and their roofline
arithmetic. Host-side description only; the data is generated on the device
by the counter-hash fill kernel (K4).

Unit of work: one decode step of one attention layer for the whole batch,
every request contributing one query token x all q heads against its whole
context. tokens/s = B / t_step.  Algorithmic bytes per step:
    sum_r 2 * Hkv * d * L_r * s_kv  +  B * Hq * d * (s_q + s_o)
(K and V read once per kv head -- GQA does not re-read per q head -- q read,
o written; partial records and block tables are implementation traffic.)
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def counter_uniform_int(seed: int, i: int, lo: int, hi: int) -> int:
    """Deterministic draw i of U[lo, hi] (inclusive) from a counter hash."""
    span = hi - lo + 1
    return lo + splitmix64((seed * 0x2545F4914F6CDD1D + i) & MASK64) % span


@dataclass
class Workload:
    name: str
    lens: List[int]
    hq: int
    hkv: int
    d: int
    dtype: int  # 0 bf16, 1 fp32
    rblocks: int = 1  # rBlocks per request on one GPU (config 1 splits into 4)
    page_tokens: int = 16
    seed: int = 20261018
    amp_k: float = 1.0
    amp_v: float = 2.0
    note: str = ""
    placement: str = "equal"  # "equal": plan_rank_ranges; "gmanager": the reference control plane's placement
    queued: int = 0  # config 5: debtor queue at the long request's home (gmanager placement input)
    n_layers: int = 32  # model depth for model-equivalent TPS (7B: 32, 70B: 80)
    meta: dict = field(default_factory=dict)

    @property
    def batch(self) -> int:
        return len(self.lens)

    @property
    def elem_bytes(self) -> int:
        return 2 if self.dtype == 0 else (4 if self.dtype == 1 else 8)

    @property
    def total_tokens(self) -> int:
        return sum(self.lens)

    def kv_bytes(self) -> int:
        return 2 * self.hkv * self.d * self.total_tokens * self.elem_bytes

    def algorithmic_bytes(self) -> int:
        return self.kv_bytes() + self.batch * self.hq * self.d * 2 * self.elem_bytes

    def algorithmic_flops(self) -> int:
        return 4 * self.hq * self.d * self.total_tokens


def config(name: str, cfg5_queue: int = 64) -> Workload:
    """BASELINE.json configs by number (1..5). ``cfg5_queue`` selects config 5's
    reference placement (debtor queue 0, 64 or 512; tests/golden/cfg5_placement.json)."""
    if name in ("1", "cfg1"):
        return Workload("cfg1: 1 req, LLaMA-7B MHA 32x128, 4K fp32 KV in 4 rBlocks", [4096], 32, 32, 128, 1,
                        rblocks=4)
    if name in ("2", "cfg2"):
        seed = 20240702
        lens = [counter_uniform_int(seed, i, 1024, 32768) for i in range(64)]
        return Workload("cfg2: batch 64 decode, LLaMA2-7B MHA 32x128, ragged 1K-32K, bf16 paged KV",
                        lens, 32, 32, 128, 0, meta={"lens_seed": seed, "lens_rule": "counter_uniform_int U[1024,32768]"})
    if name in ("3", "cfg3"):
        return Workload("cfg3: LLaMA2-70B GQA 64q/8kv x128, batch 16 x 128K, bf16", [131072] * 16, 64, 8, 128, 0, n_layers=80)
    if name in ("4", "cfg4"):
        return Workload("cfg4: 1 req x 1M tokens, LLaMA-7B MHA 32x128, bf16", [1048576], 32, 32, 128, 0)
    if name in ("5", "cfg5"):
        return Workload("cfg5: skewed mix 1x512K + 256x2K, LLaMA-7B MHA 32x128, bf16, gManager placement",
                        [524288] + [2048] * 256, 32, 32, 128, 0, placement="gmanager", queued=cfg5_queue,
                        meta={"placement": "reference control plane (oracle/_ref): most-free dispatch, "
                                           "rManager heartbeats, GManager::plan + execute_move_sync until no "
                                           "move; tests/golden/cfg5_placement.json",
                              "debtor_queue": cfg5_queue, "capacity_blocks": 32768})
    raise ValueError(f"unknown config {name!r}")


def rank_shares(w: Workload, nranks: int):
    """Per-rank token ranges of every request (sharding.RankRange lists)."""
    from .sharding import gmanager_placement, placement_from_moves, plan_rank_ranges
    if w.placement == "gmanager" and nranks > 1:
        homes, lent = gmanager_placement(w.lens, nranks, w.queued, w.page_tokens)
        return placement_from_moves(w.lens, homes, lent, nranks, w.page_tokens)
    return plan_rank_ranges(w.lens, nranks, w.page_tokens)
