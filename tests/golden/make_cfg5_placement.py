"""Generate tests/golden/cfg5_placement.json: config 5's rBlock placement as the
REFERENCE control plane decides it.

BASELINE config 5 is "1 request at 512K plus 256 requests at 2K, with rBlocks
lent across GPUs per gManager placement". The placement is produced by the
unmodified reference (oracle/_ref/libkvsched_ref.so, ref_bridge.cpp
``ref_cfg5_place``), not restated:

  1. dispatch -- requests in order (the 512K one first), each homed on the
     instance with the most free blocks, ties to the lowest id
     (simengine.cpp:252-257), blocks taken with RManager::alloc_local
     (controlplane.cpp:38-44);
  2. rManager heartbeats -> GManager (controlplane.cpp:109-142, 374-410,
     500-516), with batch = the instance's home requests and a debtor queue of
     Q requests at the 512K request's home;
  3. planning rounds: GManager::plan -> plan_round (reclaims, then the greedy
     pass; scheduler.cpp:483-493) -> every MoveKvCache executed by
     execute_move_sync (controlplane.cpp:518-540). The freed blocks admit
     queued requests of expected_new_request_tokens (512) each
     (scheduler.cpp:62-80), which take their prompt blocks at the home; rounds
     repeat until one plans no move.

Documented inputs:
  * model: default_cluster_config (config.cpp:71-87; default perf curves,
    block 16 tokens) and the default SchedulerConfig (scheduler.hpp:52-58:
    batch threshold 8, creditor utilisation 0.8, retain_local_fraction 0.5);
  * capacity per instance: 32,768 blocks = the 512K request exactly. Its home
    is then full, so the queued requests are really blocked. With any free
    block left at the home, the reference's reclaim pass (scheduler.cpp:144-178)
    pulls lent blocks back in the next round;
  * debtor queue Q in {0, 64, 512}. Q = 64 is the default workload
    (the planner lends <= 2,048 blocks, about 1.0 ms per step on
    the home GPU). Q = 0 lends nothing: the gain is positive only while freed
    blocks admit queued requests. Q = 512 reaches the 50 % retain floor.

The result per (N, Q): every request's home and its blocks per instance (local
on the home, hosted elsewhere), plus the move list. sharding.placement_from_moves
turns the block counts into token ranges: the home keeps the prefix, and hosts take
the following blocks in ascending instance order.

Usage (in the container that has /root/reference):
    python tests/golden/make_cfg5_placement.py
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cfg5_placement.json")
LENS = [524288] + [2048] * 256
CAPACITY = 32768
QUEUES = (0, 64, 512)
NS = (2, 4, 8)  # one GPU holds the whole batch: no placement
MAX_ROUNDS = 8


def generate() -> dict:
    out = {"lens": {"long": 524288, "short": 2048, "n_short": 256}, "capacity_blocks": CAPACITY,
           "block_tokens": 16, "default_queue": 64, "placements": {}}
    for n in NS:
        for q in QUEUES:
            homes, blocks, moves = oracle.ref_cfg5_place(LENS, n, CAPACITY, q, MAX_ROUNDS)
            hosted = [[r, i, b] for r, row in enumerate(blocks) for i, b in enumerate(row)
                      if i != homes[r] and b > 0]
            for r, row in enumerate(blocks):  # every block of every request is placed
                assert sum(row) == -(-LENS[r] // 16), (n, q, r)
            out["placements"][f"n{n}_q{q}"] = {
                "n_instances": n, "queued": q, "homes": homes, "hosted": hosted,
                "home_blocks": [row[homes[r]] for r, row in enumerate(blocks)][:1],
                "per_instance_blocks": [sum(row[i] for row in blocks) for i in range(n)],
                "moves": moves}
    return out


def main():
    if not oracle.ref_available():
        raise SystemExit("oracle/_ref is not built (needs /root/reference)")
    with open(OUT, "w") as f:
        json.dump(generate(), f, indent=1)
        f.write("\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
