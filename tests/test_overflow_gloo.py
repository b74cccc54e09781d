"""CPU, world_size 2 and 4 over gloo: the overflow-borrowing decode loop as
separate processes. Every rank keeps its own replica of the cluster block
ledger (dattn_ledger_*) and applies the same admissions, ensure_slot calls
(simengine.cpp:318-354) and advances; the replicas must stay identical with
no messages (checked by all-gathering their state every step). Each rank
reduces the token ranges it holds (dattn_ledger_segments) to one partial
record per (request, q head) -- the oracle standing in for the MA kernel --,
the records are all-gathered (K5's exchange) and merged; the result must
equal the unsplit reference at the grown lengths."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import paper_2401_02669_b200 as pb

    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        seed, hq, hkv, d, bs = 77, 2, 1, 16, 16
        prompts = [150, 60, 33, 90, 7]
        caps = [pb.blocks_for_tokens(150, bs)] + [30] * (world - 1)  # instance 0 is full after admission
        led = pb.Ledger(caps, bs)
        assert led.admit(0, 0, prompts[0])
        for i, L in enumerate(prompts[1:], 1):
            free = [led.free_blocks(j) for j in range(world)]
            assert led.admit(i, max(range(world), key=lambda j: (free[j], -j)), L)
        ok, worst = True, 0.0
        for t in range(60):
            for r in range(len(prompts)):
                if led.ensure_slot(r) >= 0:
                    led.advance(r)
            state = [(led.segments(r), led.request(r)) for r in range(len(prompts))] + \
                    [led.instance(j) for j in range(world)]
            states = [None] * world
            dist.all_gather_object(states, state)
            ok &= all(s == states[0] for s in states)
            if t % 20 != 19:
                continue
            rec = np.zeros((len(prompts), hq, d + 4))
            rec[:, :, 0] = -np.inf
            for r in range(len(prompts)):
                parts = {h: [] for h in range(hq)}
                for inst, lo, hi in led.segments(r):
                    if inst != rank:
                        continue
                    for h in range(hq):
                        k, v = oracle.synth_kv(seed, r, oracle.gqa_kv_head(h, hq, hkv), lo, hi - lo, d, 1.0, 2.0,
                                               oracle.F32)
                        qv = oracle.synth_q(seed, r, h, d, 1.0, oracle.F32)
                        parts[h].append(oracle.micro_attention(qv, k, v))
                for h in range(hq):
                    if parts[h]:  # this rank's local merge (K5 phase A)
                        m, e, ma = _fold(oracle, parts[h])
                        rec[r, h, :4] = [m, e, sum(p[3] for p in parts[h]), 0.0]
                        rec[r, h, 4:] = ma
            mine = torch.from_numpy(rec)
            gathered = [torch.zeros_like(mine) for _ in range(world)]
            dist.all_gather(gathered, mine)
            lens = [led.request(r)[1] for r in range(len(prompts))]
            ref = oracle.decode_ranges(seed, [0] * len(prompts), lens, list(range(len(prompts))), hq, hkv, d,
                                       dtype=oracle.F32)
            for r in range(len(prompts)):
                for h in range(hq):
                    recs = [(g[r, h, 0].item(), g[r, h, 1].item(), g[r, h, 4:].numpy(), int(g[r, h, 2].item()))
                            for g in gathered]
                    out = oracle.aggregate(recs)
                    worst = max(worst, oracle.rel_err(out, ref[r, h]))
        spans = len({s[0] for s in led.segments(0)})
        q.put((rank, ok, worst, led.borrowed(), spans, None))
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, False, None, 0, 0, traceback.format_exc()))


def _fold(oracle, parts):
    """combine_partials over one rank's segments (distattention.cpp:131-148)."""
    acc = parts[0]
    for p in parts[1:]:
        acc = oracle.combine(acc, p)
    return acc[0], acc[1], acc[2]


@pytest.mark.parametrize("world", [2, 4])
def test_overflow_loop_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, worst, borrowed, spans, exc in res:
        assert exc is None, (rank, exc)
        assert ok, rank  # ledger replicas identical at every step
        assert borrowed > 0 and spans > 1  # request 0 really spans GPUs
        assert worst < 1e-12, (rank, worst)
