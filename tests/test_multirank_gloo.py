"""CPU, world_size 2 over gloo: the N>1 protocol of dattn_decode_sharded.

Each rank holds its block-aligned share of every request (plan_rank_ranges /
placement_from_moves), reduces it to ONE partial record [m, e, tokens, 0,
ma[d]] per (request, q head) -- computed here with the oracle standing in for
K1 + local K3 --, all-gathers the packed records (the ncclAllGather of the
GPU path) and merges them in rank order (K3's rank merge). The merged output
must equal the unsplit reference computation."""
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


def _worker(rank, world, port, mode, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    from paper_2401_02669_b200.sharding import placement_from_moves, plan_rank_ranges

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seed, hq, hkv, d = 31, 4, 2, 32
    lens = [1, 40, 300, 517]
    if mode == "equal":
        shares = plan_rank_ranges(lens, world, 16)[rank]
    else:  # placement: request 3 homed on rank 0, 20 of its 33 blocks lent to rank 1
        shares = placement_from_moves(lens, [0, 1, 0, 0], {(3, 1): 20, (2, 1): 3}, world, 16)[rank]
    rec = np.zeros((len(lens), hq, d + 4))
    for rr in shares:
        for h in range(hq):
            kvh = oracle.gqa_kv_head(h, hq, hkv)
            k, v = oracle.synth_kv(seed, rr.request, kvh, rr.tok_begin, rr.tokens, d, 1.0, 2.0, oracle.F32)
            qv = oracle.synth_q(seed, rr.request, h, d, 1.0, oracle.F32)
            m, e, ma, sp = oracle.micro_attention(qv, k, v)
            rec[rr.request, h, :4] = [m, e, sp, 0.0]
            rec[rr.request, h, 4:] = ma
    mine = torch.from_numpy(rec)
    gathered = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine)
    out = np.zeros((len(lens), hq, d))
    for b in range(len(lens)):
        for h in range(hq):
            parts = [(g[b, h, 0].item(), g[b, h, 1].item(), g[b, h, 4:].numpy(), int(g[b, h, 2].item()))
                     for g in gathered]
            out[b, h] = oracle.aggregate(parts)
    ref = oracle.decode_ranges(seed, [0] * len(lens), lens, list(range(len(lens))), hq, hkv, d,
                               dtype=oracle.F32, threads=2)
    err = max(oracle.rel_err(out[b, h], ref[b, h]) for b in range(len(lens)) for h in range(hq))
    q.put((rank, err))
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["equal", "placement"])
def test_two_rank_partial_exchange(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err in res:
        assert err < 1e-12, (rank, err)
