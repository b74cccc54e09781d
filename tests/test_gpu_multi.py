"""Multi-GPU parity of dattn_decode_sharded (one process per GPU, NCCL
allgather of (m, e, ma) records between ranks). Needs >= 2 visible GPUs;
skipped otherwise (the single-GPU round-end run cannot exercise it)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = {
    "gqa_bf16": dict(lens=[5000, 37, 20000, 1, 16], hq=64, hkv=8, d=128, dtype=0, tol=2e-2),
    "mha_f32": dict(lens=[4096, 3, 777], hq=32, hkv=32, d=128, dtype=1, tol=1e-3),
}


def _worker(rank, world, port, case, placement, fused, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import oracle
    import paper_2401_02669_b200 as pb
    from paper_2401_02669_b200.sharding import placement_from_moves, plan_rank_ranges

    try:
        os.environ["DATTN_FUSED_MERGE"] = "1" if fused else "0"
        torch.cuda.set_device(rank)
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        c = CASES[case]
        lens, hq, hkv, d, dt = c["lens"], c["hq"], c["hkv"], c["d"], c["dtype"]
        seed = 404
        if placement:
            nb = -(-lens[2] // 16)
            lent = {(2, (r + 1) % world): nb // (world + 1) for r in range(world - 1)}
            shares = placement_from_moves(lens, [0] * len(lens), lent, world, 16)[rank]
        else:
            shares = plan_rank_ranges(lens, world, 16)[rank]
        pages = sum(-(-rr.tokens // 16) for rr in shares) + 8
        st = pb.Store(d, hq, hkv, dt, 16, pages, max_seqs=len(lens) + 2,
                      max_pages_per_seq=max(-(-rr.tokens // 16) for rr in shares) + 2, device=rank)
        st.set_stream(torch.cuda.current_stream().cuda_stream)
        ranges = []
        for rr in shares:
            s = st.seq_create(rr.tokens)
            st.fill_synthetic(s, seed, rr.request, rr.tok_begin, 1.0, 2.0)
            ranges.append(pb.Range(s, rr.request, 0, rr.tokens))
        tdt = {0: torch.bfloat16, 1: torch.float32}[dt]
        qd = torch.empty(len(lens), hq, st.padded_dim, dtype=tdt, device=f"cuda:{rank}")
        st.q_fill_synthetic(qd, len(lens), seed)
        out = torch.zeros_like(qd)
        uid = [pb.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        st.comm_init(uid[0], rank, world)
        st.decode_sharded(ranges, len(lens), qd, out)
        torch.cuda.synchronize()
        assert st.stats().last_exchange == (2 if fused else 1)
        # repeated steps reuse the exchange buffers (epoch flags)
        for _ in range(3):
            st.decode_sharded(ranges, len(lens), qd, out)
        torch.cuda.synchronize()
        # host-memory path gives the same bytes
        qh = qd.cpu().pin_memory()
        oh = torch.zeros_like(qh).pin_memory()
        st.decode_sharded(ranges, len(lens), qh, oh, mem=pb.MEM_HOST)
        same = bool(torch.equal(oh, out.cpu()))
        got = out[..., :d].double().cpu().numpy()
        err = None
        if rank == 0:
            ref = oracle.decode_ranges(seed, [0] * len(lens), lens, list(range(len(lens))), hq, hkv, d, dtype=dt)
            err = max(oracle.rel_err(got[b, h], ref[b, h]) for b in range(len(lens)) for h in range(hq))
        # every rank holds the same merged output
        g = torch.from_numpy(got)
        allg = [torch.zeros_like(g) for _ in range(world)]
        dist.all_gather(allg, g)
        agree = all(torch.equal(allg[0], x) for x in allg)
        q.put((rank, err, agree, same, None))
        dist.destroy_process_group()
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, None, False, False, repr(e)))


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("placement", [False, True])
@pytest.mark.parametrize("fused", [True, False], ids=["k5_nvlink", "nccl"])
def test_sharded_decode_matches_oracle(case, placement, fused):
    import torch.multiprocessing as mp
    world = min(_ngpus(), 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, placement, fused, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for rank, err, agree, same, exc in res:
        assert exc is None, (rank, exc)
        assert agree and same
        if rank == 0:
            assert err < CASES[case]["tol"], err
