"""The cluster block ledger and the overflow-borrowing slot rule
(dattn_ledger_*, include/dattn.h) pinned to the reference: (1) the per-
instance ledger against the compiled RManager (controlplane.cpp:38-79) op by
op, (2) ensure_slot against the reference cluster simulator itself
(run_simulation, simengine.cpp:318-354): its JSONL event log is replayed
through the B200 ledger -- admissions, every decode step's slot requests in
the simulator's running order, completions -- and every borrow decision
(request, host, blocks) and every step's batch must be identical. CPU only."""
import random

import pytest

import oracle
import paper_2401_02669_b200 as pb

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def replay(capacities, requests, policy, log):
    """Drive pb.Ledger through the reference simulator's event log; returns
    the ledger and counts. Asserts the borrow decisions and batches match."""
    led = pb.Ledger(capacities, 16)
    n = len(capacities)
    running = {i: [] for i in range(n)}
    home = {}
    pending = {i: [] for i in range(n)}  # participants of the instance's step in flight
    ref_borrows = []
    counts = {"steps": 0, "borrows": 0, "stalls": 0, "completes": 0}

    def settle(inst):  # on_step_done: ctx++ of the step's participants (simengine.cpp:444-452)
        for rid in pending[inst]:
            if rid in home:
                led.advance(rid, 1)
        pending[inst] = []

    for e in log:
        ev = e["ev"]
        if ev == "admit":
            rid, inst = e["req"], e["inst"]
            assert led.admit(rid, inst, requests[rid][1]), e
            assert led.blocks(rid, inst) == e["blocks"] == oracle.ref_blocks_for_tokens(requests[rid][1], 16)
            home[rid] = inst
        elif ev == "prefill_done":
            running[home[e["req"]]].append(e["req"])
        elif ev == "borrow":
            ref_borrows.append((e["req"], e["host"], e["blocks"]))
        elif ev == "step":
            inst = e["inst"]
            settle(inst)
            mine, parts = [], []
            for rid in running[inst]:
                before = led.borrowed()
                w = led.ensure_slot(rid, allow_borrow=policy != oracle.SIM_STATIC)
                if w < 0:
                    counts["stalls"] += 1
                    continue
                parts.append(rid)
                if led.borrowed() > before:
                    mine.append((rid, w, led.borrowed() - before))
            assert mine == ref_borrows, (e, mine, ref_borrows)
            assert len(parts) == e["batch"], (e, parts)
            counts["borrows"] += len(mine)
            ref_borrows = []
            pending[inst] = parts
            counts["steps"] += 1
        elif ev == "complete":
            rid = e["req"]
            settle(home[rid])
            led.release(rid)
            running[home[rid]].remove(rid)
            del home[rid]
            counts["completes"] += 1
    assert not ref_borrows
    return led, counts


def test_ledger_matches_reference_rmanager_ops():
    """admit / overflow allocations / release vs RManager alloc_local,
    alloc_hosted, free_request on the same sequence (per instance)."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = random.Random(5)
    caps = [40, 25, 60]
    led = pb.Ledger(caps, 16)
    ops = {i: [] for i in range(3)}  # reference op traces per instance
    live = {}
    nxt = 0
    for _ in range(400):
        act = rng.random()
        if act < 0.3 or not live:
            home, toks = rng.randrange(3), rng.randint(1, 200)
            ok = led.admit(nxt, home, toks)
            ops[home].append((oracle.LEDGER_ALLOC_LOCAL, nxt, pb.blocks_for_tokens(toks, 16), -1, int(ok)))
            if ok:
                live[nxt] = home
            nxt += 1
        elif act < 0.85:
            rid = rng.choice(sorted(live))
            held = {j: led.blocks(rid, j) for j in range(3)}
            w = led.ensure_slot(rid, allow_borrow=True)
            if w >= 0:
                for j in range(3):
                    d = led.blocks(rid, j) - held[j]
                    if d:
                        op = oracle.LEDGER_ALLOC_LOCAL if j == live[rid] else oracle.LEDGER_ALLOC_HOSTED
                        ops[j].append((op, rid, d, live[rid], 1))
                led.advance(rid, 1)
        else:
            rid = rng.choice(sorted(live))
            per = {j: led.blocks(rid, j) for j in range(3)}
            led.release(rid)
            for j in range(3):
                ops[j].append((oracle.LEDGER_FREE, rid, 0, -1, per[j]))
            del live[rid]
    for j in range(3):
        if not ops[j]:
            continue
        ref = oracle.ref_rmanager_trace(caps[j], [o[:4] for o in ops[j]])
        assert [r[0] for r in ref] == [o[4] for o in ops[j]], j
        _, used, free = led.instance(j)
        assert (ref[-1][1], ref[-1][2]) == (used, free), j


SCENARIOS = {
    # home runs out while others have room: borrows go to the most free
    # clean instance, then stick to the existing host
    "one_overflow": ([30, 60, 45], [(0.0, 400, 800), (0.0, 100, 50)]),
    # several instances overflow at once; borrowing instances are avoided
    # while a clean one has room, then used when nothing clean is left
    "mutual": ([30, 20, 25], [(0.0, 300, 700), (0.0, 200, 300), (0.0, 100, 600), (0.5, 64, 100)]),
    "four_inst_churn": ([24, 24, 40, 16], [(0.0, 250, 200), (0.0, 200, 150), (0.1, 120, 400),
                                           (0.2, 60, 90), (0.4, 200, 40), (1.0, 30, 300)]),
    "ragged_many": ([64, 48, 80, 32, 56],
                    [(0.05 * i, 40 + 37 * (i % 7), 60 + 53 * (i % 5)) for i in range(14)]),
}


@needs_ref
@pytest.mark.parametrize("policy", [oracle.SIM_STRAWMAN, oracle.SIM_STATIC])
@pytest.mark.parametrize("name", sorted(SCENARIOS))
def test_ensure_slot_replays_reference_simulator(name, policy):
    caps, reqs = SCENARIOS[name]
    log = oracle.ref_sim_log(caps, reqs, policy, horizon_s=3000)
    led, counts = replay(caps, reqs, policy, log)
    assert counts["steps"] > 20
    if policy == oracle.SIM_STRAWMAN and name != "ragged_many":
        assert counts["borrows"] > 0, counts
    if policy == oracle.SIM_STATIC:
        assert counts["borrows"] == 0


def test_segments_follow_block_order():
    led = pb.Ledger([3, 10], 16)
    assert led.admit(0, 0, 40)  # 3 blocks: home full
    assert led.segments(0) == [(0, 0, 40)]
    for t in range(40, 48):  # fits the last home block
        assert led.ensure_slot(0) == 0
        led.advance(0)
    assert led.ensure_slot(0) == 1  # position 48 -> block 3 borrowed on instance 1
    assert led.borrowed() == 1
    assert led.segments(0) == [(0, 0, 48)]  # the borrowed block is not written yet
    led.advance(0)
    assert led.segments(0) == [(0, 0, 48), (1, 48, 49)]
    assert led.request(0) == (0, 49, 4)
    assert led.instance(1) == (10, 1, 9)
    assert led.ensure_slot(0, allow_borrow=False) == 1  # block already held
    for _ in range(15):
        led.ensure_slot(0)
        led.advance(0)
    assert led.ensure_slot(0, allow_borrow=False) == -1  # static policy: home full -> stall
    assert led.release(0) == 4
    assert led.instance(0) == (3, 0, 3) and led.instance(1) == (10, 0, 10)


def test_ledger_contract_errors():
    led = pb.Ledger([4], 16)
    with pytest.raises(pb.ContractError):
        led.admit(0, 1, 10)  # no such instance
    with pytest.raises(pb.ContractError):
        led.admit(0, 0, 0)  # allocation must be >= 1 block (controlplane.cpp:39)
    assert led.admit(0, 0, 64)
    with pytest.raises(pb.ContractError):
        led.admit(0, 0, 1)  # already live
    assert not led.admit(1, 0, 1)  # full: not admitted, nothing changes
    with pytest.raises(pb.CapacityError):
        led.advance(0, 1)  # no block for position 64
    with pytest.raises(pb.ContractError):
        led.ensure_slot(7)


@needs_ref
@pytest.mark.parametrize("seed", range(12))
def test_ensure_slot_replays_reference_simulator_random(seed):
    """Random clusters (2-6 instances, tight capacities) and traces."""
    rng = random.Random(1000 + seed)
    n = rng.randint(2, 6)
    caps = [rng.randint(12, 70) for _ in range(n)]
    reqs = [(round(rng.uniform(0, 2.0), 3), rng.randint(1, 16 * min(caps)), rng.randint(1, 700))
            for _ in range(rng.randint(2, 12))]
    log = oracle.ref_sim_log(caps, reqs, oracle.SIM_STRAWMAN, horizon_s=2000)
    replay(caps, reqs, oracle.SIM_STRAWMAN, log)


def test_segments_partition_the_context():
    """After any mix of growth, borrowing and releases, every live request's
    segments tile [0, ctx) in order, each switch of instance falls on a block
    boundary (so a hosted sequence's pages are whole blocks), and each
    instance's used blocks equal the blocks its segments cover."""
    rng = random.Random(9)
    caps = [30, 18, 25, 12]
    led = pb.Ledger(caps, 16)
    live, nxt = [], 0
    for _ in range(3000):
        a = rng.random()
        if a < 0.05 or not live:
            home = max(range(4), key=lambda i: (led.free_blocks(i), -i))
            if led.admit(nxt, home, rng.randint(1, 150)):
                live.append(nxt)
            nxt += 1
        elif a < 0.97:
            r = rng.choice(live)
            if led.ensure_slot(r) >= 0:
                led.advance(r)
        else:
            led.release(live.pop(rng.randrange(len(live))))
        if rng.random() < 0.02:
            used = [0] * 4
            for r in live:
                segs = led.segments(r)
                _, ctx, held = led.request(r)
                assert segs[0][1] == 0 and segs[-1][2] == ctx
                for (i0, _, e0), (i1, b1, _) in zip(segs, segs[1:]):
                    assert e0 == b1 and i0 != i1 and b1 % 16 == 0
                for i in range(4):
                    used[i] += led.blocks(r, i)
                assert sum(led.blocks(r, i) for i in range(4)) == held
            assert used == [led.instance(i)[1] for i in range(4)]


def test_batched_step_equals_slot_then_advance():
    """dattn_ledger_step (one call per decode step) = ensure_slot for every
    request in order, then advance the ones that got a slot."""
    rng = random.Random(21)
    caps = [20, 14, 30]
    a, b = pb.Ledger(caps, 16), pb.Ledger(caps, 16)
    reqs = []
    for i in range(7):
        L = rng.randint(1, 120)
        h = rng.randrange(3)
        if a.admit(i, h, L):
            assert b.admit(i, h, L)
            reqs.append(i)
    for _ in range(200):
        got = a.step(reqs)
        want = [b.ensure_slot(r) for r in reqs]
        for r, w in zip(reqs, want):
            if w >= 0:
                b.advance(r)
        assert got == want
    assert [a.segments(r) for r in reqs] == [b.segments(r) for r in reqs]
    assert [a.instance(j) for j in range(3)] == [b.instance(j) for j in range(3)]


def test_batched_step_rejects_unknown_request_without_side_effects():
    led = pb.Ledger([2, 8], 16)
    assert led.admit(0, 0, 32)  # home full
    before = (led.segments(0), led.instance(0), led.instance(1), led.borrowed())
    with pytest.raises(pb.ContractError):
        led.step([0, 99])
    assert (led.segments(0), led.instance(0), led.instance(1), led.borrowed()) == before
    assert led.step([0]) == [1]  # the slot is then borrowed on instance 1 as usual
