"""CPU model of K5's flag-free exchange, with adversarial
schedules.

Every rank pushes one record per (row, q head) group into every rank's
exchange buffer in self-validating words: an empty word holds all ones, which
no pushed value has (x_enc maps that one NaN pattern to 0x7FFFFFFF). The
receiver polls each word until it is non-empty, merges, and writes the empty
pattern back. Identity records carry only their header, and payload words are
read only for live records. Buffers have two halves used by alternate steps.

The model runs N ranks as coroutines under a random scheduler. Every remote
word write is delivered after an arbitrary delay and in arbitrary order, and
ranks are skewed by random stalls. It checks three things:
(1) every step's merged result equals the expected one (no stale or torn
    record is ever consumed);
(2) after the last step every word is empty again;
(3) two halves are enough: a rank never writes into a half that a peer has
    not finished reading.
The model follows dattn_merge.cuh (x_enc, x_poll, x_clear, xchg_rank_merge)
and the push in merge_exchange_kernel.
"""
import random
import struct

import numpy as np
import pytest

EMPTY = 0xFFFFFFFF


def x_enc(v: float) -> int:
    b = struct.unpack("<I", struct.pack("<f", v))[0]
    return 0x7FFFFFFF if b == EMPTY else b


def x_dec(b: int) -> float:
    return struct.unpack("<f", struct.pack("<I", b))[0]


def test_encoding_never_produces_the_empty_word():
    nan_all_ones = struct.unpack("<f", struct.pack("<I", EMPTY))[0]
    assert x_enc(nan_all_ones) == 0x7FFFFFFF
    assert np.isnan(x_dec(x_enc(nan_all_ones)))
    for v in (0.0, -0.0, 1.5, -np.inf, np.inf, float("nan"), 3.4e38):
        assert x_enc(v) != EMPTY
    assert x_dec(x_enc(-0.0)) == 0.0 and np.signbit(x_dec(x_enc(-0.0)))


def _run(nranks, groups, payload, steps, seed):
    rng = random.Random(seed)
    rec = 4 + payload
    # exchange buffers: [rank][half][src rank][group][word]
    buf = [np.full((2, nranks, groups, rec), EMPTY, dtype=np.uint64) for _ in range(nranks)]
    inflight = []  # (dst rank, half, src, group, word, value)
    results = {}

    def record(step, src, g):
        # identity for some (step, src, group) combinations, else a live record
        if (step * 7 + src * 3 + g) % 5 == 0:
            return None
        base = step * 1000 + src * 100 + g
        return [float(base), 1.0 + src, float(src + 1)] + [float(base + w) for w in range(payload)]

    def rank_proc(r):
        for step in range(steps):
            half = step & 1
            # K5 phase A: push this rank's records to every rank, word by word
            for dst in range(nranks):
                for g in range(groups):
                    v = record(step, r, g)
                    hdr = [v[0], v[1], v[2], 0.0] if v else [-np.inf, 0.0, 0.0, 0.0]
                    words = [(w, x_enc(x)) for w, x in enumerate(hdr)]
                    if v:
                        words += [(4 + w, x_enc(x)) for w, x in enumerate(v[3:])]
                    for w, val in words:
                        inflight.append((dst, half, r, g, w, val))
                yield
            # phase D: poll headers, then live payloads, merge, empty the slots
            out = []
            for g in range(groups):
                got = []
                for src in range(nranks):
                    for w in range(4):  # x_poll of the header
                        while buf[r][half, src, g, w] == EMPTY:
                            yield
                    tok = x_dec(int(buf[r][half, src, g, 2]))
                    words = [x_dec(int(buf[r][half, src, g, w])) for w in range(3)]
                    if tok != 0.0:
                        for w in range(4, rec):
                            while buf[r][half, src, g, w] == EMPTY:
                                yield
                        words += [x_dec(int(buf[r][half, src, g, w])) for w in range(4, rec)]
                    got.append(words)
                for src in range(nranks):  # x_clear of what was read
                    buf[r][half, src, g, :4] = EMPTY
                    if x_dec(int(got[src][2])) != 0.0:
                        buf[r][half, src, g, 4:] = EMPTY
                out.append(got)
            results[(r, step)] = out
            yield

    procs = [rank_proc(r) for r in range(nranks)]
    live = list(range(nranks))
    while live or inflight:
        # deliver a random in-flight write or advance a random rank; stall ranks at random
        if inflight and (not live or rng.random() < 0.5):
            i = rng.randrange(len(inflight))
            dst, half, src, g, w, val = inflight.pop(i)
            # (3): the half being written is not being read by dst for an older step
            assert buf[dst][half, src, g, w] == EMPTY, "overwrote an unread word"
            buf[dst][half, src, g, w] = val
            continue
        r = rng.choice(live)
        if rng.random() < 0.2:
            continue  # this rank stalls
        try:
            next(procs[r])
        except StopIteration:
            live.remove(r)
    # (1) every step's merged records are the ones pushed for that step
    for (r, step), out in results.items():
        for g, got in enumerate(out):
            for src, words in enumerate(got):
                v = record(step, src, g)
                if v is None:
                    assert words[2] == 0.0 and words[0] == -np.inf
                else:
                    assert words[:3] == v[:3] and words[3:] == v[3:]
    # (2) all words empty again
    for b in buf:
        assert (b == EMPTY).all()


@pytest.mark.parametrize("nranks,seed", [(2, 1), (2, 2), (3, 3), (4, 4), (4, 5), (8, 6)])
def test_exchange_protocol_under_adversarial_schedules(nranks, seed):
    _run(nranks, groups=3, payload=4, steps=9, seed=seed)
