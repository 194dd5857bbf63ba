"""Host-side bookkeeping of the FSDP symmetric pool (no GPU): placement must
be a pure function of the allocate/release sequence, so every rank of an SPMD
program lands its all-gather outputs at the same offsets."""

import random

from paper_2402_06787_b200.fsdp import Extents


def test_best_fit_and_coalescing():
    e = Extents(1000)
    a = e.alloc(100)
    b = e.alloc(300)
    c = e.alloc(100)
    assert (a, b, c) == (0, 100, 400)
    e.release(b, 300)
    assert e.alloc(50) == 100          # best fit: the 300-byte hole, not the tail
    e.release(100, 50)
    e.release(a, 100)
    e.release(c, 100)
    assert e.extents() == [(0, 1000)]  # fully coalesced
    assert e.alloc(1001) is None


def test_placement_is_deterministic_across_replays():
    def replay(seed):
        rng = random.Random(seed)
        e = Extents(1 << 20)
        live, trace = [], []
        for _ in range(2000):
            if live and rng.random() < 0.45:
                off, n = live.pop(rng.randrange(len(live)))
                e.release(off, n)
            else:
                n = rng.choice([4096, 8192, 65536, 3 * 4096])
                off = e.alloc(n)
                trace.append(off)
                if off is not None:
                    live.append((off, n))
        for off, n in live:
            e.release(off, n)
        assert e.free_bytes == 1 << 20 and e.extents() == [(0, 1 << 20)]
        return trace

    assert replay(3) == replay(3)   # same call sequence -> same offsets (every rank)


def test_no_overlap_between_live_blocks():
    rng = random.Random(5)
    e = Extents(1 << 16)
    live = []
    for _ in range(500):
        if live and rng.random() < 0.5:
            e.release(*live.pop(rng.randrange(len(live))))
        else:
            n = rng.choice([512, 1024, 4096])
            off = e.alloc(n)
            if off is not None:
                for o, m in live:
                    assert off + n <= o or o + m <= off
                live.append((off, n))
