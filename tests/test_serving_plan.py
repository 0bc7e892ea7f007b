"""Config E host logic (bench.py): the seeded 256-request list and its request sharding over
ranks (independent requests, no collective)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def test_serving_requests_are_seeded_and_shaped():
    h1, r1 = bench.serving_requests(32000)
    h2, r2 = bench.serving_requests(32000)
    assert h1 == h2 and [im for _, im in r1] == [im for _, im in r2]
    assert len(r1) == bench.E_REQUESTS and len(h1) == bench.E_POOL
    for segs, imgs in r1:
        assert 1 <= len(imgs) <= 4
        assert [s[0] for s in segs] == ["text", "image"] * len(imgs) + ["text"]
        assert all(len(s[1]) == 32 + 7 * i for i, s in enumerate(segs[0:-1:2]))
        assert all(s[2] == 576 and s[1] == h1[c] for s, c in zip(segs[1::2], imgs))


def test_shard_requests_partitions_and_balances():
    _, reqs = bench.serving_requests(32000)
    for world in (1, 2, 4, 8):
        parts = [bench.shard_requests(reqs, world, r) for r in range(world)]
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(reqs)))  # every request exactly once
        cost = lambda i: len(reqs[i][1]) * 32 + sum(len(s[1]) for s in reqs[i][0] if s[0] == "text")
        loads = [sum(cost(i) for i in p) for p in parts]
        assert max(loads) - min(loads) <= max(cost(i) for i in range(len(reqs)))
