"""Multi-process host logic of the request-sharded path, world_size 2 over gloo on CPU:
every rank derives the same LPT plan locally, the shards are disjoint and complete, and
timings reduce by max over ranks (what bench.py --gpus N reports)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_01960_b200 import dist as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        costs = [pdist.request_cost(32, 4096, np.sort(rng.choice(9000, 100 + 50 * (i % 5), replace=False)))
                 for i in range(37)]
        plan = pdist.shard_requests(costs, world)
        mine = plan[rank]
        t = float(sum(costs[i] for i in mine)) * 1e-12 + rank  # a fake per-rank time
        tmax = pdist.max_over_ranks(t)
        total = pdist.sum_over_ranks(len(mine))
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        q.put((rank, plan, mine, tmax, total, gathered))
    finally:
        dist.destroy_process_group()


def test_request_sharding_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    (_, plan0, mine0, tmax0, tot0, gath0), (_, plan1, mine1, tmax1, tot1, gath1) = res
    assert plan0 == plan1  # deterministic plan on every rank
    assert sorted(mine0 + mine1) == list(range(37)) and not set(mine0) & set(mine1)
    assert tmax0 == tmax1 and tmax0 >= 1.0  # rank 1's fake time includes +1
    assert tot0 == tot1 == 37
    assert gath0 == gath1 == [mine0, mine1]


def test_lpt_balance():
    costs = [10, 9, 8, 7, 6, 5, 4, 3, 2, 1]
    plan = pdist.shard_requests(costs, 3)
    loads = [sum(costs[i] for i in p) for p in plan]
    assert max(loads) - min(loads) <= 2
    assert pdist.shard_requests([1.0], 4) == [[0], [], [], []]
