"""Request sharding across the GPUs of one box: independent MPIC requests
need no collective, so each rank owns a disjoint subset of the requests, balanced by the
predicted recompute cost. Only the timing reduction (max over ranks) crosses processes.

Pure host logic on purpose: it is exercised with the gloo backend on CPU by
tests/test_dist.py and drives bench.py --gpus N under torchrun (NCCL)."""
from __future__ import annotations

import heapq

import numpy as np


def request_cost(n_layers: int, hidden: int, rows, vocab: int = 0) -> float:
    """Algorithmic FLOPs of one selective pass: L·(24·m·h² + 4·h·Σ(pos_i+1))
    + 2·h·V for lm_head."""
    rows = np.asarray(rows, np.float64)
    m = float(rows.size)
    return n_layers * (24.0 * m * hidden * hidden + 4.0 * hidden * float(np.sum(rows + 1.0))) + \
        2.0 * hidden * vocab


def shard_requests(costs, world: int) -> list[list[int]]:
    """Longest-processing-time-first assignment of request indices to `world` ranks.
    Deterministic (ties by index), so every rank computes the same plan locally."""
    order = sorted(range(len(costs)), key=lambda i: (-float(costs[i]), i))
    heap = [(0.0, r) for r in range(world)]
    heapq.heapify(heap)
    out: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + float(costs[i]), r))
    for lst in out:
        lst.sort()
    return out


def max_over_ranks(value: float, group=None) -> float:
    """Max of a per-rank timing across the process group (identity when not distributed)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(value: float, group=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())
