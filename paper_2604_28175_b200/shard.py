"""Sharding of independent replays across ranks (one process per GPU) and
the end-of-run counter reduction — the multi-GPU plumbing of SURVEY §8(e).

Replays never communicate: replay r runs on rank r mod world (the analogue of
`infersim sweep`'s process pool, cli.py:64-103), and the only collective is
one all-reduce (NCCL on GPUs, gloo in the CPU tests) of the per-class
counters at the end.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np

from .replay import RC

COUNT_KEYS = ("HP_ARR", "LP_ARR", "HP_VIOL", "LP_VIOL", "HP_DROP", "LP_DROP", "BATCHES", "COMPLETED", "RESOLVED")


def shard(items: Sequence, world: int, rank: int) -> list:
    """Items of this rank: r -> rank r mod world."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    return list(items[rank::world])


def lpt(costs: Sequence[float], world: int) -> list[list[int]]:
    """Longest-processing-time-first assignment of independent replays to
    ranks: replays in decreasing cost, each to the rank with the least
    assigned cost so far (ties: lowest rank).  Returns each rank's replay
    indices in decreasing cost."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [0.0] * world
    out: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        out[r].append(i)
        load[r] += costs[i]
    return out


def shard_lpt(items: Sequence, costs: Sequence[float], world: int, rank: int) -> list:
    """This rank's items under lpt()."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    return [items[i] for i in lpt(costs, world)[rank]]


def local_counts(counters: np.ndarray) -> np.ndarray:
    """Sum of the per-replay counters [R, STRAIT_RC_N] over this rank's replays."""
    c = np.asarray(counters).reshape(-1, np.asarray(counters).shape[-1])
    if (c[:, RC["ERROR"]] != 0).any():
        raise RuntimeError("a replay reported an error")
    return np.array([c[:, RC[k]].sum() for k in COUNT_KEYS], dtype=np.int64)


def global_counts(counters: np.ndarray, dist=None, device=None) -> dict:
    """Counters summed over every rank's replays (one all-reduce)."""
    import torch

    v = torch.from_numpy(local_counts(counters))
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        if device is not None:
            v = v.to(device)
        dist.all_reduce(v, op=dist.ReduceOp.SUM)
    out = dict(zip(COUNT_KEYS, (int(x) for x in v.cpu().tolist())))
    out["hp_violation_pct"] = 100.0 * out["HP_VIOL"] / out["HP_ARR"] if out["HP_ARR"] else 0.0
    out["lp_violation_pct"] = 100.0 * out["LP_VIOL"] / out["LP_ARR"] if out["LP_ARR"] else 0.0
    return out
