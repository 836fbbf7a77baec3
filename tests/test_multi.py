"""CPU, world_size 2 over gloo: the replay sharding (replay r -> rank r mod N)
and the end-of-run counter all-reduce used by bench.py's multi-GPU leg give the
same global HP/LP counts as one process replaying everything (C oracle as the
replay engine, since the CPU suite has no GPU)."""
import json
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _specs():
    from paper_2604_28175_b200.configs import c4_point
    from paper_2604_28175_b200.replay import ReplaySpec

    pts = [(0.5, 0.2), (1.0, 0.5), (2.0, 0.8)]
    return [ReplaySpec(c4_point(lam, f, duration=200), s) for lam, f in pts for s in range(3)]


def _worker(rank, world, port, out):
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from oracle import oracle
    from paper_2604_28175_b200.replay import ReplayBatch
    from paper_2604_28175_b200.shard import global_counts, shard

    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard(_specs(), world, rank)
    res = oracle.replay(ReplayBatch(mine))
    g = global_counts(res.counters, dist)
    if rank == 0:
        with open(out, "w") as f:
            json.dump(g, f)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_counts_equal_single_process(oracle, tmp_path):
    from paper_2604_28175_b200.replay import ReplayBatch
    from paper_2604_28175_b200.shard import global_counts, shard

    out = str(tmp_path / "g.json")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = json.load(open(out))
    want = global_counts(oracle.replay(ReplayBatch(_specs())).counters)
    assert got == want
    assert want["HP_ARR"] + want["LP_ARR"] == want["RESOLVED"] > 0
    # every replay lands on exactly one rank
    items = list(range(11))
    assert sorted(shard(items, 4, 0) + shard(items, 4, 1) + shard(items, 4, 2) + shard(items, 4, 3)) == items
    with pytest.raises(ValueError):
        shard(items, 2, 2)


# ----------------------------------------------------------------------------- C3 strong partition
def _c3_worker(rank, world, port, out, segs):
    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import numpy as np
    import torch.distributed as dist

    from oracle import oracle
    from paper_2604_28175_b200.microbench import c3_feedback, c3_round

    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = c3_round(0, n_segments=segs, gpus=16, slots=4, concurrency_limit=5)
    s0, s1 = rank * segs // world, (rank + 1) * segs // world  # contiguous whole segments
    P = np.array([0.1, np.e, 0.0] + [0.1] * 5 + [0.1, 0.1, 0.5, 1.0])
    mine = oracle.sweep(full.slice_segments(s0, s1), P)
    # the refit chain runs redundantly on every rank: no parameter exchange
    state = np.concatenate([P, np.zeros(24)])
    state, _, _, _, _ = oracle.refit(state, 0, c3_feedback(0), nm=5)
    got = [None] * world
    dist.all_gather_object(got, {"range": (s0, s1), "out": {k: v.tolist() for k, v in mine.items()},
                                 "state": state.tolist()})
    if rank == 0:
        with open(out, "w") as f:
            json.dump(got, f)
    dist.barrier()
    dist.destroy_process_group()


def test_c3_strong_partition_equals_single_round(oracle, tmp_path):
    """Each rank scores a contiguous slice of whole segments (a segment's pairs
    never split) and refits redundantly; the concatenated slices equal one
    process scoring the whole round, and every rank holds the same predictor."""
    import numpy as np

    from paper_2604_28175_b200.microbench import c3_feedback, c3_round

    segs = 96
    out = str(tmp_path / "c3.json")
    mp.spawn(_c3_worker, args=(2, _free_port(), out, segs), nprocs=2, join=True)
    got = json.load(open(out))
    P = np.array([0.1, np.e, 0.0] + [0.1] * 5 + [0.1, 0.1, 0.5, 1.0])
    want = oracle.sweep(c3_round(0, n_segments=segs, gpus=16, slots=4, concurrency_limit=5), P)
    assert [g["range"] for g in got] == [[0, 48], [48, 96]]
    for k, v in want.items():
        cat = np.concatenate([np.asarray(g["out"][k], dtype=v.dtype) for g in got])
        assert np.array_equal(cat, v, equal_nan=v.dtype.kind == "f"), k
    state, _, _, _, _ = oracle.refit(np.concatenate([P, np.zeros(24)]), 0, c3_feedback(0), nm=5)
    assert all(g["state"] == state.tolist() for g in got)


def test_lpt_assignment_balances_and_covers():
    """C4's longest-first assignment: every replay on exactly one rank, each
    rank's share in decreasing cost, loads within one replay of each other."""
    from paper_2604_28175_b200.configs import c4_grid
    from paper_2604_28175_b200.shard import lpt

    grid = c4_grid(seeds=2)
    costs = [sum(w.rate_per_s for w in c.workload.models.values()) * c.workload.duration_ms / 1e3 for c, _ in grid]
    for world in (1, 2, 4, 8):
        parts = lpt(costs, world)
        assert sorted(i for p in parts for i in p) == list(range(len(grid)))
        loads = [sum(costs[i] for i in p) for p in parts]
        assert max(loads) - min(loads) <= max(costs) + 1e-9
        for p in parts:
            assert [costs[i] for i in p] == sorted((costs[i] for i in p), reverse=True)
