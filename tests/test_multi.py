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
