"""GPU: bench.py's multi-rank paths on the device engine — two ranks launched
by torchrun sharing cuda:0 over gloo (STRAIT_DIST_BACKEND=gloo; one GPU per
gpurun box).  C3 weak (a round per rank) and strong (contiguous slices of
whole segments of one round, redundant refit), C4 LPT-sharded replays with
the end-of-run counter all-reduce; every rank's outputs parity-checked
against the CPU oracle on its own inputs."""
import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_on_device(cuda):
    env = dict(os.environ, STRAIT_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", "bench.py", "--gpus", "2", "--steps", "5",
           "--warmup", "3", "--segments", "4096", "--e2e-steps", "2", "--replay-steps", "1", "--replay-seeds", "1",
           "--no-single", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert all(v is True for v in line["parity"].values()), line["parity"]
    assert line["c3_strong"]["segments_rank0"] == [0, 2048]
    c4 = line["c4"]
    assert c4["replays"] == 64 and len(c4["assignment"]["ranks"]) == 2
    assert sum(rk["replays"] for rk in c4["assignment"]["ranks"]) == 64
    assert c4["parity"]["ok"] is True
    assert line["value"] > 0 and c4["value"] > 0
