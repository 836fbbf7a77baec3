"""GPU: parity on exactly the inputs bench.py times (VERDICT r1 "parity on
what is benched"): the C3 round 0 in full (2^16 segments x 64 GPUs x 4 slots,
the headline kernel's input) and all 1,024 replays of the C4 load x
HP-fraction grid, device vs the CPU oracle, every decision and float
bit-exact.  bench.py re-checks the same on each run and reports it under
"parity"."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

P_INIT = np.array([0.1, np.e, 0.0] + [0.1] * 5 + [0.1, 0.1, 0.5, 1.0])  # PredictorParams() defaults


def _threads():
    return len(os.sched_getaffinity(0))


def test_c3_round0_full_matches_oracle(cuda, oracle):
    from paper_2604_28175_b200 import sweep as SW
    from paper_2604_28175_b200.microbench import C3_SEGMENTS, c3_round

    soa = c3_round(0, n_segments=C3_SEGMENTS)
    got = SW.sweep(soa, P_INIT)
    assert SW.last_sweep_path() == "tma-tensor"  # the benched kernel
    want = oracle.sweep(soa, P_INIT, threads=_threads())
    for k, v in want.items():
        assert np.array_equal(got[k], v, equal_nan=v.dtype.kind == "f"), k
    placed = (want["seg_gpu"] >= 0).mean()
    assert 0.05 < placed < 0.99, placed  # a round with both placed and unplaceable segments


def test_c4_grid_matches_oracle(cuda, oracle):
    from paper_2604_28175_b200.configs import c4_grid
    from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec

    specs = [ReplaySpec(c, s) for c, s in c4_grid(seeds=16)]
    assert len(specs) == 1024
    dev = ReplayBatch(specs, generate="device").run(metrics=False)  # streams drawn on the device
    host = ReplayBatch(specs)  # numpy streams, as the reference draws them
    ref = oracle.replay(host, threads=_threads())
    assert host.N == dev.batch.N
    keys = ("req_status", "req_violated", "req_completion", "req_batch", "dec_time", "dec_pass", "dec_model",
            "dec_size", "dec_gpu", "dec_est_latency", "dec_intf", "b_kernel_start", "b_kernel_end", "fb_predicted",
            "fb_actual", "cap_time", "cap_gpu", "cap_pct", "pred_state", "pred_step")
    counters = [0, 1, 2, 3, 4, 6, 7, 8, 9, 10, 11, 12]  # all but EVENTS (the reference's stale pops) and TRACE
    for r in range(len(specs)):
        a, b = ref.replay_slice(r), dev.replay_slice(r)
        for k in keys:
            x, y = np.asarray(a[k]), np.asarray(b[k])
            assert x.shape == y.shape and np.array_equal(x, y, equal_nan=x.dtype.kind == "f"), (r, k)
        assert np.array_equal(np.asarray(a["counters"])[counters], np.asarray(b["counters"])[counters]), r
