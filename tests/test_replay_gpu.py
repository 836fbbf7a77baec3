"""GPU parity of the device trace-replay engine (strait_replay, one warp per
replay) through the C-ABI:

* every golden replay produced by the reference itself (tests/golden/replay,
  see tests/golden/gen_golden.py): decisions (pass, model, size, gpu), queue
  outcomes (per-request status / violated / batch), completion order, feedback
  flags, cap-row GPUs and HP/LP arrival/drop/violation counts bit-exact, and —
  because the device exp/log/pow restate the reference host's glibc — every
  float bit-identical too (the north_star bar is 1e-5 relative);
* many replays in one launch (seed / variant / load sweeps) against the C
  oracle run on the same buffers;
* BASELINE config 2 at full size (1M requests, 6 models x 4 GPUs) against the
  C oracle, plus size-independent invariants (every request resolved once,
  drops + violations consistent, work conservation);
* the reference's error behaviour for unsupported geometry.
"""
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN
from replay_cases import CASES, DEC_KEYS, FLOAT_KEYS, REQ_KEYS, case_config, overload_doc

pytestmark = pytest.mark.gpu

REL = 1e-5


def load(name):
    return dict(np.load(os.path.join(GOLDEN, "replay", f"{name}.npz")))


def close(got, want, rel=REL, atol=0.0, what=""):
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, f"{what}: shape {got.shape} vs {want.shape}"
    both_nan = np.isnan(got) & np.isnan(want)
    ok = both_nan | (got == want) | (np.abs(got - want) <= rel * np.abs(want) + atol)
    assert ok.all(), (f"{what}: {np.count_nonzero(~ok)} of {ok.size} beyond {rel} rel; first at "
                      f"{np.flatnonzero(~ok)[:5]}: {got[~ok][:3]} vs {want[~ok][:3]}")


def device_run(specs):
    from paper_2604_28175_b200.replay import ReplayBatch

    batch = ReplayBatch(specs)
    res = batch.run()
    return batch, res


def assert_categorical_equal(s, o, what):
    for k in REQ_KEYS + DEC_KEYS + ("b_done_order", "fb_flags", "cap_gpu"):
        np.testing.assert_array_equal(s[k], o[k], err_msg=f"{what}: {k}")


@pytest.mark.parametrize("name", CASES)
def test_replay_device_vs_reference_golden(cuda, name):
    from paper_2604_28175_b200.replay import ReplaySpec

    g = load(name)
    _, res = device_run([ReplaySpec(case_config(name))])
    res.check()
    s = res.replay_slice(0)
    assert len(s["dec_time"]) == len(g["dec_time"]), "number of batches differs"
    assert_categorical_equal(s, g, name)
    for k in FLOAT_KEYS:  # the device libm is the reference host's (strait_libm.cuh): bit-identical
        np.testing.assert_array_equal(s[k], g[k], err_msg=f"{name}: {k}")
    close(s["b_work"], g["b_work"], rel=1e-12, what=f"{name}: b_work")  # reference: compensated sum()
    np.testing.assert_array_equal(s["pred_state"], g["pred_state"], err_msg=f"{name}: pred_state")
    assert s["pred_step"] == int(g["pred_step"])
    c, cc = s["counters"], g["class_counts"]
    assert (c[6], c[7]) == (cc[0][0], cc[1][0])  # HP / LP arrivals
    assert (c[10], c[11]) == (cc[0][1], cc[1][1])  # drops
    assert (c[8], c[9]) == (cc[0][2], cc[1][2])  # violations (drops included, metrics.py:103-121)


def _sweep_specs():
    """A small C4-shaped sweep: overload seeds x variants x loads, one batch."""
    from paper_2604_28175_b200 import config as MC
    from paper_2604_28175_b200.replay import ReplaySpec

    specs = []
    for seed in range(8):
        specs.append(ReplaySpec(MC.config_from_dict(overload_doc(400)), seed))
    for v in ("no_meet", "no_violate_aimd", "no_priority_scan", "no_gamma_advantage"):
        specs.append(ReplaySpec(MC.config_from_dict(overload_doc(300, policy_variant=v)), 3))
    for lam in (0.5, 1.5, 2.5):
        doc = overload_doc(300)
        doc["workload"] = {m: dict(w, rate=w["rate"] * lam) for m, w in doc["workload"].items()}
        specs.append(ReplaySpec(MC.config_from_dict(doc), 11))
    specs.append(ReplaySpec(MC.config_from_dict(overload_doc(300, n_gpus=2)), 5))  # mixed geometry
    specs.append(ReplaySpec(MC.config_from_dict(overload_doc(300, n_gpus=7, concurrency_limit=3)), 6))
    return specs


def test_replay_many_in_one_launch_vs_oracle(cuda, oracle):
    specs = _sweep_specs()
    batch, res = device_run(specs)
    res.check()
    ores = oracle.replay(batch, threads=4)
    for r in range(batch.R):
        s, o = res.replay_slice(r), ores.replay_slice(r)
        assert len(s["dec_time"]) == len(o["dec_time"]), f"replay {r}: batches differ"
        assert_categorical_equal(s, o, f"replay {r}")
        for k in FLOAT_KEYS:
            np.testing.assert_array_equal(s[k], o[k], err_msg=f"replay {r}: {k}")
        np.testing.assert_array_equal(s["counters"][6:13], o["counters"][6:13], err_msg=f"replay {r}")


def test_replay_c2_full_size_vs_oracle(cuda, oracle):
    """BASELINE configs[1]: overload.yaml at 166.667 s => ~1.0M requests."""
    from paper_2604_28175_b200 import config as MC
    from paper_2604_28175_b200.replay import ReplaySpec

    batch, res = device_run([ReplaySpec(MC.config_from_dict(overload_doc(166667)))])
    res.check()
    assert batch.N > 990_000
    ores = oracle.replay(batch)
    s, o = res.replay_slice(0), ores.replay_slice(0)
    c = s["counters"]
    np.testing.assert_array_equal(c[6:13], o["counters"][6:13])
    assert_categorical_equal(s, o, "C2")
    for k in FLOAT_KEYS:
        np.testing.assert_array_equal(s[k], o[k], err_msg=f"C2: {k}")
    # size-independent invariants
    status = s["req_status"]
    assert np.all(status > 0), "unresolved requests"
    assert c[12] == batch.N
    assert np.count_nonzero(status == 2) == c[10] + c[11]
    assert np.count_nonzero(s["req_violated"]) == c[8] + c[9]
    assert int(np.bincount(s["req_batch"][s["req_batch"] >= 0]).sum()) == int(s["dec_size"].astype(np.int64).sum())
    # work conservation: every batch consumed exactly its isolated kernel latency
    from paper_2604_28175_b200.replay import model_tables

    tab = batch.tab
    kern = tab["kernel"][s["dec_model"].astype(np.int64) * tab["B"] + s["dec_size"].astype(np.int64) - 1]
    close(s["b_work"], kern, rel=1e-9, what="work conservation")
    assert np.all(s["b_kernel_start"] >= s["b_transfer_end"] - 1e-9)


def test_replay_wide_geometry_vs_oracle(cuda, oracle):
    """Concurrency limits up to 32 per GPU, and nodes past the one-warp
    shared-memory budget (128 GPUs: one replay per CTA of 8 warps, traced and
    untraced), against the oracle."""
    from paper_2604_28175_b200 import config as MC
    from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec

    specs = [ReplaySpec(MC.config_from_dict(overload_doc(200, concurrency_limit=c, n_gpus=g)), c)
             for c, g in ((9, 4), (12, 2), (32, 1))]
    batch, res = device_run(specs)
    res.check()
    ores = oracle.replay(batch, threads=3)
    for r in range(batch.R):
        s, o = res.replay_slice(r), ores.replay_slice(r)
        assert_categorical_equal(s, o, f"replay {r}")
        for k in FLOAT_KEYS:
            np.testing.assert_array_equal(s[k], o[k], err_msg=f"replay {r}: {k}")
    # 128 GPUs x 4 slots; 76 GPUs x 8 slots (past the one-warp budget: CTA layout only)
    for g, c in ((128, 4), (76, 8)):
        big = [ReplaySpec(MC.config_from_dict(overload_doc(150, n_gpus=g, concurrency_limit=c)), 1)]
        for trace in (False, True):
            b = ReplayBatch(big, trace=trace)
            rb = b.run()
            rb.check()
            s, o = rb.replay_slice(0), oracle.replay(b, threads=1).replay_slice(0)
            assert_categorical_equal(s, o, f"{g} GPUs x {c} trace={trace}")
            for k in FLOAT_KEYS:
                np.testing.assert_array_equal(s[k], o[k], err_msg=f"{g} GPUs x {c} trace={trace}: {k}")


def test_replay_rejects_unsupported_geometry(cuda):
    """Past 32 running batches per GPU (one lane per list position), or past
    the 227 KB a CTA can hold, the launch raises instead of running."""
    from paper_2604_28175_b200 import config as MC
    from paper_2604_28175_b200.replay import ReplaySpec

    with pytest.raises(ValueError):
        device_run([ReplaySpec(MC.config_from_dict(overload_doc(100, concurrency_limit=33)))])
    with pytest.raises(ValueError):
        device_run([ReplaySpec(MC.config_from_dict(overload_doc(100, n_gpus=1024)))])


@pytest.mark.parametrize("name", CASES)
def test_replay_metrics_vs_reference(cuda, name):
    """Device compute_metrics (strait_replay_metrics) equals the reference's
    MetricsReport.to_dict() of the same replay — counts, exact nearest-rank
    percentiles, goodput windows and the error-series statistics."""
    import json

    from paper_2604_28175_b200.replay import ReplaySpec

    g = load(name)
    _, res = device_run([ReplaySpec(case_config(name))])
    got = res.metrics(0)
    want = json.loads(str(g["metrics_json"]))
    want.pop("window_ms"), got.pop("window_ms")
    assert got == want
