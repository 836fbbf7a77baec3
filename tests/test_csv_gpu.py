"""GPU: byte-identical run outputs.  A traced device replay's six run-directory
CSVs (report.py:40-47 — trace, requests, decisions, feedback, caps, batches)
have the same SHA-256 as the reference's for the same config and seed.

Fingerprints: tests/golden/replay_csv_sha.json, made by running the reference
itself (tests/golden/gen_golden.py csvsha).  They cover every golden replay
case and overload.yaml seeds 0-15, whose trace hashes are also SURVEY.md
Appendix A's (checked on CPU in test_replay_oracle.py).  Byte identity of
trace.csv pins the event order (including the interleaving of arrivals, drops,
submissions, kernel starts/completions, AIMD ticks and resets). Byte identity
of batches.csv pins every execution segment (d, slowdown). Byte identity of
requests.csv pins the resolution order.
"""
import hashlib
import json
import os

import pytest

from conftest import GOLDEN
from replay_cases import CASES, case_config, overload_doc

pytestmark = pytest.mark.gpu

SHA = json.load(open(os.path.join(GOLDEN, "replay_csv_sha.json")))


def _sha(res):
    from paper_2604_28175_b200.report import csv_texts

    return {k: hashlib.sha256(t.encode()).hexdigest() for k, t in csv_texts(res).items()}


@pytest.mark.parametrize("name", CASES)
def test_run_directory_csvs_match_reference(name):
    from paper_2604_28175_b200 import Simulation

    res = Simulation(case_config(name)).run()
    got = _sha(res)
    assert got == SHA["cases"][name], {k: (got[k][:12], SHA["cases"][name][k][:12]) for k in got}
    assert res.trace_hash() == SHA["cases"][name]["trace"]


def test_overload_seed_sweep_one_launch_matches_reference():
    """overload.yaml seeds 0-15 as ONE traced launch of 16 replays."""
    from paper_2604_28175_b200 import config as MC
    from paper_2604_28175_b200.replay import ReplaySpec
    from paper_2604_28175_b200.simulation import run_many

    cfg = MC.config_from_dict(overload_doc())
    results = run_many([ReplaySpec(cfg, s) for s in range(16)])
    for s, res in enumerate(results):
        got = _sha(res)
        assert got == SHA["overload_seeds"][str(s)], (s, {k: got[k][:12] for k in got})


def test_trace_log_overflow_reruns_with_exact_capacity():
    """A too-small trace_max is detected from the device counter and the batch
    re-runs with the exact capacity; the log is the same."""
    from paper_2604_28175_b200 import config as MC
    from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec
    from paper_2604_28175_b200.simulation import SimResult, _report

    cfg = MC.config_from_dict(overload_doc(300))
    b = ReplayBatch([ReplaySpec(cfg)], trace=True, trace_max=100)
    res = b.run()
    assert b.trace_max > 100
    r = SimResult(cfg.policy, cfg.policy_variant, cfg.seed, res, 0, _report(res, 0))
    want = ReplayBatch([ReplaySpec(cfg)], trace=True).run()
    assert (res.trace_records(0) == want.trace_records(0)).all()
    assert len(r.trace_rows) > 0


def test_untraced_run_has_no_event_log():
    from paper_2604_28175_b200 import Simulation

    res = Simulation(case_config("demo")).run(trace=False)
    assert res.trace_rows == [] and not res.traced
    assert all(b["segments"] == "" for b in res.batch_rows)


@pytest.mark.parametrize("name", ["demo", "overload", "ov_no_meet", "ov_reactive", "c5_slice"])
def test_compute_metrics_and_report_from_run_dir_match_reference(name, tmp_path):
    """compute_metrics over the SimResult rows (device launch over row arrays)
    and report_from_run_dir over the written CSVs both equal the reference's
    MetricsReport.to_dict() of the same replay (golden metrics_json)."""
    import numpy as np

    from paper_2604_28175_b200 import Simulation, compute_metrics
    from paper_2604_28175_b200.report import report_from_run_dir, write_run_dir

    g = dict(np.load(os.path.join(GOLDEN, "replay", f"{name}.npz")))
    want = json.loads(str(g["metrics_json"]))
    w = float(g["goodput_window_ms"])
    res = Simulation(case_config(name)).run()
    m = compute_metrics(res.request_rows, res.batch_rows, res.feedback_rows, res.cap_rows, window_ms=w)
    assert m.to_dict() == want
    assert m.cap_timeline == res.metrics.cap_timeline
    assert m.intf_error == res.metrics.intf_error and m.kernel_overhead == res.metrics.kernel_overhead
    write_run_dir(res, tmp_path / "run")
    assert report_from_run_dir(tmp_path / "run", window_ms=w).to_dict() == want


def test_compute_metrics_partial_and_empty():
    from paper_2604_28175_b200 import compute_metrics

    rows = [{"priority": "high", "arrival": 1.0, "dropped": 0, "completion": "", "violated": 0, "latency": ""},
            {"priority": "low", "arrival": 2.0, "dropped": 1, "completion": "", "violated": 1, "latency": ""},
            {"priority": "low", "arrival": 3.0, "dropped": 0, "completion": 2500.0, "violated": 0,
             "latency": 2497.0}]
    d = compute_metrics(rows, window_ms=1000.0).to_dict()
    assert d["partial"] is True
    assert d["high"]["arrivals"] == 1 and d["high"]["completed"] == 0 and d["high"]["p50_latency_ms"] is None
    assert d["low"] == {"arrivals": 2, "completed": 1, "dropped": 1, "violations": 1, "violation_rate_pct": 50.0,
                        "p50_latency_ms": 2497.0, "p95_latency_ms": 2497.0, "p99_latency_ms": 2497.0,
                        "goodput_counts": [0, 0, 1]}
    assert d["intf_error"] == {"count": 0} and d["kernel_overhead"] == {"count": 0}
    e = compute_metrics([]).to_dict()
    assert e["high"]["arrivals"] == 0 and e["partial"] is False


def test_ground_truth_slowdown_bit_exact():
    """ground_truth_slowdown (strait_gt_slowdown) equals the reference's
    oracle.py:55-77 on 4,000 random inputs (tests/golden/gt.npz), both families."""
    import numpy as np

    from paper_2604_28175_b200 import GroundTruthParams, PriorityLevel, ground_truth_slowdown
    from paper_2604_28175_b200.ground_truth import ground_truth_slowdown_batch

    g = dict(np.load(os.path.join(GOLDEN, "gt.npz")))
    got = np.empty(len(g["out"]))
    for i in range(len(got)):
        p = GroundTruthParams(family="quadratic" if g["family"][i] else "exponential", scale=float(g["scale"][i]),
                              base=float(g["base"][i]), offset=float(g["offset"][i]),
                              weights=tuple(g["w"][i].tolist()), self_compute_weight=float(g["w_cmp"][i]),
                              self_memory_weight=float(g["w_mem"][i]),
                              priority_factor={PriorityLevel.HIGH: float(g["pf"][i][0]),
                                               PriorityLevel.LOW: float(g["pf"][i][1])})
        got[i] = ground_truth_slowdown(p, g["co"][i].tolist(), float(g["cmp"][i]), float(g["mem"][i]),
                                       PriorityLevel(int(g["prio"][i])), float(g["noise"][i]))
    assert np.array_equal(got, g["out"]), np.flatnonzero(got != g["out"])[:5]
    # one params set, many inputs in one launch
    p = GroundTruthParams()
    co = np.random.default_rng(0).uniform(0, 2, (1000, 5))
    b = ground_truth_slowdown_batch(p, co, np.full(1000, 0.5), np.full(1000, 0.4), np.zeros(1000, np.int8))
    assert b[0] == ground_truth_slowdown(p, co[0].tolist(), 0.5, 0.4, PriorityLevel.HIGH)
    with pytest.raises(ValueError, match="metrics"):
        ground_truth_slowdown(p, [1.0, 2.0], 0.5, 0.4, PriorityLevel.HIGH)
