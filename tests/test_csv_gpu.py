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
