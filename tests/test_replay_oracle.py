"""CPU: the C replay oracle (oracle/strait_replay_oracle.c) reproduces the
reference simulator bit for bit on every golden replay — decisions, request
outcomes, batch lifecycles, feedback, cap rows and the final predictor — and
the host-side inputs (arrival streams) match the reference's streams."""
import os

import numpy as np
import pytest

from conftest import GOLDEN
from replay_cases import CASES, DEC_KEYS, FLOAT_KEYS, REQ_KEYS, case_config

SMALL = [c for c in CASES if c not in ("overload",)]


def load(name):
    return dict(np.load(os.path.join(GOLDEN, "replay", f"{name}.npz")))


def run_oracle(oracle, name):
    from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec

    batch = ReplayBatch([ReplaySpec(case_config(name))])
    res = oracle.replay(batch)
    return batch, res


@pytest.mark.parametrize("name", CASES)
def test_replay_oracle_bit_exact(oracle, name):
    g = load(name)
    batch, res = run_oracle(oracle, name)
    assert int(res.counters[0][0]) == 0
    s = res.replay_slice(0)
    assert len(s["dec_time"]) == len(g["dec_time"])
    for k in REQ_KEYS + DEC_KEYS + ("b_done_order", "fb_flags", "cap_gpu"):
        np.testing.assert_array_equal(s[k], g[k], err_msg=k)
    for k in FLOAT_KEYS:
        np.testing.assert_array_equal(s[k], g[k], err_msg=k)
    np.testing.assert_allclose(s["b_work"], g["b_work"], rtol=1e-12, atol=0)
    np.testing.assert_array_equal(s["pred_state"], g["pred_state"])
    assert s["pred_step"] == int(g["pred_step"])
    c = s["counters"]
    cc = g["class_counts"]
    assert (c[6], c[7]) == (cc[0][0], cc[1][0])  # arrivals
    assert (c[10], c[11]) == (cc[0][1], cc[1][1])  # drops
    assert (c[8], c[9]) == (cc[0][2], cc[1][2])  # violations


def test_replay_batch_many_seeds_parallel(oracle):
    """Threads over independent replays give the same results as one thread."""
    from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec
    from replay_cases import overload_doc
    from paper_2604_28175_b200 import config as MC

    specs = [ReplaySpec(MC.config_from_dict(overload_doc(200)), seed) for seed in range(6)]
    b = ReplayBatch(specs)
    r1 = oracle.replay(b, threads=1)
    r4 = oracle.replay(b, threads=4)
    for k in ("req_status", "dec_gpu", "dec_est_latency", "counters", "pred_state"):
        np.testing.assert_array_equal(r1.a[k], r4.a[k])


def test_csv_fingerprints_are_the_surveys():
    """The reference CSV fingerprints the GPU byte-identity tests compare against
    (tests/golden/replay_csv_sha.json) carry the trace hashes SURVEY.md recorded
    independently: §8(c) for demo / overload / C1, Appendix A for overload seeds 0-15."""
    import json
    import re

    from conftest import REPO

    sha = json.load(open(os.path.join(GOLDEN, "replay_csv_sha.json")))
    survey = open(os.path.join(REPO, "SURVEY.md")).read()
    app = dict(re.findall(r"^\| (\d+) \| [\d.]+ \| [\d.]+ \| `([0-9a-f]{64})` \|$", survey, flags=re.M))
    assert len(app) == 16
    for s, h in app.items():
        assert sha["overload_seeds"][s]["trace"] == h, s
    for case, tag in (("demo", "`demo.yaml` seed 1"), ("overload", "`overload.yaml` seed 0"),
                      ("c1", "C1 restated")):
        m = re.search(re.escape(tag) + r"[^`]*`([0-9a-f]{64})`", survey)
        assert m and sha["cases"][case]["trace"] == m.group(1), case
    assert set(sha["cases"]) == set(CASES)
    assert all(set(v) == {"trace", "requests", "decisions", "feedback", "caps", "batches"}
               for v in list(sha["cases"].values()) + list(sha["overload_seeds"].values()))


def test_launch_api_is_for_untraced_batches():
    """ReplayBatch.launch() (asynchronous) rejects traced batches before any
    device work: a trace may overflow and need a synchronous re-run."""
    from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec

    b = ReplayBatch([ReplaySpec(case_config("demo"))], trace=True)
    with pytest.raises(ValueError, match="untraced"):
        b.launch()
    assert b.trace_max > 0 and ReplayBatch([ReplaySpec(case_config("demo"))]).trace_max == 0
