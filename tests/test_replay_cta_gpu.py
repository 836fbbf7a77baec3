"""GPU parity of both replay-engine layouts on every reference golden replay:
one warp per replay (STRAIT_REPLAY_NW=1) and one CTA of 8 warps per replay
(STRAIT_REPLAY_NW=8: the master warp runs the event loop, the helper warps
join the intf_cur and propose jobs).  The launcher picks the CTA
layout by itself only for wide geometries (more running-batch slots than a
warp has lanes, e.g. C5's 64 GPUs); forcing it here runs the CTA jobs on
every geometry, including the all-sizes propose job (few GPUs) and the
probe-by-probe one (many GPUs).  Decisions, outcomes and every float must be
bit-identical to the reference.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN
from replay_cases import CASES, DEC_KEYS, FLOAT_KEYS, REQ_KEYS, case_config

pytestmark = pytest.mark.gpu


def load(name):
    return dict(np.load(os.path.join(GOLDEN, "replay", f"{name}.npz")))


@pytest.mark.parametrize("nw", ["1", "8"])
@pytest.mark.parametrize("name", CASES)
def test_engine_layouts_vs_reference_golden(cuda, monkeypatch, name, nw):
    from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec

    monkeypatch.setenv("STRAIT_REPLAY_NW", nw)
    g = load(name)
    res = ReplayBatch([ReplaySpec(case_config(name))]).run()
    res.check()
    s = res.replay_slice(0)
    assert len(s["dec_time"]) == len(g["dec_time"]), "number of batches differs"
    for k in REQ_KEYS + DEC_KEYS + ("b_done_order", "fb_flags", "cap_gpu"):
        np.testing.assert_array_equal(s[k], g[k], err_msg=f"{name} nw={nw}: {k}")
    for k in FLOAT_KEYS:
        np.testing.assert_array_equal(s[k], g[k], err_msg=f"{name} nw={nw}: {k}")
    np.testing.assert_array_equal(s["pred_state"], g["pred_state"], err_msg=f"{name} nw={nw}: pred_state")


def test_cta_layout_many_replays_vs_oracle(cuda, oracle, monkeypatch):
    """Several CTA replays in one launch (one per CTA), mixed geometries, vs the oracle."""
    from paper_2604_28175_b200 import config as MC
    from paper_2604_28175_b200.configs import c5
    from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec
    from replay_cases import overload_doc

    monkeypatch.setenv("STRAIT_REPLAY_NW", "8")
    specs = [ReplaySpec(MC.config_from_dict(overload_doc(300, n_gpus=g, concurrency_limit=c)), s)
             for s, (g, c) in enumerate([(4, 4), (2, 3), (7, 3), (12, 4), (1, 4)])]
    batch = ReplayBatch(specs)
    res = batch.run()
    res.check()
    ores = oracle.replay(batch, threads=4)
    for r in range(batch.R):
        s, o = res.replay_slice(r), ores.replay_slice(r)
        for k in REQ_KEYS + DEC_KEYS + FLOAT_KEYS:
            np.testing.assert_array_equal(s[k], o[k], err_msg=f"replay {r}: {k}")
    c5b = ReplayBatch([ReplaySpec(c5(60.0), 0), ReplaySpec(c5(60.0), 1)])
    cres = c5b.run()
    cres.check()
    ores = oracle.replay(c5b, threads=2)
    for r in range(2):
        s, o = cres.replay_slice(r), ores.replay_slice(r)
        for k in REQ_KEYS + DEC_KEYS + FLOAT_KEYS:
            np.testing.assert_array_equal(s[k], o[k], err_msg=f"c5 replay {r}: {k}")
