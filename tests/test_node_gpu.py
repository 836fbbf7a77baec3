"""GPU: the object-API propose (strait_node_propose, one launch over the
GPUs' page-locked records) against the REFERENCE's answers on random node
states (tests/golden/node_propose.json, made by gen_node_golden.py):

* PredictivePolicy.propose: the plan (size, gpu_id, latency, intf, assumed)
  or the reference's ValueError for a malformed running entry;
* check_violate / check_meet of every (size, GPU) pair, full GPUs included.

Decisions and every float bit-exact."""
import json
import os
import types

import pytest

from conftest import GOLDEN
from node_scenarios import build, fx

pytestmark = pytest.mark.gpu


def api():
    from paper_2604_28175_b200 import domain, predictor, runtime, scheduler

    return types.SimpleNamespace(
        PriorityLevel=domain.PriorityLevel, ModelProfile=domain.ModelProfile, Request=domain.Request,
        Batch=domain.Batch, ThroughputTimeline=domain.ThroughputTimeline, GpuRuntimeState=runtime.GpuRuntimeState,
        RunningTaskEntry=runtime.RunningTaskEntry, TaskQueue=scheduler.TaskQueue,
        PredictorParams=predictor.PredictorParams, InterferencePredictor=predictor.InterferencePredictor)


CASES = json.load(open(os.path.join(GOLDEN, "node_propose.json")))["cases"]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_propose_matches_reference(cuda, i):
    from paper_2604_28175_b200 import _abi
    from paper_2604_28175_b200.scheduler import PredictivePolicy

    case = CASES[i]
    scn, want = case["scenario"], case["expected"]
    o = build(scn, api())
    policy = PredictivePolicy(o["predictor"], use_meet=scn["use_meet"], use_violate=scn["use_violate"])
    launches = _abi.lib().strait_kernel_launches()
    if isinstance(want["plan"], dict):
        with pytest.raises(ValueError, match="no samples|precedes"):
            policy.propose(o["queue"], o["gpus"], o["now"])
        return
    plan = policy.propose(o["queue"], o["gpus"], o["now"])
    assert _abi.lib().strait_kernel_launches() == launches + 1  # one device launch per propose
    if want["plan"] is None:
        assert plan is None
    else:
        size, gid, lat, intf, assumed = want["plan"]
        assert (plan.size, plan.gpu_id) == (size, gid)
        assert plan.est_latency == fx(lat) and plan.intf_pred == fx(intf)
        assert plan.assumed == tuple(fx(v) for v in assumed)


@pytest.mark.parametrize("i", range(len(CASES)))
def test_check_violate_and_meet_match_reference(cuda, i):
    from paper_2604_28175_b200.scheduler import check_meet, check_violate

    case = CASES[i]
    o = build(case["scenario"], api())
    prof, now, pred = o["cand"], o["now"], o["predictor"]
    front = o["queue"].front().arrival_time
    for k, row in enumerate(case["expected"]["pairs"], start=1):
        for g, (viol, ok, lat, intf) in zip(o["gpus"], row):
            if viol == "error":
                with pytest.raises(ValueError):
                    check_violate(g, prof, k, now, pred)
            else:
                assert check_violate(g, prof, k, now, pred) is viol, (k, g.gpu_id)
            got = check_meet(g, prof, k, front, now, pred)
            assert got[0] is ok and got[1] == fx(lat) and got[2] == fx(intf), (k, g.gpu_id)


def test_propose_sees_record_mutations_without_export(cuda):
    """The device reads the records in place: a reservation or an AIMD reset
    made through the object API changes the very next propose."""
    from paper_2604_28175_b200.scheduler import PredictivePolicy

    case = next(c for c in CASES if len(c["scenario"]["gpus"]) == 64 and isinstance(c["expected"]["plan"], list))
    o = build(case["scenario"], api())
    pol = PredictivePolicy(o["predictor"], use_meet=case["scenario"]["use_meet"],
                           use_violate=case["scenario"]["use_violate"])
    plan = pol.propose(o["queue"], o["gpus"], o["now"])
    g = o["gpus"][plan.gpu_id]
    g.pcie.reserve(o["now"], 1000.0)  # this GPU's link is now busy for a second
    plan2 = pol.propose(o["queue"], o["gpus"], o["now"])
    assert plan2 is None or plan2.gpu_id != plan.gpu_id or plan2.est_latency > plan.est_latency
