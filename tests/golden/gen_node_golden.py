"""Golden answers of the REFERENCE's object-API scheduling functions on random
node states (tests/node_scenarios.py), for the device propose
(strait_node_propose) and the record bookkeeping (strait_node_*):

* PredictivePolicy(...).propose(queue, gpus, now)     scheduler.py:257-285
* check_violate / check_meet for every (size, GPU)    scheduler.py:118-185
* aggregate_throughput, low_priority_aggregate,       runtime.py:104-122
  link t_available / pending, every entry's TWA       pcie.py, domain.py:250-264

    python tests/golden/gen_node_golden.py      -> tests/golden/node_propose.json

Run in the build container (imports /root/reference/pkg/src read-only).
"""
from __future__ import annotations

import json
import os
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(REPO, "tests"))

import infersim.domain as RD  # noqa: E402
import infersim.predictor as RP  # noqa: E402
import infersim.runtime as RR  # noqa: E402
import infersim.scheduler as RS  # noqa: E402
from node_scenarios import build, hx, random_scenario  # noqa: E402

API = types.SimpleNamespace(
    PriorityLevel=RD.PriorityLevel, ModelProfile=RD.ModelProfile, Request=RD.Request, Batch=RD.Batch,
    ThroughputTimeline=RD.ThroughputTimeline, GpuRuntimeState=RR.GpuRuntimeState,
    RunningTaskEntry=RR.RunningTaskEntry, TaskQueue=RS.TaskQueue, PredictorParams=RP.PredictorParams,
    InterferencePredictor=RP.InterferencePredictor)


def answers(scn: dict) -> dict:
    o = build(scn, API)
    gpus, q, prof, now, pred = o["gpus"], o["queue"], o["cand"], o["now"], o["predictor"]
    out = {"state": []}
    for g in gpus:
        twas = []
        for e in g.running:
            try:
                twas.append([hx(v) for v in e.timeline.time_weighted_average(now)])
            except ValueError as exc:
                twas.append(str(exc))
        out["state"].append({"agg": [hx(v) for v in g.aggregate_throughput],
                             "lp": [hx(v) for v in g.low_priority_aggregate()],
                             "t_available": hx(g.pcie.t_available), "pending": [hx(v) for v in g.pcie.pending],
                             "twa": twas})
    policy = RS.PredictivePolicy(pred, use_meet=scn["use_meet"], use_violate=scn["use_violate"])
    try:
        plan = policy.propose(q, gpus, now)
        out["plan"] = None if plan is None else [plan.size, plan.gpu_id, hx(plan.est_latency), hx(plan.intf_pred),
                                                 [hx(v) for v in plan.assumed]]
    except ValueError as exc:
        out["plan"] = {"error": str(exc)}
    k_max = min(len(q.pending), prof.max_batch_size)
    pairs = []
    for k in range(1, k_max + 1):
        row = []
        for g in gpus:
            try:
                v = RS.check_violate(g, prof, k, now, pred)
            except ValueError:
                v = "error"
            ok, lat, intf, _ = RS.check_meet(g, prof, k, q.front().arrival_time, now, pred)
            row.append([v, ok, hx(lat), hx(intf)])
        pairs.append(row)
    out["pairs"] = pairs
    return out


def main():
    rng = np.random.default_rng(20260417)
    cases = []
    for i, G in enumerate([1, 1, 2, 4, 4, 4, 4, 8, 8, 16, 16, 64, 64, 4, 64]):
        scn = random_scenario(rng, G)
        cases.append({"scenario": scn, "expected": answers(scn)})
    for err in ("empty_timeline", "future_sample"):
        for G in (2, 8):
            scn = random_scenario(rng, G, error=err)
            cases.append({"scenario": scn, "expected": answers(scn)})
    path = os.path.join(HERE, "node_propose.json")
    with open(path, "w") as f:
        json.dump({"generator": "tests/golden/gen_node_golden.py", "cases": cases}, f, separators=(",", ":"))
    print(f"wrote {len(cases)} cases to {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
