"""Per-call latency of the object-API propose (one strait_node_propose launch
over page-locked node records) on random node states of 4 and 64 GPUs:
p50 / p99 wall time of PredictivePolicy.propose, host call to BatchPlan.
Where the reference is installed (baseline/_ref), its own
PredictivePolicy.propose is timed on the identical state (same scenario
built with its classes) on the same host, and the two plans are compared.

    python scripts/propose_latency.py [calls]
"""
import json
import os
import sys
import time
import types

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

from node_scenarios import build, random_scenario  # noqa: E402


def main():
    from paper_2604_28175_b200 import domain, predictor, runtime, scheduler

    api = types.SimpleNamespace(
        PriorityLevel=domain.PriorityLevel, ModelProfile=domain.ModelProfile, Request=domain.Request,
        Batch=domain.Batch, ThroughputTimeline=domain.ThroughputTimeline, GpuRuntimeState=runtime.GpuRuntimeState,
        RunningTaskEntry=runtime.RunningTaskEntry, TaskQueue=scheduler.TaskQueue,
        PredictorParams=predictor.PredictorParams, InterferencePredictor=predictor.InterferencePredictor)
    calls = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    ref = _ref_api()
    out = {}
    for G in (4, 64):
        scn = random_scenario(np.random.default_rng(7), G)
        scn["k_queue"] = 8
        o = build(scn, api)
        pol = scheduler.PredictivePolicy(o["predictor"])
        ts = _time(lambda: pol.propose(o["queue"], o["gpus"], o["now"]), calls)
        row = {"p50_us": float(np.percentile(ts, 50)), "p99_us": float(np.percentile(ts, 99)),
               "mean_us": float(ts.mean()), "calls": calls, "sizes": 8, "pairs": 8 * G}
        if ref is not None:
            RS, rapi = ref
            ro = build(scn, rapi)
            rpol = RS.PredictivePolicy(ro["predictor"])
            rts = _time(lambda: rpol.propose(ro["queue"], ro["gpus"], ro["now"]), max(calls // 10, 50))
            a, b = pol.propose(o["queue"], o["gpus"], o["now"]), rpol.propose(ro["queue"], ro["gpus"], ro["now"])
            same = (a is None and b is None) or (a is not None and b is not None and
                                                 (a.size, a.gpu_id, a.est_latency) == (b.size, b.gpu_id, b.est_latency))
            row["reference"] = {"p50_us": float(np.percentile(rts, 50)), "p99_us": float(np.percentile(rts, 99)),
                                "calls": len(rts), "same_plan": bool(same),
                                "what": "infersim PredictivePolicy.propose (pure Python), same state, 1 host core"}
        out[f"gpus_{G}"] = row
    print(json.dumps(out))


def _time(fn, n):
    for _ in range(min(50, n)):
        fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return np.array(ts) * 1e6


def _ref_api():
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "infersim")):
        return None
    sys.path.insert(0, ref)
    import infersim.domain as RD
    import infersim.predictor as RP
    import infersim.runtime as RR
    import infersim.scheduler as RS

    return RS, types.SimpleNamespace(
        PriorityLevel=RD.PriorityLevel, ModelProfile=RD.ModelProfile, Request=RD.Request, Batch=RD.Batch,
        ThroughputTimeline=RD.ThroughputTimeline, GpuRuntimeState=RR.GpuRuntimeState,
        RunningTaskEntry=RR.RunningTaskEntry, TaskQueue=RS.TaskQueue, PredictorParams=RP.PredictorParams,
        InterferencePredictor=RP.InterferencePredictor)


if __name__ == "__main__":
    main()
