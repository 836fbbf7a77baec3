"""Per-call latency of the object-API propose (one strait_node_propose launch
over page-locked node records) on random node states of 4 and 64 GPUs:
p50 / p99 wall time of PredictivePolicy.propose, host call to BatchPlan.

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
    out = {}
    for G in (4, 64):
        scn = random_scenario(np.random.default_rng(7), G)
        scn["k_queue"] = 8
        o = build(scn, api)
        pol = scheduler.PredictivePolicy(o["predictor"])
        for _ in range(50):
            pol.propose(o["queue"], o["gpus"], o["now"])
        ts = []
        for _ in range(calls):
            t0 = time.perf_counter()
            pol.propose(o["queue"], o["gpus"], o["now"])
            ts.append(time.perf_counter() - t0)
        ts = np.array(ts) * 1e6
        out[f"gpus_{G}"] = {"p50_us": float(np.percentile(ts, 50)), "p99_us": float(np.percentile(ts, 99)),
                            "mean_us": float(ts.mean()), "calls": calls, "sizes": 8,
                            "pairs": 8 * G}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
