"""CPU: the object-API runtime records (include/strait_node.h, runtime.py,
pcie.py) against the reference.

* Golden: the states of tests/golden/node_propose.json built on this package
  reproduce the reference's aggregates, LP aggregates, link state and every
  running entry's TWA bit for bit (fixture made by gen_node_golden.py).
* Differential (where /root/reference is mounted): random operation sequences
  — add/remove entries, timeline records, link reserve/calibrate, AIMD
  advance/reset, submit_plan / complete_batch, raw list edits — applied to the
  reference's objects and to ours, compared after every step, errors included.
"""
import json
import os
import sys
import types

import numpy as np
import pytest

from conftest import GOLDEN
from node_scenarios import build, fx

REF = "/root/reference/pkg/src"


def our_api():
    from paper_2604_28175_b200 import domain, predictor, runtime, scheduler

    return types.SimpleNamespace(
        PriorityLevel=domain.PriorityLevel, ModelProfile=domain.ModelProfile, Request=domain.Request,
        Batch=domain.Batch, ThroughputTimeline=domain.ThroughputTimeline, GpuRuntimeState=runtime.GpuRuntimeState,
        RunningTaskEntry=runtime.RunningTaskEntry, TaskQueue=scheduler.TaskQueue,
        PredictorParams=predictor.PredictorParams, InterferencePredictor=predictor.InterferencePredictor)


def cases():
    with open(os.path.join(GOLDEN, "node_propose.json")) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("i", range(19))
def test_node_state_matches_reference_golden(i):
    case = cases()[i]
    o = build(case["scenario"], our_api())
    for g, want in zip(o["gpus"], case["expected"]["state"]):
        assert g.aggregate_throughput == tuple(fx(v) for v in want["agg"])
        assert g.low_priority_aggregate() == tuple(fx(v) for v in want["lp"])
        assert g.pcie.t_available == fx(want["t_available"])
        assert list(g.pcie.pending) == [fx(v) for v in want["pending"]]
        for e, tw in zip(g.running, want["twa"]):
            if isinstance(tw, str):
                with pytest.raises(ValueError):
                    e.timeline.time_weighted_average(o["now"])
            else:
                assert e.timeline.time_weighted_average(o["now"]) == tuple(fx(v) for v in tw)


# ----------------------------------------------------------------------------- differential vs the reference

def _ref_api():
    sys.path.insert(0, REF)
    try:
        import infersim.domain as RD
        import infersim.pcie as RPC
        import infersim.predictor as RP
        import infersim.runtime as RR
        import infersim.scheduler as RS
    finally:
        sys.path.remove(REF)
    return types.SimpleNamespace(PriorityLevel=RD.PriorityLevel, ModelProfile=RD.ModelProfile, Request=RD.Request,
                                 Batch=RD.Batch, ThroughputTimeline=RD.ThroughputTimeline,
                                 GpuRuntimeState=RR.GpuRuntimeState, RunningTaskEntry=RR.RunningTaskEntry,
                                 TaskQueue=RS.TaskQueue, PredictorParams=RP.PredictorParams,
                                 InterferencePredictor=RP.InterferencePredictor, AimdState=RR.AimdState,
                                 PcieLinkState=RPC.PcieLinkState, submit_plan=RS.submit_plan,
                                 complete_batch=RS.complete_batch, early_drop=RS.early_drop, BatchPlan=RS.BatchPlan)


def _our_full_api():
    from paper_2604_28175_b200 import pcie, runtime, scheduler

    api = our_api()
    api.AimdState, api.PcieLinkState = runtime.AimdState, pcie.PcieLinkState
    api.submit_plan, api.complete_batch, api.early_drop = (scheduler.submit_plan, scheduler.complete_batch,
                                                          scheduler.early_drop)
    api.BatchPlan = scheduler.BatchPlan
    return api


def _digest(gpus):
    out = []
    for g in gpus:
        out.append((g.aggregate_throughput, g.low_priority_aggregate(), g.pcie.t_available, list(g.pcie.pending),
                    g.aimd.cap_pct, g.aimd.last_tick, len(g.running),
                    [(e.batch.batch_id, e.kernel_start_estimate, e.kernel_started, len(e.timeline),
                      e.timeline.times[-1] if len(e.timeline) else None,
                      tuple(e.timeline.values[-1]) if len(e.timeline) else None) for e in g.running]))
    return out


def _outcome(fn):
    try:
        return ("ok", fn())
    except Exception as exc:  # noqa: BLE001 - the exception TYPE is part of the contract
        return ("raise", type(exc).__name__)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
@pytest.mark.parametrize("seed", range(6))
def test_random_runtime_ops_match_reference(seed):
    ref, ours = _ref_api(), _our_full_api()
    rng = np.random.default_rng(seed)
    nm = int(rng.integers(1, 6))
    worlds = []
    for api in (ref, ours):
        P = api.PriorityLevel
        prof = [api.ModelProfile(f"m{i}", P(i % 2), 30.0, 1.0, 8, [1.0 + j for j in range(8)],
                                 [0.2 + 0.1 * j for j in range(8)], [0.5 + 0.5 * j for j in range(8)],
                                 [tuple(0.05 * (i + 1) + 0.01 * j + 0.003 * m for m in range(nm)) for j in range(8)],
                                 [0.3] * 8, [0.4] * 8, tuple(f"x{m}" for m in range(nm))) for i in range(3)]
        gpus = [api.GpuRuntimeState(g, nm, int(rng.integers(1, 4)) if False else 3) for g in range(3)]
        queues = [api.TaskQueue(p) for p in prof]
        worlds.append(types.SimpleNamespace(api=api, prof=prof, gpus=gpus, queues=queues, entries=[], n=0))
    now = 0.0
    for step in range(400):
        op = int(rng.choice(10, p=[.22, .22, .06, .1, .08, .06, .06, .04, .06, .1]))
        g = int(rng.integers(0, 3))
        now_before = now
        now += float(rng.choice([0.0, rng.uniform(0, 3.0)]))
        t_arg = float(now if rng.uniform() < 0.9 else now_before - 1.0)  # sometimes backwards in time
        m = int(rng.integers(0, 3))
        k = int(rng.integers(1, 9))
        d = float(rng.uniform(-0.5, 2.0))
        vec = tuple(float(v) for v in rng.uniform(0, 1, nm))
        pick = float(rng.uniform())
        results = []
        for w in worlds:
            api, gpu = w.api, w.gpus[g]

            def act():
                if op == 0:  # request arrival
                    w.n += 1
                    return w.queues[m].push(api.Request(f"r{w.n}", f"m{m}", now, now + 30.0 * pick + 1.0))
                if op == 1:  # submit a plan from a queue
                    q = w.queues[m]
                    if len(q.pending) < 1:
                        return None
                    size = min(k, len(q.pending))
                    b, e, win = api.submit_plan(q, api.BatchPlan(size, g, 1.0, 1.1, ()), w.gpus, t_arg, f"b{step}")
                    w.entries.append((g, e))
                    return win
                if op == 2 and w.entries:  # complete a running batch
                    gi, e = w.entries[int(pick * len(w.entries))]
                    s, _ = api.complete_batch(w.gpus[gi], e, 1.0 + pick, t_arg)
                    w.entries = [x for x in w.entries if x[1] is not e]
                    return (s.colocated_twa, s.actual)
                if op == 3 and w.entries:  # a co-location record on some entry's timeline
                    gi, e = w.entries[int(pick * len(w.entries))]
                    e.timeline.record(t_arg, vec)
                    return None
                if op == 4:
                    return gpu.pcie.reserve(t_arg, d)
                if op == 5:
                    return gpu.pcie.calibrate(t_arg)
                if op == 6:
                    return gpu.aimd.advance(t_arg)
                if op == 7:
                    return gpu.aimd.reset()
                if op == 8:
                    return [r.request_id for r in api.early_drop(w.queues[m], t_arg)]
                if op == 9 and w.entries:  # TWA of an entry
                    gi, e = w.entries[int(pick * len(w.entries))]
                    return e.timeline.time_weighted_average(t_arg)
                return None

            results.append((_outcome(act), _digest(w.gpus)))
        assert results[0] == results[1], (step, op)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
def test_raw_running_list_edits_match_reference():
    """`gpu.running.clear()` / `.remove()` edit the list only (no recompute), as
    on the reference's plain list (test_scheduler.py:418)."""
    ref, ours = _ref_api(), _our_full_api()
    states = []
    for api in (ref, ours):
        P = api.PriorityLevel
        prof = api.ModelProfile("m", P.HIGH, 30.0, 1.0, 2, [1.0, 2.0], [0.1, 0.2], [0.5, 1.0], [(0.3,), (0.5,)],
                                [0.3, 0.3], [0.3, 0.3], ("x",))
        gpu = api.GpuRuntimeState(0, 1, 4)
        es = []
        for i in range(3):
            r = api.Request(f"r{i}", "m", 0.0, 30.0)
            b = api.Batch(f"b{i}", "m", 1, P.HIGH, 0.0, [r])
            e = api.RunningTaskEntry(b, (0.3 + i,), 0.3, 0.3, 0.5, 30.0, 1.0, 1.0)
            gpu.add_entry(e, float(i))
            es.append(e)
        gpu.running.remove(es[1])
        s1 = (gpu.aggregate_throughput, len(gpu.running))
        gpu.running.clear()
        s2 = (gpu.aggregate_throughput, len(gpu.running), gpu.running == [])
        with pytest.raises(RuntimeError):
            gpu.remove_entry(es[0], 5.0)
        states.append((s1, s2))
    assert states[0] == states[1]
