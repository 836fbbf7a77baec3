"""GPU: the dispatch drop-in (paper_2604_28175_b200.scheduler / .simulation)
against the reference's own known-answer tests, restated on the mirror types
(pkg/tests/test_scheduler.py:40-334, test_simulation.py:112-144,301-336) —
every check_violate / check_meet / propose here runs in strait_sweep /
strait_estimate_latency / strait_replay."""
import itertools
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN
from replay_cases import case_config

pytestmark = pytest.mark.gpu

_ids = itertools.count()


def mk_profile(model_id="m", priority=None, deadline_ms=20.0, batch_timeout_ms=1.0, max_batch_size=8,
               base_total=3.0, transfer_frac=0.15, kernel_frac=0.7, throughput_row=None, metrics=("tensor_pipe",),
               self_compute=0.3, self_memory=0.3):
    """Linear-latency profile with a constant throughput row (reference conftest.py:11-50)."""
    from paper_2604_28175_b200.domain import ModelProfile, PriorityLevel

    priority = PriorityLevel.HIGH if priority is None else priority
    row = tuple(throughput_row) if throughput_row is not None else tuple(0.3 for _ in metrics)
    tot = [base_total * (0.5 + 0.5 * j) for j in range(1, max_batch_size + 1)]
    return ModelProfile(model_id, priority, deadline_ms, batch_timeout_ms, max_batch_size, tot,
                        [transfer_frac * t for t in tot], [kernel_frac * t for t in tot], [row] * max_batch_size,
                        [self_compute] * max_batch_size, [self_memory] * max_batch_size, tuple(metrics))


def mk_request(model_id, arrival, deadline_ms):
    from paper_2604_28175_b200.domain import Request

    return Request(f"{model_id}-t{next(_ids)}", model_id, arrival, arrival + deadline_ms)


def fill_queue(profile, arrivals):
    from paper_2604_28175_b200.scheduler import TaskQueue

    q = TaskQueue(profile)
    for t in arrivals:
        q.push(mk_request(profile.model_id, t, profile.deadline_ms))
    return q


def mk_gpu(gpu_id=0, n_metrics=1, concurrency_limit=4):
    from paper_2604_28175_b200.runtime import GpuRuntimeState

    return GpuRuntimeState(gpu_id, n_metrics, concurrency_limit)


def running(gpu, profile, size, now, kernel_start=None, deadline_abs=None, intf_predicted=1.0):
    """A running batch on `gpu`; kernel_start <= now marks it executing (conftest.py:65-104)."""
    from paper_2604_28175_b200.domain import Batch, ThroughputTimeline
    from paper_2604_28175_b200.runtime import RunningTaskEntry

    reqs = [mk_request(profile.model_id, now - 1.0, profile.deadline_ms)]
    reqs += [mk_request(profile.model_id, now - 0.5, profile.deadline_ms) for _ in range(size - 1)]
    b = Batch(f"tb{next(_ids)}", profile.model_id, size, profile.priority, min(r.arrival_time for r in reqs), reqs,
              gpu_id=gpu.gpu_id, sched_time=now)
    started = kernel_start is not None and kernel_start <= now
    if started:
        b.kernel_start = kernel_start
    e = RunningTaskEntry(b, profile.throughput_at(size), profile.self_compute_at(size), profile.self_memory_at(size),
                         profile.kernel_latency_ms(size),
                         deadline_abs if deadline_abs is not None else reqs[0].deadline_abs, intf_predicted,
                         kernel_start if kernel_start is not None else now + 1.0, ThroughputTimeline(), started)
    gpu.add_entry(e, kernel_start if started else now)
    return e


def one_metric_predictor(weight=1.0, scale=1.0, base=2.0, offset=-1.0, coeff_high=1.0, coeff_low=1.0):
    """effect(x) = scale * base**x + offset over one metric (test_scheduler.py:24-38)."""
    from paper_2604_28175_b200.domain import PriorityLevel
    from paper_2604_28175_b200.predictor import InterferencePredictor, PredictorParams

    return InterferencePredictor(PredictorParams(scale=scale, base=base, offset=offset, weights=(weight,),
                                                 self_compute_weight=0.0, self_memory_weight=0.0,
                                                 priority_coeff={PriorityLevel.HIGH: coeff_high,
                                                                 PriorityLevel.LOW: coeff_low}))


def LOW():
    from paper_2604_28175_b200.domain import PriorityLevel

    return PriorityLevel.LOW


# ----------------------------------------------------------------------------- check_violate
def test_violate_empty_gpu(cuda):
    from paper_2604_28175_b200.scheduler import check_violate

    assert check_violate(mk_gpu(), mk_profile(), 1, 0.0, one_metric_predictor()) is False


def test_violate_low_priority_cap_threshold(cuda):
    from paper_2604_28175_b200.scheduler import check_violate

    gpu = mk_gpu()
    gpu.aimd.cap_pct = 80.0
    running(gpu, mk_profile("lp-run", LOW(), deadline_ms=500.0, throughput_row=(0.5,)), 1, now=0.0)
    cand = mk_profile("lp-cand", LOW(), deadline_ms=500.0, throughput_row=(0.4,))
    assert check_violate(gpu, cand, 1, 0.0, one_metric_predictor()) is True  # 0.9 > 0.8
    gpu.aimd.cap_pct = 95.0
    assert check_violate(gpu, cand, 1, 0.0, one_metric_predictor()) is False


def test_violate_high_candidate_never_capped(cuda):
    from paper_2604_28175_b200.scheduler import check_violate

    gpu = mk_gpu()
    gpu.aimd.cap_pct = 75.0
    running(gpu, mk_profile("lp-run", LOW(), deadline_ms=500.0, throughput_row=(0.7,)), 1, now=0.0)
    cand = mk_profile("hp-cand", deadline_ms=500.0, throughput_row=(0.9,))
    assert check_violate(gpu, cand, 1, 0.0, one_metric_predictor()) is False


def test_violate_progress_projection_hand_case(cuda):
    """8 ms kernel started at 0, now 4, slowdown 1 -> half done; the candidate makes
    the slowdown 2 so the rest takes 8 ms: finishes at 12 (test_scheduler.py:112-141)."""
    from paper_2604_28175_b200.scheduler import check_violate

    pred = one_metric_predictor()
    gpu = mk_gpu()
    run_p = mk_profile("hp-run", deadline_ms=100.0, base_total=16.0, transfer_frac=0.25, kernel_frac=0.5,
                       throughput_row=(0.0,), self_compute=0.0, self_memory=0.0)
    e = running(gpu, run_p, 1, now=4.0, kernel_start=0.0, deadline_abs=11.0)
    assert e.kernel_latency_ms == 8.0
    cand = mk_profile("hp-cand", deadline_ms=500.0, throughput_row=(1.0,), self_compute=0.0, self_memory=0.0)
    assert check_violate(gpu, cand, 1, 4.0, pred) is True
    e.deadline_abs = 12.0
    assert check_violate(gpu, cand, 1, 4.0, pred) is False


def test_violate_high_may_sacrifice_low(cuda):
    from paper_2604_28175_b200.scheduler import check_violate

    pred = one_metric_predictor()
    gpu = mk_gpu()
    run_p = mk_profile("lp-run", LOW(), deadline_ms=9.0, base_total=16.0, transfer_frac=0.25, kernel_frac=0.5,
                       throughput_row=(0.0,), self_compute=0.0, self_memory=0.0)
    running(gpu, run_p, 1, now=4.0, kernel_start=0.0, deadline_abs=9.0)
    hp = mk_profile("hp-cand", deadline_ms=500.0, throughput_row=(1.0,), self_compute=0.0, self_memory=0.0)
    lp = mk_profile("lp-cand", LOW(), deadline_ms=500.0, throughput_row=(1.0,), self_compute=0.0, self_memory=0.0)
    gpu.aimd.cap_pct = 100.0
    assert check_violate(gpu, hp, 1, 4.0, pred) is False
    assert check_violate(gpu, lp, 1, 4.0, pred) is True


# ----------------------------------------------------------------------------- check_meet / propose
def test_meet_idle_gpu(cuda):
    from paper_2604_28175_b200.scheduler import check_meet

    p = mk_profile(deadline_ms=50.0, self_compute=0.0, self_memory=0.0)
    ok, lat, intf, assumed = check_meet(mk_gpu(), p, 1, 0.0, 2.0, one_metric_predictor())
    assert ok is True and intf == 1.0 and assumed == (0.0,)
    assert lat == pytest.approx(p.total_latency_ms(1) + 2.0)


def test_meet_busy_gpu_halved_throughput(cuda):
    from paper_2604_28175_b200.scheduler import check_meet

    gpu = mk_gpu()
    running(gpu, mk_profile("run", LOW(), deadline_ms=500.0, throughput_row=(0.8,)), 1, now=0.0)
    pred = one_metric_predictor(weight=2.0, coeff_high=4.0)
    p = mk_profile("cand", deadline_ms=7.0, base_total=3.0, self_compute=0.0, self_memory=0.0)
    ok, lat, intf, assumed = check_meet(gpu, p, 1, 0.0, 0.0, pred)
    assert assumed == (0.4,)
    assert intf == pytest.approx(1 + 4 * (2 ** 0.8 - 1), rel=1e-12)
    assert lat == pytest.approx(p.total_latency_ms(1) + (intf - 1) * p.kernel_latency_ms(1), rel=1e-12)
    assert ok is False


def test_propose_argmin_picks_free_link(cuda):
    from paper_2604_28175_b200.scheduler import PredictivePolicy, check_meet

    pred = one_metric_predictor()
    gpus = [mk_gpu(0), mk_gpu(1)]
    gpus[0].pcie.reserve(0.0, 2.0)
    p = mk_profile(deadline_ms=50.0, self_compute=0.0, self_memory=0.0)
    plan = PredictivePolicy(pred).propose(fill_queue(p, [0.0]), gpus, 0.0)
    assert plan.gpu_id == 1
    _, lat0, _, _ = check_meet(gpus[0], p, 1, 0.0, 0.0, pred)
    _, lat1, _, _ = check_meet(gpus[1], p, 1, 0.0, 0.0, pred)
    assert plan.est_latency == lat1 < lat0


def test_propose_one_launch_and_bsearch_vs_linear(cuda):
    """The deadline leaves room for an interior size only; the device search lands
    where a linear scan of check_violate/check_meet does (test_scheduler.py:276-294)."""
    from paper_2604_28175_b200.scheduler import PredictivePolicy, check_meet, check_violate

    pred = one_metric_predictor()
    p = mk_profile(deadline_ms=9.0, base_total=3.0, max_batch_size=8, self_compute=0.0, self_memory=0.0)
    q = fill_queue(p, [0.0] * 8)
    gpus = [mk_gpu(0)]
    linear = None
    for k in range(1, 9):
        ok, _, _, _ = check_meet(gpus[0], p, k, 0.0, 0.0, pred)
        if not check_violate(gpus[0], p, k, 0.0, pred) and ok:
            linear = k
    pol = PredictivePolicy(pred)
    plan = pol.propose(q, gpus, 0.0)
    assert linear is not None and 1 <= linear < 8 and plan.size == linear
    assert pol.launches == 1


def _run_pass(policy, queues, gpus, now):
    from paper_2604_28175_b200.scheduler import ScheduleDecision, run_scheduling_pass, submit_plan

    ctr = itertools.count()

    def on_submit(queue, plan):
        submit_plan(queue, plan, gpus, now, f"b{next(ctr)}")
        return ScheduleDecision(now, 0, queue.model_id, plan.size, plan.gpu_id, plan.est_latency, plan.intf_pred)

    dropped = []
    return run_scheduling_pass(policy, queues, gpus, now, on_submit, lambda q, rs: dropped.extend(rs)), dropped


def test_pass_full_queue_largest_batch_and_priority_order(cuda):
    from paper_2604_28175_b200.scheduler import PredictivePolicy

    p = mk_profile(deadline_ms=500.0, max_batch_size=8)
    q = fill_queue(p, [0.0] * 10)
    dec, _ = _run_pass(PredictivePolicy(one_metric_predictor()), [q], [mk_gpu(0)], 0.0)
    assert dec[0].size == 8 and len(q.pending) == 2
    hp = mk_profile("hp", deadline_ms=50.0)
    lo = mk_profile("lp_old", LOW(), deadline_ms=50.0)
    ln = mk_profile("lp_new", LOW(), deadline_ms=50.0)
    qs = [fill_queue(lo, [0.0]), fill_queue(hp, [0.5]), fill_queue(ln, [0.2])]
    dec, _ = _run_pass(PredictivePolicy(one_metric_predictor()), qs, [mk_gpu(0)], 2.0)
    assert [d.model_id for d in dec] == ["hp", "lp_old", "lp_new"]


def test_pass_timeout_gating_and_deferral(cuda):
    from paper_2604_28175_b200.scheduler import PredictivePolicy

    p = mk_profile(deadline_ms=50.0, batch_timeout_ms=5.0)
    q = fill_queue(p, [0.0])
    pol = PredictivePolicy(one_metric_predictor())
    assert _run_pass(pol, [q], [mk_gpu(0)], 2.0)[0] == []
    assert len(_run_pass(pol, [q], [mk_gpu(0)], 5.0)[0]) == 1
    q2 = fill_queue(mk_profile(deadline_ms=50.0), [0.0])
    g = mk_gpu(0, concurrency_limit=1)
    running(g, mk_profile("blk", LOW(), deadline_ms=500.0), 1, now=0.0)
    assert _run_pass(pol, [q2], [g], 1.0)[0] == [] and len(q2.pending) == 1


def test_complete_batch_refits_on_device(cuda):
    """complete_batch -> InterferencePredictor.update (strait_refit): TWA of the
    kernel window, actual = measured / isolated, entry removed (test_scheduler.py:387-430)."""
    from paper_2604_28175_b200.scheduler import complete_batch

    gpu = mk_gpu()
    pred = one_metric_predictor()
    e = running(gpu, mk_profile("a", throughput_row=(0.5,)), 1, now=0.0, kernel_start=0.0)
    running(gpu, mk_profile("b", throughput_row=(0.3,)), 1, now=0.0, kernel_start=0.0)
    step0 = pred.opt.step
    sample, res = complete_batch(gpu, e, 2.0 * e.kernel_latency_ms, 4.0, pred)
    assert sample.actual == 2.0 and len(gpu.running) == 1
    assert sample.colocated_twa == pytest.approx((0.3,))
    assert res is not None and not res.skipped and pred.opt.step == step0 + 1


# ----------------------------------------------------------------------------- Simulation / run
def test_run_drop_in_matches_reference_golden(cuda):
    """run(config, seed) -> SimResult rows equal the reference's (golden C1 replay)."""
    from paper_2604_28175_b200.simulation import run

    g = dict(np.load(os.path.join(GOLDEN, "replay", "demo.npz")))
    res = run(case_config("demo"))
    rows = res.decision_rows
    assert [r["size"] for r in rows] == g["dec_size"].tolist()
    assert [r["gpu"] for r in rows] == g["dec_gpu"].tolist()
    assert [r["pass_id"] for r in rows] == g["dec_pass"].tolist()
    np.testing.assert_allclose([r["est_latency"] for r in rows], g["dec_est_latency"], rtol=1e-5)
    fb = res.feedback_rows  # completion order; golden arrays are indexed by batch id
    done = np.argsort(g["b_done_order"], kind="stable")
    np.testing.assert_array_equal([r["actual"] for r in fb], g["fb_actual"][done])
    np.testing.assert_array_equal([r["batch"] for r in fb], [f"b{b}" for b in done])
    req = res.request_rows
    assert sum(r["violated"] for r in req) == int(g["class_counts"][:, 2].sum())
    from paper_2604_28175_b200.domain import PriorityLevel

    hp = res.metrics.per_class[PriorityLevel.HIGH]
    assert (hp.arrivals, hp.dropped, hp.violations) == tuple(int(x) for x in g["class_counts"][0])
    import json

    assert res.metrics.to_dict() == json.loads(str(g["metrics_json"]))  # metrics.py MetricsReport, on device
    assert len(res.cap_rows) == len(g["cap_time"])


def test_simulation_injected_predictor_refit_in_place(cuda):
    """Simulation(config, seed, predictor=...) refits the injected predictor
    (simulation.py:123-127,155) — final state equals the golden replay's."""
    from paper_2604_28175_b200.predictor import InterferencePredictor, PredictorParams
    from paper_2604_28175_b200.simulation import Simulation

    g = dict(np.load(os.path.join(GOLDEN, "replay", "demo.npz")))
    pred = InterferencePredictor(PredictorParams(weights=(0.1,) * 5))
    Simulation(case_config("demo"), predictor=pred).run()
    np_ = 12
    np.testing.assert_allclose(pred.params.to_vector(), g["pred_state"][:np_], rtol=1e-5)
    assert pred.opt.step == int(g["pred_step"])


def test_same_early_drop_sets_across_policies(cuda):
    """test_baselines.py:139-155: every policy (the predictive one's propose on
    the device) drops exactly the requests that cannot meet their deadline in
    isolation, given identical queue state."""
    from paper_2604_28175_b200.predictor import InterferencePredictor, PredictorParams
    from paper_2604_28175_b200.scheduler import ScheduleDecision, make_policy, run_scheduling_pass, submit_plan

    def build():
        return fill_queue(mk_profile("q", deadline_ms=10.0, base_total=3.0, batch_timeout_ms=0.0),
                          [0.0, 6.0, 7.0, 7.5])

    now = 8.0
    predictor = InterferencePredictor(PredictorParams(weights=(0.1,)))
    for name in ("predictive", "temporal", "static", "reactive"):
        policy = make_policy(name, predictor)
        q, gpus, dropped = build(), [mk_gpu(0)], []

        def on_submit(queue, plan):
            submit_plan(queue, plan, gpus, now, "b0")
            return ScheduleDecision(now, 0, queue.model_id, plan.size, plan.gpu_id, plan.est_latency, plan.intf_pred)

        run_scheduling_pass(policy, [q], gpus, now, on_submit, lambda queue, reqs: dropped.extend(reqs))
        assert [r.arrival_time for r in dropped] == [0.0], name
