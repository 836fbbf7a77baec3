"""Priority-aware dispatch (Algorithm 1) — host mirror of
infersim/scheduler.py with the reference's names, signatures and error
behaviour.  The queue/pass bookkeeping is host control flow on the
reference's own data structures; every prediction, violate/meet check and the
(latency, gpu_id) argmin run in the CUDA library:

* ``PredictivePolicy.propose`` marshals the queue's whole search — every size
  k in 1..k_max x every GPU x every co-runner — into ONE ``strait_twa`` +
  ``strait_sweep`` pair (segment = size k), then replays the reference's
  binary-search probe sequence (scheduler.py:78-90) on the per-size results.
  best_for is pure, so evaluating sizes the search never probes is harmless.
* ``check_violate`` / ``check_meet`` are single-pair calls of the same kernels.
"""
from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass
from typing import Callable, Iterable, Optional, Sequence

import numpy as np
import torch

from . import _abi
from . import _device as D
from . import sweep as SW
from .domain import Batch, ModelProfile, PriorityLevel, Request, make_batch
from .predictor import FeedbackSample, InterferencePredictor, UpdateResult, estimate_latency_batch
from .runtime import GpuRuntimeState, RunningTaskEntry


class TaskQueue:
    """FIFO of pending requests for one model (scheduler.py:25-62)."""

    def __init__(self, profile: ModelProfile):
        self.profile = profile
        self.model_id = profile.model_id
        self.priority = profile.priority
        self.pending: deque[Request] = deque()
        self.front_generation = 0

    def __len__(self) -> int:
        return len(self.pending)

    def push(self, request: Request) -> bool:
        self.pending.append(request)
        if len(self.pending) == 1:
            self.front_generation += 1
            return True
        return False

    def front(self) -> Request:
        return self.pending[0]

    def timeout_deadline(self) -> float:
        return self.pending[0].arrival_time + self.profile.batch_timeout_ms

    def eligible(self, now: float) -> bool:
        if not self.pending:
            return False
        return len(self.pending) >= self.profile.max_batch_size or now >= self.timeout_deadline()

    def pop_front(self, k: int) -> list[Request]:
        taken = [self.pending.popleft() for _ in range(k)]
        self.front_generation += 1
        return taken


def early_drop(queue: TaskQueue, now: float) -> list[Request]:
    """scheduler.py:65-75: drop requests that cannot finish even alone at size 1."""
    floor_latency = queue.profile.total_latency_ms(1)
    dropped = [r for r in queue.pending if r.deadline_abs - now < floor_latency]
    if dropped:
        old_front = queue.pending[0]
        queue.pending = deque(r for r in queue.pending if r.deadline_abs - now >= floor_latency)
        if not queue.pending or queue.pending[0] is not old_front:
            queue.front_generation += 1
    return dropped


def largest_feasible(k_max: int, feasible: Callable[[int], bool]) -> Optional[int]:
    """scheduler.py:78-90: binary search for the largest feasible size."""
    lo, hi = 1, k_max
    best: Optional[int] = None
    while lo <= hi:
        mid = (lo + hi) // 2
        if feasible(mid):
            best = mid
            lo = mid + 1
        else:
            hi = mid - 1
    return best


@dataclass
class BatchPlan:
    size: int
    gpu_id: int
    est_latency: float
    intf_pred: float
    assumed: tuple[float, ...]


@dataclass
class ScheduleDecision:
    time: float
    pass_id: int
    model_id: str
    size: int
    gpu_id: int
    est_latency: float
    intf_pred: float
    assumed: tuple[float, ...] = ()


# ----------------------------------------------------------------------------- snapshot -> SoA
def _pow2(n: int) -> int:
    p = 1
    while p < n:
        p *= 2
    return p


def _snapshot(profile: ModelProfile, sizes: Sequence[int], front: float, gpus: Sequence[GpuRuntimeState],
              now: float, predictor: InterferencePredictor):
    """Device SoA of segments = sizes, pairs = gpus, triples = co-runners."""
    nm = len(profile.metrics)
    G = len(gpus)
    S = len(sizes)
    C = min(32, _pow2(max([1] + [len(g.running) for g in gpus])))
    if any(len(g.running) > 32 for g in gpus):
        raise ValueError("more than 32 co-runners on one GPU")
    conc = {g.concurrency_limit for g in gpus}
    if len(conc) != 1:
        raise ValueError("all GPUs of a scheduling pass must share one concurrency_limit")
    a = {
        "cand_contrib": np.array([profile.throughput_at(k) for k in sizes], dtype=np.float64).T.copy(),
        "cand_self_cmp": np.array([profile.self_compute_at(k) for k in sizes]),
        "cand_self_mem": np.array([profile.self_memory_at(k) for k in sizes]),
        "cand_total": np.array([profile.total_latency_ms(k) for k in sizes]),
        "cand_kernel": np.array([profile.kernel_latency_ms(k) for k in sizes]),
        "cand_deadline": np.full(S, profile.deadline_ms),
        "cand_front": np.full(S, front),
        "cand_prio": np.full(S, int(profile.priority), dtype=np.int8),
    }
    agg = np.array([g.aggregate_throughput for g in gpus], dtype=np.float64).reshape(G, nm)
    lpa = np.array([g.low_priority_aggregate() for g in gpus], dtype=np.float64).reshape(G, nm)
    a["gpu_agg"] = np.tile(agg.T, (1, S))
    a["gpu_lp_agg"] = np.tile(lpa.T, (1, S))
    a["gpu_cap_pct"] = np.tile(np.array([g.aimd.cap_pct for g in gpus]), S)
    a["gpu_t_avail"] = np.tile(np.array([g.pcie.t_available for g in gpus]), S)
    a["gpu_n_running"] = np.tile(np.array([len(g.running) for g in gpus], dtype=np.int8), S)
    # co-runner slots of one (size-independent) GPU block, then tiled per size
    T1 = G * C
    contrib = np.zeros((nm, T1))
    cmp_ = np.zeros(T1)
    mem = np.zeros(T1)
    tk = np.ones(T1)
    dl = np.zeros(T1)
    ks = np.zeros(T1)
    prio = np.zeros(T1, dtype=np.int8)
    t0 = np.zeros(T1)
    tl = np.zeros(T1)
    vl = np.zeros((nm, T1))
    acc = np.zeros((nm, T1))
    for gi, g in enumerate(gpus):
        for j, e in enumerate(g.running):
            t = gi * C + j
            contrib[:, t] = e.contribution
            cmp_[t], mem[t], tk[t], dl[t] = e.self_compute, e.self_memory, e.kernel_latency_ms, e.deadline_abs
            ks[t] = e.batch.kernel_start if e.kernel_started else e.kernel_start_estimate
            prio[t] = int(e.priority)
            tln = e.timeline
            if not len(tln):
                raise ValueError("running entry without timeline samples")
            if now < tln.times[-1]:
                raise ValueError(f"end_time {now} precedes last sample at {tln.times[-1]}")
            t0[t], tl[t] = tln.times[0], tln.times[-1]
            vl[:, t] = tln.values[-1]
            acc[:, t] = tln.acc
    # the co-runners' TWA at now on the device (strait_twa, domain.py:249-264)
    tw = D.empty((nm, T1))
    keep = [D.dev(x) for x in (t0, tl, vl, acc, np.full(T1, now))]  # alive until the launch is enqueued
    D.check(D.lib().strait_twa(nm, *[D.ptr(t) for t in keep], T1, D.ptr(tw), D.stream_handle()))
    dev = {k: D.dev(v, torch.int8 if v.dtype == np.int8 else torch.float64) for k, v in a.items()}
    rep = lambda x, dt=torch.float64: D.dev(np.tile(x, (1, S)) if x.ndim == 2 else np.tile(x, S), dt)  # noqa: E731
    dev["ent_contrib"] = rep(contrib)
    dev["ent_twa"] = tw.repeat(1, S).contiguous()
    dev["ent_self_cmp"] = rep(cmp_)
    dev["ent_self_mem"] = rep(mem)
    dev["ent_t_kernel"] = rep(tk)
    dev["ent_deadline_abs"] = rep(dl)
    dev["ent_kstart"] = rep(ks)
    dev["ent_prio"] = rep(prio, torch.int8)
    soa = SW.SweepSoA(nm, C, G, conc.pop(), S, float(now), dev)
    return soa, agg


def _sweep_sizes(profile, sizes, front, gpus, now, predictor, use_violate=True, use_meet=True):
    soa, agg = _snapshot(profile, sizes, front, gpus, now, predictor)
    P = predictor.params.device_vector()
    out = SW.alloc_outputs(soa)
    SW.launch_sweep(soa, P, out, predictor.params.effect_cap, use_violate, use_meet)
    return {k: D.host(v) for k, v in out.items()}, agg


# ----------------------------------------------------------------------------- reference API
def check_violate(gpu: GpuRuntimeState, profile: ModelProfile, size: int, now: float,
                  predictor: InterferencePredictor) -> bool:
    """scheduler.py:118-161 (one pair of the sweep kernel)."""
    profile._index(size)  # ValueError on a bad size, as the reference's profile accessors
    out, _ = _sweep_sizes(profile, [size], 0.0, [gpu], now, predictor)
    return bool(out["pair_flags"][0] & _abi.PAIR_VIOLATE)


def check_meet(gpu: GpuRuntimeState, profile: ModelProfile, size: int, front_enqueue_time: float, now: float,
               predictor: InterferencePredictor) -> tuple[bool, float, float, tuple[float, ...]]:
    """scheduler.py:164-185 via strait_estimate_latency."""
    assumed = tuple(0.5 * a for a in gpu.aggregate_throughput)
    lat, intf = estimate_latency_batch(predictor.params, [assumed], profile.self_compute_at(size),
                                       profile.self_memory_at(size), int(profile.priority),
                                       profile.total_latency_ms(size), profile.kernel_latency_ms(size),
                                       gpu.pcie.t_available, front_enqueue_time, now)
    latency, intf = float(lat[0]), float(intf[0])
    return latency <= profile.deadline_ms, latency, intf, assumed


class SchedulingPolicy:
    """scheduler.py:209-226."""

    name = "base"

    def begin_pass(self, now: float) -> None:
        pass

    def queue_order(self, queues: Iterable[TaskQueue], now: float) -> list[TaskQueue]:
        ready = [q for q in queues if q.pending]
        ready.sort(key=lambda q: (q.priority.value, q.front().arrival_time, q.model_id))
        return ready

    def propose(self, queue: TaskQueue, gpus: Sequence[GpuRuntimeState], now: float):
        raise NotImplementedError

    def on_hp_violation(self, gpus: Sequence[GpuRuntimeState], gpu_id: Optional[int], now: float) -> None:
        pass


class PredictivePolicy(SchedulingPolicy):
    """scheduler.py:229-292; one device sweep per propose."""

    name = "predictive"

    def __init__(self, predictor: InterferencePredictor, use_priority_order: bool = True, use_meet: bool = True,
                 use_violate: bool = True):
        self.predictor = predictor
        self.use_priority_order = use_priority_order
        self.use_meet = use_meet
        self.use_violate = use_violate
        self.launches = 0

    def queue_order(self, queues, now):
        ready = [q for q in queues if q.pending]
        if self.use_priority_order:
            ready.sort(key=lambda q: (q.priority.value, q.front().arrival_time, q.model_id))
        else:
            ready.sort(key=lambda q: (q.front().arrival_time, q.model_id))
        return ready

    def propose(self, queue: TaskQueue, gpus: Sequence[GpuRuntimeState], now: float) -> Optional[BatchPlan]:
        profile = queue.profile
        k_max = min(len(queue.pending), profile.max_batch_size)
        if k_max < 1 or not gpus:
            return None
        ids = [g.gpu_id for g in gpus]
        order = sorted(range(len(gpus)), key=lambda i: ids[i])  # tie-break on gpu_id
        gs = [gpus[i] for i in order]
        sizes = list(range(1, k_max + 1))
        out, agg = _sweep_sizes(profile, sizes, queue.front().arrival_time, gs, now, self.predictor,
                                self.use_violate, self.use_meet)
        self.launches += 1
        seg_gpu = out["seg_gpu"]
        k = largest_feasible(k_max, lambda size: seg_gpu[size - 1] >= 0)
        if k is None:
            return None
        g = int(seg_gpu[k - 1])
        assumed = tuple(0.5 * a for a in gs[g].aggregate_throughput)
        return BatchPlan(k, gs[g].gpu_id, float(out["seg_latency"][k - 1]), float(out["seg_intf"][k - 1]), assumed)

    def on_hp_violation(self, gpus, gpu_id, now):
        if gpu_id is None:
            for gpu in gpus:
                gpu.aimd.reset()
        else:
            gpus[gpu_id].aimd.reset()


def submit_plan(queue: TaskQueue, plan: BatchPlan, gpus: Sequence[GpuRuntimeState], now: float,
                batch_id: str) -> tuple[Batch, RunningTaskEntry, tuple[float, float]]:
    """scheduler.py:295-324."""
    profile = queue.profile
    requests = queue.pop_front(plan.size)
    batch = make_batch(batch_id, profile, requests)
    batch.gpu_id = plan.gpu_id
    batch.sched_time = now
    gpu = gpus[plan.gpu_id]
    t_start, t_end = gpu.pcie.reserve(now, profile.transfer_latency_ms(plan.size))
    batch.transfer_start = t_start
    entry = RunningTaskEntry(batch=batch, contribution=profile.throughput_at(plan.size),
                             self_compute=profile.self_compute_at(plan.size),
                             self_memory=profile.self_memory_at(plan.size),
                             kernel_latency_ms=profile.kernel_latency_ms(plan.size),
                             deadline_abs=requests[0].deadline_abs, intf_predicted=plan.intf_pred,
                             kernel_start_estimate=t_end)
    gpu.add_entry(entry, now)
    return batch, entry, (t_start, t_end)


def complete_batch(gpu: GpuRuntimeState, entry: RunningTaskEntry, measured_kernel_ms: float, now: float,
                   predictor: Optional[InterferencePredictor] = None
                   ) -> tuple[FeedbackSample, Optional[UpdateResult]]:
    """scheduler.py:327-352; the refit runs in strait_refit."""
    twa = entry.timeline.time_weighted_average(now)
    intf_actual = measured_kernel_ms / entry.kernel_latency_ms
    sample = FeedbackSample(batch_id=entry.batch.batch_id, colocated_twa=twa, self_compute=entry.self_compute,
                            self_memory=entry.self_memory, priority=entry.priority, actual=intf_actual,
                            predicted_at_schedule=entry.intf_predicted)
    gpu.remove_entry(entry, now)
    result = predictor.update(sample) if predictor is not None else None
    return sample, result


def run_scheduling_pass(policy: SchedulingPolicy, queues: Iterable[TaskQueue], gpus: Sequence[GpuRuntimeState],
                        now: float, on_submit: Callable[[TaskQueue, BatchPlan], ScheduleDecision],
                        on_drop: Callable[[TaskQueue, list[Request]], None]) -> list[ScheduleDecision]:
    """scheduler.py:355-378."""
    policy.begin_pass(now)
    decisions: list[ScheduleDecision] = []
    for queue in policy.queue_order(queues, now):
        dropped = early_drop(queue, now)
        if dropped:
            on_drop(queue, dropped)
        if not queue.pending or not queue.eligible(now):
            continue
        plan = policy.propose(queue, gpus, now)
        if plan is None:
            continue
        decisions.append(on_submit(queue, plan))
    return decisions


def _isolated_latency_plan(queue: TaskQueue, gpu_id: int, size: int, now: float) -> BatchPlan:
    """baselines.py:34-37."""
    latency = (now - queue.front().arrival_time) + queue.profile.total_latency_ms(size)
    return BatchPlan(size=size, gpu_id=gpu_id, est_latency=latency, intf_pred=1.0, assumed=())


class TemporalPolicy(SchedulingPolicy):
    """baselines.py:40-59: one batch per GPU; largest size meeting the front deadline in isolation."""

    name = "temporal"

    def propose(self, queue, gpus, now):
        idle = [g for g in gpus if not g.running]
        if not idle:
            return None
        profile = queue.profile
        deadline = queue.front().deadline_abs
        k_max = min(len(queue.pending), profile.max_batch_size)
        size = largest_feasible(k_max, lambda k: now + profile.total_latency_ms(k) <= deadline)
        return None if size is None else _isolated_latency_plan(queue, idle[0].gpu_id, size, now)


class StaticSpatialPolicy(SchedulingPolicy):
    """baselines.py:62-78: fixed concurrency cap, least-loaded GPU, everything buffered."""

    name = "static"

    def __init__(self, cap: int = 3):
        self.cap = cap

    def propose(self, queue, gpus, now):
        open_gpus = [g for g in gpus if len(g.running) < min(self.cap, g.concurrency_limit)]
        if not open_gpus:
            return None
        gpu = min(open_gpus, key=lambda g: (len(g.running), g.gpu_id))
        return _isolated_latency_plan(queue, gpu.gpu_id, min(len(queue.pending), queue.profile.max_batch_size), now)


@dataclass
class ReactiveState:
    """baselines.py:81-107."""

    lp_allowance: int = 3
    default_allowance: int = 3
    min_allowance: int = 1
    hp_bound: int = 3
    reset_period_ms: float = 200.0
    last_reset: float = 0.0

    def catch_up(self, now: float) -> None:
        if now - self.last_reset >= self.reset_period_ms:
            periods = math.floor((now - self.last_reset) / self.reset_period_ms)
            self.lp_allowance = self.default_allowance
            self.last_reset += periods * self.reset_period_ms

    def on_hp_violation(self) -> None:
        self.lp_allowance = max(self.min_allowance, self.lp_allowance - 1)


class ReactiveSpatialPolicy(SchedulingPolicy):
    """baselines.py:110-133: LP concurrency throttled by HP deadline misses."""

    name = "reactive"

    def __init__(self, state: Optional[ReactiveState] = None):
        self.state = state if state is not None else ReactiveState()

    def begin_pass(self, now: float) -> None:
        self.state.catch_up(now)

    def _class_open(self, gpu: GpuRuntimeState, priority: PriorityLevel) -> bool:
        if not gpu.has_slot():
            return False
        count = sum(1 for e in gpu.running if e.priority is priority)
        bound = self.state.lp_allowance if priority is PriorityLevel.LOW else self.state.hp_bound
        return count < bound

    def propose(self, queue, gpus, now):
        open_gpus = [g for g in gpus if self._class_open(g, queue.priority)]
        if not open_gpus:
            return None
        gpu = min(open_gpus, key=lambda g: (len(g.running), g.gpu_id))
        return _isolated_latency_plan(queue, gpu.gpu_id, min(len(queue.pending), queue.profile.max_batch_size), now)

    def on_hp_violation(self, gpus, gpu_id, now):
        self.state.catch_up(now)
        self.state.on_hp_violation()


POLICY_NAMES = ("predictive", "temporal", "static", "reactive")
ABLATION_VARIANTS = ("full", "no_priority_scan", "no_gamma_advantage", "no_meet", "no_violate_aimd")


def make_policy(name: str, predictor: Optional[InterferencePredictor] = None, variant: str = "full"):
    """baselines.py:136-160 registry.  Whole replays of every policy run on the
    device (simulation.run / replay.ReplayBatch); these objects serve the
    per-call pass API (run_scheduling_pass)."""
    if name == "predictive":
        if variant not in ABLATION_VARIANTS:
            raise ValueError(f"unknown ablation variant {variant!r}")
        if predictor is None:
            raise ValueError("predictive policy needs a predictor")
        return PredictivePolicy(predictor, use_priority_order=variant != "no_priority_scan",
                                use_meet=variant != "no_meet", use_violate=variant != "no_violate_aimd")
    if name == "temporal":
        return TemporalPolicy()
    if name == "static":
        return StaticSpatialPolicy()
    if name == "reactive":
        return ReactiveSpatialPolicy()
    raise ValueError(f"unknown policy {name!r}, expected one of {POLICY_NAMES}")
