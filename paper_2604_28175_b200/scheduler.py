"""Priority-aware dispatch (Algorithm 1) — the object API of
infersim/scheduler.py over node records.

What runs where:

* ``PredictivePolicy.propose`` is ONE ``strait_node_propose`` launch.  The
  GPUs' records (page-locked, see runtime.py) are read in place by the device,
  which evaluates every (size, GPU) pair — has_slot, the LP cap, the projection
  of every running co-runner under its timeline TWA (check_violate), check_meet
  — then best_for's argmin per size and largest_feasible's probe sequence.  The
  host writes the candidate's profile rows and reads back one small struct.
* ``check_violate`` / ``check_meet`` are the same launch for one (size, GPU).
* ``submit_plan`` / ``complete_batch`` and the AIMD tick mutate records
  through the library's ``strait_node_*`` entry points (runtime.py).
* Queues hold the caller's ``Request`` objects (callers mutate them in place,
  e.g. a deadline), so ``TaskQueue`` / ``early_drop`` stay host control flow.
"""
from __future__ import annotations

import ctypes as C
from collections import deque
from dataclasses import dataclass
from typing import Callable, Iterable, Optional, Sequence

import numpy as np

from ._abi import PAIR_MEET, PAIR_VIOLATE, STRAIT_OK, StraitUnavailable, check
from ._node_abi import ENTRY_BYTES, HDR_BYTES, ProposeArgs, ProposeOut, nlib
from .domain import Batch, ModelProfile, PriorityLevel, Request, make_batch
from .predictor import FeedbackSample, InterferencePredictor, UpdateResult
from .runtime import GpuRuntimeState, RunningTaskEntry


# ----------------------------------------------------------------------------- queues

class TaskQueue:
    """Per-model FIFO of pending requests (scheduler.py:25-62).  The queue is
    schedulable once a full batch waits or its front has aged past the
    batching timeout.  ``front_generation`` changes whenever a different
    request becomes the front (the simulator's timeout validity key)."""

    def __init__(self, profile: ModelProfile):
        self.profile = profile
        self.model_id = profile.model_id
        self.priority = profile.priority
        self.pending: deque[Request] = deque()
        self.front_generation = 0

    def __len__(self) -> int:
        return len(self.pending)

    def push(self, request: Request) -> bool:
        """Enqueue; True when `request` is now the front."""
        was_empty = not self.pending
        self.pending.append(request)
        self.front_generation += was_empty
        return was_empty

    def front(self) -> Request:
        return self.pending[0]

    def timeout_deadline(self) -> float:
        return self.front().arrival_time + self.profile.batch_timeout_ms

    def eligible(self, now: float) -> bool:
        n = len(self.pending)
        return n > 0 and (n >= self.profile.max_batch_size or now >= self.timeout_deadline())

    def pop_front(self, k: int) -> list[Request]:
        q = self.pending
        taken = [q.popleft() for _ in range(k)]
        self.front_generation += 1
        return taken


def early_drop(queue: TaskQueue, now: float) -> list[Request]:
    """scheduler.py:65-75: requests whose remaining slack is below the
    isolated size-1 latency cannot be served; remove them, keeping the order of
    the rest.  The front generation moves when the front changes."""
    floor = queue.profile.total_latency_ms(1)
    keep, gone = deque(), []
    for r in queue.pending:
        slack = r.deadline_abs - now
        if slack < floor:
            gone.append(r)
        elif slack >= floor:  # (a NaN slack is in neither list, as in the reference's two comprehensions)
            keep.append(r)
    if gone:
        head = queue.pending[0]
        queue.pending = keep
        if not keep or keep[0] is not head:
            queue.front_generation += 1
    return gone


def largest_feasible(k_max: int, feasible: Callable[[int], bool]) -> Optional[int]:
    """scheduler.py:78-90: the largest k in 1..k_max with feasible(k), found by
    bisection (feasibility is monotone); None when k = 1 fails.  The probe
    sequence is the reference's: mid = (lo + hi) // 2."""
    found, window = None, (1, k_max)
    while window[0] <= window[1]:
        mid = (window[0] + window[1]) // 2
        if feasible(mid):
            found, window = mid, (mid + 1, window[1])
        else:
            window = (window[0], mid - 1)
    return found


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


# ----------------------------------------------------------------------------- device propose

def _require_device():
    try:
        import torch
    except ImportError as exc:  # pragma: no cover
        raise StraitUnavailable("torch is required for the device path") from exc
    if not torch.cuda.is_available():
        raise StraitUnavailable("no CUDA device: strait_node_propose has no CPU fallback")
    return torch


class _ProposeBuffers:
    """Page-locked argument/result blocks of strait_node_propose, grown on
    demand and reused across calls (the device reads and writes them in place)."""

    def __init__(self):
        self.cap_g = self.cap_k = 0
        self.block = None

    def ensure(self, G: int, K: int, nm: int) -> None:
        if G <= self.cap_g and K <= self.cap_k and self.block is not None:
            return
        torch = _require_device()
        self.cap_g, self.cap_k = max(G, 2 * self.cap_g, 8), max(K, self.cap_k, 8)
        cg, ck = self.cap_g, self.cap_k
        sizes = {"recs": 8 * cg, "params": 8 * 16, "cand": 8 * (8 + 4) * ck, "flags": ck * cg,
                 "lat": 8 * ck * cg, "intf": 8 * ck * cg, "seg_gpu": 4 * ck, "seg_lat": 8 * ck,
                 "seg_intf": 8 * ck, "out": C.sizeof(ProposeOut)}
        offs, o = {}, 0
        for k, n in sizes.items():
            offs[k] = o
            o += (n + 63) & ~63
        self.block = torch.empty(o, dtype=torch.uint8, pin_memory=True)
        base = self.block.data_ptr()
        self.addr = {k: base + v for k, v in offs.items()}
        self.recs = (C.c_uint64 * cg).from_address(self.addr["recs"])
        self.params = (C.c_double * 16).from_address(self.addr["params"])
        self.out = ProposeOut.from_address(self.addr["out"])
        self.np = {
            "cand": np.frombuffer((C.c_double * (12 * ck)).from_address(self.addr["cand"]), dtype=np.float64),
            "flags": np.frombuffer((C.c_uint8 * (ck * cg)).from_address(self.addr["flags"]), dtype=np.uint8),
            "lat": np.frombuffer((C.c_double * (ck * cg)).from_address(self.addr["lat"]), dtype=np.float64),
            "intf": np.frombuffer((C.c_double * (ck * cg)).from_address(self.addr["intf"]), dtype=np.float64),
            "seg_gpu": np.frombuffer((C.c_int32 * ck).from_address(self.addr["seg_gpu"]), dtype=np.int32),
            "seg_lat": np.frombuffer((C.c_double * ck).from_address(self.addr["seg_lat"]), dtype=np.float64),
            "seg_intf": np.frombuffer((C.c_double * ck).from_address(self.addr["seg_intf"]), dtype=np.float64),
        }


_BUFS = _ProposeBuffers()
_TWA_ERRORS = {1: "no samples", 2: "end_time {now!r} precedes the last timeline sample"}


def node_propose(profile: ModelProfile, k_max: int, front_arrival: float, gpus: Sequence[GpuRuntimeState],
                 now: float, predictor: InterferencePredictor, use_violate: bool = True, use_meet: bool = True,
                 fixed_size: int = 0, want_pairs: bool = False, stream=None):
    """One strait_node_propose launch; returns (ProposeOut fields as a dict,
    per-pair/per-size arrays when `want_pairs`)."""
    torch = _require_device()
    nm = len(predictor.params.weights)
    G, K = len(gpus), k_max
    for g in gpus:
        if g.n_metrics != nm:
            raise ValueError(f"aggregate throughput has {g.n_metrics} metrics, model expects {nm}")
    if len(profile.throughput[0]) != nm:
        raise ValueError(f"candidate throughput has {len(profile.throughput[0])} metrics, model expects {nm}")
    B = _BUFS
    B.ensure(G, K, nm)
    for i, g in enumerate(gpus):
        B.recs[i] = g._rec.dev_addr
    vec = predictor.params.to_vector()
    for i, v in enumerate(vec):
        B.params[i] = v
    cand = B.np["cand"]
    rows = np.asarray(profile.throughput[:K], dtype=np.float64)  # [K][nm]
    cand[:nm * K] = rows.T.reshape(-1)
    for f, arr in enumerate((profile.self_compute, profile.self_memory, profile.total_latency,
                             profile.kernel_latency)):
        cand[(nm + f) * K:(nm + f + 1) * K] = arr[:K]
    slots = max(g._rec.hdr.slot_cap for g in gpus)
    stride = (HDR_BYTES + ENTRY_BYTES * slots + 15) & ~15
    L = nlib()
    if L.strait_node_propose_smem(K, G, stride) > 200 * 1024:
        stride = 0  # read the records in place instead of staging them
    a = ProposeArgs()
    a.n_metrics, a.n_gpus, a.k_max, a.cand_prio = nm, G, K, int(profile.priority)
    a.use_violate, a.use_meet, a.fixed_size, a.stage_stride = int(use_violate), int(use_meet), fixed_size, stride
    a.now, a.effect_cap = now, float(predictor.params.effect_cap)
    a.deadline_ms, a.front_arrival = profile.deadline_ms, front_arrival
    ad = B.addr
    a.params, a.recs, a.out = ad["params"], ad["recs"], ad["out"]
    a.cand_contrib = ad["cand"]
    for f, name in enumerate(("cand_self_cmp", "cand_self_mem", "cand_total", "cand_kernel")):
        setattr(a, name, ad["cand"] + 8 * (nm + f) * K)
    if want_pairs:
        a.pair_flags, a.pair_latency, a.pair_intf = ad["flags"], ad["lat"], ad["intf"]
        a.seg_gpu, a.seg_latency, a.seg_intf = ad["seg_gpu"], ad["seg_lat"], ad["seg_intf"]
    s = stream if stream is not None else torch.cuda.current_stream()
    check(L.strait_node_propose(C.byref(a), s.cuda_stream))
    s.synchronize()
    o = B.out
    if o.status != STRAIT_OK:
        raise ValueError(_TWA_ERRORS.get(o.err_kind, "malformed running entry").format(now=now) +
                         f" (gpu {gpus[o.err_gpu].gpu_id}, running entry {o.err_pos})")
    res = {"size": o.size, "gpu_index": o.gpu_index, "latency": o.latency, "intf": o.intf, "probes": o.probes}
    if not want_pairs:
        return res, None
    n = K * G
    pairs = {"flags": B.np["flags"][:n].reshape(K, G).copy(), "latency": B.np["lat"][:n].reshape(K, G).copy(),
             "intf": B.np["intf"][:n].reshape(K, G).copy(), "seg_gpu": B.np["seg_gpu"][:K].copy(),
             "seg_latency": B.np["seg_lat"][:K].copy(), "seg_intf": B.np["seg_intf"][:K].copy()}
    return res, pairs


def _one_pair(gpu: GpuRuntimeState, profile: ModelProfile, size: int, front: float, now: float,
              predictor: InterferencePredictor, violate: bool):
    profile._index(size)  # ValueError on a bad size, as the reference's profile accessors
    _, pairs = node_propose(profile, size, front, [gpu], now, predictor, use_violate=violate, fixed_size=size,
                            want_pairs=True)
    return int(pairs["flags"][size - 1, 0]), float(pairs["latency"][size - 1, 0]), float(pairs["intf"][size - 1, 0])


def check_violate(gpu: GpuRuntimeState, profile: ModelProfile, size: int, now: float,
                  predictor: InterferencePredictor) -> bool:
    """scheduler.py:118-161 — one (size, GPU) pair of strait_node_propose."""
    flags, _, _ = _one_pair(gpu, profile, size, 0.0, now, predictor, violate=True)
    return bool(flags & PAIR_VIOLATE)


def check_meet(gpu: GpuRuntimeState, profile: ModelProfile, size: int, front_enqueue_time: float, now: float,
               predictor: InterferencePredictor) -> tuple[bool, float, float, tuple[float, ...]]:
    """scheduler.py:164-185 — (ok, latency, intf, assumed) of one pair."""
    flags, lat, intf = _one_pair(gpu, profile, size, front_enqueue_time, now, predictor, violate=False)
    return bool(flags & PAIR_MEET), lat, intf, tuple(0.5 * a for a in gpu.aggregate_throughput)


# ----------------------------------------------------------------------------- policies

class SchedulingPolicy:
    """The pass-level plug-in seam (scheduler.py:209-226)."""

    name = "base"

    def begin_pass(self, now: float) -> None:
        pass

    def queue_order(self, queues: Iterable[TaskQueue], now: float) -> list[TaskQueue]:
        return _ordered(queues, by_priority=True)

    def propose(self, queue: TaskQueue, gpus: Sequence[GpuRuntimeState], now: float) -> Optional[BatchPlan]:
        raise NotImplementedError

    def on_hp_violation(self, gpus: Sequence[GpuRuntimeState], gpu_id: Optional[int], now: float) -> None:
        pass


def _ordered(queues: Iterable[TaskQueue], by_priority: bool) -> list[TaskQueue]:
    """Non-empty queues by (priority, front arrival, model id), or without the
    priority term (the no_priority_scan ablation); stable."""
    ready = [q for q in queues if q.pending]
    if by_priority:
        return sorted(ready, key=lambda q: (q.priority.value, q.front().arrival_time, q.model_id))
    return sorted(ready, key=lambda q: (q.front().arrival_time, q.model_id))


class PredictivePolicy(SchedulingPolicy):
    """The interference-predictive policy (scheduler.py:229-292): the largest
    admitted batch size, on the GPU with the lowest estimated latency — one
    device launch per propose.  Flags switch mechanisms off for ablations."""

    name = "predictive"

    def __init__(self, predictor: InterferencePredictor, use_priority_order: bool = True, use_meet: bool = True,
                 use_violate: bool = True):
        self.predictor = predictor
        self.use_priority_order = use_priority_order
        self.use_meet = use_meet
        self.use_violate = use_violate
        self.launches = 0

    def queue_order(self, queues, now):
        return _ordered(queues, by_priority=self.use_priority_order)

    def propose(self, queue: TaskQueue, gpus: Sequence[GpuRuntimeState], now: float) -> Optional[BatchPlan]:
        k_max = min(len(queue.pending), queue.profile.max_batch_size)
        if k_max < 1 or not gpus:
            return None
        res, _ = node_propose(queue.profile, k_max, queue.front().arrival_time, gpus, now, self.predictor,
                              self.use_violate, self.use_meet)
        self.launches += 1
        if res["size"] == 0:
            return None
        g = gpus[res["gpu_index"]]
        return BatchPlan(res["size"], g.gpu_id, res["latency"], res["intf"],
                         tuple(0.5 * a for a in g.aggregate_throughput))

    def on_hp_violation(self, gpus, gpu_id, now):
        for gpu in (gpus if gpu_id is None else [gpus[gpu_id]]):
            gpu.aimd.reset()


# ----------------------------------------------------------------------------- pass driver

def submit_plan(queue: TaskQueue, plan: BatchPlan, gpus: Sequence[GpuRuntimeState], now: float,
                batch_id: str) -> tuple[Batch, RunningTaskEntry, tuple[float, float]]:
    """scheduler.py:295-324: pop the plan's requests into a batch, reserve the
    GPU's link for its transfer and register it as running — the last two in
    one library call (GpuRuntimeState.submit_entry)."""
    prof, k = queue.profile, plan.size
    requests = queue.pop_front(k)
    batch = make_batch(batch_id, prof, requests)
    batch.gpu_id, batch.sched_time = plan.gpu_id, now
    entry = RunningTaskEntry(batch, prof.throughput_at(k), prof.self_compute_at(k), prof.self_memory_at(k),
                             prof.kernel_latency_ms(k), requests[0].deadline_abs, plan.intf_pred,
                             kernel_start_estimate=0.0)
    window = gpus[plan.gpu_id].submit_entry(entry, prof.transfer_latency_ms(k), now)
    batch.transfer_start = window[0]
    return batch, entry, window


def complete_batch(gpu: GpuRuntimeState, entry: RunningTaskEntry, measured_kernel_ms: float, now: float,
                   predictor: Optional[InterferencePredictor] = None
                   ) -> tuple[FeedbackSample, Optional[UpdateResult]]:
    """scheduler.py:327-352: the feedback sample (TWA of the kernel window,
    measured / isolated kernel latency), the entry's removal with departure
    samples on the survivors, then the device refit step."""
    if not any(e is entry for e in gpu._order):
        raise RuntimeError(f"gpu {gpu.gpu_id}: batch {entry.batch.batch_id} is not running here")
    twa = entry.timeline.time_weighted_average(now)
    sample = FeedbackSample(entry.batch.batch_id, twa, entry.self_compute, entry.self_memory, entry.priority,
                            measured_kernel_ms / entry.kernel_latency_ms, entry.intf_predicted)
    gpu.remove_entry(entry, now)
    return sample, (None if predictor is None else predictor.update(sample))


def run_scheduling_pass(policy: SchedulingPolicy, queues: Iterable[TaskQueue], gpus: Sequence[GpuRuntimeState],
                        now: float, on_submit: Callable[[TaskQueue, BatchPlan], ScheduleDecision],
                        on_drop: Callable[[TaskQueue, list[Request]], None]) -> list[ScheduleDecision]:
    """scheduler.py:355-378: queues in policy order; each is early-dropped,
    then — if still eligible — proposed for and submitted at most once."""
    policy.begin_pass(now)
    out: list[ScheduleDecision] = []
    for q in policy.queue_order(queues, now):
        lost = early_drop(q, now)
        if lost:
            on_drop(q, lost)
        plan = policy.propose(q, gpus, now) if q.eligible(now) else None
        if plan is not None:
            out.append(on_submit(q, plan))
    return out


from .baselines import (ABLATION_VARIANTS, POLICY_NAMES, ReactiveSpatialPolicy, ReactiveState,  # noqa: E402,F401
                        StaticSpatialPolicy, TemporalPolicy, make_policy)
