"""Trace replay — host mirror of infersim/simulation.py (``Simulation``,
``run``, ``SimResult``).  The whole discrete-event replay executes on the
device in one ``strait_replay`` launch (csrc/strait_replay_impl.cuh); this
module only builds the inputs (replay.ReplayBatch) and rebuilds the
reference's row schemas (simulation.py:100-119, report.py:14-30) from the
device arrays.

Differences from the reference, all outside the parity contract:
* ``trace_rows`` is empty: the event log is a debugging aid whose SHA-256 is
  not a parity criterion (floats are within 1e-5, not byte-identical).
* ``batch_rows[*]["segments"]`` is empty; the consumed isolated work is
  returned as ``work`` instead (work conservation, simulation.py:58-69).
* ``request_rows`` are ordered by arrival (the reference appends them in
  resolution order); their content is identical.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .config import ExperimentConfig
from .domain import PriorityLevel
from .predictor import InterferencePredictor
from .replay import ReplayBatch, ReplayResult, ReplaySpec, RC

EV_KERNEL_COMPLETE, EV_TRANSFER_COMPLETE, EV_ARRIVAL, EV_BATCH_TIMEOUT, EV_AIMD_TICK = range(5)


@dataclass
class ClassMetrics:
    arrivals: int
    dropped: int
    violations: int

    @property
    def violation_rate_pct(self) -> float:
        return 100.0 * self.violations / self.arrivals if self.arrivals else 0.0


@dataclass
class MetricsReport:
    """The per-class counts of metrics.compute_metrics (metrics.py:88-158) that
    the parity contract covers; percentiles/goodput are host post-processing."""

    per_class: dict = field(default_factory=dict)


@dataclass
class SimResult:
    policy: str
    policy_variant: str
    seed: int
    _res: ReplayResult
    _r: int
    metrics: MetricsReport
    trace_rows: list = field(default_factory=list)

    # -- reference row schemas ---------------------------------------------
    @property
    def _s(self):
        return self._res.replay_slice(self._r)

    @property
    def decision_rows(self) -> list[dict]:
        s, tab = self._s, self._res.batch.tab
        return [{"time": float(s["dec_time"][b]), "pass_id": int(s["dec_pass"][b]),
                 "model": tab["ids"][int(s["dec_model"][b])], "size": int(s["dec_size"][b]),
                 "gpu": int(s["dec_gpu"][b]), "est_latency": float(s["dec_est_latency"][b]),
                 "intf_pred": float(s["dec_intf"][b])} for b in range(len(s["dec_time"]))]

    def _done_order(self):
        return np.argsort(self._s["b_done_order"], kind="stable")

    @property
    def feedback_rows(self) -> list[dict]:
        s = self._s
        return [{"time": float(s["b_kernel_end"][b]), "batch": f"b{b}", "predicted": float(s["fb_predicted"][b]),
                 "actual": float(s["fb_actual"][b]), "residual": float(s["fb_residual"][b]),
                 "predicted_at_schedule": float(s["dec_intf"][b]), "skipped": int(s["fb_flags"][b] & 1),
                 "saturated": int((s["fb_flags"][b] >> 1) & 1)} for b in self._done_order()]

    @property
    def batch_rows(self) -> list[dict]:
        s, tab = self._s, self._res.batch.tab
        out = []
        for b in self._done_order():
            m, k = int(s["dec_model"][b]), int(s["dec_size"][b])
            mid = tab["ids"][m]
            kern = float(tab["kernel"][m * tab["B"] + k - 1])
            ks, ke, comp = float(s["b_kernel_start"][b]), float(s["b_kernel_end"][b]), float(s["b_completion"][b])
            out.append({"batch": f"b{b}", "model": mid, "priority": PriorityLevel(int(tab["prio"][m])).label,
                        "size": k, "gpu": int(s["dec_gpu"][b]), "front_enqueue": float(s["b_front"][b]),
                        "sched_time": float(s["dec_time"][b]), "transfer_start": float(s["b_transfer_start"][b]),
                        "kernel_start": ks, "kernel_end": ke, "completion": comp, "isolated_kernel": kern,
                        "measured_kernel": ke - ks, "intf_pred": float(s["dec_intf"][b]),
                        "intf_actual": float(s["fb_actual"][b]), "est_latency": float(s["dec_est_latency"][b]),
                        "actual_latency": comp - float(s["b_front"][b]), "segments": "",
                        "work": float(s["b_work"][b])})
        return out

    @property
    def request_rows(self) -> list[dict]:
        res, r = self._res, self._r
        batch = res.batch
        tab = batch.tab
        lo, hi = int(batch.inputs["req_off"][r]), int(batch.inputs["req_off"][r + 1])
        M = tab["M"]
        kidx = np.empty(hi - lo, dtype=np.int64)
        for m in range(M):
            a, b = int(batch.inputs["mr_off"][r * M + m]), int(batch.inputs["mr_off"][r * M + m + 1])
            kidx[batch.inputs["model_req"][a:b] - lo] = np.arange(b - a)
        rows = []
        arr = batch.inputs["arr_time"]
        for i in range(hi - lo):
            gi = lo + i
            m = int(batch.inputs["arr_model"][gi])
            mid = tab["ids"][m]
            t = float(arr[gi])
            dl = t + float(tab["deadline"][m])
            dropped = int(res.a["req_status"][gi]) == 2
            comp = float(res.a["req_completion"][gi])
            rows.append({"request": f"{mid}-{int(kidx[i])}", "model": mid,
                         "priority": PriorityLevel(int(tab["prio"][m])).label, "arrival": t, "deadline_abs": dl,
                         "batch": "" if dropped else f"b{int(res.a['req_batch'][gi])}",
                         "completion": "" if dropped else comp, "latency": "" if dropped else comp - t,
                         "dropped": int(dropped), "violated": int(res.a["req_violated"][gi])})
        return rows

    @property
    def cap_rows(self) -> list[dict]:
        s = self._s
        return [{"time": float(t), "gpu": int(g), "cap_pct": float(c)}
                for t, g, c in zip(s["cap_time"], s["cap_gpu"], s["cap_pct"])]

    @property
    def counters(self) -> np.ndarray:
        return self._s["counters"]


class Simulation:
    """simulation.py:122-513: Simulation(config, seed=None, predictor=None).run().
    An injected predictor is refit in place, as in the reference."""

    def __init__(self, config: ExperimentConfig, seed: Optional[int] = None,
                 predictor: Optional[InterferencePredictor] = None):
        config.validate()
        self.cfg = config
        self.seed = config.seed if seed is None else seed
        self.predictor = predictor

    def run(self) -> SimResult:
        return run_many([ReplaySpec(self.cfg, self.seed, self.predictor)])[0]


def _metrics(c) -> MetricsReport:
    return MetricsReport({
        "high": ClassMetrics(int(c[RC["HP_ARR"]]), int(c[RC["HP_DROP"]]), int(c[RC["HP_VIOL"]])),
        "low": ClassMetrics(int(c[RC["LP_ARR"]]), int(c[RC["LP_DROP"]]), int(c[RC["LP_VIOL"]])),
    })


def run_many(specs: list[ReplaySpec]) -> list[SimResult]:
    """Many independent replays in ONE device launch (the analogue of
    `infersim sweep`, cli.py:64-103).  Injected predictors are refit in place."""
    batch = ReplayBatch(specs)
    res = batch.run()
    res.check()
    out = []
    np_ = batch.tab["nm"] + 7
    for r, s in enumerate(specs):
        sl = res.replay_slice(r)
        if s.predictor is not None:  # mirror the in-place refit of an injected predictor
            st = sl["pred_state"]
            s.predictor.params.apply_vector(list(st[:np_]))
            s.predictor.opt.m = list(st[np_:2 * np_])
            s.predictor.opt.v = list(st[2 * np_:])
            s.predictor.opt.step = int(sl["pred_step"])
        seed = s.config.seed if s.seed is None else s.seed
        out.append(SimResult(s.config.policy, s.config.policy_variant, seed, res, r, _metrics(sl["counters"])))
    return out


def run(config: ExperimentConfig, seed: Optional[int] = None) -> SimResult:
    """simulation.py:516-519."""
    return Simulation(config, seed).run()
