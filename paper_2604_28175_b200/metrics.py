"""Run metrics — host mirror of infersim/metrics.py (metrics.py:16-200).

``compute_metrics`` aggregates outcome rows exactly as the reference does,
with the arithmetic on the device: the rows become the arrays of one
``strait_replay_metrics`` launch (counts, nearest-rank percentiles by radix
select, CPython floor-division goodput windows, signed error series;
csrc/strait_metrics.cu).  ``perturb_profiles`` prepares replay INPUTS (numpy
draws, like the workload generator) and stays on the host.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _device as D
from ._replay_abi import RC, RC_N, MS_N, MetricsArgs
from .domain import ModelProfile, PriorityLevel


def nearest_rank(sorted_values: Sequence[float], pct: float) -> Optional[float]:
    """metrics.py:16-22: the ceil(p/100 * N)-th smallest value (host helper for
    already-sorted host lists; the report's percentiles come from the device)."""
    n = len(sorted_values)
    if n == 0:
        return None
    rank = max(1, math.ceil(pct / 100.0 * n))
    return sorted_values[min(rank, n) - 1]


@dataclass
class ClassMetrics:
    """metrics.py:25-50."""

    arrivals: int = 0
    completed: int = 0
    dropped: int = 0
    violations: int = 0
    violation_rate_pct: float = 0.0
    p50_latency: Optional[float] = None
    p95_latency: Optional[float] = None
    p99_latency: Optional[float] = None
    goodput_counts: list = field(default_factory=list)

    def to_dict(self) -> dict:
        return {"arrivals": self.arrivals, "completed": self.completed, "dropped": self.dropped,
                "violations": self.violations, "violation_rate_pct": self.violation_rate_pct,
                "p50_latency_ms": self.p50_latency, "p95_latency_ms": self.p95_latency,
                "p99_latency_ms": self.p99_latency, "goodput_counts": list(self.goodput_counts)}


@dataclass
class MetricsReport:
    """metrics.py:53-85, computed on the device (strait_replay_metrics)."""

    per_class: dict
    window_ms: float
    intf_error: list
    latency_error: list
    kernel_overhead: list
    cap_timeline: list
    partial: bool = False
    _stats: dict = field(default_factory=dict, repr=False)

    def goodput_per_s(self, priority: PriorityLevel) -> list[float]:
        scale = 1000.0 / self.window_ms
        return [c * scale for c in self.per_class[priority].goodput_counts]

    def to_dict(self) -> dict:
        d = {"window_ms": self.window_ms, "partial": self.partial,
             "high": self.per_class[PriorityLevel.HIGH].to_dict(), "low": self.per_class[PriorityLevel.LOW].to_dict()}
        for k in ("intf_error", "latency_error", "kernel_overhead"):
            # device statistics of the run; for a report built by hand from host
            # lists, error_stats (metrics.py:64-74) over those lists
            d[k] = self._stats[k] if k in self._stats else _error_stats(getattr(self, k))
        return d


def _error_stats(errors: list) -> dict:
    if not errors:
        return {"count": 0}
    s = sorted(abs(e) for e in errors)
    return {"count": len(s), "median_abs": nearest_rank(s, 50), "p95_abs": nearest_rank(s, 95),
            "p99_abs": nearest_rank(s, 99)}


def _stats_of(out: dict, s: int) -> dict:
    n = int(out["series_count"][s])
    if not n:
        return {"count": 0}
    q = out["pct"].reshape(MS_N, 3)[s]
    return {"count": n, "median_abs": float(q[0]), "p95_abs": float(q[1]), "p99_abs": float(q[2])}


def _metrics_launch(n_req, arr, prio, status, violated, completion, n_series, est, lat_end, meas_end, iso,
                    fb_pred, fb_act, window_ms, max_windows):
    """One strait_replay_metrics launch over a single synthetic replay.  Batch
    b's actual latency is passed as b_completion[b] - 0 and its measured kernel
    as b_kernel_end[b] - 0, so the device forms exactly the row values."""
    nb = max(n_series, 1)
    table, inv = np.unique(np.asarray(iso, dtype=np.float64), return_inverse=True) if n_series else (np.ones(1), [])
    if len(table) > 32767:
        raise ValueError("more than 32767 distinct isolated kernel latencies")
    counters = np.zeros(RC_N, np.int64)
    counters[RC["COMPLETED"]] = n_series
    z = np.zeros(nb)

    def col(x, dt=np.float64):
        x = np.asarray(x, dtype=dt)
        return x if len(x) else np.zeros(1, dt)

    dz = D.dev(z)
    din = {"window_ms": D.dev(np.array([window_ms])), "req_off": D.dev(np.array([0, n_req], np.int64), torch.int64),
           "arr_time": D.dev(col(arr)), "arr_model": D.dev(col(prio, np.int16), torch.int16),
           "model_prio": D.dev(np.array([0, 1], np.int8), torch.int8),
           "req_status": D.dev(col(status, np.int8), torch.int8),
           "req_violated": D.dev(col(violated, np.uint8), torch.uint8), "req_completion": D.dev(col(completion)),
           "counters": D.dev(counters, torch.int64),
           "dec_model": D.dev(col(np.asarray(inv, np.int16), np.int16), torch.int16),
           "dec_size": D.dev(np.ones(nb, np.int8), torch.int8), "dec_est_latency": D.dev(col(est)),
           "b_front": dz, "b_kernel_start": dz, "b_kernel_end": D.dev(col(meas_end)),
           "b_completion": D.dev(col(lat_end)), "fb_predicted": D.dev(col(fb_pred)), "fb_actual": D.dev(col(fb_act)),
           "kernel_table": D.dev(table)}
    W = max_windows
    mout = {"class_counts": D.empty(8, torch.int64), "partial": D.empty(1, torch.uint8),
            "pct": D.empty(MS_N * 3), "series_count": D.empty(MS_N, torch.int64),
            "goodput": D.empty(2 * W, torch.int64), "goodput_len": D.empty(2, torch.int32),
            "intf_error": D.empty(nb), "latency_error": D.empty(nb), "kernel_overhead": D.empty(nb)}
    m = MetricsArgs()
    m.n_replays, m.max_windows, m.table_stride = 1, W, 1
    for k, v in list(din.items()) + list(mout.items()):
        setattr(m, k, D.ptr(v))
    D.check(D.lib().strait_replay_metrics(C.byref(m), D.stream_handle()))
    return {k: D.host(v) for k, v in mout.items()}


def compute_metrics(request_rows: list[dict], batch_rows: Optional[list[dict]] = None,
                    feedback_rows: Optional[list[dict]] = None, cap_rows: Optional[list[dict]] = None,
                    window_ms: float = 1000.0) -> MetricsReport:
    """metrics.py:88-158 on the device: early drops count as violations,
    latency percentiles over completed requests, goodput buckets on-time
    completions by int(completion // window_ms), predictor / latency error and
    kernel-overhead series.  Accepts the row dicts of a SimResult or of
    report.read_rows (cells "" = unresolved)."""
    n = len(request_rows)
    prio = np.empty(n, np.int16)
    arr = np.empty(n)
    status = np.zeros(n, np.int8)
    viol = np.zeros(n, np.uint8)
    comp = np.full(n, np.nan)
    for i, row in enumerate(request_rows):
        prio[i] = int(PriorityLevel.from_name(row["priority"]))
        arr[i] = float(row["arrival"])
        if int(row["dropped"]):
            status[i] = 2
        elif row["completion"] != "":
            status[i] = 1
            comp[i] = float(row["completion"])
            viol[i] = 1 if int(row["violated"]) else 0
    done = comp[status == 1]
    max_windows = int(np.max(done) // window_ms) + 2 if len(done) else 1
    fb = feedback_rows or []
    bt = batch_rows or []
    fb_pred = [float(r["predicted"]) for r in fb]
    fb_act = [float(r["actual"]) for r in fb]
    # launch 1: request classes, latency percentiles, goodput, intf_error series
    a = _metrics_launch(n, arr, prio, status, viol, comp, len(fb), np.ones(len(fb)), np.ones(len(fb)),
                        np.ones(len(fb)), np.ones(len(fb)), fb_pred, fb_act, window_ms, max_windows)
    # launch 2: latency_error and kernel_overhead series of the batch rows
    b = _metrics_launch(0, [], [], [], [], [], len(bt), [float(r["est_latency"]) for r in bt],
                        [float(r["actual_latency"]) for r in bt], [float(r["measured_kernel"]) for r in bt],
                        [float(r["isolated_kernel"]) for r in bt], np.ones(len(bt)), np.ones(len(bt)), window_ms, 1)
    cc = a["class_counts"].reshape(2, 4)
    pct = a["pct"].reshape(MS_N, 3)
    gp = a["goodput"].reshape(2, max_windows)
    per = {}
    for p in PriorityLevel:
        arrivals, completed, dropped, violations = (int(x) for x in cc[int(p)])
        q = pct[int(p)]

        def opt(x):
            return None if np.isnan(x) else float(x)

        per[p] = ClassMetrics(arrivals, completed, dropped, violations,
                              100.0 * violations / arrivals if arrivals else 0.0, opt(q[0]), opt(q[1]), opt(q[2]),
                              [int(x) for x in gp[int(p)][:int(a["goodput_len"][int(p)])]])
    caps = [(float(r["time"]), int(r["gpu"]), float(r["cap_pct"])) for r in cap_rows or []]
    stats = {"intf_error": _stats_of(a, 2), "latency_error": _stats_of(b, 3), "kernel_overhead": _stats_of(b, 4)}
    return MetricsReport(per, window_ms, a["intf_error"][:len(fb)].tolist(), b["latency_error"][:len(bt)].tolist(),
                         b["kernel_overhead"][:len(bt)].tolist(), caps, bool(a["partial"][0] & 1), stats)


def perturb_profiles(profiles: dict[str, ModelProfile], magnitude_pct: float, seed) -> dict[str, ModelProfile]:
    """metrics.py:161-195: every profiled throughput / self-compute / self-memory
    value times (1 + u), u ~ U(-m%, +m%) in model-sorted, row-major draw order,
    clamped to [0, 1]; latencies untouched.  Replay input preparation (numpy)."""
    if not 0 <= magnitude_pct <= 100:
        raise ValueError(f"magnitude must be within [0, 100], got {magnitude_pct}")
    rng = np.random.default_rng(seed)
    m = magnitude_pct / 100.0

    def wobble(v: float) -> float:
        return min(1.0, max(0.0, v * (1.0 + float(rng.uniform(-m, m)))))

    out = {}
    for mid in sorted(profiles):
        p = profiles[mid]
        out[mid] = ModelProfile(model_id=p.model_id, priority=p.priority, deadline_ms=p.deadline_ms,
                                batch_timeout_ms=p.batch_timeout_ms, max_batch_size=p.max_batch_size,
                                total_latency=list(p.total_latency), transfer_latency=list(p.transfer_latency),
                                kernel_latency=list(p.kernel_latency),
                                throughput=[tuple(wobble(v) for v in row) for row in p.throughput],
                                self_compute=[wobble(v) for v in p.self_compute],
                                self_memory=[wobble(v) for v in p.self_memory], metrics=p.metrics)
    return out
