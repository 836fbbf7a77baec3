"""Trace replay — host mirror of infersim/simulation.py (``Simulation``,
``run``, ``SimResult``).  The whole discrete-event replay executes on the
device in one ``strait_replay`` launch (csrc/strait_replay_impl.cuh); this
module only builds the inputs (replay.ReplayBatch) and rebuilds the
reference's row schemas (simulation.py:100-119, report.py:14-30) from the
device arrays.

With the event log on (the default of ``run`` / ``Simulation.run`` /
``run_many``), every row list is the reference's exactly: ``trace_rows``
(Simulation._trace) and the batch rows' ``segments`` come from the device's
event log, request rows are in resolution order, and every float is
bit-identical, so the run-directory CSVs (report.py) and ``trace_hash()`` are
byte-identical to the reference's (tests/test_csv_gpu.py).  Without it
(``trace=False``), ``trace_rows`` is empty, ``segments`` is empty and request
rows are in arrival order.  Batch rows carry one extra key, ``work`` (the
consumed isolated work, simulation.py:58-69), which no CSV column selects.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .config import ExperimentConfig
from .domain import PriorityLevel
from .predictor import InterferencePredictor
from ._replay_abi import TR
from .metrics import ClassMetrics, MetricsReport
from .replay import ReplayBatch, ReplayResult, ReplaySpec

TRACE_EVENTS = ("arrival", "submit", "drop", "kernel_start", "kernel_complete", "aimd_tick", "aimd_reset")

EV_KERNEL_COMPLETE, EV_TRANSFER_COMPLETE, EV_ARRIVAL, EV_BATCH_TIMEOUT, EV_AIMD_TICK = range(5)


def _report(res: ReplayResult, r: int) -> MetricsReport:
    d = res.metrics(r)
    per = {}
    for p, name in ((PriorityLevel.HIGH, "high"), (PriorityLevel.LOW, "low")):
        c = d[name]
        per[p] = ClassMetrics(c["arrivals"], c["completed"], c["dropped"], c["violations"], c["violation_rate_pct"],
                              c["p50_latency_ms"], c["p95_latency_ms"], c["p99_latency_ms"], c["goodput_counts"])
    sl = res.replay_slice(r)
    lo = int(res.batch.inputs["req_off"][r])
    nb = len(sl["dec_time"])
    order = np.argsort(sl["b_done_order"], kind="stable")  # feedback / batch rows are in completion order
    series = {k: res.a["m_" + k][lo:lo + nb][order].tolist() for k in ("intf_error", "latency_error",
                                                                       "kernel_overhead")}
    caps = [(float(t), int(g), float(c)) for t, g, c in zip(sl["cap_time"], sl["cap_gpu"], sl["cap_pct"])]
    return MetricsReport(per, d["window_ms"], series["intf_error"], series["latency_error"],
                         series["kernel_overhead"], caps, d["partial"],
                         {k: d[k] for k in ("intf_error", "latency_error", "kernel_overhead")})


@dataclass
class SimResult:
    policy: str
    policy_variant: str
    seed: int
    _res: ReplayResult
    _r: int
    metrics: MetricsReport

    # -- reference row schemas ---------------------------------------------
    @property
    def _s(self):
        return self._res.replay_slice(self._r)

    @property
    def traced(self) -> bool:
        return "trace" in self._res.a

    def _kidx(self) -> np.ndarray:
        """Per-model arrival index k of each request (request_id = f"{model}-{k}", simulation.py:188)."""
        batch, r = self._res.batch, self._r
        M = batch.tab["M"]
        lo, hi = int(batch.inputs["req_off"][r]), int(batch.inputs["req_off"][r + 1])
        kidx = np.empty(hi - lo, dtype=np.int64)
        for m in range(M):
            a, b = int(batch.inputs["mr_off"][r * M + m]), int(batch.inputs["mr_off"][r * M + m + 1])
            kidx[batch.inputs["model_req"][a:b] - lo] = np.arange(b - a)
        return kidx

    def _rows_log(self):
        """The event log without the segment records, as Python scalars."""
        rec = self._res.trace_records(self._r)
        rec = rec[rec["event"] != TR["SEGMENT"]]
        return (rec["time"].tolist(), rec["event"].tolist(), rec["gpu"].tolist(), rec["batch"].tolist(),
                rec["request"].tolist(), rec["size"].tolist(), rec["x"].tolist())

    @property
    def trace_rows(self) -> list[dict]:
        """Simulation._trace rows (simulation.py:207-218) from the device event log."""
        if not self.traced:
            return []
        batch = self._res.batch
        ids = batch.tab["ids"]
        lo = int(batch.inputs["req_off"][self._r])
        kidx = self._kidx()
        arr_model = batch.inputs["arr_model"]
        dec_model = self._s["dec_model"]
        rows = []
        for t, ev, g, b, q, k, x in zip(*self._rows_log()):
            row = {"time": t, "event": TRACE_EVENTS[ev], "gpu": "", "model": "", "batch": "", "request": "",
                   "detail": ""}
            if ev == TR["ARRIVAL"] or ev == TR["DROP"]:
                mid = ids[int(arr_model[q])]
                row["model"], row["request"] = mid, f"{mid}-{int(kidx[q - lo])}"
            elif ev == TR["RESET"]:
                row["gpu"], row["detail"] = g, f"cap={x[0]!r}"
            elif ev != TR["TICK"]:
                row["gpu"], row["model"], row["batch"] = g, ids[int(dec_model[b])], f"b{b}"
                if ev == TR["SUBMIT"]:
                    row["detail"] = f"size={k} transfer={x[0]!r}..{x[1]!r} est={x[2]!r}"
                elif ev == TR["KSTART"]:
                    row["detail"] = f"slowdown={x[0]!r}"
                else:
                    row["detail"] = f"measured={x[0]!r} intf={x[1]!r}"
            rows.append(row)
        return rows

    def trace_csv_text(self) -> str:
        """simulation.py:114-116."""
        from .report import TRACE_COLUMNS, rows_to_csv_text

        return rows_to_csv_text(self.trace_rows, TRACE_COLUMNS)

    def trace_hash(self) -> str:
        """simulation.py:118-119."""
        return hashlib.sha256(self.trace_csv_text().encode()).hexdigest()

    def _segments(self) -> dict:
        """ExecutionState.segments per batch (simulation.py:56-66), formatted as _fmt_segments (:85-86)."""
        if not self.traced:
            return {}
        rec = self._res.trace_records(self._r)
        rec = rec[rec["event"] == TR["SEGMENT"]]
        out: dict = {}
        for b, x in zip(rec["batch"].tolist(), rec["x"].tolist()):
            out.setdefault(b, []).append(f"{x[0]!r}:{x[1]!r}")
        return {b: "|".join(v) for b, v in out.items()}

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
        segs = self._segments()
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
                        "actual_latency": comp - float(s["b_front"][b]), "segments": segs.get(int(b), ""),
                        "work": float(s["b_work"][b])})
        return out

    @property
    def request_rows(self) -> list[dict]:
        res, r = self._res, self._r
        batch = res.batch
        tab = batch.tab
        lo, hi = int(batch.inputs["req_off"][r]), int(batch.inputs["req_off"][r + 1])
        kidx = self._kidx()
        rows = []
        arr = batch.inputs["arr_time"]
        for i in self._resolution_order():
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

    def _resolution_order(self):
        """Replay-local request indices in the order the reference appends request
        rows: drops as they happen, a batch's requests (queue order) at its
        kernel completion (simulation.py:240-277,353-355,413-415).  Arrival
        order without the event log."""
        res, r = self._res, self._r
        lo, hi = int(res.batch.inputs["req_off"][r]), int(res.batch.inputs["req_off"][r + 1])
        if not self.traced:
            return range(hi - lo)
        rb = res.a["req_batch"][lo:hi]
        idx = np.argsort(rb, kind="stable")  # per batch, ascending request index = queue order
        starts = np.searchsorted(rb[idx], np.arange(len(self._s["dec_time"]) + 1))
        out = []
        _, ev, _, b, q, _, _ = self._rows_log()
        for e, bb, qq in zip(ev, b, q):
            if e == TR["DROP"]:
                out.append(qq - lo)
            elif e == TR["KDONE"]:
                out.extend(idx[starts[bb]:starts[bb + 1]].tolist())
        return out

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

    def run(self, trace: bool = True) -> SimResult:
        return run_many([ReplaySpec(self.cfg, self.seed, self.predictor)], trace=trace)[0]


def run_many(specs: list[ReplaySpec], trace: bool = True) -> list[SimResult]:
    """Many independent replays in ONE device launch (the analogue of
    `infersim sweep`, cli.py:64-103).  Injected predictors are refit in place.
    trace=False skips the event log (trace_rows / segments) and runs the
    faster untraced engine."""
    batch = ReplayBatch(specs, trace=trace)
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
        out.append(SimResult(s.config.policy, s.config.policy_variant, seed, res, r, _report(res, r)))
    return out


def run(config: ExperimentConfig, seed: Optional[int] = None) -> SimResult:
    """simulation.py:516-519."""
    return Simulation(config, seed).run()
