"""Batched trace replays on the device (reference: infersim/simulation.py).

``ReplayBatch`` turns (ExperimentConfig, seed[, predictor]) replays into the
flat host arrays of include/strait_replay.h — arrival streams and batch noise
drawn exactly as the reference draws them — and ``ReplayBatch.run()``
executes every replay to completion in ONE launch of the CUDA engine
(strait_replay, one warp per replay).  Results come back as numpy arrays;
``ReplayResult.sim_result(r)`` rebuilds the reference's row schemas.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import math
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _device as D
from ._replay_abi import (ARG_ARRAYS, METRIC_OUTPUTS, MS_N, POLICY_CODES, RC, RC_N, MetricsArgs, ReplayArgs,
                          ReplayConfig, ReplayModels, TRACE_DTYPE)
from .config import ExperimentConfig
from .domain import PriorityLevel
from .predictor import InterferencePredictor, PredictorParams, bias_correction_tables, refit_mode

NOISE_STREAM = 1_000_003  # simulation.py:163

# output arrays: name -> (dtype, per) with per in {"req", "batch", "cap", "replay"}
OUTPUTS = {
    "req_status": (np.int8, "req"), "req_violated": (np.uint8, "req"), "req_completion": (np.float64, "req"),
    "req_batch": (np.int32, "req"),
    "dec_time": (np.float64, "req"), "dec_pass": (np.int32, "req"), "dec_model": (np.int16, "req"),
    "dec_size": (np.int8, "req"), "dec_gpu": (np.int16, "req"), "dec_est_latency": (np.float64, "req"),
    "dec_intf": (np.float64, "req"), "b_front": (np.float64, "req"), "b_transfer_start": (np.float64, "req"),
    "b_transfer_end": (np.float64, "req"), "b_kernel_start": (np.float64, "req"),
    "b_kernel_end": (np.float64, "req"), "b_completion": (np.float64, "req"), "b_work": (np.float64, "req"),
    "b_done_order": (np.int32, "req"), "fb_predicted": (np.float64, "req"), "fb_actual": (np.float64, "req"),
    "fb_residual": (np.float64, "req"), "fb_flags": (np.uint8, "req"),
    "cap_time": (np.float64, "cap"), "cap_gpu": (np.int16, "cap"), "cap_pct": (np.float64, "cap"),
    "counters": (np.int64, "replay"),
}


@dataclass
class ReplaySpec:
    config: ExperimentConfig
    seed: Optional[int] = None
    predictor: Optional[InterferencePredictor] = None


def device_exp(z: torch.Tensor) -> torch.Tensor:
    """exp of a device array with the glibc-exact device exp (strait_math fn 0,
    csrc/strait_libm.cuh): the bits of the reference's ``math.exp``
    (simulation.py:309-311)."""
    out = torch.empty_like(z)
    D.check(D.lib().strait_math(0, D.ptr(z), None, z.numel(), D.ptr(out), D.stream_handle()))
    return out


def model_tables(profiles: dict) -> dict:
    ids = sorted(profiles)
    M = len(ids)
    nm = len(profiles[ids[0]].metrics)
    B = max(p.max_batch_size for p in profiles.values())
    t = {k: np.zeros(M * B) for k in ("total", "transfer", "kernel", "self_cmp", "self_mem")}
    thr = np.zeros((nm, M * B))
    for m, mid in enumerate(ids):
        p = profiles[mid]
        n = p.max_batch_size
        t["total"][m * B:m * B + n] = p.total_latency
        t["transfer"][m * B:m * B + n] = p.transfer_latency
        t["kernel"][m * B:m * B + n] = p.kernel_latency
        t["self_cmp"][m * B:m * B + n] = p.self_compute
        t["self_mem"][m * B:m * B + n] = p.self_memory
        thr[:, m * B:m * B + n] = np.asarray(p.throughput, dtype=np.float64).T
    t["throughput"] = thr
    t["max_batch"] = np.array([profiles[i].max_batch_size for i in ids], dtype=np.int32)
    t["prio"] = np.array([int(profiles[i].priority) for i in ids], dtype=np.int8)
    t["deadline"] = np.array([profiles[i].deadline_ms for i in ids], dtype=np.float64)
    t["timeout"] = np.array([profiles[i].batch_timeout_ms for i in ids], dtype=np.float64)
    return dict(ids=ids, M=M, nm=nm, B=B, **t)


def _check_predictor(pred: InterferencePredictor, nm: int) -> None:
    """The engine reads 3 * (nm + 7) doubles of predictor state per replay; a
    predictor sized for another metric count raises, as the reference's
    pressure_exponent does on a metric-count mismatch (predictor.py:169-172)."""
    n = pred.params.n_params()
    if n != nm + 7:
        raise ValueError(f"predictor has {n - 7} metric weights, the profiles have {nm} metrics")
    if not (len(pred.opt.m) == len(pred.opt.v) == n):
        raise ValueError(f"optimizer moments have {len(pred.opt.m)}/{len(pred.opt.v)} entries, expected {n}")


# baselines.py defaults: StaticSpatialPolicy(cap=3), ReactiveState() (lines 62-110)
STATIC_CAP = 3
REACTIVE = dict(default=3, min=1, hp_bound=3, period=200.0)


def replay_config(cfg: ExperimentConfig, pred: InterferencePredictor) -> ReplayConfig:
    if cfg.policy not in POLICY_CODES:
        raise ValueError(f"unknown policy {cfg.policy!r}, expected one of {tuple(POLICY_CODES)}")
    variant = cfg.policy_variant
    predictive = cfg.policy == "predictive"
    # simulation.py:160-161: the no_gamma_advantage ablation only applies to the predictive policy
    gt = (cfg.ground_truth.without_priority_advantage() if predictive and variant == "no_gamma_advantage"
          else cfg.ground_truth)
    c = ReplayConfig()
    c.n_gpus, c.concurrency_limit = cfg.n_gpus, cfg.concurrency_limit
    c.policy = POLICY_CODES[cfg.policy]
    # the baselines scan queues in the base priority order (scheduler.py:214-217)
    c.use_priority_order = int(not predictive or variant != "no_priority_scan")
    c.use_meet = int(variant != "no_meet")
    c.use_violate = int(variant != "no_violate_aimd")
    c.static_cap = STATIC_CAP
    c.reactive_default, c.reactive_min = REACTIVE["default"], REACTIVE["min"]
    c.reactive_hp_bound, c.reactive_period = REACTIVE["hp_bound"], REACTIVE["period"]
    c.gt_family = 0 if gt.family == "exponential" else 1
    c.has_noise = int(gt.noise_sigma > 0)
    c.effect_cap = pred.params.effect_cap
    o = pred.opt
    c.learning_rate, c.beta1, c.beta2, c.eps, c.huber_delta = o.learning_rate, o.beta1, o.beta2, o.eps, o.huber_delta
    c.gt_scale, c.gt_base, c.gt_offset = gt.scale, gt.base, gt.offset
    c.gt_w_cmp, c.gt_w_mem = gt.self_compute_weight, gt.self_memory_weight
    c.gt_pf_high, c.gt_pf_low = gt.priority_factor[PriorityLevel.HIGH], gt.priority_factor[PriorityLevel.LOW]
    for i, w in enumerate(gt.weights):
        c.gt_w[i] = w
    a = cfg.aimd
    c.aimd_floor, c.aimd_ceiling, c.aimd_increase, c.aimd_interval = a.floor, a.ceiling, a.increase_pct, a.interval_ms
    return c


class ReplayBatch:
    """Host inputs of a batch of replays sharing one profile set."""

    def __init__(self, specs: Sequence[ReplaySpec], cap_rows_max: Optional[int] = None, generate: str = "host",
                 trace: bool = False, trace_max: Optional[int] = None):
        """generate="host": draw the arrival / noise streams with numpy here;
        generate="device": draw the same streams on the GPU (devgen.py).
        trace=True also records the event log (SimResult.trace_rows) and the
        execution segments; `trace_max` records per replay (default: an
        estimate, grown and re-run if a replay overflows it)."""
        if not specs:
            raise ValueError("empty replay batch")
        if generate not in ("host", "device"):
            raise ValueError(f"generate must be 'host' or 'device', got {generate!r}")
        self.generate = generate
        self._dev = {}
        self.specs = list(specs)
        prof = self.specs[0].config.profiles
        for s in self.specs:
            s.config.validate()
            if sorted(s.config.profiles) != sorted(prof):
                raise ValueError("all replays of a batch must share one profile set")
        self.tab = model_tables(prof)
        M, nm = self.tab["M"], self.tab["nm"]
        self.preds = []
        arr_t, arr_m, model_req, mr_off, noise, req_off, cfgs, states, steps = [], [], [], [0], [], [0], [], [], []
        for s in self.specs:
            cfg = s.config
            seed = cfg.seed if s.seed is None else s.seed
            pred = s.predictor or InterferencePredictor(PredictorParams(weights=(0.1,) * nm))
            _check_predictor(pred, nm)
            self.preds.append(pred)
            cfgs.append(replay_config(cfg, pred))
            cfgs[-1].refit_frozen = int(s.predictor is not None and refit_mode(pred) == "frozen")
            states.append(pred.params.to_vector() + list(pred.opt.m) + list(pred.opt.v))
            steps.append(pred.opt.step)
            if generate == "device":
                continue
            streams = cfg.workload.generate_arrays(seed)
            per = [np.asarray(streams.get(mid, np.empty(0)), dtype=np.float64) for mid in self.tab["ids"]]
            counts = np.array([len(x) for x in per], dtype=np.int64)
            times = np.concatenate(per) if len(per) else np.empty(0)
            models = np.repeat(np.arange(M, dtype=np.int16), counts)
            order = np.argsort(times, kind="stable")  # heap order: (time, model-sorted k seq)
            pos = np.empty(len(times), dtype=np.int64)
            pos[order] = np.arange(len(times))
            base = req_off[-1]
            arr_t.append(times[order])
            arr_m.append(models[order])
            model_req.append((pos + base).astype(np.int32))
            starts = np.concatenate([[0], np.cumsum(counts)])
            mr_off.extend((base + starts[1:]).tolist())
            n = len(times)
            if cfg.ground_truth.noise_sigma > 0 and n:
                rng = np.random.default_rng(np.random.SeedSequence([seed, NOISE_STREAM]))
                # the normal draws; exp(z) is applied on the device (device_inputs), bit-exact
                noise.append(rng.normal(0.0, cfg.ground_truth.noise_sigma, n))
            else:
                noise.append(np.zeros(n))  # exp(0.0) == 1.0: the reference's noise-free factor
            req_off.append(base + n)
        if generate == "device":
            from . import devgen

            items = [(s.config.workload, s.config.seed if s.seed is None else s.seed, s.config.ground_truth.noise_sigma)
                     for s in self.specs]
            g = devgen.generate(items, self.tab["ids"])
            self._dev = {k: g[k] for k in ("arr_time", "arr_model", "model_req", "noise")}
            req_off, mr_off = g["req_off"].tolist(), g["mr_off"].tolist()
        betas = {(p.opt.beta1, p.opt.beta2) for p in self.preds}
        if len(betas) != 1:
            raise ValueError("all replays of a batch must share the Adam betas")
        b1, b2 = betas.pop()
        N = req_off[-1]
        bc1, bc2 = bias_correction_tables(b1, b2, max(steps) + N + 1)
        self.N = int(N)
        self.R = len(self.specs)
        if cap_rows_max is None:
            cap_rows_max = max(
                s.config.n_gpus * (2 * (int(s.config.workload.duration_ms / s.config.aimd.interval_ms) + 400) + 3)
                for s in self.specs)
        self.cap_rows_max = int(cap_rows_max)
        self.trace = bool(trace)
        if trace_max is None:  # arrivals + drops + 3 rows per batch + segments + ticks / resets
            n_max = int(np.max(np.diff(np.asarray(req_off, dtype=np.int64)))) if len(req_off) > 1 else 0
            trace_max = max(6 * n_max + (int(s.config.workload.duration_ms / s.config.aimd.interval_ms) + 8)
                            * (s.config.n_gpus + 1) for s in self.specs) + 256
        self.trace_max = int(min(trace_max, 2**31 - 1)) if self.trace else 0
        self.inputs = {
            "req_off": np.asarray(req_off, dtype=np.int64), "mr_off": np.asarray(mr_off, dtype=np.int64),
            "bc1": bc1, "bc2": bc2,
            "pred_state": np.asarray(states, dtype=np.float64).ravel(),
            "pred_step": np.asarray(steps, dtype=np.int64),
            "cfg": (ReplayConfig * self.R)(*cfgs),
            # launch heaviest replays first so the first CTA wave spreads them over the SMs
            "order": np.argsort(-np.diff(np.asarray(req_off, dtype=np.int64)), kind="stable").astype(np.int32),
        }
        if generate == "host":
            self.inputs.update(arr_time=np.concatenate(arr_t), arr_model=np.concatenate(arr_m),
                               model_req=np.concatenate(model_req), noise_z=np.concatenate(noise))

    # ------------------------------------------------------------------ buffers
    def alloc_outputs(self, device: bool):
        sizes = {"req": max(self.N, 1), "cap": self.R * self.cap_rows_max, "replay": self.R * RC_N}
        out = {}
        for k, (dt, per) in OUTPUTS.items():
            if device:  # zeroed: rows past a replay's batch count are never written
                out[k] = D.empty(sizes[per], getattr(torch, np.dtype(dt).name)).zero_()
            else:
                out[k] = np.zeros(sizes[per], dtype=dt)
        if self.trace:
            nbytes = max(self.R * self.trace_max, 1) * TRACE_DTYPE.itemsize
            out["trace"] = D.empty(nbytes, torch.uint8) if device else np.zeros(nbytes, np.uint8)
        return out

    def args(self, inputs: dict, outputs: dict, ptr) -> ReplayArgs:
        a = ReplayArgs()
        a.n_replays, a.cap_rows_max, a.n_bc = self.R, self.cap_rows_max, len(self.inputs["bc1"])
        a.max_gpus = max(s.config.n_gpus for s in self.specs)
        a.max_concurrency = max(s.config.concurrency_limit for s in self.specs)
        a.trace_max = self.trace_max
        a.policies = 0
        for s in self.specs:
            a.policies |= 1 << POLICY_CODES[s.config.policy]
        a.uniform = int(all(s.config.n_gpus == a.max_gpus and s.config.concurrency_limit == a.max_concurrency
                            for s in self.specs))
        t = self.tab
        md = a.models
        md.n_models, md.n_metrics, md.stride = t["M"], t["nm"], t["B"]
        for k in ("max_batch", "prio", "deadline", "timeout", "total", "transfer", "kernel", "self_cmp",
                  "self_mem", "throughput"):
            setattr(md, k, ptr(inputs["tab_" + k]))
        for k in ARG_ARRAYS:
            if k == "trace" and "trace" not in outputs:
                continue  # NULL: no event log
            src = outputs if k in outputs else inputs
            setattr(a, k, ptr(src[k]))
        return a

    def _host_small(self) -> dict:
        d = dict(self.inputs)
        for k in ("max_batch", "prio", "deadline", "timeout", "total", "transfer", "kernel", "self_cmp",
                  "self_mem", "throughput"):
            d["tab_" + k] = np.ascontiguousarray(self.tab[k])
        return d

    def host_inputs(self) -> dict:
        """Host copies of the inputs.  Host-drawn batches hold the noise as the
        normal draws ``noise_z`` (the factor is exp(z), applied where the replay
        runs); device-generated batches hold the factors ``noise``."""
        d = self._host_small()
        for k, v in self._dev.items():  # device-generated streams (copied back for host checkers)
            d[k] = D.host(v)[:max(self.N, 1)]
        return d

    def device_inputs(self) -> dict:
        out = dict(self._dev)  # device-generated streams stay where they are
        for k, v in self._host_small().items():
            if k == "cfg":
                buf = np.frombuffer(bytes(v), dtype=np.uint8)
                out[k] = D.dev(buf, torch.uint8)
            else:
                v = np.asarray(v)
                if not v.size:  # a replay batch without requests still passes valid (1-element) buffers
                    v = np.zeros(1, v.dtype)
                out[k] = D.dev(v, getattr(torch, v.dtype.name))
        for k, t in out.items():
            if isinstance(t, torch.Tensor) and not t.numel():
                out[k] = D.empty(1, t.dtype)
        if "noise_z" in out:  # host-drawn normals -> the per-batch factors exp(z), on the device
            out["noise"] = device_exp(out.pop("noise_z"))
        return out

    # ------------------------------------------------------------------ metrics
    def max_windows(self) -> int:
        """Goodput bins that can be non-empty: on-time completions finish by
        their deadline, i.e. before duration + the largest deadline_ms."""
        dl = float(np.max(self.tab["deadline"]))
        return max(int((s.config.workload.duration_ms + dl) // s.config.goodput_window_ms) + 2 for s in self.specs)

    def metrics_args(self, din: dict, dout: dict, mout: dict, ptr) -> MetricsArgs:
        m = MetricsArgs()
        m.n_replays, m.max_windows, m.table_stride = self.R, self.max_windows(), self.tab["B"]
        src = {"window_ms": din["window_ms"], "model_prio": din["tab_prio"], "kernel_table": din["tab_kernel"]}
        for k in ("req_off", "arr_time", "arr_model"):
            src[k] = din[k]
        for k in ("req_status", "req_violated", "req_completion", "counters", "dec_model", "dec_size",
                  "dec_est_latency", "b_front", "b_kernel_start", "b_kernel_end", "b_completion", "fb_predicted",
                  "fb_actual"):
            src[k] = dout[k]
        for k, v in list(src.items()) + list(mout.items()):
            setattr(m, k, ptr(v))
        return m

    def alloc_metrics(self) -> dict:
        W = self.max_windows()
        sizes = {"class_counts": (self.R * 8, torch.int64), "partial": (self.R, torch.uint8),
                 "pct": (self.R * MS_N * 3, torch.float64), "series_count": (self.R * MS_N, torch.int64),
                 "goodput": (self.R * 2 * W, torch.int64), "goodput_len": (self.R * 2, torch.int32),
                 "intf_error": (max(self.N, 1), torch.float64), "latency_error": (max(self.N, 1), torch.float64),
                 "kernel_overhead": (max(self.N, 1), torch.float64)}
        return {k: D.empty(n, dt) for k, (n, dt) in sizes.items()}

    def _enqueue(self, metrics: bool):
        """Inputs, outputs, replay and metrics launches, all on the current stream."""
        din = self.device_inputs()
        dout = self.alloc_outputs(device=True)
        args = self.args(din, dout, D.ptr)
        D.check(D.lib().strait_replay(C.byref(args), D.stream_handle()))
        mout = None
        if metrics:
            din["window_ms"] = D.dev(np.array([s.config.goodput_window_ms for s in self.specs], dtype=np.float64))
            mout = self.alloc_metrics()
            margs = self.metrics_args(din, dout, mout, D.ptr)
            D.check(D.lib().strait_replay_metrics(C.byref(margs), D.stream_handle()))
        return din, dout, mout

    def _overflow(self, counters: np.ndarray) -> bool:
        """Grow the cap-row / event-log capacity if a replay overflowed it
        (the kernel counts every row but stores only the first `*_max`);
        True means the launch must be repeated."""
        c = counters.reshape(self.R, RC_N)
        grow = False
        need = int(c[:, RC["CAP_ROWS"]].max()) if self.R else 0
        if need > self.cap_rows_max:
            self.cap_rows_max, grow = need, True
        if self.trace:
            need = int(c[:, RC["TRACE"]].max())
            if need > self.trace_max:
                if need > 2**31 - 1:
                    raise ValueError(f"event log of {need} records exceeds the trace capacity")
                self.trace_max, grow = need, True
        return grow

    def launch(self, stream=None, metrics: bool = True) -> "PendingReplay":
        """Enqueue the replay (+ device metrics) on `stream` (default: the current
        stream) without waiting: the host is free to build the next batch while
        this one runs (`PendingReplay.result` collects it).  Untraced batches
        only (a trace may need a re-run)."""
        if self.trace:
            raise ValueError("launch() is for untraced batches; use run() with trace=True")
        with _on(stream):
            din, dout, mout = self._enqueue(metrics)
            done = torch.cuda.Event()
            done.record()
        return PendingReplay(self, din, dout, mout, stream, metrics, done)

    def run(self, stream=None, metrics: bool = True, fetch=None) -> "ReplayResult":
        """Host in, device replay (+ device metrics), host out, every step on
        `stream` (default: the current stream).  `fetch` limits the
        device->host copy to those output arrays (default: all)."""
        with _on(stream):
            din, dout, mout = self._enqueue(metrics)
            if self._overflow(D.host(dout["counters"])):  # cap rows / event log overflowed: exact re-run
                return self.run(stream, metrics, fetch)
            return ReplayResult(self, _collect(din, dout, mout, fetch))


def _on(stream):
    return torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()


def _collect(din, dout, mout, fetch) -> dict:
    res = {}
    if mout is not None:
        series = ("intf_error", "latency_error", "kernel_overhead")  # per-batch arrays: only on request
        res.update({"m_" + k: D.host(v) for k, v in mout.items()
                    if fetch is None or k not in series or "m_" + k in fetch})
    res.update({k: D.host(v) for k, v in dout.items() if fetch is None or k in fetch or k == "counters"})
    if "trace" in res:
        res["trace"] = res["trace"].view(TRACE_DTYPE)
    res["pred_state"] = D.host(din["pred_state"])
    res["pred_step"] = D.host(din["pred_step"])
    return res


class PendingReplay:
    """A launched replay batch (ReplayBatch.launch); result() copies it back."""

    def __init__(self, batch, din, dout, mout, stream, metrics=True, done=None):
        self.batch, self.din, self.dout, self.mout, self.stream = batch, din, dout, mout, stream
        self.metrics, self.done = metrics, done

    def result(self, fetch=None, copy_stream=None) -> "ReplayResult":
        """Wait for this replay and copy it back.  With `copy_stream` the copies
        run there, ordered after this launch only, so a batch launched since on
        the launch stream keeps running while they proceed."""
        on = copy_stream if copy_stream is not None else self.stream
        with _on(on):
            if copy_stream is not None and self.done is not None:
                copy_stream.wait_event(self.done)
            if self.batch._overflow(D.host(self.dout["counters"])):  # cap rows overflowed: exact re-run
                return self.batch.run(self.stream, self.metrics, fetch)
            return ReplayResult(self.batch, _collect(self.din, self.dout, self.mout, fetch))


class ReplayResult:
    """Outputs of a replay batch (numpy), with reference-shaped views."""

    def __init__(self, batch: ReplayBatch, arrays: dict):
        self.batch = batch
        self.a = arrays
        self.counters = arrays["counters"].reshape(batch.R, RC_N)

    def check(self):
        from ._abi import check_code

        for r in range(self.batch.R):
            check_code(int(self.counters[r, RC["ERROR"]]), f"replay {r}")

    def metrics(self, r: int) -> dict:
        """The replay's metrics in the reference's MetricsReport.to_dict() schema
        (metrics.py:63-85), from the device metrics kernels."""
        if "m_pct" not in self.a:
            raise ValueError("replay ran without metrics")
        b = self.batch
        W = b.max_windows()
        cc = self.a["m_class_counts"].reshape(b.R, 2, 4)[r]
        pct = self.a["m_pct"].reshape(b.R, MS_N, 3)[r]
        cnt = self.a["m_series_count"].reshape(b.R, MS_N)[r]
        gp = self.a["m_goodput"].reshape(b.R, 2, W)[r]
        glen = self.a["m_goodput_len"].reshape(b.R, 2)[r]

        def opt(x):
            return None if np.isnan(x) else float(x)

        out = {"window_ms": float(b.specs[r].config.goodput_window_ms), "partial": bool(self.a["m_partial"][r] & 1)}
        for c, name in ((0, "high"), (1, "low")):
            arr, comp, drop, viol = (int(x) for x in cc[c])
            out[name] = {"arrivals": arr, "completed": comp, "dropped": drop, "violations": viol,
                         "violation_rate_pct": 100.0 * viol / arr if arr else 0.0,
                         "p50_latency_ms": opt(pct[c][0]), "p95_latency_ms": opt(pct[c][1]),
                         "p99_latency_ms": opt(pct[c][2]), "goodput_counts": [int(x) for x in gp[c][:glen[c]]]}
        for s_, name in ((2, "intf_error"), (3, "latency_error"), (4, "kernel_overhead")):
            n = int(cnt[s_])
            out[name] = {"count": n, "median_abs": opt(pct[s_][0]), "p95_abs": opt(pct[s_][1]),
                         "p99_abs": opt(pct[s_][2])} if n else {"count": 0}
        return out

    def violation_rates(self, r: int) -> tuple[float, float]:
        c = self.counters[r]
        hp = 100.0 * c[RC["HP_VIOL"]] / c[RC["HP_ARR"]] if c[RC["HP_ARR"]] else 0.0
        lp = 100.0 * c[RC["LP_VIOL"]] / c[RC["LP_ARR"]] if c[RC["LP_ARR"]] else 0.0
        return hp, lp

    def replay_slice(self, r: int) -> dict:
        """Per-replay views: request arrays (global order) and batch arrays (submission order)."""
        b = self.batch
        lo, hi = int(b.inputs["req_off"][r]), int(b.inputs["req_off"][r + 1])
        nb = int(self.counters[r, RC["BATCHES"]])
        out = {}
        for k, (_, per) in OUTPUTS.items():
            if per == "req":
                out[k] = self.a[k][lo:hi] if k.startswith("req") else self.a[k][lo:lo + nb]
            elif per == "cap":
                n = min(int(self.counters[r, RC["CAP_ROWS"]]), b.cap_rows_max)
                out[k] = self.a[k][r * b.cap_rows_max:r * b.cap_rows_max + n]
        np_ = b.tab["nm"] + 7
        out["pred_state"] = self.a["pred_state"][r * 3 * np_:(r + 1) * 3 * np_]
        out["pred_step"] = int(self.a["pred_step"][r])
        out["counters"] = self.counters[r]
        return out

    def trace_records(self, r: int) -> np.ndarray:
        """Replay r's event log (StraitTraceRec, TRACE_DTYPE) in the reference's append order."""
        if "trace" not in self.a:
            raise ValueError("replay ran without trace=True")
        tm = self.batch.trace_max
        n = int(self.counters[r, RC["TRACE"]])
        return self.a["trace"][r * tm:r * tm + n]
