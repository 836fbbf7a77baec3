"""Interference predictor with online refit — host mirror of
/root/reference/pkg/src/infersim/predictor.py whose arithmetic runs in the
CUDA library (strait_predict*, strait_estimate_latency, strait_refit).

Names, signatures, dataclasses and error behaviour follow the reference so
existing callers and tests keep working; ``InterferencePredictor.update``
executes the reference's Adam/Huber step (predictor.py:345-363) on the device
and mirrors the resulting parameters/moments back into ``params``/``opt``.
Batched entry points (``predict_batch``, ``update_batch``) amortise the
host<->device round trip over many samples.
"""
from __future__ import annotations

import ctypes as C
import copy
import json
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _device as D
from ._abi import RefitArgs
from .domain import ModelProfile, PriorityLevel
from .pcie import PcieLinkState

EFFECT_CAP = 50.0  # predictor.py:22
MIN_SCALE = 1e-6
MIN_BASE = 1.0 + 1e-6
MIN_PRIORITY_COEFF = 1e-6


@dataclass
class PredictorParams:
    """predictor.py:30-102; canonical flat layout
    [scale, base, offset, *weights, w_cmp, w_mem, coeff_high, coeff_low]."""

    scale: float = 0.1
    base: float = math.e
    offset: float = 0.0
    weights: tuple[float, ...] = (0.1, 0.1, 0.1, 0.1, 0.1)
    self_compute_weight: float = 0.1
    self_memory_weight: float = 0.1
    priority_coeff: dict[PriorityLevel, float] = field(
        default_factory=lambda: {PriorityLevel.HIGH: 0.5, PriorityLevel.LOW: 1.0}
    )
    effect_cap: float = EFFECT_CAP

    def copy(self) -> "PredictorParams":
        return PredictorParams(self.scale, self.base, self.offset, tuple(self.weights), self.self_compute_weight,
                               self.self_memory_weight, dict(self.priority_coeff), self.effect_cap)

    def to_vector(self) -> list[float]:
        return [self.scale, self.base, self.offset, *self.weights, self.self_compute_weight,
                self.self_memory_weight, self.priority_coeff[PriorityLevel.HIGH],
                self.priority_coeff[PriorityLevel.LOW]]

    def apply_vector(self, vec: Sequence[float]) -> None:
        n = len(self.weights)
        if len(vec) != n + 7:
            raise ValueError(f"expected {n + 7} parameters, got {len(vec)}")
        self.scale, self.base, self.offset = vec[0], vec[1], vec[2]
        self.weights = tuple(vec[3:3 + n])
        self.self_compute_weight, self.self_memory_weight = vec[3 + n], vec[4 + n]
        self.priority_coeff[PriorityLevel.HIGH] = vec[5 + n]
        self.priority_coeff[PriorityLevel.LOW] = vec[6 + n]

    def n_params(self) -> int:
        return len(self.weights) + 7

    def coeff_index(self, priority: PriorityLevel) -> int:
        return len(self.weights) + (5 if priority is PriorityLevel.HIGH else 6)

    def enforce_floors(self) -> None:
        self.scale = max(self.scale, MIN_SCALE)
        self.base = max(self.base, MIN_BASE)
        for p in self.priority_coeff:
            self.priority_coeff[p] = max(self.priority_coeff[p], MIN_PRIORITY_COEFF)

    def device_vector(self) -> torch.Tensor:
        return D.dev(np.asarray(self.to_vector(), dtype=np.float64))


@dataclass
class OptimizerState:
    """predictor.py:105-121 — Adam moments + Huber threshold."""

    m: list[float]
    v: list[float]
    step: int = 0
    learning_rate: float = 0.0075
    beta1: float = 0.7
    beta2: float = 0.9
    eps: float = 1e-8
    huber_delta: float = 0.50

    @classmethod
    def for_params(cls, params: PredictorParams, **hyper) -> "OptimizerState":
        n = params.n_params()
        return cls(m=[0.0] * n, v=[0.0] * n, **hyper)


@dataclass
class FeedbackSample:
    """predictor.py:245-260."""

    batch_id: str
    colocated_twa: tuple[float, ...]
    self_compute: float
    self_memory: float
    priority: PriorityLevel
    actual: float
    predicted_at_schedule: Optional[float] = None

    def __post_init__(self):
        if not self.actual > 0:
            raise ValueError(f"sample {self.batch_id}: measured slowdown must be positive")


@dataclass
class UpdateResult:
    predicted: float
    residual: float
    skipped: bool = False
    saturated: bool = False


# ----------------------------------------------------------------------------- bias-correction tables

_BC_CACHE: dict[tuple[float, float], tuple[np.ndarray, np.ndarray, bool]] = {}
_BC_MAX = 1 << 22


def bias_correction_tables(beta1: float, beta2: float, upto: int) -> tuple[np.ndarray, np.ndarray]:
    """``1.0 - beta**t`` for t = 1..L computed with Python's float pow — the
    reference's exact operation (predictor.py:136-137).  L covers ``upto``
    steps, or stops early once both terms are exactly 1.0 (beta**t below
    2**-54), after which the device uses 1.0 — identical by construction."""
    key = (float(beta1), float(beta2))
    tab1, tab2, complete = _BC_CACHE.get(key, (np.empty(0), np.empty(0), False))
    if complete or len(tab1) >= upto:
        return tab1, tab2
    n = max(upto, 2 * len(tab1), 512)
    n = min(n, _BC_MAX)
    b1, b2 = key
    t1 = [1.0 - b1 ** t for t in range(1, n + 1)]
    t2 = [1.0 - b2 ** t for t in range(1, n + 1)]
    complete = False
    for i in range(n):  # 1 - beta**t is non-decreasing: once both are 1.0 they stay 1.0
        if t1[i] == 1.0 and t2[i] == 1.0:
            t1, t2, complete = t1[: i + 1], t2[: i + 1], True
            break
    if not complete and upto > _BC_MAX:
        raise ValueError(f"Adam betas ({b1}, {b2}) need more than {_BC_MAX} bias-correction entries")
    tab1, tab2 = np.asarray(t1, dtype=np.float64), np.asarray(t2, dtype=np.float64)
    _BC_CACHE[key] = (tab1, tab2, complete)
    return tab1, tab2


# ----------------------------------------------------------------------------- device batch helpers

def _coloc_matrix(colocated, n_metrics: int) -> np.ndarray:
    """[n][nm] or [nm]-per-row input -> metric-major [nm][n] float64."""
    a = np.asarray(colocated, dtype=np.float64)
    if a.ndim == 1:
        a = a[None, :]
    if a.shape[1] != n_metrics:
        raise ValueError(f"aggregate throughput has {a.shape[1]} metrics, model expects {n_metrics}")
    return np.ascontiguousarray(a.T)


def predict_parts_batch(params: PredictorParams, colocated, self_compute, self_memory, priority):
    """Device evaluation of Eq.4-5 for n inputs -> (exponent, effect, intf, saturated) numpy arrays."""
    nm = len(params.weights)
    A = _coloc_matrix(colocated, nm)
    n = A.shape[1]
    dA = D.dev(A)
    cmp_ = D.dev(np.broadcast_to(np.asarray(self_compute, dtype=np.float64), (n,)))
    mem = D.dev(np.broadcast_to(np.asarray(self_memory, dtype=np.float64), (n,)))
    pr = D.dev(np.broadcast_to(np.asarray(priority, dtype=np.int8), (n,)), torch.int8)
    P = params.device_vector()
    x, eff, intf = D.empty(n), D.empty(n), D.empty(n)
    sat = D.empty(n, torch.uint8)
    D.check(D.lib().strait_predict_parts(D.ptr(P), nm, float(params.effect_cap), D.ptr(dA), D.ptr(cmp_),
                                         D.ptr(mem), D.ptr(pr), n, D.ptr(x), D.ptr(eff), D.ptr(intf), D.ptr(sat),
                                         D.stream_handle()))
    return D.host(x), D.host(eff), D.host(intf), D.host(sat).astype(bool)


def predict_interference_batch(params: PredictorParams, colocated, self_compute, self_memory, priority):
    """Batched predict_interference -> (intf[n], saturated[n])."""
    _, _, intf, sat = predict_parts_batch(params, colocated, self_compute, self_memory, priority)
    return intf, sat


# ----------------------------------------------------------------------------- reference-named functions

def pressure_exponent(params: PredictorParams, colocated: Sequence[float], self_compute: float,
                      self_memory: float) -> float:
    """predictor.py:161-176 (device)."""
    if len(colocated) != len(params.weights):
        raise ValueError(f"aggregate throughput has {len(colocated)} metrics, model expects {len(params.weights)}")
    return float(predict_parts_batch(params, [colocated], self_compute, self_memory, 0)[0][0])


def _raw_effect(params: PredictorParams, exponent: float) -> tuple[float, bool]:
    """predictor.py:179-185 — (effect as clamped by kernel_effect, saturated)."""
    nm = len(params.weights)
    P = params.device_vector()
    x = D.dev(np.asarray([exponent], dtype=np.float64))
    out, sat = D.empty(1), D.empty(1, torch.uint8)
    D.check(D.lib().strait_kernel_effect(D.ptr(P), nm, float(params.effect_cap), D.ptr(x), 1, D.ptr(out),
                                         D.ptr(sat), D.stream_handle()))
    return float(D.host(out)[0]), bool(D.host(sat)[0])


def kernel_effect(params: PredictorParams, exponent: float) -> float:
    """predictor.py:188-195 (device)."""
    return _raw_effect(params, exponent)[0]


def interference_degree(params: PredictorParams, effect: float, priority: PriorityLevel) -> float:
    """predictor.py:198-200 — API shim; the product path computes this inside
    the device predictor."""
    return 1.0 + effect * params.priority_coeff[priority]


def kernel_delay(intf: float, kernel_latency_ms: float) -> float:
    """predictor.py:203-205 — API shim (used on device by strait_estimate_latency)."""
    return (intf - 1.0) * kernel_latency_ms


def predict_interference(params: PredictorParams, colocated: Sequence[float], self_compute: float,
                         self_memory: float, priority: PriorityLevel) -> float:
    """predictor.py:208-216 (device)."""
    if len(colocated) != len(params.weights):
        raise ValueError(f"aggregate throughput has {len(colocated)} metrics, model expects {len(params.weights)}")
    return float(predict_interference_batch(params, [colocated], self_compute, self_memory, int(priority))[0][0])


def estimate_latency_batch(params: PredictorParams, assumed, self_compute, self_memory, priority, total, kernel,
                           t_avail, front, now):
    """Batched Eq.1 (predictor.py:219-242) -> (latency[n], intf[n])."""
    nm = len(params.weights)
    A = _coloc_matrix(assumed, nm)
    n = A.shape[1]

    def f(v, dt=torch.float64, np_dt=np.float64):
        return D.dev(np.broadcast_to(np.asarray(v, dtype=np_dt), (n,)), dt)

    dA = D.dev(A)
    args = [f(self_compute), f(self_memory), f(priority, torch.int8, np.int8), f(total), f(kernel), f(t_avail),
            f(front), f(now)]
    lat, intf = D.empty(n), D.empty(n)
    P = params.device_vector()
    D.check(D.lib().strait_estimate_latency(D.ptr(P), nm, float(params.effect_cap), D.ptr(dA),
                                            *[D.ptr(t) for t in args], n, D.ptr(lat), D.ptr(intf),
                                            D.stream_handle()))
    return D.host(lat), D.host(intf)


def estimate_latency(params: PredictorParams, profile: ModelProfile, size: int, front_enqueue_time: float,
                     link: PcieLinkState, now: float, assumed_colocated: Sequence[float]) -> float:
    """predictor.py:219-242 (device)."""
    total = profile.total_latency_ms(size)  # raises ValueError on a bad size, as the reference
    if len(assumed_colocated) != len(params.weights):
        raise ValueError(f"aggregate throughput has {len(assumed_colocated)} metrics, "
                         f"model expects {len(params.weights)}")
    lat, _ = estimate_latency_batch(params, [assumed_colocated], profile.self_compute_at(size),
                                    profile.self_memory_at(size), int(profile.priority), total,
                                    profile.kernel_latency_ms(size), link.t_available, front_enqueue_time, now)
    return float(lat[0])


# ----------------------------------------------------------------------------- refit building blocks

def huber_batch(residuals, delta: float):
    """(huber_loss[n], huber_grad[n]) on the device (predictor.py:148-158)."""
    r = np.atleast_1d(np.asarray(residuals, dtype=np.float64))
    dr, loss, grad = D.dev(r), D.empty(max(len(r), 1)), D.empty(max(len(r), 1))
    D.check(D.lib().strait_huber(D.ptr(dr), float(delta), len(r), D.ptr(loss), D.ptr(grad), D.stream_handle()))
    return D.host(loss)[:len(r)], D.host(grad)[:len(r)]


def huber_loss(residual: float, delta: float) -> float:
    """predictor.py:148-152."""
    return float(huber_batch([residual], delta)[0][0])


def huber_grad(residual: float, delta: float) -> float:
    """predictor.py:155-158."""
    return float(huber_batch([residual], delta)[1][0])


def loss_gradient_batch(params: PredictorParams, samples: Sequence["FeedbackSample"], delta: float):
    """loss_gradient of many samples under one parameter vector, one launch:
    (predicted[n], residual[n], saturated[n], grads[n][n_params])."""
    nm = len(params.weights)
    n = len(samples)
    tw = np.empty((nm, max(n, 1)))
    for i, s in enumerate(samples):
        if len(s.colocated_twa) != nm:
            raise ValueError(f"aggregate throughput has {len(s.colocated_twa)} metrics, model expects {nm}")
        tw[:, i] = s.colocated_twa
    col = lambda f, dt=np.float64: np.array([f(s) for s in samples] or [0], dtype=dt)  # noqa: E731
    ins = [D.dev(tw), D.dev(col(lambda s: s.self_compute)), D.dev(col(lambda s: s.self_memory)),
           D.dev(col(lambda s: int(s.priority), np.int8), torch.int8), D.dev(col(lambda s: s.actual))]
    m = max(n, 1)
    pred, res, sat, grad = D.empty(m), D.empty(m), D.empty(m, torch.uint8), D.empty(params.n_params() * m)
    P = params.device_vector()
    D.check(D.lib().strait_loss_gradient(D.ptr(P), nm, float(params.effect_cap), float(delta),
                                         *[D.ptr(t) for t in ins], n, D.ptr(pred), D.ptr(res), D.ptr(sat),
                                         D.ptr(grad), D.stream_handle()))
    g = D.host(grad).reshape(params.n_params(), m)[:, :n].T
    return D.host(pred)[:n], D.host(res)[:n], D.host(sat)[:n].astype(bool), g


def loss_gradient(params: PredictorParams, sample: "FeedbackSample", delta: float):
    """predictor.py:303-309: (predicted, residual, saturated, dLoss/dtheta)."""
    p, r, s, g = loss_gradient_batch(params, [sample], delta)
    return float(p[0]), float(r[0]), bool(s[0]), [float(x) for x in g[0]]


def adam_step(opt: OptimizerState, values: list, grads: Sequence[float],
              active: Optional[Sequence[bool]] = None) -> None:
    """predictor.py:124-145: one Adam update in place on the device; inactive
    entries keep value and moments, the shared step counter advances once.
    The bias corrections 1 - beta**t are the reference's Python float powers."""
    opt.step += 1
    t = opt.step
    bc1, bc2 = 1.0 - opt.beta1 ** t, 1.0 - opt.beta2 ** t
    n = len(grads)
    if n == 0:
        return
    dv, dm, dvv = (D.dev(np.asarray(x[:n], dtype=np.float64)) for x in (values, opt.m, opt.v))
    dg = D.dev(np.asarray(grads, dtype=np.float64))
    da = D.dev(np.asarray(active, dtype=np.uint8), torch.uint8) if active is not None else None
    D.check(D.lib().strait_adam_step(D.ptr(dv), D.ptr(dm), D.ptr(dvv), D.ptr(dg), D.ptr(da), n, bc1, bc2,
                                     opt.learning_rate, opt.beta1, opt.beta2, opt.eps, D.stream_handle()))
    values[:n] = D.host(dv).tolist()
    opt.m[:n] = D.host(dm).tolist()
    opt.v[:n] = D.host(dvv).tolist()


# ----------------------------------------------------------------------------- the predictor

class InterferencePredictor:
    """predictor.py:312-428 — one global model serving all GPUs of a node.

    ``params``/``opt`` are the host view; every update runs on the device
    (strait_refit) and writes the new vector/moments back into them."""

    def __init__(self, params: Optional[PredictorParams] = None, opt: Optional[OptimizerState] = None):
        self.params = params if params is not None else PredictorParams()
        self.opt = opt if opt is not None else OptimizerState.for_params(self.params)

    def predict(self, colocated, self_compute, self_memory, priority) -> float:
        return predict_interference(self.params, colocated, self_compute, self_memory, priority)

    def predict_batch(self, colocated, self_compute, self_memory, priority):
        return predict_interference_batch(self.params, colocated, self_compute, self_memory, priority)[0]

    def estimate_latency(self, profile, size, front_enqueue_time, link, now, assumed_colocated) -> float:
        return estimate_latency(self.params, profile, size, front_enqueue_time, link, now, assumed_colocated)

    # -- refit ---------------------------------------------------------------

    def device_state(self) -> tuple[torch.Tensor, torch.Tensor]:
        """Upload (params | m | v) and the step counter."""
        vec = self.params.to_vector() + list(self.opt.m) + list(self.opt.v)
        return D.dev(np.asarray(vec, dtype=np.float64)), D.dev(np.asarray([self.opt.step]), torch.int64)

    def absorb_device_state(self, state: torch.Tensor, step: torch.Tensor) -> None:
        vals = D.host(state).tolist()
        n = self.params.n_params()
        self.params.apply_vector(vals[:n])
        self.opt.m = vals[n:2 * n]
        self.opt.v = vals[2 * n:3 * n]
        self.opt.step = int(D.host(step)[0])

    def refit_args(self, state, step, n, tw, cmp_, mem, prio, actual, out_pred=None, out_res=None,
                   out_flags=None, bc=None) -> tuple[RefitArgs, tuple]:
        """C-ABI argument block for strait_refit over device sample arrays."""
        if bc is None:
            t1, t2 = bias_correction_tables(self.opt.beta1, self.opt.beta2, self.opt.step + n)
            bc = (D.dev(t1), D.dev(t2))
        a = RefitArgs()
        a.n_metrics = len(self.params.weights)
        a.n_bc = int(bc[0].numel())
        a.n = int(n)
        a.effect_cap = float(self.params.effect_cap)
        a.learning_rate, a.beta1, a.beta2 = self.opt.learning_rate, self.opt.beta1, self.opt.beta2
        a.eps, a.huber_delta = self.opt.eps, self.opt.huber_delta
        a.state, a.step = D.ptr(state), D.ptr(step)
        a.bc1, a.bc2 = D.ptr(bc[0]), D.ptr(bc[1])
        a.twa, a.self_cmp, a.self_mem, a.actual, a.prio = (D.ptr(tw), D.ptr(cmp_), D.ptr(mem), D.ptr(actual),
                                                           D.ptr(prio))
        a.out_predicted, a.out_residual, a.out_flags = D.ptr(out_pred), D.ptr(out_res), D.ptr(out_flags)
        return a, bc

    def update_batch(self, samples: Sequence[FeedbackSample]) -> list[UpdateResult]:
        """Apply ``update`` to each sample in order, in one device launch."""
        n = len(samples)
        if n == 0:
            return []
        nm = len(self.params.weights)
        tw = np.empty((nm, n))
        for i, s in enumerate(samples):
            if len(s.colocated_twa) != nm:
                raise ValueError(f"aggregate throughput has {len(s.colocated_twa)} metrics, model expects {nm}")
            tw[:, i] = s.colocated_twa
        dtw = D.dev(tw)
        cmp_ = D.dev(np.array([s.self_compute for s in samples], dtype=np.float64))
        mem = D.dev(np.array([s.self_memory for s in samples], dtype=np.float64))
        actual = D.dev(np.array([s.actual for s in samples], dtype=np.float64))
        prio = D.dev(np.array([int(s.priority) for s in samples], dtype=np.int8), torch.int8)
        state, step = self.device_state()
        pred, res, flags = D.empty(n), D.empty(n), D.empty(n, torch.uint8)
        args, _bc = self.refit_args(state, step, n, dtw, cmp_, mem, prio, actual, pred, res, flags)
        D.check(D.lib().strait_refit(C.byref(args), D.stream_handle()))
        self.absorb_device_state(state, step)
        p, r, f = D.host(pred), D.host(res), D.host(flags)
        return [UpdateResult(float(p[i]), float(r[i]), bool(f[i] & 1), bool(f[i] & 2)) for i in range(n)]

    def update(self, sample: FeedbackSample) -> UpdateResult:
        """predictor.py:345-363 (device)."""
        return self.update_batch([sample])[0]

    # -- checkpointing (predictor.py:365-428) --------------------------------

    def checkpoint_dict(self) -> dict:
        return {
            "params": {
                "scale": self.params.scale,
                "base": self.params.base,
                "offset": self.params.offset,
                "weights": list(self.params.weights),
                "self_compute_weight": self.params.self_compute_weight,
                "self_memory_weight": self.params.self_memory_weight,
                "priority_coeff": {p.label: c for p, c in sorted(self.params.priority_coeff.items())},
                "effect_cap": self.params.effect_cap,
            },
            "optimizer": {
                "m": list(self.opt.m), "v": list(self.opt.v), "step": self.opt.step,
                "learning_rate": self.opt.learning_rate, "beta1": self.opt.beta1, "beta2": self.opt.beta2,
                "eps": self.opt.eps, "huber_delta": self.opt.huber_delta,
            },
        }

    def save(self, path) -> None:
        with open(path, "w") as f:
            json.dump(self.checkpoint_dict(), f, indent=2)

    @classmethod
    def from_checkpoint_dict(cls, doc: dict) -> "InterferencePredictor":
        p = doc["params"]
        params = PredictorParams(
            scale=p["scale"], base=p["base"], offset=p["offset"], weights=tuple(p["weights"]),
            self_compute_weight=p["self_compute_weight"], self_memory_weight=p["self_memory_weight"],
            priority_coeff={PriorityLevel.from_name(k): c for k, c in p["priority_coeff"].items()},
            effect_cap=p.get("effect_cap", EFFECT_CAP),
        )
        o = doc["optimizer"]
        opt = OptimizerState(m=list(o["m"]), v=list(o["v"]), step=o["step"], learning_rate=o["learning_rate"],
                             beta1=o["beta1"], beta2=o["beta2"], eps=o["eps"], huber_delta=o["huber_delta"])
        return cls(params, opt)

    @classmethod
    def load(cls, path) -> "InterferencePredictor":
        with open(path) as f:
            return cls.from_checkpoint_dict(json.load(f))


# ----------------------------------------------------------------------------- injection seam

_ENGINE_METHODS = ("predict", "predict_batch", "estimate_latency")


def refit_mode(predictor: InterferencePredictor) -> str:
    """How the device replay engine runs an injected predictor
    (``Simulation(config, predictor=...)``, simulation.py:127,155).

    The engine evaluates the stock estimator and refit on the device, so an
    injected object is accepted only where that is exactly what the object
    does; anything else raises instead of being silently replaced:

    * ``"adam"``: ``update`` is the stock Adam/Huber step (predictor.py:345-363),
      inherited or overridden with the same effect;
    * ``"frozen"``: ``update`` evaluates the loss but never changes ``params``
      or ``opt`` — the reference's own FrozenPredictor
      (tests/test_simulation.py:316-323);
    * ``NotImplementedError`` for overridden ``predict``/``estimate_latency`` or
      any other ``update``.

    An overridden ``update`` is classified by running it on copies of the
    predictor over probe samples and comparing the resulting state with the
    stock update's.
    """
    cls = type(predictor)
    for name in _ENGINE_METHODS:
        if getattr(cls, name) is not getattr(InterferencePredictor, name):
            raise NotImplementedError(f"{cls.__name__}.{name} is overridden; the device replay engine evaluates "
                                      f"the stock estimator (predictor.py:208-242) and cannot run it")
    if cls.update is InterferencePredictor.update:
        return "adam"
    nm = len(predictor.params.weights)
    probes = [FeedbackSample(f"probe{i}", tuple(0.1 * (i + 1 + k) for k in range(nm)), 0.2 + 0.1 * i,
                             0.3, PriorityLevel(i % 2), 1.0 + 0.7 * i) for i in range(3)]

    def state(p):
        return (p.params.to_vector(), list(p.opt.m), list(p.opt.v), p.opt.step)

    custom, stock = copy.deepcopy(predictor), copy.deepcopy(predictor)
    before = state(custom)
    for smp in probes:
        custom.update(smp)
        InterferencePredictor.update(stock, smp)
    after = state(custom)
    if after == before:
        return "frozen"
    if after == state(stock):
        return "adam"
    raise NotImplementedError(f"{cls.__name__}.update changes the predictor differently from the stock "
                              f"Adam/Huber refit (predictor.py:345-363); the device replay engine cannot run it")
