"""The reference's shipped experiment configs and the BASELINE.json
workloads as ExperimentConfig builders.

* ``demo`` / ``overload`` / ``trace_replay``: pkg/configs/demo.yaml,
  overload.yaml, trace_replay.yaml (+ example_trace.csv) restated as dicts.
* C1: demo minus the uniform stream, 26.316 s (9,858 requests).
* C2: overload at 166.667 s (~1.0M requests).
* C4: load x HP-fraction sweep, 8 loads x 8 HP fractions x 16 seeds = 1,024
  replays of overload's 3 s horizon (~26M requests).
* C5: 64 GPUs, 20 random_profile models, bursty HP trace.
"""
from __future__ import annotations

import math

import numpy as np

from . import config as MC
from .domain import PriorityLevel
from .profiles import random_profile
from .workload import ModelWorkload

# pkg/configs/example_trace.csv (per-minute counts)
EXAMPLE_TRACE = {"vision_gate": {0: 7654.0, 1: 11412.0, 2: 7322.0, 3: 7268.0, 4: 8189.0},
                 "doc_reader": {0: 2514.0, 1: 3306.0, 2: 2307.0, 3: 3713.0, 4: 3644.0}}

DEMO = {"profiles": "default6", "duration_ms": 1000, "seed": 1, "n_gpus": 1, "policy": "predictive",
        "ground_truth": {"noise_sigma": 0.05},
        "workload": {"resnet50": {"mode": "poisson", "rate": 300}, "yolo_v8n": {"mode": "uniform", "rate": 150},
                     "roberta_b": {"mode": "poisson", "rate": 80}}}
C1 = {"profiles": "default6", "duration_ms": 26316, "seed": 1, "n_gpus": 1, "policy": "predictive",
      "ground_truth": {"noise_sigma": 0.05},
      "workload": {"resnet50": {"mode": "poisson", "rate": 300}, "roberta_b": {"mode": "poisson", "rate": 80}}}
OVERLOAD_GT = {"family": "exponential", "scale": 0.5, "base": 2.718281828459045, "offset": -0.7686,
               "weights": [0.3] * 5, "self_compute_weight": 0.25, "self_memory_weight": 0.2,
               "priority_factor": {"high": 0.6, "low": 1.0}, "noise_sigma": 0.05}
OVERLOAD_WL = {"resnet50": {"mode": "poisson", "rate": 2200}, "vit_b16": {"mode": "poisson", "rate": 800},
               "yolo_v8n": {"mode": "poisson", "rate": 1300}, "convnext_b": {"mode": "poisson", "rate": 650},
               "vgg19": {"mode": "poisson", "rate": 650}, "roberta_b": {"mode": "poisson", "rate": 400}}
OVERLOAD_HP = ("resnet50", "vit_b16")  # the HIGH-priority models of default6
C4_LOADS = (0.5, 0.75, 1.0, 1.25, 1.5, 1.75, 2.0, 2.5)
C4_HP_FRACTIONS = (0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8)
C4_SEEDS = 16


def overload_doc(duration=3000, **kw) -> dict:
    d = {"profiles": "default6", "duration_ms": duration, "seed": 0, "n_gpus": 4, "concurrency_limit": 4,
         "policy": "predictive", "goodput_window_ms": 1000, "ground_truth": dict(OVERLOAD_GT),
         "workload": {k: dict(v) for k, v in OVERLOAD_WL.items()}}
    d.update(kw)
    return d


def demo():
    return MC.config_from_dict(DEMO)


def c1():
    return MC.config_from_dict(C1)


def overload(duration=3000, **kw):
    return MC.config_from_dict(overload_doc(duration, **kw))


def c2():
    return overload(166667)


def trace_replay(duration=30000):
    doc = {"profiles": "default6", "duration_ms": duration, "seed": 2, "n_gpus": 2, "policy": "predictive",
           "ground_truth": {"noise_sigma": 0.05}, "workload": {"yolo_v8n": {"mode": "poisson", "rate": 100}}}
    cfg = MC.config_from_dict(doc)
    cfg.workload.models["resnet50"] = ModelWorkload("trace", function_id="vision_gate", scale=1.0,
                                                    trace_table=EXAMPLE_TRACE)
    cfg.workload.models["roberta_b"] = ModelWorkload("trace", function_id="doc_reader", scale=0.5,
                                                     trace_table=EXAMPLE_TRACE)
    cfg.validate()
    return cfg


def c4_point(load: float, hp_fraction: float, duration=3000):
    """One C4 grid point: HP models' rates x 2*f*load, LP models' x 2*(1-f)*load
    (overload's base HP share is exactly 3000 / 6000 req/s)."""
    doc = overload_doc(duration)
    for m, w in doc["workload"].items():
        w["rate"] = w["rate"] * (2.0 * hp_fraction * load if m in OVERLOAD_HP else 2.0 * (1.0 - hp_fraction) * load)
    return MC.config_from_dict(doc)


def c4_grid(duration=3000, seeds=C4_SEEDS):
    """[(config, seed)] of the 64-point x `seeds` sweep, point-major."""
    out = []
    for lam in C4_LOADS:
        for f in C4_HP_FRACTIONS:
            cfg = c4_point(lam, f, duration)
            out.extend((cfg, s) for s in range(seeds))
    return out


C5_DURATION_MS = 1_923_000.0  # >= 33 trace minutes: ~100M requests
C5_MINUTES = 33
C5_PREFIX_MS = 19_230.0  # the first ~1.0M requests of that replay


def c5_prefix(duration=C5_PREFIX_MS, seed=0):
    """The timed prefix of the 100M-request C5 replay: the full run's inputs
    (33-minute trace table, same RNG consumption), cut at `duration` — its
    arrivals, and so its decisions, are the full run's first ones."""
    return c5(duration=duration, minutes=C5_MINUTES, seed=seed)


def c5(duration=150.0, minutes=2, seed=0, n_gpus=64):
    """C5 shape: 20 random_profile models (m00-m05 HP bursty
    trace, m06-m19 LP Poisson 2600/s), 64 GPUs."""
    rng = np.random.default_rng(2604)
    profs = {f"m{i:02d}": random_profile(rng, f"m{i:02d}", PriorityLevel.HIGH if i < 6 else PriorityLevel.LOW)
             for i in range(20)}
    table = {}
    for i in range(6):
        for m in range(minutes):
            table.setdefault(f"hp{i}", {})[m] = float(int(rng.lognormal(math.log(150000), 0.6)))
    wl = {f"m{i:02d}": ({"mode": "poisson", "rate": 2600}) for i in range(6, 20)}
    doc = {"profiles": profs, "duration_ms": duration, "seed": seed, "n_gpus": n_gpus, "concurrency_limit": 4,
           "policy": "predictive", "ground_truth": {"noise_sigma": 0.05}, "workload": wl}
    cfg = MC.config_from_dict(doc)
    for i in range(6):
        cfg.workload.models[f"m{i:02d}"] = ModelWorkload("trace", function_id=f"hp{i}", scale=1.0, trace_table=table)
    cfg.validate()
    return cfg
